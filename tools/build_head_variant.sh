#!/bin/bash
# build libf3s_<name>.so from the committed sources of <rev> (default HEAD) for same-box A/B runs
NAME=${1:-old}; REV=${2:-HEAD}
set -e
T=$(mktemp -d)
cp -r paper_2505_08098_b200/csrc $T/cur
for f in paper_2505_08098_b200/csrc/*.cu paper_2505_08098_b200/csrc/*.h paper_2505_08098_b200/csrc/*.cuh; do
  git show $REV:$f > $f
done
python paper_2505_08098_b200/_build.py $NAME > /dev/null
cp $T/cur/* paper_2505_08098_b200/csrc/
rm -rf $T
touch paper_2505_08098_b200/csrc/*.cu
