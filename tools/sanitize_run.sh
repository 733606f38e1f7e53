#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck over tools/sanitize_small.py -> gpurun_out/$1
OUT=gpurun_out/${1:-sanitizer.txt}
mkdir -p gpurun_out
echo "compute-sanitizer (memcheck, synccheck, racecheck) on tools/sanitize_small.py" > $OUT
for t in memcheck synccheck racecheck; do
  echo "== $t" >> $OUT
  timeout -s KILL 600 /usr/local/cuda/bin/compute-sanitizer --tool $t python tools/sanitize_small.py 2>&1 | grep -v "^=========$" | tail -14 >> $OUT
done
grep -i "summary\|ok fwd" $OUT
