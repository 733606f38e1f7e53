#!/bin/bash
# saved-stats backward time per experiment library (libf3s_<v>.so; "base" = libf3s.so), round-robin
for c in ${CONFIGS:-arxiv reddit batched}; do for r in 1 2; do for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset F3S_LIB_VARIANT; else export F3S_LIB_VARIANT=$v; fi
  echo "$c $v $(timeout -s KILL 300 python tools/bench_backward.py --config $c --variant saved 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["ms_per_step"])')"
done; done; done
