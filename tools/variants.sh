#!/bin/bash
# bench several experiment builds (libf3s_<v>.so) back to back: VARIANTS="a b" CONFIGS="arxiv batched"
# [BENCH_ARGS="--dtype e4m3"]
mkdir -p gpurun_out
for v in ${VARIANTS}; do
  for c in ${CONFIGS:-arxiv batched}; do
    if [ "$v" = base ]; then unset F3S_LIB_VARIANT; else export F3S_LIB_VARIANT=$v; fi
    timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/var_${v}_$c.json 2> gpurun_out/var_${v}_$c.err
    python -c "
import json
try:
  j=json.loads(open('gpurun_out/var_${v}_$c.json').read().strip().splitlines()[-1]); print('$v', '$c', j['ms_per_step'], j['roofline']['frac'])
except Exception as e: print('$v $c ERR', e)
"
  done
done
unset F3S_LIB_VARIANT
