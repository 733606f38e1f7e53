#!/bin/bash
# one-call check of a kernel change: gpu tests, then the bench line of each config (tag = $1)
T=${1:-q}
CONFIGS=${CONFIGS:-products arxiv reddit batched cora}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -3 gpurun_out/${T}_gpu_tests.txt
for c in $CONFIGS; do
  timeout -s KILL 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
  python -c "
import json
try:
  j=json.loads(open('gpurun_out/${T}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', j['ms_per_step'], j['roofline']['frac'])
except Exception as e: print('$c ERR', e)
"
done
