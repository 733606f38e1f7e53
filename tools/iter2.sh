#!/bin/bash
# GPU iteration: parity tests, bench lines, per-role profile (tag = $1)
TAG=${1:-x}
timeout -s KILL 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -2
for c in ${CONFIGS:-arxiv batched cora}; do
  timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
for c in ${PROF:-arxiv batched}; do timeout -s KILL 300 python tools/prof.py --config $c > gpurun_out/prof_${TAG}_$c.txt 2>&1; done
