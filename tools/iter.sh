#!/bin/bash
# one GPU iteration: parity tests of the fused kernel, bench lines and F3S_TRACE dumps (tag = $1)
TAG=${1:-x}; shift
CONFIGS=${CONFIGS:-"arxiv batched cora"}
timeout -s KILL 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -2
for c in $CONFIGS; do
  timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
for c in ${TRACE:-arxiv batched}; do
  timeout -s KILL 300 python tools/trace.py --config $c --out gpurun_out/trace_${TAG}_$c.npz > /dev/null 2>&1
done
