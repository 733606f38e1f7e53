#!/bin/bash
# GPU iteration: attention parity tests + bench lines (tag = $1), printed compactly
TAG=${1:-x}
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -3
for c in ${CONFIGS:-arxiv batched cora}; do
  timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err || tail -5 gpurun_out/bench_${TAG}_$c.err
done
bash tools/show.sh $TAG
for c in ${PROF:-}; do timeout -s KILL 300 python tools/prof.py --config $c > gpurun_out/prof_${TAG}_$c.txt 2>&1; done
