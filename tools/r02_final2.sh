#!/bin/bash
# late round-2 checkpoint without ncu reports (gpurun copies back <= 64 MiB): gpu tests, smoke, fp16 bench
# lines of every config, the reference arm, backward lines, backward launch times, shard balance.
T=${1:-r02w}
mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -2 gpurun_out/${T}_gpu_tests.txt
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.txt 2>&1; tail -2 gpurun_out/${T}_smoke.txt
timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
for c in arxiv reddit batched cora; do
  timeout -s KILL 600 python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
for c in arxiv reddit batched cora; do for v in saved saved_lp tc; do timeout -s KILL 300 python tools/bench_backward.py --config $c --variant $v 2>/dev/null | tail -1; done; done > gpurun_out/${T}_bench_backward.jsonl
CONFIGS="arxiv reddit batched" bash tools/bwd_launches.sh ${T} > gpurun_out/${T}_bwd_launches.txt 2>&1
python tools/shard_balance.py > gpurun_out/${T}_shard_balance.txt 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_launches_products.csv python bench.py --config products --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-batch 0 > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
