#!/bin/bash
# round-2 checkpoint on one GPU (tag = $1): all gpu tests, smoke, every bench line (fp16, bf16, e4m3),
# the reference arm, backward lines, launch lists and ncu --set full of the fused kernel per config.
T=${1:-r02f}
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -2 gpurun_out/${T}_gpu_tests.txt
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.txt 2>&1; tail -2 gpurun_out/${T}_smoke.txt
timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
for c in arxiv reddit batched cora; do
  timeout -s KILL 600 python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
for c in products arxiv reddit batched cora; do
  timeout -s KILL 600 python bench.py --config $c --dtype bf16 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_${c}_bf16.json 2> gpurun_out/${T}_bench_${c}_bf16.err
done
for c in products arxiv reddit; do
  timeout -s KILL 600 python bench.py --config $c --dtype e4m3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_${c}_e4m3.json 2> gpurun_out/${T}_bench_${c}_e4m3.err
done
for c in arxiv reddit batched cora; do for v in saved saved_lp tc; do timeout -s KILL 300 python tools/bench_backward.py --config $c --variant $v 2>/dev/null | tail -1; done; done > gpurun_out/${T}_bench_backward.jsonl
CONFIGS="arxiv reddit batched" bash tools/bwd_launches.sh ${T} > gpurun_out/${T}_bwd_launches.txt 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd -c 3 -o gpurun_out/${T}_prof_bwd_arxiv python tools/bench_backward.py --config arxiv --variant saved --steps 1 --warmup 0 > /dev/null 2>&1
for c in products reddit arxiv batched cora; do
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-batch 0 > /dev/null 2>&1
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_f3s_sm100 -s 3 -c 1 -o gpurun_out/${T}_prof_$c python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-batch 0 > /dev/null 2>&1
done
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_f3s_sm100 -s 3 -c 1 -o gpurun_out/${T}_prof_arxiv_e4m3 python bench.py --config arxiv --dtype e4m3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-batch 0 > /dev/null 2>&1
# gpurun copies back at most 64 MiB: summarise the ncu reports here and keep only the products one
for f in gpurun_out/${T}_prof_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
python tools/update_traffic.py ${T} products reddit arxiv batched cora > /dev/null 2>&1; cp profiles/traffic.json gpurun_out/${T}_traffic.json
ls gpurun_out/${T}_prof_*.ncu-rep | grep -v "_prof_products.ncu-rep" | xargs rm -f
ls gpurun_out | grep "^${T}_" | wc -l
