#!/bin/bash
# full evaluation on one GPU: all gpu tests, smoke, the default bench line, the reference arm,
# the other configs, ablation variants, the ncu launch list and full ncu captures (tag = $1)
T=${1:-r01}
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.txt 2>&1; tail -3 gpurun_out/${T}_gpu_tests.txt
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.txt 2>&1; tail -1 gpurun_out/${T}_smoke.txt
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err; cat gpurun_out/${T}_bench_default.json
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_reference.json 2>&1
for c in cora batched products reddit; do
  timeout -s KILL 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout -s KILL 600 python bench.py --variant simt --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_arxiv_simt.json 2>&1
timeout -s KILL 600 python bench.py --variant no_reorder --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_arxiv_noreorder.json 2>&1
timeout -s KILL 600 python bench.py --dtype e4m3 > gpurun_out/${T}_bench_arxiv_e4m3.json 2>&1
timeout -s KILL 600 python bench.py --config batched --variant one_head --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_batched_onehead.json 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches_arxiv.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_f3s_sm100 -s 3 -c 1 -o gpurun_out/${T}_prof_arxiv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_f3s_sm100 -s 3 -c 1 -o gpurun_out/${T}_prof_batched python bench.py --config batched --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep "^${T}_" | head -50
for c in arxiv batched reddit cora; do timeout -s KILL 300 python tools/bench_backward.py --config $c 2>/dev/null | tail -1; done > gpurun_out/${T}_bench_backward.jsonl
