#!/bin/bash
# round-2 evaluation on one GPU (tag = $1): gpu tests, smoke, default bench line (products),
# the other configs (fp16 + bf16), launch list + ncu --set full of the fused kernel per config.
T=${1:-r02}
STAGES=${STAGES:-tests smoke bench configs ncu}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt 2>&1
for s in $STAGES; do case $s in
tests)
  timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.txt 2>&1
  tail -3 gpurun_out/${T}_gpu_tests.txt ;;
smoke)
  timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.txt 2>&1; tail -2 gpurun_out/${T}_smoke.txt ;;
bench)
  timeout -s KILL 900 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
  tail -1 gpurun_out/${T}_bench_default.json ;;
configs)
  for c in arxiv reddit batched cora; do
    timeout -s KILL 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
  done
  for c in products arxiv reddit batched cora; do
    timeout -s KILL 600 python bench.py --config $c --dtype bf16 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_bench_${c}_bf16.json 2> gpurun_out/${T}_bench_${c}_bf16.err
  done
  for f in gpurun_out/${T}_bench_*.json; do python - "$f" <<'EOF'
import json, sys
try:
    j = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], j["config"]["workload"], j.get("dtype"), j["ms_per_step"], j["roofline"]["frac"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
EOF
  done ;;
ncu)
  for c in products reddit arxiv batched cora; do
    timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${T}_launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-batch 0 > /dev/null 2>&1
    timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_f3s_sm100 -s 3 -c 1 -o gpurun_out/${T}_prof_$c python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph-batch 0 > /dev/null 2>&1
  done
  ls gpurun_out | grep "^${T}_" ;;
esac; done
