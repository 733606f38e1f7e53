timeout -s KILL 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -1
VARIANTS="base" CONFIGS="arxiv batched reddit cora" bash tools/variants.sh
for c in arxiv batched; do timeout -s KILL 300 python tools/trace.py --config $c --out gpurun_out/trace_sf_$c.npz > gpurun_out/tr_$c.log 2>&1; tail -1 gpurun_out/tr_$c.log; done
python tools/trace_stats.py gpurun_out/trace_sf_*.npz
