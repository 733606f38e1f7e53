timeout -s KILL 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -1
VARIANTS="base nosplit" CONFIGS="arxiv batched reddit cora" bash tools/variants.sh
