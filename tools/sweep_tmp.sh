F3S_LIB_VARIANT=w3l3 timeout -s KILL 300 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -1
VARIANTS="base w3l3 w3l4" CONFIGS="arxiv batched reddit" bash tools/variants.sh
