timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
VARIANTS="base" CONFIGS="arxiv batched reddit products cora" bash tools/variants.sh
