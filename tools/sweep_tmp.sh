timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
VARIANTS="base" CONFIGS="arxiv batched reddit" bash tools/variants.sh
timeout -s KILL 300 python tools/prof.py --config reddit 2>&1 | grep -E "kernel|experiment" | head -5
