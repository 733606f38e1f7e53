#!/bin/bash
TAG=$1
for f in gpurun_out/bench_${TAG}_*.json; do python -c "
import json,sys
try:
  j=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('_')[-1][:-5], j['value'], j['ms_per_step'], j['roofline']['frac'], j['roofline']['achieved'])
except Exception as e: print('$f', 'ERR', e)
"; done
python tools/trace_stats.py gpurun_out/trace_${TAG}_*.npz 2>/dev/null
