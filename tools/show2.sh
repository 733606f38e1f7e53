#!/bin/bash
TAG=$1
for f in gpurun_out/bench_${TAG}_*.json; do python -c "
import json,sys
try:
  j=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('_')[-1][:-5], j['value'], j['ms_per_step'], j['roofline']['frac'], j['roofline']['achieved'])
except Exception as e: print('$f', 'ERR', open('$f').read()[-500:])
"; done
paste gpurun_out/prof_${TAG}_arxiv.txt gpurun_out/prof_${TAG}_batched.txt 2>/dev/null | sed 's/us\/CTA//g'
