mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests/test_gpu_backward.py -q -x -p no:cacheprovider 2>&1 | tail -3
for c in ${CONFIGS:-arxiv reddit batched}; do for r in 1 2; do for v in old new; do
  if [ $v = old ]; then export F3S_LIB_VARIANT=old; else unset F3S_LIB_VARIANT; fi
  echo "$c $v $(timeout -s KILL 300 python tools/bench_backward.py --config $c --variant ${VARIANT:-saved} 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(j["ms_per_step"])')"
done; done; done
