mkdir -p gpurun_out
for c in reddit arxiv products batched; do
  timeout -s KILL 600 python tools/prof.py --config $c > gpurun_out/r02b_prof_$c.txt 2>&1
done
