#!/bin/bash
# per-kernel times of the saved-stats backward (ncu launch list, cold/serialised) for each config (tag = $1)
T=${1:-bl}
mkdir -p gpurun_out
for c in ${CONFIGS:-arxiv reddit batched}; do
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:k_bwd --csv --log-file gpurun_out/${T}_bwd_launch_$c.csv python tools/bench_backward.py --config $c --variant saved --steps 1 --warmup 0 > /dev/null 2>&1
  python - $c gpurun_out/${T}_bwd_launch_$c.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
h = rows[0]; k = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void unnamed>::", "")
    k.setdefault((d["ID"], name), {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
for (i, n), m in k.items():
    t = m["gpu__time_duration.sum"]
    print(sys.argv[1], n, "%.3f ms" % (t[0] / (1e6 if t[1] == "ns" else 1e3 if t[1] == "us" else 1)),
          " ".join("%s=%.2fGB" % (x.split("__")[1].split(".")[0], v[0] / 1e9) for x, v in m.items() if "bytes" in x))
PY
done
