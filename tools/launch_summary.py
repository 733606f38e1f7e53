"""Summarise an ncu --metrics gpu__time_duration.sum launch list: python tools/launch_summary.py list.csv [cmd]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = collections.OrderedDict()
tot = 0.0
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", ""))
        agg.setdefault(d["Kernel Name"][:90], []).append(v)
        tot += v
if len(sys.argv) > 2:
    print(f"ncu launch list of `{sys.argv[2]}` (gpu__time_duration.sum, --clock-control none; cold, serialised)")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v) / tot * 100:6.1f}%  n={len(v):4d}  mean={sum(v) / len(v) / 1e3:10.1f} us  {k}")
