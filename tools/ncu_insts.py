"""Warp-level instructions executed per source line (and per warp-role line range) from an ncu
report captured with --import-source on: which role's code the SM issue slots go to.

  python tools/ncu_insts.py rep.ncu-rep [--items N] [--top 30]
"""
import argparse
import csv
import io
import re
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--items", type=float, default=0, help="divide totals by this (e.g. work items per launch)")
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--src", default="paper_2505_08098_b200/csrc/attention_sm100.cu")
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
per = {}
fname = None
hdr = None
for row in csv.reader(io.StringIO(raw)):
    if not row:
        continue
    if row[0] in ("File Path", "File Name"):
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0].isdigit():
        continue
    try:
        n = float(row[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    if n > 0:
        per[(fname, int(row[0]))] = (n, row[1].strip())
tot = sum(v[0] for v in per.values())
div = a.items or 1.0
print(f"total warp instructions {tot:.4g}  per item {tot / div:.1f}")
# role ranges from the '=====' banners of the kernel source
src = open(a.src).read().splitlines()
marks = [(i + 1, re.sub(r"[^a-zA-Z /()-]", "", l.split("=====")[1]).strip()[:28]) for i, l in enumerate(src) if "// =====" in l]
marks.append((len(src) + 1, "end"))
role = {}
for (fn, ln), (n, s) in per.items():
    r = "other/helpers"
    if fn == a.src.split("/")[-1]:
        for (b, nm), (e, _) in zip(marks, marks[1:]):
            if b <= ln < e:
                r = nm
        if ln < marks[0][0]:
            r = "setup"
    role[r] = role.get(r, 0) + n
for r, n in sorted(role.items(), key=lambda x: -x[1]):
    print(f"  {r:30s} {100 * n / tot:5.1f}%  {n / div:8.1f} per item")
for (fn, ln), (n, s) in sorted(per.items(), key=lambda x: -x[1][0])[: a.top]:
    print(f"{fn[:14]:>14s}:{ln:<4d} {100 * n / tot:5.1f}% {n / div:8.1f}  {s[:90]}")
