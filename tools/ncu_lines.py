"""Per-source-line warp-stall samples from an ncu report captured with --import-source on and a
-lineinfo build: where each warp role of the fused kernel spends its time, without perturbing it.

  python tools/ncu_lines.py gpurun_out/src_arxiv.ncu-rep [--top 40] [--roles]
"""
import argparse
import csv
import io
import re
import subprocess

STALLS = ["barrier", "branch_resolving", "dispatch", "drain", "lg", "long_sb", "math", "membar", "mio", "misc",
          "no_inst", "not_selected", "selected", "short_sb", "sleep", "tex", "wait"]


def load(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    out = []  # (file, line, source, samples, {stall: n})
    fname = None
    hdr = None
    for row in csv.reader(io.StringIO(raw)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or row[0] == "" or row[0] == "Function Name":
            continue
        try:
            n = float(row[4])
        except (ValueError, IndexError):
            continue
        st = {}
        for s in STALLS:
            if "stall_" + s in hdr:
                try:
                    st[s] = float(row[hdr.index("stall_" + s)])
                except ValueError:
                    pass
        out.append((fname, int(row[0]), row[1].strip(), n, st))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--file", default="attention_sm100.cu")
    a = ap.parse_args()
    rows = load(a.rep)
    tot = sum(r[3] for r in rows) or 1
    print(f"total samples {tot:.0f}")
    for f, ln, src, n, st in sorted(rows, key=lambda r: -r[3])[: a.top]:
        top = sorted(st.items(), key=lambda x: -x[1])[:3]
        ts = " ".join(f"{k}:{v / n * 100:.0f}%" for k, v in top if v > 0)
        print(f"{f[:14]:>14}:{ln:<4} {n / tot * 100:5.1f}%  {ts:42s} {src[:80]}")


def roles(rep, bounds, dump=None):
    """Per-role sample totals: SASS rows are labelled by the role of the closest preceding
    attention_sm100.cu line (inlined helpers in sm100.cuh inherit their call site's role).
    bounds: list of (first_line, name) sorted by line."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, cur_line = None, None
    recs = []  # (addr, file, line, samples, stalls-dict)
    hdr = None
    for row in csv.reader(io.StringIO(raw)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or row[0] == "Function Name":
            continue
        if row[0] != "":
            cur_line = int(row[0])
            continue
        if not row[2].startswith("0x"):
            continue
        try:
            n = float(row[4])
        except ValueError:
            continue
        st = {s: float(row[hdr.index("stall_" + s)] or 0) for s in STALLS if "stall_" + s in hdr}
        recs.append((int(row[2], 16), cur_file, cur_line, n, st, row[3].strip()))
    recs.sort()
    def role_of(line):
        r = "setup"
        for b, nm in bounds:
            if line >= b:
                r = nm
        return r
    cur = "setup"
    agg = {}
    for addr, f, ln, n, st, sass in recs:
        if f == "attention_sm100.cu" and ln is not None and ln > 240:
            cur = role_of(ln)
        d = agg.setdefault(cur, {"n": 0.0, "wait_mbar": 0.0, "st": {}})
        d["n"] += n
        if "SYNCS.PHASECHK" in sass or (f == "sm100.cuh" and ln in (40, 41, 42, 43, 44, 45, 46, 47, 50, 51, 52, 53, 54, 55, 56, 57, 58)):
            d["wait_mbar"] += n
        for k, v in st.items():
            d["st"][k] = d["st"].get(k, 0) + v
        if dump == cur:
            key = (f, ln)
            d.setdefault("lines", {}).setdefault(key, [0.0, {}])
            d["lines"][key][0] += n
            for k, v in st.items():
                d["lines"][key][1][k] = d["lines"][key][1].get(k, 0) + v
    tot = sum(d["n"] for d in agg.values()) or 1
    for nm, d in sorted(agg.items(), key=lambda x: -x[1]["n"]):
        top = sorted(d["st"].items(), key=lambda x: -x[1])[:4]
        print(f"{nm:10s} {d['n'] / tot * 100:5.1f}% of samples, mbar-wait {d['wait_mbar'] / max(d['n'], 1) * 100:4.0f}%  "
              + " ".join(f"{k}:{v / max(d['n'], 1) * 100:.0f}%" for k, v in top))
    if dump and dump in agg:
        d = agg[dump]
        print(f"--- lines of role {dump}")
        for (f, ln), (n, st) in sorted(d.get("lines", {}).items(), key=lambda x: -x[1][0])[:30]:
            top = sorted(st.items(), key=lambda x: -x[1])[:3]
            print(f"{f[:16]:>16}:{ln:<4} {n / d['n'] * 100:5.1f}%  " + " ".join(f"{k}:{v / max(n, 1) * 100:.0f}%" for k, v in top))


ROLE_BOUNDS = [(246, "index"), (309, "producer"), (382, "loaders"), (426, "mma"), (518, "softmax"), (636, "correct"),
               (722, "teardown")]

if __name__ == "__main__":
    import sys
    if len(sys.argv) > 2 and sys.argv[2] == "--roles":
        roles(sys.argv[1], ROLE_BOUNDS, sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        main()
