"""Markdown rows of DESIGN.md §8 from bench JSON lines: python tools/results_table.py TAG [BASE_TAG]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(tag, name):
    p = os.path.join(ROOT, "gpurun_out", f"{tag}_bench_{name}.json")
    if not os.path.exists(p):
        p = os.path.join(ROOT, "profiles", f"{tag}_bench_{name}.json")
    try:
        return json.loads(open(p).read().strip().splitlines()[-1])
    except Exception:
        return None


tag = sys.argv[1]
base = sys.argv[2] if len(sys.argv) > 2 else None
for name in ["default", "arxiv", "reddit", "batched", "cora", "products_bf16", "arxiv_bf16", "reddit_bf16",
             "batched_bf16", "cora_bf16"]:
    j = load(tag, name)
    if not j:
        continue
    b = load(base, name) if base else None
    wl = j["config"]["workload"].split(":")[0]
    par = j.get("parity") or {}
    pt = f"{par.get('max_abs', float('nan')):.1e} / {par.get('rel_fro', float('nan')):.1e}" if par else "(bench: sampled)"
    r = j["roofline"]
    print(f"| {wl} ({j['dtype']}) | {b['ms_per_step'] if b else '—'} | {j['ms_per_step']:.3f} "
          f"(p10 {j['timing']['step_ms']['p10']:.3f}, p90 {j['timing']['step_ms']['p90']:.3f}) | {j['value']:.0f} | "
          f"{r['achieved']:.0f} ({r['frac']:.2f}) | {pt} |")
