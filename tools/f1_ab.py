"""f1 (heavy row-window split) A/B on one GPU, for the long-tailed Reddit-shaped
graph: the whole graph (1 GPU) and each of the 8 row shards of an 8-GPU run (each shard is one
GPU's whole job; the 8-GPU makespan is the slowest shard), with
  * no split (bound larger than any window),
  * the global bound (default at every GPU count: bitwise equal to the single-GPU result),
  * the shard's own bound max(16, shard chunks / (2 * SMs)) (what a shard-local plan would pick),
  * fixed bounds.
Prints ms per call (median of --reps, cold L2) and the split windows per plan.

  python tools/f1_ab.py [--config reddit] [--world 8] [--reps 10]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from f3s_inputs import configs
    from paper_2505_08098_b200 import dist, f3s
    w = configs.get(a.config)
    csr = w.graph()
    Qb, Kb, Vb = w.qkv(csr)
    dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.float16)
    Q, K, V = dev(Qb), dev(Kb), dev(Vb)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(plan, Ql, O):
        for _ in range(2):
            f3s.attention(plan, Ql, K, V, O, scale=w.scale)
        t = []
        for _ in range(a.reps):
            flush.fill_(1)
            ev[0].record()
            f3s.attention(plan, Ql, K, V, O, scale=w.scale)
            ev[1].record()
            torch.cuda.synchronize()
            t.append(ev[0].elapsed_time(ev[1]))
        return float(np.median(t))

    full = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
    total = full.info()["total_chunks"]
    gbound = f3s.default_split_chunks(total, sms)
    O = torch.empty(Q.shape, dtype=torch.float32, device="cuda")
    print(f"{a.config}: total chunks {total}, global bound {gbound} chunks, max width {full.info()['max_width']}")
    res = {}
    for name, bound in [("no split", 1 << 30), ("global bound", gbound), ("bound 256", 256), ("bound 128", 128),
                        ("bound 64", 64)]:
        full.set_split(bound)
        res[name] = timed(full, Q, O)
        print(f"  1 GPU  {name:14s} ({bound if bound < 1 << 30 else 'inf'} chunks): {res[name]:.3f} ms "
              f"split windows {full.info()['split_groups']}", flush=True)
    ref = None
    bounds = dist.partition(csr.row_ptr, a.world)
    for name in ["no split", "global bound", "shard bound"]:
        worst, per = 0.0, []
        for r in range(a.world):
            spec = dist.shard_spec(csr.row_ptr, csr.col_idx, r, a.world, bounds=bounds)
            rp = torch.from_numpy(spec.row_ptr).cuda()
            ci = torch.from_numpy(spec.col_idx).cuda()
            p = f3s.plan_rows(rp, ci, spec.row_end - spec.row_begin, spec.n_cols)
            b = {"no split": 1 << 30, "global bound": gbound,
                 "shard bound": f3s.default_split_chunks(p.info()["total_chunks"], sms)}[name]
            p.set_split(b)
            Ql = Q[spec.row_begin:spec.row_end].contiguous()
            Ol = torch.empty(Ql.shape, dtype=torch.float32, device="cuda")
            ms = timed(p, Ql, Ol)
            per.append(ms)
            worst = max(worst, ms)
            del p
        print(f"  {a.world} shards {name:14s}: slowest shard {worst:.3f} ms, mean {np.mean(per):.3f} ms, "
              f"per shard {' '.join(f'{x:.3f}' for x in per)}", flush=True)


if __name__ == "__main__":
    main()
