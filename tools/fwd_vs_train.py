"""f3s_attention vs f3s_attention_fwd (training forward: + per-row (m, l)) on the bench workloads,
cold L2, CUDA events: python tools/fwd_vs_train.py [--configs batched arxiv reddit]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["batched", "arxiv", "reddit"])
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from f3s_inputs import configs
    from paper_2505_08098_b200 import f3s
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for cfg in a.configs:
        w = configs.get(cfg)
        csr = w.graph()
        Qb, Kb, Vb = w.qkv(csr)
        dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.float16)
        Q, K, V = dev(Qb), dev(Kb), dev(Vb)
        p = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
        O = torch.empty(Q.shape, dtype=torch.float32, device="cuda")
        ml = torch.empty((Q.shape[0], Q.shape[1], 2), dtype=torch.float32, device="cuda")
        calls = {"attention": lambda: f3s.attention(p, Q, K, V, O, scale=w.scale),
                 "attention_fwd": lambda: f3s.attention_fwd(p, Q, K, V, O, ml, scale=w.scale)}
        t = {k: [] for k in calls}
        for _ in range(2):
            for k, c in calls.items():
                for _ in range(a.reps):
                    flush.fill_(1)
                    ev[0].record()
                    c()
                    ev[1].record()
                    torch.cuda.synchronize()
                    t[k].append(ev[0].elapsed_time(ev[1]))
        print(cfg, " ".join(f"{k} {np.median(v):.4f} ms" for k, v in t.items()), flush=True)


if __name__ == "__main__":
    main()
