"""F3S_TRACE capture: run the fused kernel with per-chunk globaltimer stamps and dump them.

  python tools/trace.py --config batched --out gpurun_out/trace_batched.npz
Stamps per CTA and chunk: 0 ids requested, 1 gathers issued, 2 MMA1 issued, 3 S seen,
4 P written, 5 MMA2 issued, 6 O seen, 7 rows stored (last chunk of an item).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="arxiv")
    ap.add_argument("--variant", default="default")
    ap.add_argument("--chunks", type=int, default=8192)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import torch
    from f3s_inputs import configs
    from paper_2505_08098_b200 import f3s
    w = configs.get(a.config)
    csr = w.graph()
    Qb, Kb, Vb = w.qkv(csr)
    dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.float16)
    p = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
    Q, K, V = dev(Qb), dev(Kb), dev(Vb)
    O = torch.empty(Q.shape, dtype=torch.float32, device="cuda")
    for _ in range(3):
        f3s.attention(p, Q, K, V, O, scale=w.scale, variant=a.variant)
    tr = f3s.attention_trace(p, Q, K, V, O, scale=w.scale, trace_chunks=a.chunks, variant=a.variant)
    torch.cuda.synchronize()
    np.savez_compressed(a.out, trace=tr.cpu().numpy())
    print("saved", a.out, tr.shape)


if __name__ == "__main__":
    main()
