"""Per-call times of the backward (diagnostics): python tools/bwd_percall.py CONFIG [N]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from f3s_inputs import configs
from paper_2505_08098_b200 import f3s
w = configs.get(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
csr = w.graph(); Qb, Kb, Vb = w.qkv(csr)
dev = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.float16)
p = f3s.plan(torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx).cuda(), csr.n_rows)
Q, K, V = dev(Qb), dev(Kb), dev(Vb)
dO = torch.randn(Q.shape, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n)]
for i in range(n):
    ev[2 * i].record(); f3s.attention_backward(p, Q, K, V, dO, scale=w.scale); ev[2 * i + 1].record()
torch.cuda.synchronize()
print(sys.argv[1], "back-to-back", [round(ev[2 * i].elapsed_time(ev[2 * i + 1]), 3) for i in range(n)])
t = []
for i in range(n):
    torch.cuda.synchronize(); ev[0].record(); f3s.attention_backward(p, Q, K, V, dO, scale=w.scale); ev[1].record(); torch.cuda.synchronize()
    t.append(round(ev[0].elapsed_time(ev[1]), 3))
print(sys.argv[1], "synced", t)
