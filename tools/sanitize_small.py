"""Small fused calls for compute-sanitizer runs (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import f3s_inputs as fi
from paper_2505_08098_b200 import f3s
for (n, H, d, seed) in [(200, 1, 64, 1), (100, 4, 64, 2), (150, 2, 128, 3)]:
    csr = fi.random_csr(n, n, 0, 150, seed=seed) if H != 4 else fi.molecules(6, 10, 30, seed=seed)
    rp = torch.from_numpy(csr.row_ptr).cuda(); ci = torch.from_numpy(csr.col_idx).cuda()
    p = f3s.plan(rp, ci, csr.n_rows)
    Q = torch.randn(csr.n_rows, H, d, device="cuda").half(); K = torch.randn_like(Q); V = torch.randn_like(Q)
    O = f3s.attention(p, Q, K, V, scale=0.125)
    dO = torch.randn(Q.shape, device="cuda")
    f3s.attention_backward(p, Q, K, V, dO, scale=0.125)
    torch.cuda.synchronize()
    print("ok", n, H, d, float(O.abs().sum()))
# E4M3 inputs (f4), d = 128 and 64, forward only
for (n, H, d, seed) in [(150, 2, 128, 4), (120, 3, 64, 5)]:
    csr = fi.random_csr(n, n, 0, 150, seed=seed)
    rp = torch.from_numpy(csr.row_ptr).cuda(); ci = torch.from_numpy(csr.col_idx).cuda()
    p = f3s.plan(rp, ci, csr.n_rows)
    Q, K, V = (torch.randn(csr.n_rows, H, d, device="cuda").to(torch.float8_e4m3fn) for _ in range(3))
    O = f3s.attention(p, Q, K, V, scale=0.125)
    torch.cuda.synchronize()
    print("ok e4m3", n, H, d, float(O.abs().sum()))
