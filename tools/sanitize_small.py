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
# round 2: split pieces, per-window head groups (wide head + narrow tail), partial mode with head
# groups, tensor-core and CUDA-core backward, bf16
mol = fi.molecules(8, 25, 60, seed=7)
wide = fi.random_csr(32, mol.n_rows, 60, 200, seed=7)
rp_h = np.concatenate([mol.row_ptr, mol.row_ptr[-1] + wide.row_ptr[1:]]).astype(np.int32)
ci_h = np.concatenate([mol.col_idx, wide.col_idx]).astype(np.int32)
n = mol.n_rows + 32
p = f3s.plan(torch.from_numpy(rp_h).cuda(), torch.from_numpy(ci_h).cuda(), n)
p.set_split(1)
for dt in (torch.float16, torch.bfloat16):
    Q = torch.randn(n, 4, 64, device="cuda").to(dt); K = torch.randn_like(Q); V = torch.randn_like(Q)
    O = f3s.attention(p, Q, K, V, scale=0.125)
    Op = torch.empty(Q.shape, device="cuda"); ml = torch.empty((n, 4, 2), device="cuda")
    f3s.attention_partial_raw(p, Q.data_ptr(), K.data_ptr(), V.data_ptr(), 0, Op.data_ptr(), ml.data_ptr(), 0.125, 4, 64,
                              f3s.FP16 if dt == torch.float16 else f3s.BF16, 0, torch.cuda.current_stream().cuda_stream)
    dO = torch.randn(Q.shape, device="cuda")
    f3s.attention_backward(p, Q, K, V, dO, scale=0.125, variant="tc")
    f3s.attention_backward(p, Q, K, V, dO, scale=0.125, variant="simt")
    torch.cuda.synchronize()
    print("ok mixed/split/partial/backward", dt, float(O.abs().sum()))
# round 2, later: the training pair (f3s_attention_fwd + f3s_attention_backward_saved) on the
# mixed/split plan, a head-group plan and d = 128
for (pl, nn, H, d) in [(p, n, 4, 64), (None, 0, 8, 64), (None, 0, 2, 128)]:
    if pl is None:
        g = fi.molecules(10, 20, 40, seed=H + d) if H == 8 else fi.random_csr(300, 300, 0, 200, seed=d)
        pl, nn = f3s.plan(torch.from_numpy(g.row_ptr).cuda(), torch.from_numpy(g.col_idx).cuda(), g.n_rows), g.n_rows
    Q = torch.randn(nn, H, d, device="cuda").half(); K = torch.randn_like(Q); V = torch.randn_like(Q)
    O, ml = f3s.attention_fwd(pl, Q, K, V, scale=0.125)
    dO = torch.randn(Q.shape, device="cuda")
    dQ, dK, dV = f3s.attention_backward_saved(pl, Q, K, V, O, ml, dO, scale=0.125)
    torch.cuda.synchronize()
    print("ok fwd+saved backward", nn, H, d, float(dQ.abs().sum() + dK.abs().sum() + dV.abs().sum()))
