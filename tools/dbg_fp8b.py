"""e4m3 debug: one-neighbour rows, a single CTA (grid = 1): which work items come out right."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_08098_b200 import f3s
import oracle

n, H, d = 512, 1, 128
rng = np.random.default_rng(1)
rp = np.arange(n + 1, dtype=np.int32)
ci = rng.permutation(n).astype(np.int32)
def e4(x):
    t = torch.from_numpy(x.astype(np.float32)).to(torch.float8_e4m3fn)
    return t.cuda(), t.to(torch.float64).numpy()
(Q, q), (K, k), (V, v) = (e4(rng.uniform(-1, 1, (n, H, d))) for _ in range(3))
p = f3s.plan(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), n)
ref = oracle.attention_f64(rp, ci, q, k, v, scale=0.1)
for grid in (1, 2, 0):
    for variant in ("default", "no_reorder"):
        O = torch.zeros((n, H, d), dtype=torch.float32, device="cuda")
        f3s.attention_trace(p, Q, K, V, O, scale=0.1, trace_chunks=64, grid=grid, variant=variant)
        torch.cuda.synchronize()
        Oc = O.cpu().numpy()
        okw = (np.abs(Oc - ref).max(axis=(1, 2)) < 1e-6).reshape(-1, 16).all(axis=1)
        zw = (np.abs(Oc).max(axis=(1, 2)) == 0).reshape(-1, 16).all(axis=1)
        print(grid, variant, "ok windows", "".join("1" if x else "0" for x in okw), " zero windows", "".join("1" if x else "0" for x in zw), flush=True)
# Q = 0 and V = 1 single CTA: O must be 1
Qz = torch.zeros_like(Q); V1 = torch.ones((n, H, d)).to(torch.float8_e4m3fn).cuda()
O = torch.zeros((n, H, d), dtype=torch.float32, device="cuda")
f3s.attention_trace(p, Qz, K, V1, O, scale=0.1, trace_chunks=64, grid=1)
torch.cuda.synchronize()
print("Q=0,V=1 rows equal to 1:", int((O.cpu().numpy() == 1).all(axis=(1, 2)).sum()), "zero rows", int((O.cpu().numpy() == 0).all(axis=(1, 2)).sum()))
print("O sample", O[16, 0, :4].tolist(), O[0, 0, :4].tolist())
