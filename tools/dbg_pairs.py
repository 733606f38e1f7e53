import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import f3s_inputs as fi
import oracle
from paper_2505_08098_b200 import f3s
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import make_qkv, to_dev, csr_to_dev
for (n, degmax, H, d) in [(4000, 40, 2, 64), (4000, 400, 1, 64), (20000, 6, 8, 128)]:
    csr = fi.random_csr(n, n, 0, degmax, seed=3)
    Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=5)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, n)
    O = f3s.attention(p, to_dev(Qb, "fp16"), to_dev(Kb, "fp16"), to_dev(Vb, "fp16"), scale=0.125).cpu().numpy()
    O2 = f3s.attention(p, to_dev(Qb, "fp16"), to_dev(Kb, "fp16"), to_dev(Vb, "fp16"), scale=0.125).cpu().numpy()
    ref = oracle.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.125)
    err = np.abs(O - ref).max(axis=(1, 2))
    bad = np.where(err > 1e-2)[0]
    rw = np.unique(bad // 16)
    print(n, degmax, H, d, "bad rows", len(bad), "bad windows", len(rw), rw[:10], "det", np.array_equal(O, O2), "max", err.max())
    order = p.export()[3]
    pos = np.argsort(order)
    print("   LPT positions of bad windows:", pos[rw][:10], "widths", np.diff(p.export()[0])[rw][:10])
