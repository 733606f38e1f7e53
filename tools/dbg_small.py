import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import f3s_inputs as fi
from helpers import make_qkv, to_dev, csr_to_dev
from paper_2505_08098_b200 import f3s
d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
csr = fi.random_csr(200, 200, 0, 40, seed=3)
Qb, Kb, Vb = make_qkv(200, 200, 2, d, "fp16", seed=1)
rp, ci = csr_to_dev(csr)
p = f3s.plan(rp, ci, 200)
O = f3s.attention(p, to_dev(Qb, "fp16"), to_dev(Kb, "fp16"), to_dev(Vb, "fp16"), scale=0.1)
torch.cuda.synchronize()
print("ok", d, float(O.abs().sum()))
