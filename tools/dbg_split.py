"""Debug helper: time a fused call on a config-shaped graph, report errors and timing."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import f3s_inputs as fi
from paper_2505_08098_b200 import f3s
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
csr = fi.random_csr(n, n, 1, 40, seed=1)
rp = torch.from_numpy(csr.row_ptr).cuda(); ci = torch.from_numpy(csr.col_idx).cuda()
p = f3s.plan(rp, ci, csr.n_rows)
print({k: v for k, v in p.info().items() if k in ("num_rw", "split_chunks", "split_groups")}, flush=True)
H, d = 2, 64
Q = torch.randn(csr.n_rows, H, d, device="cuda").half(); K = Q.clone(); V = Q.clone()
t0 = time.time()
try:
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
        O = f3s.attention(p, Q, K, V, scale=0.125, variant=os.environ.get('VAR', 'default'))
        torch.cuda.synchronize()
    print("ok", n, time.time() - t0, flush=True)
except Exception as e:
    print("FAIL", n, time.time() - t0, str(e)[:100], flush=True)
