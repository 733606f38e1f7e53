"""Plan statistics of the synthetic workloads at 16x8 TCBs (Tab.datasets' metrics)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from f3s_inputs import configs

def stats(csr):
    p = oracle.plan(csr.row_ptr, csr.col_idx, csr.n_cols)
    t = p.tcb8.astype(np.float64)
    rows16 = np.minimum(np.arange(1, p.num_rw + 1) * 16, csr.n_rows)
    nnz_rw = csr.row_ptr[rows16] - csr.row_ptr[rows16 - np.minimum(16, rows16 - np.arange(p.num_rw) * 16)]
    m = t > 0
    npt = nnz_rw[m] / t[m]
    q = np.sort(t)
    dec = [int(q[max(0, int(len(q) * f) - 1)]) for f in (0.1, 0.5, 0.9, 1.0)]
    return dict(n=csr.n_rows, nnz=csr.nnz, R=p.num_rw, W=len(p.cols), tcb_rw=round(t.mean(), 1), tcb_cv=round(t.std() / t.mean(), 2),
                nnz_tcb=round(npt.mean(), 1), nnz_tcb_cv=round(npt.std() / npt.mean(), 2), deciles_10_50_90_max=dec)

for name in sys.argv[1:] or list(configs.WORKLOADS):
    print(name, stats(configs.get(name).graph()), flush=True)
