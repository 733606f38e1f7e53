"""Calibrate the Reddit-shaped generator against Tab.datasets (TCB/RW 477.2, CV 1.35;
nnz/TCB 16.5, CV 0.95) and Tab.tcb_deciles.  Prints the plan statistics of one setting.

  python tools/calib_reddit.py COMM MU GAMMA TAIL_ALPHA
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from f3s_inputs import configs  # noqa: E402


def window_stats(csr):
    n = csr.n_rows
    R = (n + 15) // 16
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(csr.row_ptr))
    keys = (rows // 16) << 32 | csr.col_idx.astype(np.int64)
    u = np.unique(keys)
    w = np.bincount((u >> 32).astype(np.int64), minlength=R).astype(np.float64)
    t = np.ceil(w / 8)
    nnz_rw = np.bincount(rows // 16, minlength=R).astype(np.float64)
    m = t > 0
    npt = nnz_rw[m] / t[m]
    q = np.sort(t)
    dec = [int(q[min(len(q) - 1, int(len(q) * f / 10))]) for f in range(0, 11)]
    return dict(nnz=csr.nnz, W=int(w.sum()), tcb_rw=round(t.mean(), 1), tcb_cv=round(t.std() / t.mean(), 2),
                nnz_tcb=round(npt.mean(), 1), nnz_tcb_cv=round(npt.std() / npt.mean(), 2), deciles=dec)


if __name__ == "__main__":
    comm, mu, gamma, alpha = int(sys.argv[1]), float(sys.argv[2]), float(sys.argv[3]), float(sys.argv[4])
    t0 = time.time()
    sd = float(sys.argv[5]) if len(sys.argv) > 5 else 15.7
    mx = float(sys.argv[6]) if len(sys.argv) > 6 else 8.5
    csr = configs.reddit_windows(232965, seed=1003, tail_alpha=alpha, comm_size=comm, mu=mu, gamma=gamma, ratio_mean=mx, ratio_sd=sd)
    print(sys.argv[1:], window_stats(csr), f"{time.time() - t0:.0f}s", flush=True)
