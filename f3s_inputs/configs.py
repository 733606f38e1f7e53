"""The five BASELINE.json workloads as seeded synthetic inputs (recipes: DESIGN.md §Input recipe).

Graph shapes follow the paper's datasets (Tab.datasets, deciles P:577) and
BASELINE.json's configs; values are splitmix64 streams on a 2^-23 grid in [-1, 1), RNE-rounded
to fp16 (Tab.mixedp).  seed_graph = 1000 + index, seed_t = (seed_graph << 8) | t.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import CSR, chung_lu, dcsbm, molecules, values, windows

# Tab.tcb_deciles, Reddit: min / decile boundaries / max of TCBs (16x8) per row window
REDDIT_DECILES = (4, 46, 88, 135, 190, 265, 367, 503, 718, 1113.5, 9857)
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _uniform(count: int, seed: int) -> np.ndarray:
    """u[i] in [0, 1): 53 bits of the i-th output of a splitmix64 stream started at `seed`."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.arange(count, dtype=np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def reddit_windows(n: int, seed: int, tail_alpha: float = 2.1, comm_size: int = 4500, mu: float = 0.8,
                   gamma: float = 2.1, ratio_mean: float = 9.3, ratio_sd: float = 28.0) -> CSR:
    """Reddit-shaped A built row window by row window (f3s_inputs.windows) from the paper's own
    statistics: TCB/RW deciles of Tab.tcb_deciles and nnz/TCB mean 16.5, CV 0.95
    (Tab.datasets).

    Window k gets t_k = Q(u_k), u_k = (rank_k + 0.5) / R with ranks a seeded permutation (every
    decile holds R/10 windows); Q is log-linear between the decile boundaries and, in the last
    decile, a Pareto(tail_alpha) truncated at the table's maximum (tail_alpha = 2.1 gives the
    table's mean 477).  Its nnz/TCB target is 8 + X (8 is the floor: one row per column), X
    lognormal with mean 9.3 and standard deviation 28, clipped to 128 (all 16 rows); after the
    clip and the per-column Poisson row counts the windows' nnz/TCB has the table's mean 16.5
    and CV 0.95 (calibrated with tools/calib_reddit.py, profiles/r02_graph_stats.txt)."""
    R = (n + 15) // 16
    rank = np.argsort(_uniform(R, seed ^ 0x77), kind="stable").argsort(kind="stable")
    u = (rank + 0.5) / R
    kn = np.log(np.asarray(REDDIT_DECILES, dtype=np.float64))
    i = np.minimum((u * 10).astype(np.int64), 9)
    f = u * 10 - i
    t = np.exp(kn[i] + f * (kn[np.minimum(i + 1, 10)] - kn[i]))
    lo, hi = REDDIT_DECILES[9], REDDIT_DECILES[10]
    tail = i == 9
    c = 1.0 - (lo / hi) ** tail_alpha
    t[tail] = lo * (1.0 - f[tail] * c) ** (-1.0 / tail_alpha)
    tcb = np.rint(t).astype(np.int32)
    mx, sx = ratio_mean, ratio_sd
    sig2 = np.log1p((sx / mx) ** 2)
    u1, u2 = _uniform(R, seed ^ 0x99), _uniform(R, seed ^ 0xAA)
    z = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)  # Box-Muller
    ratio = np.minimum(8.0 + np.exp(np.log(mx) - sig2 / 2 + np.sqrt(sig2) * z), 128.0)
    return windows(n, tcb, ratio, comm_size=comm_size, mu=mu, gamma=gamma, seed=seed)


@dataclass
class Workload:
    name: str
    index: int
    H: int
    d: int
    make: Callable[[int], CSR] = field(repr=False)
    dtype: str = "fp16"
    description: str = ""

    @property
    def seed_graph(self) -> int:
        return 1000 + self.index

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.d)

    def graph(self) -> CSR:
        return self.make(self.seed_graph)

    def qkv(self, csr: CSR, dtype: str | None = None):
        dt = dtype or self.dtype
        s = self.seed_graph
        Q = values((csr.n_rows, self.H, self.d), seed=(s << 8) | 1, dtype=dt)
        K = values((csr.n_cols, self.H, self.d), seed=(s << 8) | 2, dtype=dt)
        V = values((csr.n_cols, self.H, self.d), seed=(s << 8) | 3, dtype=dt)
        return Q, K, V

    def qkv_rows(self, rows: np.ndarray, which: int, n: int, dtype: str | None = None) -> np.ndarray:
        """Regenerate only the listed rows of tensor `which` (1=Q, 2=K, 3=V): element (r, h, k) is
        element r*H*d + h*d + k of the stream, so any row can be produced alone."""
        dt = dtype or self.dtype
        s = self.seed_graph
        hd = self.H * self.d
        out = np.empty((len(rows), self.H, self.d), np.uint16)
        for i, r in enumerate(rows):
            out[i] = values((self.H, self.d), seed=(s << 8) | which, dtype=dt, offset=int(r) * hd)
        return out


WORKLOADS = {
    "cora": Workload(
        "cora", 0, 1, 64,
        lambda s: chung_lu(2708, 5278, gamma=2.7, max_deg=170, symmetrize=True, self_loops=True, permute=True, seed=s),
        description="Cora-shaped: 2,708 nodes, 5,278 undirected pairs -> 10,556 directed + 2,708 self-loops; d=64, 1 head"),
    "arxiv": Workload(
        "arxiv", 1, 8, 128,
        lambda s: chung_lu(169343, 1166243, directed=True, gamma=2.6, max_deg=500, gamma_in=2.1, max_deg_in=13000,
                           symmetrize=False, self_loops=False, permute=True, seed=s),
        description="ogbn-arxiv-shaped: 169,343 nodes, 1,166,243 directed edges (power-law in/out); d=128, 8 heads"),
    "products": Workload(
        "products", 2, 4, 64,
        lambda s: chung_lu(2449029, 61859140, gamma=2.3, max_deg=17481, symmetrize=True, permute=True, seed=s),
        description="ogbn-products-shaped: 2,449,029 nodes, 61,859,140 undirected pairs -> 123.7M nnz; d=64, 4 heads"),
    "reddit": Workload(
        "reddit", 3, 1, 64,
        lambda s: reddit_windows(232965, seed=s),
        description="Reddit-shaped: 232,965 nodes, ~115M nnz, row windows with the paper's TCB/RW deciles "
                    "(4..9857 TCBs, mean 477) and nnz/TCB 16.5; d=64, 1 head"),
    "batched": Workload(
        "batched", 4, 8, 64,
        lambda s: molecules(10000, 25, 150, self_loops=False, seed=s),
        description="10,000 molecule-like graphs (25-150 nodes) in one block-diagonal plan; d=64, 8 heads"),
}


def get(name: str) -> Workload:
    return WORKLOADS[name]
