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

from . import CSR, chung_lu, dcsbm, molecules, values


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
        lambda s: dcsbm(232965, 57_459_000, comm_size=4500, mu=0.9, gamma=2.1, max_deg=21657, seed=s),
        description="Reddit-shaped DC-SBM: 232,965 nodes, ~114.9M nnz, contiguous communities; d=64, 1 head"),
    "batched": Workload(
        "batched", 4, 8, 64,
        lambda s: molecules(10000, 25, 150, self_loops=False, seed=s),
        description="10,000 molecule-like graphs (25-150 nodes) in one block-diagonal plan; d=64, 8 heads"),
}


def get(name: str) -> Workload:
    return WORKLOADS[name]
