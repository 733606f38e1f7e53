"""Multi-GPU driver (one process per GPU, torch.distributed/NCCL for the plumbing).

Row windows are independent (node-parallel fusion), so the path shards by
rows: rank g owns the contiguous rows [bounds[g], bounds[g+1]) cut at multiples of 16 and
balanced by nnz (f3s_partition_rows), builds its plan with f3s_plan_rows over global column
ids, and holds Q/O for its rows.  K and V are produced as equal row shards and replicated by
one NCCL all-gather each over NVLink (the only exchange step).  Because
every window of a shard equals the corresponding window of the global plan, each rank's O rows
are bitwise identical to the 1-GPU result.

Batched mode: whole graphs per rank (cuts only at graph starts,
f3s_partition_at); each rank owns the K/V of its own graphs, so there is no collective.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import f3s


@dataclass
class Shard:
    rank: int
    world: int
    bounds: np.ndarray   # int32[world+1] row boundaries
    row_begin: int
    row_end: int
    n_cols: int
    shard_rows: int      # rows per K/V all-gather shard (ceil(n_cols / world))
    plan: f3s.Plan | None = None
    col_offset: int = 0  # batched mode: first global column owned by this rank


def partition(row_ptr: np.ndarray, world: int, graph_ptr: np.ndarray | None = None) -> np.ndarray:
    if graph_ptr is not None:
        return f3s.partition_at(row_ptr, graph_ptr, world)
    return f3s.partition_rows(row_ptr, world)


def make_shard(row_ptr: np.ndarray, col_idx: np.ndarray, rank: int, world: int, *, device=None,
               graph_ptr: np.ndarray | None = None) -> Shard:
    """Partition (host), then build this rank's plan on its device from its CSR slice."""
    import torch
    n = len(row_ptr) - 1
    bounds = partition(row_ptr, world, graph_ptr)
    b, e = int(bounds[rank]), int(bounds[rank + 1])
    dev = device or torch.device("cuda", torch.cuda.current_device())
    lo, hi = int(row_ptr[b]), int(row_ptr[e])
    rp = torch.from_numpy((row_ptr[b:e + 1] - lo).astype(np.int32)).to(dev)
    ci_host = col_idx[lo:hi]
    if graph_ptr is not None:
        # batched: local column ids, K/V of the own graphs only (no collective)
        ci = torch.from_numpy((ci_host - b).astype(np.int32) if hi > lo else np.zeros(1, np.int32)).to(dev)
        plan = f3s.plan_rows(rp, ci, e - b, e - b)
        return Shard(rank, world, bounds, b, e, e - b, e - b, plan, col_offset=b)
    ci = torch.from_numpy(ci_host.astype(np.int32) if hi > lo else np.zeros(1, np.int32)).to(dev)
    plan = f3s.plan_rows(rp, ci, e - b, n)
    return Shard(rank, world, bounds, b, e, n, -(-n // world), plan)


def allgather_kv(K_shard, V_shard, K_full, V_full, group=None) -> None:
    """K_full/V_full [world*shard_rows, H, d] <- concatenation of every rank's shard (NCCL)."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(K_full, K_shard, group=group)
    dist.all_gather_into_tensor(V_full, V_shard, group=group)


def attention(shard: Shard, Q_local, K_full, V_full, O_local=None, *, scale: float, stream=None, variant="default"):
    """Local fused pass over this rank's rows against the replicated K/V."""
    if shard.row_end == shard.row_begin:
        return O_local
    return f3s.attention(shard.plan, Q_local, K_full, V_full, O_local, scale=scale, stream=stream, variant=variant)
