"""Multi-GPU driver (one process per GPU, torch.distributed/NCCL for the plumbing).

Row windows are independent (node-parallel fusion), so the path shards by
rows: rank g owns the contiguous rows [bounds[g], bounds[g+1]) cut at multiples of 16 and
balanced by nnz (f3s_partition_rows), builds its plan with f3s_plan_rows over global column
ids, and holds Q/O for its rows.  K and V are produced as equal row shards of
S = ceil(n / world) rows and replicated by one NCCL all-gather each over NVLink (the only
exchange step).  Every window of a shard equals the corresponding window
of the global plan and is split (f1) by the global problem's bound, so each rank's O rows are
bitwise identical to the 1-GPU result.

Batched mode: whole graphs per rank (cuts only at graph starts,
f3s_partition_at); each rank owns the K/V rows of its own graphs, so there is no collective.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ShardSpec:
    """Host-side description of one rank's part of the problem (no device state)."""
    rank: int
    world: int
    bounds: np.ndarray    # int32[world+1] row boundaries (multiples of 16, or graph starts)
    row_begin: int
    row_end: int
    n_cols: int           # columns of the local A (global n, or own graph rows in batched mode)
    kv_rows: int          # K/V rows this rank contributes: all-gather shard size, or own rows (batched)
    kv_begin: int         # first global K/V row of this rank's contribution
    row_ptr: np.ndarray   # int32[local rows + 1], starting at 0
    col_idx: np.ndarray   # int32[local nnz], global ids (or local ids in batched mode)
    batched: bool


def partition(row_ptr: np.ndarray, world: int, graph_ptr: np.ndarray | None = None) -> np.ndarray:
    from . import f3s
    if graph_ptr is not None:
        return f3s.partition_at(row_ptr, graph_ptr, world)
    return f3s.partition_rows(row_ptr, world)


def shard_spec(row_ptr: np.ndarray, col_idx: np.ndarray, rank: int, world: int,
               graph_ptr: np.ndarray | None = None, bounds: np.ndarray | None = None) -> ShardSpec:
    """Slice the global CSR for `rank` (host only)."""
    n = len(row_ptr) - 1
    if bounds is None:
        bounds = partition(row_ptr, world, graph_ptr)
    b, e = int(bounds[rank]), int(bounds[rank + 1])
    lo, hi = int(row_ptr[b]), int(row_ptr[e])
    rp = (row_ptr[b:e + 1] - lo).astype(np.int32)
    ci = np.ascontiguousarray(col_idx[lo:hi], dtype=np.int32)
    if graph_ptr is not None:
        # batched: a rank's graphs only reference their own rows -> local column ids
        if len(ci) and (ci.min() < b or ci.max() >= e):
            raise ValueError("batched sharding needs a block-diagonal A cut at graph boundaries")
        return ShardSpec(rank, world, bounds, b, e, e - b, e - b, b, rp, (ci - b).astype(np.int32), True)
    S = -(-n // world) if n else 0
    return ShardSpec(rank, world, bounds, b, e, n, S, min(rank * S, n), rp, ci, False)


def kv_slice(spec: ShardSpec, n: int) -> tuple[int, int]:
    """Global K/V rows [lo, hi) this rank holds before the all-gather (padded to kv_rows)."""
    lo = spec.kv_begin
    hi = min(lo + spec.kv_rows, n) if not spec.batched else spec.row_end
    return lo, hi


def kv_shard(spec: ShardSpec, K: np.ndarray, V: np.ndarray, n: int) -> np.ndarray:
    """This rank's padded [K||V] shard [S, 2, H, d] (host): rows kv_slice(spec) of K and V,
    interleaved per row so that one all-gather replicates both (zero rows past n)."""
    lo, hi = kv_slice(spec, n)
    out = np.zeros((spec.kv_rows, 2) + tuple(K.shape[1:]), dtype=K.dtype)
    out[:hi - lo, 0] = K[lo:hi]
    out[:hi - lo, 1] = V[lo:hi]
    return out


def allgather_kv_into(KV_full, KV_shard, group=None) -> None:
    """KV_full [world*S, 2, H, d] <- every rank's padded [K||V] shard in rank order: ONE collective
    (NCCL over NVLink on GPUs, gloo on CPU).  K = KV_full[:, 0] and V = KV_full[:, 1] are then
    rows of stride 2*H*d, which f3s_attention_kv reads directly."""
    import torch
    import torch.distributed as dist
    if KV_full.is_cuda and dist.get_backend(group) == "gloo":
        # gloo (CPU test rigs: several ranks on one GPU) moves host tensors; 16-bit data as fp16
        tv = torch.float16 if KV_full.element_size() == 2 else torch.uint8
        host = torch.empty(KV_full.shape, dtype=tv)
        dist.all_gather_into_tensor(host, KV_shard.view(tv).cpu(), group=group)
        KV_full.view(tv).copy_(host)
        return
    dist.all_gather_into_tensor(KV_full, KV_shard, group=group)


def allgather_kv(K_shard, V_shard, K_full, V_full, group=None) -> None:
    """Separate-tensor form (two collectives): K_full/V_full [world*S, H, d] <- every rank's shard."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(K_full, K_shard, group=group)
    dist.all_gather_into_tensor(V_full, V_shard, group=group)


@dataclass
class Shard:
    spec: ShardSpec
    plan: object  # f3s.Plan


def global_chunk_count(local_chunks: int, group=None, device=None) -> int:
    """Sum of every rank's plan chunk count (the single-GPU plan's count: shards are cut at
    row-window boundaries, so every window belongs to exactly one shard)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("global_chunk_count needs an initialised process group (or pass global_chunks)")
    on_gpu = dist.get_backend(group) == "nccl"
    t = torch.tensor([int(local_chunks)], dtype=torch.int64, device=device if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def make_shard(row_ptr: np.ndarray, col_idx: np.ndarray, rank: int, world: int, *, device=None,
               graph_ptr: np.ndarray | None = None, group=None, global_chunks: int | None = None) -> Shard:
    """Partition on the host, then build this rank's plan (f3s_plan_rows) on its device.

    Row shards of one graph take the heavy-window split bound of the GLOBAL problem
    (f3s_default_split_chunks over the summed chunk counts, all-reduced over `group` unless
    `global_chunks` is given), so every window is split exactly as in the single-GPU plan and the
    shard's O rows stay bitwise equal to the single-GPU call (f3s.h, f3s_plan_set_split).
    Batched mode (whole graphs per rank) is a different problem per rank and keeps its own bound."""
    import torch

    from . import f3s
    spec = shard_spec(row_ptr, col_idx, rank, world, graph_ptr)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    rp = torch.from_numpy(spec.row_ptr).to(dev)
    ci = torch.from_numpy(spec.col_idx if len(spec.col_idx) else np.zeros(1, np.int32)).to(dev)
    plan = f3s.plan_rows(rp, ci, spec.row_end - spec.row_begin, spec.n_cols)
    if graph_ptr is None and world > 1:
        total = global_chunks if global_chunks is not None else \
            global_chunk_count(plan.info()["total_chunks"], group, dev)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        plan.set_split(f3s.default_split_chunks(total, sms))
    return Shard(spec, plan)


def attention_kv(shard: Shard, Q_local, KV_full, O_local=None, *, scale: float, stream=None):
    """Local fused pass over this rank's rows against the all-gathered [K||V] buffer."""
    from . import f3s
    if shard.spec.row_end == shard.spec.row_begin:
        return O_local
    return f3s.attention_kv(shard.plan, Q_local, KV_full, O_local, scale=scale, stream=stream)


def attention(shard: Shard, Q_local, K_full, V_full, O_local=None, *, scale: float, stream=None, variant="default"):
    """Local fused pass over this rank's rows against the replicated (or own, batched) K/V."""
    from . import f3s
    if shard.spec.row_end == shard.spec.row_begin:
        return O_local
    return f3s.attention(shard.plan, Q_local, K_full, V_full, O_local, scale=scale, stream=stream, variant=variant)
