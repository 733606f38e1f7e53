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


# ---- f2: K/V exchange overlapped with compute ------------------------------
def column_block_csr(spec: ShardSpec, parts: int) -> list:
    """The rank's local CSR split by K/V source block: block r holds the entries whose (global)
    column lies in [r*S, (r+1)*S), S = spec.kv_rows.  Host only; global column ids are kept."""
    rp, ci = spec.row_ptr, spec.col_idx
    n_loc = len(rp) - 1
    rows = np.repeat(np.arange(n_loc, dtype=np.int64), np.diff(rp))
    owner = ci // max(spec.kv_rows, 1)
    out = []
    for r in range(parts):
        sel = owner == r
        cnt = np.bincount(rows[sel], minlength=n_loc)
        out.append((np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32), np.ascontiguousarray(ci[sel], np.int32)))
    return out


def ring_schedule(rank: int, world: int) -> list:
    """Round t = 1 .. world-1 of the ring exchange: (send to, receive from) = (rank+t, rank-t).
    After round t this rank holds block (rank - t) % world; its own block needs no transfer."""
    return [((rank + t) % world, (rank - t) % world) for t in range(1, world)]


def ring_exchange(KV_full, S: int, rank: int, world: int, group=None, on_block=None) -> None:
    """Replicate every rank's [K||V] shard (rows [r*S, (r+1)*S) of KV_full) with world-1 rounds of
    paired send/recv; on_block(r) is called (on the current stream) as soon as block r is present,
    own block first.  NCCL moves device tensors; gloo (CPU test rigs) moves host copies."""
    import torch
    import torch.distributed as dist
    if on_block is not None:
        on_block(rank)
    via_host = KV_full.is_cuda and dist.get_backend(group) == "gloo"
    tv = torch.float16 if KV_full.element_size() == 2 else torch.uint8
    for dst, src in ring_schedule(rank, world):
        send = KV_full[rank * S:(rank + 1) * S]
        recv = KV_full[src * S:(src + 1) * S]
        if via_host:
            hs, hr = send.view(tv).cpu(), torch.empty(recv.shape, dtype=tv)
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, hs, dst, group), dist.P2POp(dist.irecv, hr, src, group)])
            for q in reqs:
                q.wait()
            recv.view(tv).copy_(hr)
        else:
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, send, dst, group),
                                           dist.P2POp(dist.irecv, recv, src, group)])
            for q in reqs:
                q.wait()
        if on_block is not None:
            on_block(src)


class OverlappedShard:
    """One rank of the overlapped multi-GPU pass: the K/V blocks arrive over a side stream in ring
    order while f3s_attention_partial runs on the blocks already present (own block first, with
    `reserve_sms` SMs left to the transfers until the last block), then f3s_attention_merge
    combines the block partials in block order (deterministic; tolerance-equal to the one-GPU
    result, not bitwise: the blocks change where the online softmax rescales)."""

    def __init__(self, spec: ShardSpec, heads: int, d: int, dtype, *, device=None, reserve_sms: int = 16,
                 group=None):
        import torch

        from . import f3s
        assert not spec.batched, "batched mode has no exchange"
        self.spec, self.H, self.d, self.group = spec, heads, d, group
        self.world, self.rank = spec.world, spec.rank
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.tdt = dtype
        self.code = {torch.float16: f3s.FP16, torch.bfloat16: f3s.BF16, torch.float8_e4m3fn: f3s.E4M3}[dtype]
        n_loc = spec.row_end - spec.row_begin
        self.n_loc = n_loc
        self.plans = []
        for rp, ci in column_block_csr(spec, self.world):
            self.plans.append(f3s.plan_rows(torch.from_numpy(rp).to(self.dev),
                                            torch.from_numpy(ci if len(ci) else np.zeros(1, np.int32)).to(self.dev),
                                            n_loc, spec.n_cols))
        S = spec.kv_rows
        self.KV = torch.empty((self.world * S, 2, heads, d), dtype=dtype, device=self.dev)
        self.Op = torch.empty((self.world, max(n_loc, 1), heads, d), dtype=torch.float32, device=self.dev)
        self.mlp = torch.empty((self.world, max(n_loc, 1), heads, 2), dtype=torch.float32, device=self.dev)
        self.comm = torch.cuda.Stream(device=self.dev)
        sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.cap = max(1, sms - reserve_sms) if self.world > 1 else 0

    def own_block(self):
        """The rows of KV this rank fills before run() (its padded [K||V] shard)."""
        S = self.spec.kv_rows
        return self.KV[self.rank * S:(self.rank + 1) * S]

    def run(self, Q, O, scale: float) -> None:
        import torch

        from . import f3s
        comp = torch.cuda.current_stream(self.dev)
        es = self.KV.element_size()
        kv = self.KV.data_ptr()
        H, d = self.H, self.d
        arrived = []

        def partial(r, cap):
            if self.n_loc == 0:
                return
            f3s.attention_partial_raw(self.plans[r], Q.data_ptr(), kv, kv + H * d * es, 2 * H * d,
                                      self.Op[r].data_ptr(), self.mlp[r].data_ptr(), scale, H, d, self.code, cap,
                                      comp.cuda_stream)

        events = {}

        def on_block(r):  # block r is present once the comm stream reaches this point
            if r == self.rank:
                return
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.dev))
            events[r] = ev
            arrived.append(r)

        self.comm.wait_stream(comp)          # the own shard (uploaded on comp) is in place
        partial(self.rank, self.cap)         # own block first: no transfer needed
        with torch.cuda.stream(self.comm):
            ring_exchange(self.KV, self.spec.kv_rows, self.rank, self.world, self.group, on_block)
        for i, r in enumerate(arrived):
            comp.wait_event(events[r])
            partial(r, self.cap if i < len(arrived) - 1 else 0)
        if self.n_loc:
            f3s.attention_merge(self.Op, self.mlp, O, stream=comp)
