"""Multi-GPU orchestration (paper_2505_08098_b200.dist): host-side sharding, K/V all-gather layout
over a world_size-2 gloo process group on CPU, and (GPU) bitwise equality of row-sharded results
with the single-GPU call."""
import os
import socket

import numpy as np
import pytest

import f3s_inputs as fi
from helpers import make_qkv


@pytest.fixture(scope="module")
def dist_mod():
    from paper_2505_08098_b200 import build
    build()
    from paper_2505_08098_b200 import dist
    return dist


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_specs_cover_rows(dist_mod, world):
    g = fi.chung_lu(5000, 30000, gamma=2.3, max_deg=800, seed=5)
    specs = [dist_mod.shard_spec(g.row_ptr, g.col_idx, r, world) for r in range(world)]
    assert specs[0].row_begin == 0 and specs[-1].row_end == g.n_rows
    for a, b in zip(specs, specs[1:]):
        assert a.row_end == b.row_begin
    for s in specs:
        assert s.row_begin % 16 == 0
        # the local CSR is exactly the global rows
        for r in range(s.row_begin, s.row_end, 97):
            lr = r - s.row_begin
            assert np.array_equal(s.col_idx[s.row_ptr[lr]:s.row_ptr[lr + 1]], g.col_idx[g.row_ptr[r]:g.row_ptr[r + 1]])
        lo, hi = dist_mod.kv_slice(s, g.n_rows)
        assert hi - lo <= s.kv_rows
    # K/V shards tile [0, n) in rank order
    assert sum(min(s.kv_rows, max(0, g.n_rows - s.kv_begin)) for s in specs) == g.n_rows


def test_batched_specs_are_graph_aligned(dist_mod):
    g = fi.molecules(400, seed=7)
    for world in (2, 4):
        specs = [dist_mod.shard_spec(g.row_ptr, g.col_idx, r, world, g.graph_ptr) for r in range(world)]
        for s in specs:
            assert s.row_begin in set(g.graph_ptr.tolist())
            assert len(s.col_idx) == 0 or (s.col_idx.min() >= 0 and s.col_idx.max() < s.n_cols)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist

    import oracle
    from paper_2505_08098_b200 import dist as f3sdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = fi.chung_lu(3000, 15000, gamma=2.4, max_deg=500, seed=11)
        n, H, d = g.n_rows, 2, 64
        Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=11)
        spec = f3sdist.shard_spec(g.row_ptr, g.col_idx, rank, world)
        lo, hi = f3sdist.kv_slice(spec, n)
        S = spec.kv_rows
        f16 = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.float16))
        Ks = torch.zeros((S, H, d), dtype=torch.float16)
        Vs = torch.zeros((S, H, d), dtype=torch.float16)
        Ks[:hi - lo] = f16(Kb[lo:hi])
        Vs[:hi - lo] = f16(Vb[lo:hi])
        Kf = torch.empty((world * S, H, d), dtype=torch.float16)
        Vf = torch.empty((world * S, H, d), dtype=torch.float16)
        f3sdist.allgather_kv(Ks, Vs, Kf, Vf)
        Kfull = Kf.numpy().view(np.uint16)[:n]
        Vfull = Vf.numpy().view(np.uint16)[:n]
        ok_kv = bool(np.array_equal(Kfull, Kb) and np.array_equal(Vfull, Vb))
        # the rank's rows, computed from its local CSR and the gathered K/V, equal the global rows
        O_loc = oracle.attention(spec.row_ptr, spec.col_idx, Qb[spec.row_begin:spec.row_end], Kfull, Vfull,
                                 scale=0.125, n_cols=n)
        O_ref = oracle.attention(g.row_ptr, g.col_idx, Qb, Kb, Vb, scale=0.125,
                                 rows=np.arange(spec.row_begin, spec.row_end, dtype=np.int32))
        q.put((rank, ok_kv, bool(np.array_equal(O_loc, O_ref)), spec.row_begin, spec.row_end))
    finally:
        tdist.destroy_process_group()


def test_gloo_world2_allgather_and_rows(dist_mod, oracle_mod):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    assert [r[1] for r in res] == [True, True], "K/V all-gather layout"
    assert [r[2] for r in res] == [True, True], "sharded rows != global rows"
    assert res[0][4] == res[1][3]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_row_shards_bitwise_equal_single_gpu(dist_mod, world):
    import torch

    from helpers import csr_to_dev, to_dev
    from paper_2505_08098_b200 import f3s
    g = fi.chung_lu(20000, 150000, gamma=2.2, max_deg=3000, seed=21)
    n, H, d = g.n_rows, 4, 64
    Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=21)
    Q, K, V = to_dev(Qb, "fp16"), to_dev(Kb, "fp16"), to_dev(Vb, "fp16")
    rp, ci = csr_to_dev(g)
    p1 = f3s.plan(rp, ci, n)
    O1 = f3s.attention(p1, Q, K, V, scale=0.125)
    parts = []
    for r in range(world):
        sh = dist_mod.make_shard(g.row_ptr, g.col_idx, r, world, global_chunks=p1.info()["total_chunks"])
        s = sh.spec
        Ol = dist_mod.attention(sh, Q[s.row_begin:s.row_end].contiguous(), K, V,
                                torch.empty((s.row_end - s.row_begin, H, d), dtype=torch.float32, device="cuda"),
                                scale=0.125)
        parts.append(Ol)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), O1)


@pytest.mark.gpu
def test_batched_graph_shards(dist_mod, oracle_mod):
    import torch

    from helpers import assert_close, to_dev
    g = fi.molecules(600, seed=9)
    n, H, d = g.n_rows, 8, 64
    Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=9)
    ref = oracle_mod.attention(g.row_ptr, g.col_idx, Qb, Kb, Vb, scale=0.125)
    outs = []
    for r in range(4):
        sh = dist_mod.make_shard(g.row_ptr, g.col_idx, r, 4, graph_ptr=g.graph_ptr)
        s = sh.spec
        Ol = dist_mod.attention(sh, to_dev(Qb[s.row_begin:s.row_end], "fp16"), to_dev(Kb[s.row_begin:s.row_end], "fp16"),
                                to_dev(Vb[s.row_begin:s.row_end], "fp16"),
                                torch.empty((s.row_end - s.row_begin, H, d), dtype=torch.float32, device="cuda"),
                                scale=0.125)
        outs.append(Ol.cpu().numpy())
    assert_close(np.concatenate(outs), ref)


def _hub_window_graph(n_windows=60000, hub_cols=2560, seed=3):
    """1 chunk per row window plus one window (rows 0..15) of hub_cols distinct columns: its chunk
    count (20) lies between a 2-shard plan's own split bound (16 = the floor, ~30K chunks /
    (2 * 8 * SMs)) and the global one (26, ~60K chunks)."""
    rng = np.random.default_rng(seed)
    n = 16 * n_windows
    deg = rng.integers(2, 9, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = rng.integers(0, n, len(rows))
    hub_r = np.repeat(np.arange(16, dtype=np.int64), hub_cols // 16)
    hub_c = rng.choice(n, hub_cols, replace=False)
    keys = np.unique(np.concatenate([rows[rows >= 16] * n + cols[rows >= 16], hub_r * n + hub_c]))
    rp = np.searchsorted(keys // n, np.arange(n + 1)).astype(np.int32)
    ci = (keys % n).astype(np.int32)
    return n, rp, ci


@pytest.mark.gpu
def test_shard_split_bound_is_global(dist_mod):
    """A row-shard plan takes the heavy-window split bound of the global problem, so a window the
    1-GPU plan leaves whole is left whole on its shard and the O rows stay bitwise equal
    (f3s.h f3s_plan_set_split)."""
    import torch

    from helpers import to_dev
    from paper_2505_08098_b200 import f3s
    n, rp_h, ci_h = _hub_window_graph()
    H, d = 1, 64
    Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=3)
    Q, K, V = to_dev(Qb, "fp16"), to_dev(Kb, "fp16"), to_dev(Vb, "fp16")
    p1 = f3s.plan(torch.from_numpy(rp_h).cuda(), torch.from_numpy(ci_h).cuda(), n)
    i1 = p1.info()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    assert i1["split_chunks"] == f3s.default_split_chunks(i1["total_chunks"], sms)
    assert i1["split_groups"] == 0  # the 20-chunk hub window is whole in the 1-GPU plan
    O1 = f3s.attention(p1, Q, K, V, scale=0.125)
    own = []
    parts = []
    for r in range(2):
        spec = dist_mod.shard_spec(rp_h, ci_h, r, 2)
        local = f3s.plan_rows(torch.from_numpy(spec.row_ptr).cuda(), torch.from_numpy(spec.col_idx).cuda(),
                              spec.row_end - spec.row_begin, n)
        own.append(local.info())
        sh = dist_mod.make_shard(rp_h, ci_h, r, 2, global_chunks=i1["total_chunks"])
        assert sh.plan.info()["split_chunks"] == i1["split_chunks"]
        parts.append(dist_mod.attention(sh, Q[spec.row_begin:spec.row_end].contiguous(), K, V,
                                        torch.empty((spec.row_end - spec.row_begin, H, d), dtype=torch.float32,
                                                    device="cuda"), scale=0.125))
    # the shard holding the hub would have split it with its own bound
    assert own[0]["split_groups"] == 1 and own[0]["split_chunks"] < 20 < i1["split_chunks"]
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), O1)


def _ring_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist

    from paper_2505_08098_b200 import dist as f3sdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = fi.chung_lu(2000, 9000, gamma=2.4, max_deg=300, seed=13)
        n, H, d = g.n_rows, 2, 64
        Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=13)
        spec = f3sdist.shard_spec(g.row_ptr, g.col_idx, rank, world)
        S = spec.kv_rows
        KV = torch.zeros((world * S, 2, H, d), dtype=torch.float16)
        KV[rank * S:(rank + 1) * S] = torch.from_numpy(f3sdist.kv_shard(spec, Kb, Vb, n).view(np.float16))
        order = []
        f3sdist.ring_exchange(KV, S, rank, world, on_block=order.append)
        got = KV.numpy().view(np.uint16)[:n]
        ok = bool(np.array_equal(got[:, 0], Kb) and np.array_equal(got[:, 1], Vb))
        # the column blocks of the local CSR partition its entries by K/V owner
        blocks = f3sdist.column_block_csr(spec, world)
        part_ok = sum(len(b[1]) for b in blocks) == len(spec.col_idx) and all(
            len(ci) == 0 or (ci.min() >= r * S and ci.max() < (r + 1) * S) for r, (_, ci) in enumerate(blocks))
        q.put((rank, ok, order, bool(part_ok)))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ring_exchange_order_and_blocks(dist_mod, world):
    """f2 host logic: the ring exchange (world-1 rounds of paired send/recv) replicates every
    [K||V] shard bit for bit, announces the own block first and then block rank-t in round t, and
    the column-block CSRs split the local entries by owner."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, ok, order, part_ok in res:
        assert ok and part_ok
        assert order == [rank] + [(rank - t) % world for t in range(1, world)]
