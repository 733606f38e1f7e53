"""SURVEY §8(e) row a12 on a real GPU: the multi-GPU exchange and the fused kernel running
together on device memory.  Two ranks (processes) share the one GPU of the test box over a gloo
process group (NCCL needs one GPU per rank): each builds its row-shard plan with the global split
bound (all-reduced chunk count), uploads its padded [K||V] shard, replicates it with ONE
all-gather, and runs f3s_attention_kv on the gathered buffer.  Each rank's O rows must equal the
single-GPU call bit for bit and the fp64 oracle within BASELINE.json's tolerances."""
import os
import socket

import numpy as np
import pytest

import f3s_inputs as fi
from helpers import TOL_MAX_ABS, TOL_REL_FRO, errors, make_qkv

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, graph, overlap, q):
    import torch
    import torch.distributed as tdist

    import oracle
    from paper_2505_08098_b200 import dist as f3sdist
    from paper_2505_08098_b200 import f3s
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        if graph == "power":
            g = fi.chung_lu(30000, 200000, gamma=2.2, max_deg=3000, seed=41)
            H, d = 4, 64
        else:  # dense communities: long row windows
            g = fi.dcsbm(12000, 1500000, comm_size=3000, mu=0.9, gamma=2.1, max_deg=2000, seed=43)
            H, d = 2, 128
        n = g.n_rows
        Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=41)
        f16 = lambda b: torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).to(dev).view(torch.float16)
        shard = f3sdist.make_shard(g.row_ptr, g.col_idx, rank, world, device=dev)  # global split bound via gloo
        spec = shard.spec
        Qloc = f16(Qb[spec.row_begin:spec.row_end])
        if overlap:  # f2: ring exchange on a side stream, column-block partials, merge
            ov = f3sdist.OverlappedShard(spec, H, d, torch.float16, device=dev)
            ov.own_block().copy_(f16(f3sdist.kv_shard(spec, Kb, Vb, n)))
            Ol = torch.empty((spec.row_end - spec.row_begin, H, d), dtype=torch.float32, device=dev)
            ov.run(Qloc, Ol, scale=1.0 / d ** 0.5)
        else:
            KV_sh = f16(f3sdist.kv_shard(spec, Kb, Vb, n))
            KV = torch.empty((world * spec.kv_rows, 2, H, d), dtype=torch.float16, device=dev)
            f3sdist.allgather_kv_into(KV, KV_sh)
            Ol = f3sdist.attention_kv(shard, Qloc, KV, scale=1.0 / d ** 0.5)
        # the single-GPU call on the full problem, in this process
        p1 = f3s.plan(torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col_idx).to(dev), n)
        O1 = f3s.attention(p1, f16(Qb), f16(Kb), f16(Vb), scale=1.0 / d ** 0.5)
        torch.cuda.synchronize()
        same = bool(torch.equal(Ol, O1[spec.row_begin:spec.row_end])) if not overlap else \
            bool(torch.allclose(Ol, O1[spec.row_begin:spec.row_end], rtol=0, atol=2e-3))
        same_split = shard.plan.info()["split_chunks"] == p1.info()["split_chunks"]
        ref = oracle.attention(g.row_ptr, g.col_idx, Qb, Kb, Vb, scale=1.0 / d ** 0.5,
                               rows=np.arange(spec.row_begin, spec.row_end, dtype=np.int32))
        max_abs, rel = errors(Ol.cpu().numpy(), ref)
        q.put((rank, same, same_split, max_abs, rel, spec.row_begin, spec.row_end, n))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("graph,overlap", [("power", False), ("communities", False), ("power", True),
                                           ("communities", True)])
def test_two_ranks_allgather_then_kernel(graph, overlap):
    """overlap=False: one [K||V] all-gather, then f3s_attention_kv (bitwise = 1-GPU).  overlap=True
    (f2): ring exchange of the blocks while f3s_attention_partial runs on those present, then
    f3s_attention_merge (tolerance-equal to the 1-GPU call and the oracle)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, graph, overlap, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert len(r) == 8, f"rank {r[0]} failed: {r[1]}"
    assert [r[1] for r in res] == [True, True], "shard rows != single-GPU rows"
    assert [r[2] for r in res] == [True, True], "shard split bound != single-GPU bound"
    for r in res:
        assert r[3] <= TOL_MAX_ABS and r[4] <= TOL_REL_FRO, r
    assert res[0][5] == 0 and res[0][6] == res[1][5] and res[1][6] == res[1][7]


def _column_blocks(row_ptr, col_idx, n_cols, parts):
    """The CSR entries whose column lies in block g = [g*S, (g+1)*S), S = ceil(n_cols / parts)."""
    S = -(-n_cols // parts)
    rows = np.repeat(np.arange(len(row_ptr) - 1), np.diff(row_ptr))
    out = []
    for g in range(parts):
        sel = (col_idx >= g * S) & (col_idx < (g + 1) * S)
        cnt = np.bincount(rows[sel], minlength=len(row_ptr) - 1)
        out.append((np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32), col_idx[sel].astype(np.int32)))
    return out


@pytest.mark.parametrize("parts,H,d,dtype", [(1, 2, 64, "fp16"), (3, 4, 64, "fp16"), (8, 2, 128, "bf16"),
                                             (5, 1, 64, "fp16")])
def test_column_block_partials_merge(oracle_mod, parts, H, d, dtype):
    """f2 building blocks on one GPU: the shard's columns split into `parts` K/V blocks, each block
    run by f3s_attention_partial on its own plan (a heavy-window split inside a block included),
    then f3s_attention_merge in block order: equals the fp64 oracle within the tolerances and is
    deterministic; with one block it is the plain call up to the final division."""
    import torch

    from helpers import assert_close, to_dev
    from paper_2505_08098_b200 import f3s
    g = fi.dcsbm(9000, 700000, comm_size=3000, mu=0.8, gamma=2.1, max_deg=2500, seed=parts)
    n = g.n_rows
    Qb, Kb, Vb = make_qkv(n, n, H, d, dtype, seed=7)
    Q, K, V = to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype)
    blocks = _column_blocks(g.row_ptr, g.col_idx, n, parts)
    Op = torch.empty((parts, n, H, d), dtype=torch.float32, device="cuda")
    mlp = torch.empty((parts, n, H, 2), dtype=torch.float32, device="cuda")
    plans = []
    for b, (rp, ci) in enumerate(blocks):
        p = f3s.plan_rows(torch.from_numpy(rp).cuda(), torch.from_numpy(ci if len(ci) else np.zeros(1, np.int32)).cuda(),
                          n, n)
        if b == 0:
            p.set_split(4)  # force split pieces inside a block (merge of pieces in partial mode)
        plans.append(p)
        f3s.attention_partial_raw(p, Q.data_ptr(), K.data_ptr(), V.data_ptr(), 0, Op[b].data_ptr(), mlp[b].data_ptr(),
                                  0.125, H, d, f3s.FP16 if dtype == "fp16" else f3s.BF16, 100 if b % 2 else 0,
                                  torch.cuda.current_stream().cuda_stream)
    O = f3s.attention_merge(Op, mlp)
    O2 = f3s.attention_merge(Op, mlp)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)
    ref = oracle_mod.attention(g.row_ptr, g.col_idx, Qb, Kb, Vb, scale=0.125, dtype=dtype)
    assert_close(O.cpu().numpy(), ref)
    if parts == 1:
        O1 = f3s.attention(plans[0], Q, K, V, scale=0.125)
        l = mlp[0, :, :, 1:2]
        assert torch.allclose(torch.where(l > 0, Op[0] / l, torch.zeros_like(Op[0])), O1, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("parts,H", [(1, 4), (3, 8)])
def test_column_block_partials_head_groups(oracle_mod, parts, H):
    """Partial mode on head-group plans (d = 64, H % 4 == 0, every window <= 32 columns: the
    batched-molecules shape): the head-group epilogue leaves unnormalised O and each head's (m, l);
    merged in block order they equal the oracle, and with one block O / l is the plain call."""
    import torch

    from helpers import assert_close, to_dev
    from paper_2505_08098_b200 import f3s
    g = fi.molecules(400, 25, 150, seed=parts)
    n, d = g.n_rows, 64
    Qb, Kb, Vb = make_qkv(n, n, H, d, "fp16", seed=9)
    Q, K, V = to_dev(Qb, "fp16"), to_dev(Kb, "fp16"), to_dev(Vb, "fp16")
    blocks = _column_blocks(g.row_ptr, g.col_idx, n, parts)
    Op = torch.empty((parts, n, H, d), dtype=torch.float32, device="cuda")
    mlp = torch.empty((parts, n, H, 2), dtype=torch.float32, device="cuda")
    plans = []
    for b, (rp, ci) in enumerate(blocks):
        p = f3s.plan_rows(torch.from_numpy(rp).cuda(), torch.from_numpy(ci if len(ci) else np.zeros(1, np.int32)).cuda(),
                          n, n)
        assert p.info()["max_width"] <= 32
        plans.append(p)
        f3s.attention_partial_raw(p, Q.data_ptr(), K.data_ptr(), V.data_ptr(), 0, Op[b].data_ptr(), mlp[b].data_ptr(),
                                  0.125, H, d, f3s.FP16, 0, torch.cuda.current_stream().cuda_stream)
    O = f3s.attention_merge(Op, mlp)
    torch.cuda.synchronize()
    ref = oracle_mod.attention(g.row_ptr, g.col_idx, Qb, Kb, Vb, scale=0.125, dtype="fp16")
    assert_close(O.cpu().numpy(), ref)
    if parts == 1:
        O1 = f3s.attention(plans[0], Q, K, V, scale=0.125)
        l = mlp[0, :, :, 1:2]
        assert torch.allclose(torch.where(l > 0, Op[0] / l, torch.zeros_like(Op[0])), O1, rtol=1e-5, atol=1e-6)
