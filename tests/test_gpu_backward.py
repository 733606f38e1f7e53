"""Backward of the fused 3S pass (f3s_attention_backward) against the fp64 oracle
backward (pinned in test_oracle_backward.py) on the same seeded inputs: dQ, dK, dV element by
element, plus determinism and row-shard additivity."""
import numpy as np
import pytest

import f3s_inputs as fi
from conftest import decode
from helpers import csr_to_dev, errors, make_qkv, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def f3s():
    import torch
    assert torch.cuda.is_available()
    from paper_2505_08098_b200 import f3s as mod
    return mod


def _close(got, ref):
    # fp32 arithmetic on the exact inputs: the same bar as the forward, relative to the scale
    max_abs, rel = errors(got, ref)
    scale = max(1.0, float(np.max(np.abs(ref))))
    assert np.all(np.isfinite(got)) and max_abs <= 1e-2 * scale and rel <= 5e-3, (max_abs, rel, scale)


def _bwd(f3s, p, Qb, Kb, Vb, G, dtype, scale):
    import torch
    dO = torch.from_numpy(G.astype(np.float32)).cuda()
    dQ, dK, dV = f3s.attention_backward(p, to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype), dO, scale=scale)
    torch.cuda.synchronize()
    return dQ.cpu().numpy(), dK.cpu().numpy(), dV.cpu().numpy()


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("d,H", [(64, 1), (64, 3), (128, 2)])
def test_backward_parity(f3s, oracle_mod, dtype, d, H):
    csr = fi.random_csr(1000 + 7, 1000 + 7, 0, 40, keep_dups=True, unsorted=True, seed=d + H)
    Qb, Kb, Vb = make_qkv(csr.n_rows, csr.n_cols, H, d, dtype, seed=21)
    G = np.random.default_rng(d + H).standard_normal((csr.n_rows, H, d)).astype(np.float32)
    scale = 1.0 / np.sqrt(d)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    got = _bwd(f3s, p, Qb, Kb, Vb, G, dtype, scale)
    ref = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, decode(Qb, dtype), decode(Kb, dtype),
                                        decode(Vb, dtype), G.astype(np.float64), scale=scale)
    for g, r in zip(got, ref):
        _close(g, r)
    empty = np.diff(csr.row_ptr) == 0
    assert empty.any() and np.all(got[0][empty] == 0)
    # deterministic: fixed visiting order in both passes, no atomics on the data
    again = _bwd(f3s, p, Qb, Kb, Vb, G, dtype, scale)
    assert all(np.array_equal(a, b) for a, b in zip(got, again))


def test_backward_power_law(f3s, oracle_mod):
    # hub rows and hub columns (windows of many chunks, columns with thousands of rows)
    csr = fi.chung_lu(6000, 60000, gamma=2.1, max_deg=3000, seed=21)
    Qb, Kb, Vb = make_qkv(6000, 6000, 2, 64, "fp16", seed=22)
    G = np.random.default_rng(5).standard_normal((6000, 2, 64)).astype(np.float32)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    got = _bwd(f3s, p, Qb, Kb, Vb, G, "fp16", 0.125)
    ref = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, decode(Qb, "fp16"), decode(Kb, "fp16"),
                                        decode(Vb, "fp16"), G.astype(np.float64), scale=0.125)
    for g, r in zip(got, ref):
        _close(g, r)


def test_backward_row_shards_add_up(f3s):
    # dK, dV of a row shard are that shard's partial sums: the shards' sum is the full result
    import torch
    n, H, d = 2000, 2, 64
    csr = fi.random_csr(n, n, 1, 20, seed=9)
    Qb, Kb, Vb = make_qkv(n, n, H, d, "bf16", seed=23)
    G = np.random.default_rng(7).standard_normal((n, H, d)).astype(np.float32)
    rp, ci = csr_to_dev(csr)
    full = _bwd(f3s, f3s.plan(rp, ci, n), Qb, Kb, Vb, G, "bf16", 0.125)
    bounds = [0, 992, n]
    dQ_parts, dK_sum, dV_sum = [], 0.0, 0.0
    for b, e in zip(bounds[:-1], bounds[1:]):
        lrp = torch.from_numpy((csr.row_ptr[b:e + 1] - csr.row_ptr[b]).astype(np.int32)).cuda()
        lci = torch.from_numpy(csr.col_idx[csr.row_ptr[b]:csr.row_ptr[e]].copy()).cuda()
        ps = f3s.plan_rows(lrp, lci, e - b, n)
        dO = torch.from_numpy(G[b:e]).cuda()
        dQ, dK, dV = f3s.attention_backward(ps, to_dev(Qb[b:e].copy(), "bf16"), to_dev(Kb, "bf16"), to_dev(Vb, "bf16"),
                                            dO, scale=0.125)
        torch.cuda.synchronize()
        dQ_parts.append(dQ.cpu().numpy())
        dK_sum = dK_sum + dK.cpu().numpy().astype(np.float64)
        dV_sum = dV_sum + dV.cpu().numpy().astype(np.float64)
    assert np.array_equal(np.concatenate(dQ_parts), full[0])  # rows of a window live in one shard
    assert np.max(np.abs(dK_sum - full[1])) <= 1e-5 and np.max(np.abs(dV_sum - full[2])) <= 1e-5


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("d,H", [(64, 2), (128, 1)])
def test_backward_tc_vs_simt(f3s, oracle_mod, dtype, d, H):
    """The tensor-core backward (default) and the CUDA-core kernels both meet the bar against the
    oracle on a power-law graph with multi-chunk windows and hub columns, and agree with each other."""
    import torch
    csr = fi.chung_lu(3000, 40000, gamma=2.1, max_deg=1500, seed=5 + d)
    Qb, Kb, Vb = make_qkv(csr.n_rows, csr.n_cols, H, d, dtype, seed=8)
    G = np.random.default_rng(d).standard_normal((csr.n_rows, H, d)).astype(np.float32)
    scale = 1.0 / np.sqrt(d)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    dO = torch.from_numpy(G).cuda()
    Q, K, V = to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype)
    tc = [x.cpu().numpy() for x in f3s.attention_backward(p, Q, K, V, dO, scale=scale, variant="tc")]
    simt = [x.cpu().numpy() for x in f3s.attention_backward(p, Q, K, V, dO, scale=scale, variant="simt")]
    ref = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, decode(Qb, dtype), decode(Kb, dtype),
                                        decode(Vb, dtype), G.astype(np.float64), scale=scale)
    for a, b, r in zip(tc, simt, ref):
        _close(a, r)
        _close(b, r)
        _close(a, b.astype(np.float64))


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("H", [4, 8])
def test_backward_head_groups(f3s, oracle_mod, dtype, H):
    """d = 64, H % 4 == 0, every window <= 32 columns (the batched-molecules shape): both backward
    passes run 4 heads per chunk; parity with the oracle and with the CUDA-core kernels."""
    import torch
    csr = fi.molecules(300, 25, 150, seed=H)
    n = csr.n_rows
    Qb, Kb, Vb = make_qkv(n, n, H, 64, dtype, seed=12)
    G = np.random.default_rng(H).standard_normal((n, H, 64)).astype(np.float32)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, n)
    assert p.info()["max_width"] <= 32
    dO = torch.from_numpy(G).cuda()
    Q, K, V = to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype)
    tc = [x.cpu().numpy() for x in f3s.attention_backward(p, Q, K, V, dO, scale=0.125, variant="tc")]
    again = [x.cpu().numpy() for x in f3s.attention_backward(p, Q, K, V, dO, scale=0.125, variant="tc")]
    simt = [x.cpu().numpy() for x in f3s.attention_backward(p, Q, K, V, dO, scale=0.125, variant="simt")]
    ref = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, decode(Qb, dtype), decode(Kb, dtype),
                                        decode(Vb, dtype), G.astype(np.float64), scale=0.125)
    for a, b, c, r in zip(tc, again, simt, ref):
        assert np.array_equal(a, b)
        _close(a, r)
        _close(a, c.astype(np.float64))


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("graph,d,H", [("power", 64, 2), ("power", 128, 1), ("molecules", 64, 4), ("ragged", 64, 3)])
def test_training_forward_and_saved_backward(f3s, oracle_mod, dtype, graph, d, H):
    """f3s_attention_fwd gives f3s_attention's O bit for bit plus (m, l) with LSE = m + log2(l) the
    oracle's log-sum-exp; f3s_attention_backward_saved on those saved outputs meets the oracle
    backward's bar (and matches the recomputing backward within it)."""
    import torch
    if graph == "power":
        csr = fi.chung_lu(3000, 40000, gamma=2.1, max_deg=1500, seed=5 + d)
    elif graph == "molecules":
        csr = fi.molecules(300, 25, 150, seed=H)
    else:
        csr = fi.random_csr(1000 + 7, 1000 + 7, 0, 40, keep_dups=True, unsorted=True, seed=d + H)
    n = csr.n_rows
    Qb, Kb, Vb = make_qkv(n, csr.n_cols, H, d, dtype, seed=31)
    G = np.random.default_rng(3 * d + H).standard_normal((n, H, d)).astype(np.float32)
    scale = 1.0 / np.sqrt(d)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, n)
    Q, K, V = to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype)
    O, ml = f3s.attention_fwd(p, Q, K, V, scale=scale)
    O_ref = f3s.attention(p, Q, K, V, scale=scale)
    torch.cuda.synchronize()
    assert torch.equal(O, O_ref)
    # statistics: LSE_i = m + log2(l) = log2 sum_j exp(scale q_i.k_j) over the row's distinct columns
    qd, kd = decode(Qb, dtype), decode(Kb, dtype)
    mlh = ml.cpu().numpy().astype(np.float64)
    rows = np.random.default_rng(1).choice(n, size=min(n, 300), replace=False)
    for i in rows:
        cols = np.unique(csr.col_idx[csr.row_ptr[i]:csr.row_ptr[i + 1]])
        for h in range(H):
            if cols.size == 0:
                assert mlh[i, h, 1] == 0.0
                continue
            s = scale * (kd[cols, h, :] @ qd[i, h, :])
            lse2 = (s.max() + np.log(np.exp(s - s.max()).sum())) / np.log(2.0)
            got = mlh[i, h, 0] + np.log2(mlh[i, h, 1])
            # l sums the P values rounded to the input dtype (reading c7): relative error <= u, the
            # unit roundoff (2^-11 fp16, 2^-8 bf16), so |log2 error| <= log2(1 + u) + fp32 noise
            u = 2.0 ** -11 if dtype == "fp16" else 2.0 ** -8
            assert abs(got - lse2) <= np.log2(1 + u) + 1e-4 * max(1.0, abs(lse2)), (i, h, got, lse2)
    dO = torch.from_numpy(G).cuda()
    saved = [x.cpu().numpy() for x in f3s.attention_backward_saved(p, Q, K, V, O, ml, dO, scale=scale)]
    again = [x.cpu().numpy() for x in f3s.attention_backward_saved(p, Q, K, V, O, ml, dO, scale=scale)]
    recomputed = [x.cpu().numpy() for x in f3s.attention_backward(p, Q, K, V, dO, scale=scale)]
    ref = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, qd, kd, decode(Vb, dtype), G.astype(np.float64),
                                        scale=scale)
    for a, b, c, r in zip(saved, again, recomputed, ref):
        assert np.array_equal(a, b)
        _close(a, r)
        _close(a, c.astype(np.float64))
    # dO handed over and gradients returned in the input dtype (f3s_attention_backward_saved_lp):
    # against the oracle backward of the same rounded dO (one more rounding of each gradient, RNE)
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    dO_lp = dO.to(tdt)
    lp = f3s.attention_backward_saved(p, Q, K, V, O, ml, dO_lp, scale=scale)
    assert all(x.dtype == tdt for x in lp)  # gradients in the input dtype too
    lp = [x.float().cpu().numpy() for x in lp]
    G_lp = dO_lp.double().cpu().numpy()
    ref_lp = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, qd, kd, decode(Vb, dtype), G_lp, scale=scale)
    for a, r in zip(lp, ref_lp):
        _close(a, r)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_training_pair_split_and_mixed_widths(f3s, oracle_mod, dtype):
    """The training forward on a plan with both launch kinds (wide windows one head per chunk, split
    into pieces by a forced bound; narrow windows with head groups): O bitwise equal to
    f3s_attention, and the saved-stats backward against the oracle."""
    import torch
    mol = fi.molecules(40, 25, 60, seed=3)
    wide = fi.random_csr(48, mol.n_rows, 60, 400, seed=4)
    rp = np.concatenate([mol.row_ptr, mol.row_ptr[-1] + wide.row_ptr[1:]]).astype(np.int32)
    ci = np.concatenate([mol.col_idx, wide.col_idx]).astype(np.int32)
    n = mol.n_rows + 48
    p = f3s.plan(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), n)
    p.set_split(1)
    assert p.info()["split_groups"] > 0 and p.info()["max_width"] > 32
    H, d = 4, 64
    Qb, Kb, Vb = make_qkv(n, n, H, d, dtype, seed=41)
    Q, K, V = to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype)
    O, ml = f3s.attention_fwd(p, Q, K, V, scale=0.125)
    assert torch.equal(O, f3s.attention(p, Q, K, V, scale=0.125))
    G = np.random.default_rng(11).standard_normal((n, H, d)).astype(np.float32)
    got = [x.cpu().numpy() for x in f3s.attention_backward_saved(p, Q, K, V, O, ml, torch.from_numpy(G).cuda(),
                                                                 scale=0.125)]
    ref = oracle_mod.attention_backward(rp, ci, decode(Qb, dtype), decode(Kb, dtype), decode(Vb, dtype),
                                        G.astype(np.float64), scale=0.125)
    for a, r in zip(got, ref):
        _close(a, r)
