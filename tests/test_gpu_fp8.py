"""FP8 (E4M3) inputs, SURVEY 8(f) f4 "FP8 K/V gathers" (FP8 is the paper's future work,
PAPER.md:750-751): Q, K, V stored as OCP E4M3; S on tcgen05 kind::f8f6f4 (exact products, fp32
accumulation), P rounded to E4M3 (scaled by 2^8) for the SpMM.  The oracle gets the decoded fp8
values, so the only deviation beyond fp32 rounding is the rounding of P, bounded per row by
DESIGN.md reading c24:

    |O_i - O_ref_i| <= (2^-4 + deg_i * 2^-18) * max_{j in N(i)} |V_j|   (+ fp32 slack)

(relative rounding error 2^-4 of normal e4m3 values; absolute 2^-10 below 2^-6, i.e. 2^-18 of the
row's largest weight 2^8).
"""
import numpy as np
import pytest

import f3s_inputs as fi
from conftest import decode
from helpers import csr_to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def f3s():
    import torch
    assert torch.cuda.is_available()
    from paper_2505_08098_b200 import f3s as mod
    return mod


def _e4m3(shape, seed, amp=1.0):
    """Seeded values rounded (RNE) to E4M3: (device tensor, exact decoded float64 array)."""
    import torch
    x = decode(fi.values(shape, seed=seed, dtype="fp16", amp=amp), "fp16").astype(np.float32)
    t = torch.from_numpy(x).to(torch.float8_e4m3fn)
    return t.cuda(), t.to(torch.float64).numpy()


def _run(f3s, csr, H, seed, scale, split=None, d=128):
    import torch
    (Q, Qd), (K, Kd), (V, Vd) = (_e4m3((n, H, d), (seed << 8) | t) for n, t in
                                 ((csr.n_rows, 1), (csr.n_cols, 2), (csr.n_cols, 3)))
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows) if csr.n_rows == csr.n_cols else f3s.plan_rows(rp, ci, csr.n_rows, csr.n_cols)
    if split is not None:
        p.set_split(split)
    O = f3s.attention(p, Q, K, V, scale=scale)
    torch.cuda.synchronize()
    return O.cpu().numpy(), (Q, K, V, p), (Qd, Kd, Vd)


def _check_bound(csr, O, Vd, ref):
    deg = np.diff(csr.row_ptr)
    assert np.all(np.isfinite(O))
    for i in range(csr.n_rows):
        if deg[i] == 0:
            assert np.all(O[i] == 0)
            continue
        vmax = np.abs(Vd[csr.col_idx[csr.row_ptr[i]:csr.row_ptr[i + 1]]]).max(axis=(0, 2))  # per head
        tol = (2.0 ** -4 + deg[i] * 2.0 ** -18 + 1e-5) * vmax + 1e-5
        err = np.abs(O[i].astype(np.float64) - ref[i]).max(axis=1)
        assert np.all(err <= tol), (i, deg[i], err, tol)


@pytest.mark.parametrize("d", [128, 64])
def test_fp8_parity_ragged(f3s, oracle_mod, d):
    # ragged n, duplicates, unsorted rows, empty rows, chunk tails of every length mod 32
    csr = fi.random_csr(1000 + 7, 1000 + 7, 0, 150, keep_dups=True, unsorted=True, seed=81)
    O, _, (Qd, Kd, Vd) = _run(f3s, csr, 2, 5, 1.0 / np.sqrt(d), d=d)
    ref = oracle_mod.attention_f64(csr.row_ptr, csr.col_idx, Qd, Kd, Vd, scale=1.0 / np.sqrt(d))
    _check_bound(csr, O, Vd, ref)
    diff = O - ref
    # the rounding errors of P are unbiased: far below the worst case over the whole output
    assert np.linalg.norm(diff) / np.linalg.norm(ref) <= 2e-2


@pytest.mark.parametrize("d,H", [(128, 1), (64, 3)])
def test_fp8_power_law_and_split(f3s, oracle_mod, d, H):
    # (d = 64, H = 3: the Q box of the last head reaches past the row, zero-filled by the tensor map)
    import torch
    csr = fi.chung_lu(6000, 60000, gamma=2.1, max_deg=3000, seed=82)
    O, (Q, K, V, p), (Qd, Kd, Vd) = _run(f3s, csr, H, 6, 0.125, d=d)
    ref = oracle_mod.attention_f64(csr.row_ptr, csr.col_idx, Qd, Kd, Vd, scale=0.125)
    _check_bound(csr, O, Vd, ref)
    # heavy windows split into pieces of 2 chunks: same bound, deterministic
    p.set_split(2)
    O2 = f3s.attention(p, Q, K, V, scale=0.125)
    O3 = f3s.attention(p, Q, K, V, scale=0.125)
    torch.cuda.synchronize()
    _check_bound(csr, O2.cpu().numpy(), Vd, ref)
    assert torch.equal(O2, O3)


def test_fp8_host_path_and_rectangular(f3s, oracle_mod):
    import torch
    # rectangular A (a row shard against all columns) through the host-buffer entry point
    csr = fi.random_csr(300, 2000, 1, 60, seed=83)
    O, (Q, K, V, p), (Qd, Kd, Vd) = _run(f3s, csr, 3, 7, 0.3)
    ref = oracle_mod.attention_f64(csr.row_ptr, csr.col_idx, Qd, Kd, Vd, scale=0.3)
    _check_bound(csr, O, Vd, ref)
    Oh = torch.empty(O.shape, dtype=torch.float32).pin_memory()
    hq, hk, hv = (x.cpu().pin_memory() for x in (Q, K, V))
    f3s.attention_host(p, hq, hk, hv, Oh, scale=0.3, heads=3, d=128, dtype=f3s.E4M3)
    assert np.array_equal(Oh.numpy(), O)


def test_fp8_rejected_where_unsupported(f3s):
    import torch
    csr = fi.random_csr(64, 64, 1, 4, seed=84)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, 64)
    x32 = torch.zeros((64, 1, 32), dtype=torch.float8_e4m3fn, device="cuda")
    with pytest.raises(f3s.F3SError):
        f3s.attention(p, x32, x32, x32, scale=1.0)  # d = 32
    x = torch.zeros((64, 1, 128), dtype=torch.float8_e4m3fn, device="cuda")
    with pytest.raises(f3s.F3SError):
        f3s.attention(p, x, x, x, scale=1.0, variant="simt")
    with pytest.raises(f3s.F3SError):
        f3s.attention_backward(p, x, x, x, torch.zeros((64, 1, 128), device="cuda"), scale=1.0)


@pytest.mark.parametrize("variant", ["default", "no_reorder"])
def test_fp8_eight_heads_variants(f3s, oracle_mod, variant):
    # the bench's head count (8 x 128) on an arxiv-like degree mix, both work orders
    import torch
    csr = fi.chung_lu(3000, 20000, directed=True, gamma=2.3, max_deg=400, seed=85)
    (Q, Qd), (K, Kd), (V, Vd) = (_e4m3((3000, 8, 128), (9 << 8) | t) for t in (1, 2, 3))
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, 3000)
    O = f3s.attention(p, Q, K, V, scale=1.0 / np.sqrt(128), variant=variant)
    torch.cuda.synchronize()
    ref = oracle_mod.attention_f64(csr.row_ptr, csr.col_idx, Qd, Kd, Vd, scale=1.0 / np.sqrt(128))
    _check_bound(csr, O.cpu().numpy(), Vd, ref)
