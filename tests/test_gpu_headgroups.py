"""Head groups (d = 64, every row window at most 32 compacted columns wide, e.g. batched small
graphs): the default kernel packs 4 heads of a row window into one 128-row chunk (head g in tile
rows / S^T lanes 32g .. 32g+31).  Each head's arithmetic is the one-head kernel's (same MMA
shapes and accumulation order per lane), so the result must match the oracle within the BASELINE
tolerance and the one-head variant (F3S_VARIANT_ONE_HEAD) bit for bit."""
import numpy as np
import pytest

import f3s_inputs as fi
from helpers import assert_close, csr_to_dev, make_qkv, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def f3s():
    import torch
    assert torch.cuda.is_available()
    from paper_2505_08098_b200 import f3s as mod
    return mod


def _run(f3s, p, Qb, Kb, Vb, dtype, scale, variant):
    import torch
    O = f3s.attention(p, to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype), scale=scale, variant=variant)
    torch.cuda.synchronize()
    return O.cpu().numpy()


@pytest.mark.parametrize("dtype,H", [("fp16", 4), ("bf16", 8), ("fp16", 12)])
@pytest.mark.parametrize("self_loops", [False, True])
def test_head_groups_parity(f3s, oracle_mod, dtype, H, self_loops):
    csr = fi.molecules(400, 10, 60, self_loops=self_loops, seed=7 + H)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    assert p.info()["max_width"] <= 32  # every window qualifies for head groups
    Qb, Kb, Vb = make_qkv(csr.n_rows, csr.n_cols, H, 64, dtype, seed=41)
    O = _run(f3s, p, Qb, Kb, Vb, dtype, 0.125, "default")
    ref = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.125, dtype=dtype)
    assert_close(O, ref)
    O1 = _run(f3s, p, Qb, Kb, Vb, dtype, 0.125, "one_head")
    assert np.array_equal(O, O1)


def test_head_groups_empty_rows_and_ragged(f3s, oracle_mod):
    # empty rows, empty row windows and a ragged last window (n % 16 != 0) inside head groups
    csr = fi.random_csr(16 * 40 + 9, 16 * 40 + 9, 0, 2, seed=3)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    assert p.info()["max_width"] <= 32
    Qb, Kb, Vb = make_qkv(csr.n_rows, csr.n_cols, 4, 64, "fp16", seed=42, amp_qk=8.0)
    O = _run(f3s, p, Qb, Kb, Vb, "fp16", 0.125, "default")
    ref = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.125)
    assert_close(O, ref)
    empty = np.diff(csr.row_ptr) == 0
    assert empty.any() and np.all(O[empty] == 0)
    assert np.array_equal(O, _run(f3s, p, Qb, Kb, Vb, "fp16", 0.125, "one_head"))


@pytest.mark.parametrize("H", [4, 8])
def test_head_groups_per_window(f3s, oracle_mod, H):
    """A plan with both wide windows (> 32 columns, one head per chunk) and narrow ones (head
    groups): the default call runs them in two launches and is bitwise equal to the one-head
    kernel over the whole plan (reading c22), and within the tolerances of the oracle."""
    import torch
    mol = fi.molecules(300, 25, 150, seed=H)
    n_mol = mol.n_rows
    wide = fi.random_csr(64, n_mol, 40, 120, seed=H)  # 4 windows of many distinct columns
    rp = np.concatenate([mol.row_ptr, mol.row_ptr[-1] + wide.row_ptr[1:]]).astype(np.int32)
    ci = np.concatenate([mol.col_idx, wide.col_idx]).astype(np.int32)
    n = n_mol + 64
    csr = fi.CSR(n, n, rp, ci)
    Qb, Kb, Vb = make_qkv(n, n, H, 64, "fp16", seed=3)
    p = f3s.plan(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), n)
    assert p.info()["max_width"] > 32
    O = _run(f3s, p, Qb, Kb, Vb, "fp16", 0.125, "default")
    ref = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=0.125)
    assert_close(O, ref)
    assert np.array_equal(O, _run(f3s, p, Qb, Kb, Vb, "fp16", 0.125, "one_head"))


def test_head_groups_per_window_with_split(f3s, oracle_mod):
    """Per-window head groups on a plan with split windows whose last pieces are narrow: the
    narrow-tail launch must start after the last piece (every output row written, oracle parity,
    bitwise equal to the one-head kernel)."""
    import torch
    mol = fi.molecules(200, 25, 150, seed=2)
    n_mol = mol.n_rows
    wide = fi.random_csr(64, n_mol, 300, 600, seed=2)  # windows of ~4-6 chunks
    rp = np.concatenate([mol.row_ptr, mol.row_ptr[-1] + wide.row_ptr[1:]]).astype(np.int32)
    ci = np.concatenate([mol.col_idx, wide.col_idx]).astype(np.int32)
    n = n_mol + 64
    Qb, Kb, Vb = make_qkv(n, n, 4, 64, "fp16", seed=4)
    p = f3s.plan(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), n)
    p.set_split(1)  # every wide window in 128-column pieces; the last piece of most is < 32 columns
    assert p.info()["split_groups"] > 0
    O = _run(f3s, p, Qb, Kb, Vb, "fp16", 0.125, "default")
    assert np.all(np.isfinite(O))
    assert_close(O, oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=0.125))
    assert np.array_equal(O, _run(f3s, p, Qb, Kb, Vb, "fp16", 0.125, "one_head"))
