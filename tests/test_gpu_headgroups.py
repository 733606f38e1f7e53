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
