"""Heavy row-window split (the paper's "multiple thread blocks per row window",
PAPER.md:616-618): row windows of more than `split_chunks` 128-column chunks are processed as
pieces on different CTAs and merged, in piece order, by the CTA finishing the last piece.
The result must match the fp64 oracle within the BASELINE tolerance, be bitwise deterministic,
and agree with the unsplit kernel up to fp32 rounding of the merge."""
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


def _skewed_csr(seed=3):
    # power-law graph whose hubs make row windows thousands of compacted columns wide (tens of
    # chunks), plus a ragged last window (n % 16 != 0)
    return fi.chung_lu(20000 + 5, 240000, gamma=2.0, max_deg=12000, seed=seed)


def _run(f3s, p, Qb, Kb, Vb, dtype, scale):
    import torch
    O = f3s.attention(p, to_dev(Qb, dtype), to_dev(Kb, dtype), to_dev(Vb, dtype), scale=scale)
    torch.cuda.synchronize()
    return O.cpu().numpy()


@pytest.mark.parametrize("split_chunks", [1, 2, 5])
@pytest.mark.parametrize("dtype,d,H", [("fp16", 64, 1), ("bf16", 64, 3), ("fp16", 128, 2)])
def test_split_parity(f3s, oracle_mod, split_chunks, dtype, d, H):
    csr = _skewed_csr()
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    p.set_split(split_chunks)
    info = p.info()
    assert info["split_chunks"] == split_chunks and info["split_groups"] > 0
    Qb, Kb, Vb = make_qkv(csr.n_rows, csr.n_cols, H, d, dtype, seed=31)
    scale = 1.0 / np.sqrt(d)
    O = _run(f3s, p, Qb, Kb, Vb, dtype, scale)
    ref = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=scale, dtype=dtype)
    assert_close(O, ref)
    # deterministic merge order: a second call is bitwise identical
    O2 = _run(f3s, p, Qb, Kb, Vb, dtype, scale)
    assert np.array_equal(O, O2)
    # same result as the unsplit kernel up to rounding: P is cast to the input dtype relative to
    # each piece's own row max instead of the running max, so the two differ by about one
    # rounding unit u of that dtype (2^-11 fp16, 2^-8 bf16) times |V| <= 1
    p.set_split(0)
    assert p.info()["split_groups"] == 0
    O0 = _run(f3s, p, Qb, Kb, Vb, dtype, scale)
    u = 2.0 ** -11 if dtype == "fp16" else 2.0 ** -8
    assert np.max(np.abs(O - O0)) <= 2 * u


def test_split_large_scores_and_empty_rows(f3s, oracle_mod):
    # scores ~1e2..1e3 (inputs x16): the merge's max-rescaling must stay finite; rows without
    # entries stay exactly 0 even inside split windows
    csr = _skewed_csr(seed=4)
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    p.set_split(1)
    Qb, Kb, Vb = make_qkv(csr.n_rows, csr.n_cols, 2, 64, "fp16", seed=32, amp_qk=16.0)
    O = _run(f3s, p, Qb, Kb, Vb, "fp16", 0.125)
    ref = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.125)
    assert_close(O, ref)
    empty = np.diff(csr.row_ptr) == 0
    assert np.all(O[empty] == 0)


def test_default_split_threshold(f3s):
    # f3s_plan's default bound: max(16, ceil(total chunks / (2 * 8 * SMs))) chunks per piece (the
    # per-SM share of an 8-GPU row-sharded run, f3s.h f3s_default_split_chunks)
    import torch
    csr = _skewed_csr()
    rp, ci = csr_to_dev(csr)
    p = f3s.plan(rp, ci, csr.n_rows)
    rw_ptr, _, _, _ = p.export()
    w = np.diff(rw_ptr.astype(np.int64))
    chunks = np.maximum(1, (w + 127) // 128)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    t = max(16, int(-(-int(chunks.sum()) // (2 * 8 * sms))))
    info = p.info()
    assert info["split_chunks"] == t
    assert info["split_groups"] == int(np.count_nonzero(chunks > t))
