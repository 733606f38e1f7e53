"""Device plan builder (f3s_plan / f3s_plan_rows) vs the oracle's independent block builder:
bit-exact on random and adversarial CSRs, plus CSR error detection.  Calls go through the C ABI."""
import numpy as np
import pytest

import f3s_inputs as fi
from helpers import csr_to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def f3s():
    import torch
    assert torch.cuda.is_available()
    from paper_2505_08098_b200 import f3s as mod
    return mod


def check_plan(f3s, oracle_mod, csr, n_cols=None, rows_api=False):
    import torch
    n_cols = csr.n_cols if n_cols is None else n_cols
    rp, ci = csr_to_dev(csr)
    p = f3s.plan_rows(rp, ci, csr.n_rows, n_cols) if rows_api else f3s.plan(rp, ci, csr.n_rows)
    torch.cuda.synchronize()
    rw_ptr, cols, masks, order = p.export()
    ref = oracle_mod.plan(csr.row_ptr - csr.row_ptr[0], csr.col_idx[csr.row_ptr[0]:], n_cols)
    assert np.array_equal(rw_ptr, ref.rw_ptr)
    assert np.array_equal(cols, ref.cols)
    assert np.array_equal(masks, ref.masks)
    assert np.array_equal(order, ref.rw_order)
    info = p.info()
    assert info["num_rw"] == ref.num_rw and info["total_cols"] == len(ref.cols)
    assert info["total_tcb8"] == int(ref.tcb8.sum())
    assert info["nnz"] == int(sum(bin(int(m)).count("1") for m in ref.masks))
    return p


@pytest.mark.parametrize("n,dmin,dmax,seed", [(1, 1, 1, 1), (15, 0, 3, 2), (16, 0, 5, 3), (17, 1, 4, 4),
                                              (33, 0, 0, 5), (1000, 0, 30, 6), (5000, 2, 9, 7), (20011, 0, 60, 8)])
def test_plan_random_raw_csr(f3s, oracle_mod, n, dmin, dmax, seed):
    # duplicates and unsorted rows are merged (reading c2)
    csr = fi.random_csr(n, n, dmin, dmax, keep_dups=True, unsorted=True, seed=seed)
    check_plan(f3s, oracle_mod, csr)


def test_plan_hub_row_and_ragged(f3s, oracle_mod):
    n = 70_003
    rp = [0]
    cols = []
    rng = np.random.default_rng(0)
    for r in range(n):
        if r == 5:
            c = np.arange(n)  # hub row: every column (> 64K compacted columns in one RW)
        elif r % 97 == 0:
            c = rng.integers(0, n, 40)
        else:
            c = np.zeros(0, np.int64)
        cols.extend(c.tolist())
        rp.append(len(cols))
    csr = fi.CSR(n, n, np.array(rp, np.int32), np.array(cols, np.int32))
    check_plan(f3s, oracle_mod, csr)


def test_plan_generators(f3s, oracle_mod):
    check_plan(f3s, oracle_mod, fi.chung_lu(2708, 5278, gamma=2.7, max_deg=170, self_loops=True, seed=1001))
    check_plan(f3s, oracle_mod, fi.molecules(300, seed=5))


def test_plan_rows_rectangular_with_base(f3s, oracle_mod):
    import torch
    g = fi.chung_lu(4000, 20000, gamma=2.5, max_deg=200, seed=3)
    for b, e in [(0, 4000), (16, 1000), (1600, 4000), (48, 48)]:
        sub = fi.CSR(e - b, 4000, g.row_ptr[b:e + 1], g.col_idx)
        rp = torch.from_numpy(g.row_ptr).cuda()[b:e + 1]
        ci = torch.from_numpy(g.col_idx).cuda()
        p = f3s.plan_rows(rp, ci, e - b, 4000)
        rw_ptr, cols, masks, order = p.export()
        ref = oracle_mod.plan(sub.row_ptr - sub.row_ptr[0], g.col_idx[sub.row_ptr[0]:sub.row_ptr[-1]], 4000)
        assert np.array_equal(rw_ptr, ref.rw_ptr) and np.array_equal(cols, ref.cols)
        assert np.array_equal(masks, ref.masks) and np.array_equal(order, ref.rw_order)


def test_plan_empty(f3s, oracle_mod):
    csr = fi.CSR(0, 0, np.zeros(1, np.int32), np.zeros(0, np.int32))
    import torch
    p = f3s.plan(torch.zeros(1, dtype=torch.int32, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda"), 0)
    assert p.info()["num_rw"] == 0
    check_plan(f3s, oracle_mod, fi.CSR(40, 40, np.zeros(41, np.int32), np.zeros(0, np.int32)))


def test_plan_invalid_csr(f3s):
    import torch
    dev = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    with pytest.raises(f3s.F3SError) as e:
        f3s.plan(dev([0, 2]), dev([0, 3]), 1)  # column 3 >= n = 1
    assert e.value.status == f3s.INVALID_CSR
    with pytest.raises(f3s.F3SError) as e:
        f3s.plan(dev([1, 2]), dev([0, 0]), 1)  # row_ptr[0] != 0
    assert e.value.status == f3s.INVALID_CSR
    with pytest.raises(f3s.F3SError) as e:
        f3s.plan(dev([0, 2, 1]), dev([0, 1]), 2)  # decreasing
    assert e.value.status == f3s.INVALID_CSR
    with pytest.raises(f3s.F3SError) as e:
        f3s.plan(dev([0, 1]), dev([-1]), 1)
    assert e.value.status == f3s.INVALID_CSR
    # the library stays usable after errors
    p = f3s.plan(dev([0, 1]), dev([0]), 1)
    assert p.info()["nnz"] == 1


def test_plan_deterministic(f3s):
    csr = fi.random_csr(3000, 3000, 0, 25, keep_dups=True, unsorted=True, seed=9)
    rp, ci = csr_to_dev(csr)
    a = f3s.plan(rp, ci, 3000).export()
    b = f3s.plan(rp, ci, 3000).export()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
