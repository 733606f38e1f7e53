"""Pins for oracle.plan (BSB-equivalent plan, RW reordering P:402).

Worked examples from SPEC.md, brute-force support
round-trips, and the invariants of S:111-116 / S:168.
"""
import numpy as np
import pytest

from conftest import csr_from_dense, dense_from_csr


def plan_of_dense(oracle_mod, A):
    rp, ci = csr_from_dense(A)
    return oracle_mod.plan(rp, ci, A.shape[1])


def support_from_plan(p, n_rows, n_cols):
    """to_dense of the plan: (16k+i, cols[q]) for every set bit i of masks[q] in RW k."""
    A = np.zeros((n_rows, n_cols), bool)
    for k in range(p.num_rw):
        for q in range(p.rw_ptr[k], p.rw_ptr[k + 1]):
            for i in range(16):
                if (int(p.masks[q]) >> i) & 1:
                    A[16 * k + i, p.cols[q]] = True
    return A


def test_empty_16x16(oracle_mod):
    p = plan_of_dense(oracle_mod, np.zeros((16, 16), bool))
    assert p.num_rw == 1 and list(p.rw_ptr) == [0, 0] and len(p.cols) == 0 and list(p.rw_order) == [0]


def test_identity_16(oracle_mod):
    p = plan_of_dense(oracle_mod, np.eye(16, dtype=bool))
    assert list(p.rw_ptr) == [0, 16] and list(p.cols) == list(range(16))
    assert list(p.masks) == [1 << i for i in range(16)]
    assert list(p.tcb8) == [2]
    assert sum(bin(int(m)).count("1") for m in p.masks) == 16
    # BSB footprint 32(N/r + bc) + b*r*c (Tab.format_compare) = 800 bits on this matrix
    N, r, c = 16, 16, 8
    bc, b = len(p.cols), int(p.tcb8.sum())
    assert 32 * (N // r + bc) + b * r * c == 800


def test_lpt_example(oracle_mod):  # TCB counts [2,5,5,1] -> order [1,2,0,3]
    widths = [16, 40, 33, 8]
    A = np.zeros((64, 64), bool)
    for k, w in enumerate(widths):
        A[16 * k, :w] = True
    p = plan_of_dense(oracle_mod, A)
    assert list(p.tcb8) == [2, 5, 5, 1]
    assert list(p.rw_order) == [1, 2, 0, 3]


def test_lpt_ties_identity(oracle_mod):
    A = np.zeros((64, 64), bool)
    for k in range(4):
        A[16 * k + 3, 10:20] = True
    assert list(plan_of_dense(oracle_mod, A).rw_order) == [0, 1, 2, 3]


@pytest.mark.parametrize("n_rows,n_cols,dmax,seed", [(1, 1, 1, 1), (15, 15, 4, 2), (16, 30, 9, 3), (17, 17, 5, 4),
                                                     (100, 100, 12, 5), (333, 80, 20, 6), (64, 5000, 3, 7)])
def test_roundtrip_and_invariants(oracle_mod, inputs_mod, n_rows, n_cols, dmax, seed):
    raw = inputs_mod.random_csr(n_rows, n_cols, 0, dmax, keep_dups=True, unsorted=True, seed=seed)
    A = dense_from_csr(raw.row_ptr, raw.col_idx, n_rows, n_cols)
    p = oracle_mod.plan(raw.row_ptr, raw.col_idx, n_cols)
    R = (n_rows + 15) // 16
    assert p.num_rw == R and p.rw_ptr[0] == 0 and np.all(np.diff(p.rw_ptr) >= 0)
    # exact support reconstruction and popcount = nnz of the deduplicated A
    assert np.array_equal(support_from_plan(p, n_rows, n_cols), A)
    assert sum(bin(int(m)).count("1") for m in p.masks) == int(A.sum())
    for k in range(R):
        cols = p.cols[p.rw_ptr[k]:p.rw_ptr[k + 1]]
        # strictly increasing; exactly the columns with >= 1 nonzero in the RW
        assert np.all(np.diff(cols) > 0)
        assert set(cols.tolist()) == set(np.nonzero(A[16 * k:16 * k + 16].any(0))[0].tolist())
        assert np.all(p.masks[p.rw_ptr[k]:p.rw_ptr[k + 1]] != 0)
        # width bound: 8(t-1) < w <= 8t
        w, t = len(cols), int(p.tcb8[k])
        assert (w == 0 and t == 0) or (8 * (t - 1) < w <= 8 * t)
    # reorder: permutation sorted by (tcb desc, index asc), checked with Python's stable sort
    assert sorted(p.rw_order.tolist()) == list(range(R))
    assert p.rw_order.tolist() == sorted(range(R), key=lambda k: -int(p.tcb8[k]))
    # duplicates / unsorted rows give the same canonical plan as the clean CSR
    rp, ci = csr_from_dense(A)
    q = oracle_mod.plan(rp, ci, n_cols)
    for a, b in [(p.rw_ptr, q.rw_ptr), (p.cols, q.cols), (p.masks, q.masks), (p.rw_order, q.rw_order)]:
        assert np.array_equal(a, b)


def test_invalid_csr(oracle_mod):
    with pytest.raises(ValueError):
        oracle_mod.plan(np.array([0, 2], np.int32), np.array([0, 3], np.int32), 3)
    with pytest.raises(ValueError):
        oracle_mod.plan(np.array([1, 2], np.int32), np.array([0, 0], np.int32), 3)
    with pytest.raises(ValueError):
        oracle_mod.plan(np.array([0, 2, 1], np.int32), np.array([0, 1], np.int32), 3)


def test_zero_rows(oracle_mod):
    p = oracle_mod.plan(np.array([0], np.int32), np.zeros(0, np.int32), 0)
    assert p.num_rw == 0 and list(p.rw_ptr) == [0]
