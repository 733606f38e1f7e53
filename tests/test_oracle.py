"""Pins for oracle.attention (Eq.1 / Eq.7) against things other than itself.

Each check is chosen so that a plausible mistake in the oracle (dropped max subtraction,
softmax over non-edges, wrong operand index, transposed K, head mix-up, missing dedup,
NaN on empty rows) fails at least one of them.
"""
import numpy as np
import pytest
import scipy.special
import torch

from conftest import csr_from_dense, decode, dense_from_csr, encode

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def rand_bits(rng, shape, dtype, amp=1.0):
    return encode(rng.uniform(-amp, amp, size=shape), dtype)


def dense_bruteforce(A, Q, K, V, scale):
    """Materialise S = scale*Q K^T (n x n) per head, -inf off the support of A, library
    softmax per row (scipy), dense product with V.  Rows without support give 0."""
    n, H, d = Q.shape
    O = np.zeros((n, H, d))
    for h in range(H):
        S = scale * Q[:, h, :] @ K[:, h, :].T
        S = np.where(A, S, -np.inf)
        has = A.any(1)
        E = np.zeros_like(S)
        E[has] = scipy.special.softmax(S[has], axis=1)
        O[:, h, :] = E @ V[:, h, :]
    return O


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
@pytest.mark.parametrize("n,density,H,d", [(1, 1.0, 1, 8), (17, 0.3, 2, 16), (48, 0.1, 3, 32), (64, 0.05, 1, 64)])
def test_dense_bruteforce(oracle_mod, dtype, n, density, H, d):
    rng = np.random.default_rng(n * 7 + H)
    A = rng.random((n, n)) < density
    A[rng.integers(0, n)] = False  # at least one empty row
    Qb, Kb, Vb = (rand_bits(rng, (n, H, d), dtype) for _ in range(3))
    rp, ci = csr_from_dense(A)
    scale = 1.0 / np.sqrt(d)
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=scale, dtype=dtype)
    ref = dense_bruteforce(A, decode(Qb, dtype), decode(Kb, dtype), decode(Vb, dtype), scale)
    np.testing.assert_allclose(O, ref, rtol=0, atol=1e-12)


def sdpa(Qf, Kf, Vf, scale, **kw):
    """torch SDPA in fp64 on CPU over heads: inputs [n, H, d] -> [n, H, d]."""
    q, k, v = (torch.from_numpy(np.ascontiguousarray(x.transpose(1, 0, 2))) for x in (Qf, Kf, Vf))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, scale=scale, **kw)
    return o.numpy().transpose(1, 0, 2)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_sdpa_all_ones(oracle_mod, dtype):
    rng = np.random.default_rng(1)
    n, H, d = 40, 2, 32
    Qb, Kb, Vb = (rand_bits(rng, (n, H, d), dtype) for _ in range(3))
    rp, ci = csr_from_dense(np.ones((n, n), bool))
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=0.3, dtype=dtype)
    ref = sdpa(decode(Qb, dtype), decode(Kb, dtype), decode(Vb, dtype), 0.3)
    np.testing.assert_allclose(O, ref, rtol=0, atol=1e-12)


def test_sdpa_causal(oracle_mod):
    rng = np.random.default_rng(2)
    n, H, d = 50, 3, 16
    Qb, Kb, Vb = (rand_bits(rng, (n, H, d), "fp16", 2.0) for _ in range(3))
    rp, ci = csr_from_dense(np.tril(np.ones((n, n), bool)))
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=1.0, dtype="fp16")
    ref = sdpa(decode(Qb, "fp16"), decode(Kb, "fp16"), decode(Vb, "fp16"), 1.0, is_causal=True)
    np.testing.assert_allclose(O, ref, rtol=0, atol=1e-12)


def test_sdpa_bool_mask_and_block_diagonal(oracle_mod):
    rng = np.random.default_rng(3)
    n, H, d = 60, 2, 8
    Qb, Kb, Vb = (rand_bits(rng, (n, H, d), "fp16") for _ in range(3))
    Q, K, V = (decode(x, "fp16") for x in (Qb, Kb, Vb))
    # random boolean mask, every row non-empty (SDPA gives NaN on empty rows)
    A = rng.random((n, n)) < 0.2
    A[np.arange(n), rng.integers(0, n, n)] = True
    rp, ci = csr_from_dense(A)
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=0.5, dtype="fp16")
    ref = sdpa(Q, K, V, 0.5, attn_mask=torch.from_numpy(A))
    np.testing.assert_allclose(O, ref, rtol=0, atol=1e-12)
    # block-diagonal (batched graphs): per-block dense SDPA
    sizes = [7, 13, 1, 20, 19]
    A = np.zeros((n, n), bool)
    b = 0
    for s in sizes:
        A[b:b + s, b:b + s] = True
        b += s
    rp, ci = csr_from_dense(A)
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=0.25, dtype="fp16")
    b = 0
    for s in sizes:
        ref = sdpa(Q[b:b + s], K[b:b + s], V[b:b + s], 0.25)
        np.testing.assert_allclose(O[b:b + s], ref, rtol=0, atol=1e-12)
        b += s


def test_self_loops_copy_v_exactly(oracle_mod):
    rng = np.random.default_rng(4)
    n, H, d = 33, 2, 16
    Qb, Kb, Vb = (rand_bits(rng, (n, H, d), "fp16", 4.0) for _ in range(3))
    rp = np.arange(n + 1, dtype=np.int32)
    ci = np.arange(n, dtype=np.int32)
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=1.0, dtype="fp16")
    assert np.array_equal(O, decode(Vb, "fp16"))  # softmax of one finite score is exactly 1


def test_single_neighbour_copies_v(oracle_mod):
    rng = np.random.default_rng(5)
    n, H, d = 20, 1, 8
    Qb, Kb, Vb = (rand_bits(rng, (n, H, d), "bf16") for _ in range(3))
    nb = rng.integers(0, n, n).astype(np.int32)
    O = oracle_mod.attention(np.arange(n + 1, dtype=np.int32), nb, Qb, Kb, Vb, scale=2.0, dtype="bf16")
    assert np.array_equal(O, decode(Vb, "bf16")[nb])


@pytest.mark.parametrize("how", ["q_zero", "scale_zero", "k_identical"])
def test_uniform_weights_give_neighbour_mean(oracle_mod, how):
    rng = np.random.default_rng(6)
    n, H, d = 30, 2, 16
    Qb, Kb, Vb = (rand_bits(rng, (n, H, d), "fp16") for _ in range(3))
    scale = 0.7
    if how == "q_zero":
        Qb[:] = 0
    elif how == "scale_zero":
        scale = 0.0
    else:
        Kb[:] = Kb[0]
    A = rng.random((n, n)) < 0.25
    A[0] = False
    rp, ci = csr_from_dense(A)
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=scale, dtype="fp16")
    V = decode(Vb, "fp16")
    for i in range(n):
        ref = V[A[i]].mean(0) if A[i].any() else np.zeros((H, d))
        np.testing.assert_allclose(O[i], ref, rtol=0, atol=1e-14)


def test_two_neighbours_sigmoid(oracle_mod):
    # scores differ by delta -> weights sigma(delta), 1 - sigma(delta)
    d = 4
    Qb = encode(np.array([[[1.0, 0, 0, 0]]] * 3), "fp16")
    Kb = encode(np.array([[[0.0, 0, 0, 0]], [[0.75, 0, 0, 0]], [[-1.5, 0, 0, 0]]]), "fp16")
    Vb = encode(np.array([[[0.0] * d], [[1.0, 2.0, -1.0, 0.5]], [[-2.0, 0.25, 1.0, 3.0]]]), "fp16")
    rp = np.array([0, 2, 2, 2], np.int32)
    ci = np.array([1, 2], np.int32)
    scale = 1.5
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=scale, dtype="fp16")
    delta = scale * (0.75 - (-1.5))
    w = 1.0 / (1.0 + np.exp(-delta))
    ref = w * decode(Vb, "fp16")[1, 0] + (1 - w) * decode(Vb, "fp16")[2, 0]
    np.testing.assert_allclose(O[0, 0], ref, rtol=0, atol=1e-15)
    assert np.all(O[1:] == 0)  # empty rows -> exact zeros (reading c4)


def test_invariants(oracle_mod, inputs_mod):
    csr = inputs_mod.random_csr(70, 70, 0, 9, seed=7)
    n, H, d = 70, 3, 16
    rng = np.random.default_rng(7)
    # values on a 2^-4 grid in [-2, 2) so that K + u stays exact in fp16
    grid = lambda: encode(np.round(rng.uniform(-2, 2, (n, H, d)) * 16) / 16, "fp16")
    Qb, Kb, Vb = grid(), grid(), grid()
    O = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.5, dtype="fp16")
    nonempty = np.diff(csr.row_ptr) > 0
    assert np.all(O[~nonempty] == 0)
    # V == 1 -> O == 1 on non-empty rows (weights sum to 1)
    ones = encode(np.ones((n, H, d)), "fp16")
    O1 = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, ones, scale=0.5, dtype="fp16")
    np.testing.assert_allclose(O1[nonempty], 1.0, rtol=0, atol=1e-14)
    # shifting every K row by the same u changes each row's scores by a constant
    u = np.round(rng.uniform(-1, 1, (1, H, d)) * 16) / 16
    Ks = encode(decode(Kb, "fp16") + u, "fp16")
    assert np.array_equal(decode(Ks, "fp16"), decode(Kb, "fp16") + u)
    Os = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Ks, Vb, scale=0.5, dtype="fp16")
    np.testing.assert_allclose(Os, O, rtol=0, atol=1e-12)
    # relabelling nodes permutes O
    perm = rng.permutation(n)
    inv = np.argsort(perm)
    A = dense_from_csr(csr.row_ptr, csr.col_idx, n, n)
    rp2, ci2 = csr_from_dense(A[perm][:, perm])
    Op = oracle_mod.attention(rp2, ci2, Qb[perm], Kb[perm], Vb[perm], scale=0.5, dtype="fp16")
    np.testing.assert_allclose(Op[inv], O, rtol=0, atol=1e-12)
    # heads are independent
    Kh = Kb.copy()
    Kh[:, 1] = grid()[:, 1]
    Oh = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kh, Vb, scale=0.5, dtype="fp16")
    assert np.array_equal(Oh[:, 0], O[:, 0]) and np.array_equal(Oh[:, 2], O[:, 2])


def test_duplicates_and_unsorted_rows_merge(oracle_mod, inputs_mod):
    raw = inputs_mod.random_csr(40, 40, 1, 12, keep_dups=True, unsorted=True, seed=8)
    A = dense_from_csr(raw.row_ptr, raw.col_idx, 40, 40)
    rp, ci = csr_from_dense(A)
    rng = np.random.default_rng(8)
    Qb, Kb, Vb = (rand_bits(rng, (40, 2, 8), "fp16") for _ in range(3))
    O1 = oracle_mod.attention(raw.row_ptr, raw.col_idx, Qb, Kb, Vb, scale=1.0)
    O2 = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=1.0)
    assert np.array_equal(O1, O2)


def test_large_scores_stay_finite(oracle_mod):
    # Eq.6 would overflow beyond ~e^89 in fp32; Eq.7 must not.
    rng = np.random.default_rng(9)
    n, H, d = 32, 1, 64
    Qb, Kb = (rand_bits(rng, (n, H, d), "fp16", 16.0) for _ in range(2))
    Vb = rand_bits(rng, (n, H, d), "fp16")
    A = rng.random((n, n)) < 0.5
    rp, ci = csr_from_dense(A)
    O = oracle_mod.attention(rp, ci, Qb, Kb, Vb, scale=1.0)
    S = decode(Qb, "fp16")[:, 0] @ decode(Kb, "fp16")[:, 0].T
    assert np.abs(S[A]).max() > 500  # scores far beyond the fp32 exp range
    assert np.all(np.isfinite(O))
    ref = dense_bruteforce(A, decode(Qb, "fp16"), decode(Kb, "fp16"), decode(Vb, "fp16"), 1.0)
    np.testing.assert_allclose(O, ref, rtol=0, atol=1e-12)


def test_row_subset_and_rectangular(oracle_mod, inputs_mod):
    csr = inputs_mod.random_csr(37, 90, 0, 6, seed=10)
    rng = np.random.default_rng(10)
    Qb = rand_bits(rng, (37, 2, 16), "bf16")
    Kb, Vb = (rand_bits(rng, (90, 2, 16), "bf16") for _ in range(2))
    O = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.25, dtype="bf16")
    A = dense_from_csr(csr.row_ptr, csr.col_idx, 37, 90)
    Q, K, V = decode(Qb, "bf16"), decode(Kb, "bf16"), decode(Vb, "bf16")
    ref = np.zeros_like(O)
    for h in range(2):
        S = np.where(A, 0.25 * Q[:, h] @ K[:, h].T, -np.inf)
        has = A.any(1)
        ref[has, h] = scipy.special.softmax(S[has], axis=1) @ V[:, h]
    np.testing.assert_allclose(O, ref, rtol=0, atol=1e-12)
    rows = np.array([36, 0, 5, 5], np.int32)
    Os = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.25, dtype="bf16", rows=rows)
    assert np.array_equal(Os, O[rows])


def test_invalid_csr_rejected(oracle_mod):
    Qb = np.zeros((2, 1, 8), np.uint16)
    with pytest.raises(ValueError):
        oracle_mod.attention(np.array([0, 1, 2], np.int32), np.array([0, 5], np.int32), Qb, Qb, Qb, scale=1.0)
