"""CPU pin of reading c24 (FP8 inputs): the per-row error bound the GPU
tests use for E4M3 P,

    |O_i - O_ref_i| <= (2^-4 + deg_i * 2^-18) * max_{j in N(i)} |V_j|,

checked on a plain numpy emulation of the reading (E = 2^8 e^{S - m} rounded to E4M3 by torch's
cast, l summing the unrounded E) against the fp64 oracle, including the adversarial cases the bound
is derived for: weights just above a rounding tie (relative error -> 2^-4) and weights below E4M3's
normal range (absolute error 2^-10 on the 2^8 scale).  No GPU."""
import numpy as np
import pytest

import f3s_inputs as fi


def _e4m3(x):
    import torch
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.float8_e4m3fn).to(torch.float64).numpy()


def _emulate(row_ptr, col_idx, Q, K, V, scale, offset=8.0):
    n, H, d = Q.shape
    O = np.zeros((n, H, d))
    for i in range(n):
        cols = np.unique(col_idx[row_ptr[i]:row_ptr[i + 1]])  # A is 0/1: duplicates count once (reading c2)
        if len(cols) == 0:
            continue
        for h in range(H):
            s = scale * (K[cols, h] @ Q[i, h])
            e = np.exp2((s - s.max()) * np.log2(np.e) + offset)  # 2^8 e^{S - m}
            O[i, h] = (_e4m3(e) @ V[cols, h]) / e.sum()
    return O


def _bound(row_ptr, col_idx, V):
    deg = np.diff(row_ptr)
    out = np.zeros((len(deg), V.shape[1]))
    for i, k in enumerate(deg):
        if k:
            out[i] = (2.0 ** -4 + k * 2.0 ** -18) * np.abs(V[col_idx[row_ptr[i]:row_ptr[i + 1]]]).max(axis=(0, 2))
    return out


def test_bound_holds_on_random_inputs(oracle_mod):
    csr = fi.random_csr(200, 200, 0, 60, keep_dups=True, seed=31)
    rng = np.random.default_rng(3)
    Q, K, V = (_e4m3(rng.uniform(-1, 1, (200, 2, 16))) for _ in range(3))
    ref = oracle_mod.attention_f64(csr.row_ptr, csr.col_idx, Q, K, V, scale=0.5)
    got = _emulate(csr.row_ptr, csr.col_idx, Q, K, V, 0.5)
    err = np.abs(got - ref).max(axis=2)
    b = _bound(csr.row_ptr, csr.col_idx, V)
    assert np.all(err <= b * (1 + 1e-9) + 1e-12)
    assert err.max() > 1e-3  # the rounding of P is really there (not a vacuous comparison)


def test_bound_is_reached_by_a_tie_case(oracle_mod):
    # one row, two neighbours: E = 2^8 and 2^8 * (1 - 2^-5) -> rounds to 2^8 (1 - 2^-4) ... the second
    # weight's relative error approaches 2^-4; O moves by about 2^-5 of |V| (half the bound)
    rp = np.array([0, 2], np.int32)
    ci = np.array([0, 1], np.int32)
    d = 1
    V = np.array([[[1.0]], [[-1.0]]])
    K = np.zeros((2, 1, d))
    Q = np.zeros((1, 1, d))
    s1 = np.log(1 - 2.0 ** -5 * 1.01)  # score gap that puts E_2 just past a rounding tie
    K[1, 0, 0] = s1
    Q[0, 0, 0] = 1.0
    ref = oracle_mod.attention_f64(rp, ci, Q, K, V, scale=1.0)
    got = _emulate(rp, ci, Q, K, V, 1.0)
    err = float(np.abs(got - ref).max())
    b = float(_bound(rp, ci, V).max())
    assert 0.2 * b < err <= b


@pytest.mark.parametrize("offset", [8.0, 0.0])
def test_tiny_weights_and_the_offset(oracle_mod, offset):
    # one dominant neighbour and many with weights e^-12 ~ 6e-6: below E4M3's normal range (2^-6)
    # without the 2^8 offset (they flush towards 0 / coarse subnormals), inside it with the offset
    n_nb = 200
    rp = np.array([0, n_nb], np.int32)
    ci = np.arange(n_nb, dtype=np.int32)
    Q = np.ones((1, 1, 1))
    K = np.full((n_nb, 1, 1), -12.0)
    K[0] = 0.0
    V = np.ones((n_nb, 1, 1))
    V[0] = -1.0
    ref = oracle_mod.attention_f64(rp, ci, Q, K, V, scale=1.0)
    got = _emulate(rp, ci, Q, K, V, 1.0, offset=offset)
    err = float(np.abs(got - ref).max())
    if offset == 8.0:
        assert err <= float(_bound(rp, ci, V).max())
    else:
        # the reading's offset is what keeps these weights: without it the error is far larger
        assert err > 3 * float(np.abs(_emulate(rp, ci, Q, K, V, 1.0) - ref).max())
