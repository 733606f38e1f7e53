"""Pins of the oracle's backward (oracle_attention_backward) against things other
than itself: central finite differences of the fp64 forward, torch autograd of dense masked
attention in fp64 (library routine), and closed forms / invariants of the softmax Jacobian."""
import numpy as np
import pytest

import f3s_inputs as fi
from conftest import decode


def _graph(n, seed, deg_min=0, deg_max=5):
    return fi.random_csr(n, n, deg_min, deg_max, keep_dups=True, unsorted=True, seed=seed)


def _inputs(n, H, d, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, H, d)), rng.standard_normal((n, H, d)), rng.standard_normal((n, H, d)),
            rng.standard_normal((n, H, d)))


def test_f64_forward_equals_the_fp16_oracle(oracle_mod):
    csr = _graph(40, 1)
    Qb, Kb, Vb = (fi.values((40, 2, 8), seed=s, dtype="fp16") for s in (11, 12, 13))
    ref = oracle_mod.attention(csr.row_ptr, csr.col_idx, Qb, Kb, Vb, scale=0.3)
    got = oracle_mod.attention_f64(csr.row_ptr, csr.col_idx, decode(Qb, "fp16"), decode(Kb, "fp16"),
                                   decode(Vb, "fp16"), scale=0.3)
    assert np.max(np.abs(got - ref)) <= 1e-13


@pytest.mark.parametrize("seed", [2, 3])
def test_central_finite_differences(oracle_mod, seed):
    # L = <O, G>: dL/dX from the backward vs (L(X + eps e) - L(X - eps e)) / 2 eps per entry
    n, H, d, scale = 12, 2, 3, 0.7
    csr = _graph(n, seed)
    Q, K, V, G = _inputs(n, H, d, seed)
    dQ, dK, dV = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, Q, K, V, G, scale=scale)
    L = lambda q, k, v: float(np.sum(oracle_mod.attention_f64(csr.row_ptr, csr.col_idx, q, k, v, scale=scale) * G))
    eps = 1e-6
    for X, dX, which in ((Q, dQ, 0), (K, dK, 1), (V, dV, 2)):
        fd = np.zeros_like(X)
        for idx in np.ndindex(X.shape):
            Xp, Xm = X.copy(), X.copy()
            Xp[idx] += eps
            Xm[idx] -= eps
            args_p = [Q, K, V]
            args_m = [Q, K, V]
            args_p[which], args_m[which] = Xp, Xm
            fd[idx] = (L(*args_p) - L(*args_m)) / (2 * eps)
        assert np.max(np.abs(fd - dX)) <= 1e-7 * max(1.0, float(np.max(np.abs(dX))))


def test_torch_autograd_dense_masked_attention(oracle_mod):
    import torch
    n, H, d, scale = 48, 3, 8, 0.25
    csr = _graph(n, 5, deg_min=1, deg_max=9)  # every row has a neighbour (SDPA of an empty row is NaN)
    Q, K, V, G = _inputs(n, H, d, 9)
    mask = np.zeros((n, n), bool)
    for i in range(n):
        mask[i, csr.col_idx[csr.row_ptr[i]:csr.row_ptr[i + 1]]] = True
    tq, tk, tv = (torch.tensor(x.transpose(1, 0, 2), requires_grad=True) for x in (Q, K, V))
    out = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=torch.tensor(mask), scale=scale)
    out.backward(torch.tensor(G.transpose(1, 0, 2)))
    dQ, dK, dV = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, Q, K, V, G, scale=scale)
    for ours, t in ((dQ, tq), (dK, tk), (dV, tv)):
        assert np.max(np.abs(ours - t.grad.numpy().transpose(1, 0, 2))) <= 1e-12


def test_closed_forms_and_invariants(oracle_mod):
    n, H, d, scale = 64, 2, 5, 0.5
    csr = _graph(n, 7)
    Q, K, V, G = _inputs(n, H, d, 4)
    dQ, dK, dV = oracle_mod.attention_backward(csr.row_ptr, csr.col_idx, Q, K, V, G, scale=scale)
    nonempty = np.diff(csr.row_ptr) > 0
    # sum_j ds_ij = 0 for every row, so the key gradients of each head sum to zero ...
    assert np.max(np.abs(dK.sum(0))) <= 1e-12
    # ... and the softmax weights sum to one, so the value gradients sum to the non-empty rows' dO
    assert np.max(np.abs(dV.sum(0) - G[nonempty].sum(0))) <= 1e-12
    assert np.all(dQ[~nonempty] == 0)
    # a single neighbour: p = 1 is constant, dQ = dK = 0 and dV_j collects dO_i
    rp = np.arange(n + 1, dtype=np.int32)
    ci = ((np.arange(n) * 7) % n).astype(np.int32)  # a permutation
    dQ1, dK1, dV1 = oracle_mod.attention_backward(rp, ci, Q, K, V, G, scale=scale)
    assert np.all(dQ1 == 0) and np.all(dK1 == 0)
    assert np.array_equal(dV1[ci], G)
