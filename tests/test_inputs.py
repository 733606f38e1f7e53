"""The seeded input generators: bit-exact against a numpy re-implementation of the
counter-based splitmix64 stream + library RNE casts, and structural checks of the graphs."""
import numpy as np
import pytest

from conftest import dense_from_csr, encode

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def np_splitmix(seed: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


@pytest.mark.parametrize("dtype,amp", [("fp16", 1.0), ("bf16", 1.0), ("fp16", 16.0), ("bf16", 0.0625)])
def test_values_match_numpy(inputs_mod, dtype, amp):
    n = 50_000
    got = inputs_mod.values((n,), seed=12345, dtype=dtype, amp=amp, offset=77)
    z = np_splitmix(12345, np.arange(n) + 77)
    f = ((z >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)) * np.float32(amp)
    assert np.array_equal(got, encode(f, dtype))


def test_values_slices_regenerate(inputs_mod):
    full = inputs_mod.values((1000,), seed=5)
    part = inputs_mod.values((100,), seed=5, offset=450)
    assert np.array_equal(full[450:550], part)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_rne_rounding_edges(inputs_mod, dtype):
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 3,
                        rng.uniform(-1e-6, 1e-6, 2000).astype(np.float32),     # fp16 subnormals
                        np.array([65504, 65519.99, 65520, -7e4, 0.0, -0.0, 2 ** -24, 2 ** -25, 3 * 2 ** -26], np.float32)])
    assert np.array_equal(inputs_mod.round_f32(x, dtype), encode(x, dtype))


def check_csr(csr, n_cols):
    assert csr.row_ptr[0] == 0 and np.all(np.diff(csr.row_ptr) >= 0)
    for r in range(csr.n_rows):
        c = csr.col_idx[csr.row_ptr[r]:csr.row_ptr[r + 1]]
        assert np.all(np.diff(c) > 0) and (len(c) == 0 or (c[0] >= 0 and c[-1] < n_cols))


def test_chung_lu_undirected(inputs_mod):
    c = inputs_mod.chung_lu(500, 1200, gamma=2.7, max_deg=60, seed=3)
    check_csr(c, 500)
    A = dense_from_csr(c.row_ptr, c.col_idx, 500, 500)
    assert np.array_equal(A, A.T) and not A.diagonal().any() and c.nnz == 2400
    c2 = inputs_mod.chung_lu(500, 1200, gamma=2.7, max_deg=60, seed=3, self_loops=True)
    assert c2.nnz == 2900 and dense_from_csr(c2.row_ptr, c2.col_idx, 500, 500).diagonal().all()
    assert np.array_equal(inputs_mod.chung_lu(500, 1200, gamma=2.7, max_deg=60, seed=3).col_idx, c.col_idx)


def test_chung_lu_directed(inputs_mod):
    c = inputs_mod.chung_lu(800, 3000, directed=True, gamma=2.5, max_deg=80, gamma_in=2.2, max_deg_in=150,
                            symmetrize=False, seed=4)
    check_csr(c, 800)
    assert c.nnz == 3000


def test_molecules(inputs_mod):
    c = inputs_mod.molecules(50, 25, 150, seed=9)
    check_csr(c, c.n_cols)
    gp = c.graph_ptr
    assert gp[0] == 0 and gp[-1] == c.n_rows and np.all(np.diff(gp) >= 25) and np.all(np.diff(gp) <= 150)
    A = dense_from_csr(c.row_ptr, c.col_idx, c.n_rows, c.n_rows)
    assert np.array_equal(A, A.T)
    g = np.searchsorted(gp, np.arange(c.n_rows), side="right") - 1
    r, col = np.nonzero(A)
    assert np.all(g[r] == g[col])  # block-diagonal
    # every graph is connected (tree backbone)
    for k in range(len(gp) - 1):
        b, e = gp[k], gp[k + 1]
        seen, stack = {b}, [b]
        while stack:
            u = stack.pop()
            for v in c.col_idx[c.row_ptr[u]:c.row_ptr[u + 1]]:
                if v not in seen:
                    seen.add(int(v)); stack.append(int(v))
        assert len(seen) == e - b


def test_dcsbm(inputs_mod):
    c = inputs_mod.dcsbm(2000, 20000, comm_size=200, mu=0.8, gamma=2.3, max_deg=300, seed=11)
    check_csr(c, 2000)
    A = dense_from_csr(c.row_ptr, c.col_idx, 2000, 2000)
    assert np.array_equal(A, A.T) and c.nnz == 40000
    r, col = np.nonzero(A)
    assert np.mean(r // 200 == col // 200) > 0.6
