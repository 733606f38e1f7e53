"""CPU-side checks of libf3s.so: it loads, exports every function include/f3s.h declares, and
its host-only entry points (partitioner, status strings, argument validation) behave."""
import ctypes
import os
import re

import numpy as np
import pytest

import f3s_inputs as fi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def f3s():
    from paper_2505_08098_b200 import build
    build()
    from paper_2505_08098_b200 import f3s as mod
    return mod


def test_exports_every_declared_symbol(f3s):
    header = open(os.path.join(ROOT, "include", "f3s.h")).read()
    declared = set(re.findall(r"^\s*(?:const char\*|f3s_status|int64_t|int32_t)\s+(f3s_\w+)\s*\(", header, re.M))
    assert len(declared) >= 13
    lib = ctypes.CDLL(f3s.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(f3s.EXPORTED)


def test_sass_is_blackwell_native(f3s):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", f3s.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out          # tcgen05.mma (both contractions)
    assert "UTMALDG.2D" in out       # TMA tile load (Q tiles)
    assert "UBLKCP" in out           # cp.async.bulk (column ids / masks into chunk slots)
    assert "LDGSTS" in out           # cp.async gathers of K/V rows
    assert "LDTM" in out             # tcgen05.ld (S^T and O^T out of TMEM)
    assert "UTCQMMA" in out          # tcgen05.mma kind::f8f6f4 (E4M3 inputs, f4)
    assert re.search(r"\s HMMA", out) is None  # no legacy mma.sync path (UTCHMMA is tcgen05)


def test_dtype_codes_match_the_header(f3s):
    import torch
    header = open(os.path.join(ROOT, "include", "f3s.h")).read()
    enum = dict((k, int(v)) for k, v in re.findall(r"(F3S_(?:FP16|BF16|E4M3)) = (\d+)", header))
    assert enum == {"F3S_FP16": f3s.FP16, "F3S_BF16": f3s.BF16, "F3S_E4M3": f3s.E4M3}
    for dt, code in ((torch.float16, f3s.FP16), (torch.bfloat16, f3s.BF16), (torch.float8_e4m3fn, f3s.E4M3)):
        assert f3s._dtype_code(torch.zeros(1, dtype=dt)) == code
    with pytest.raises(TypeError):
        f3s._dtype_code(torch.zeros(1, dtype=torch.float32))


def test_status_strings(f3s):
    assert f3s._lib.f3s_status_string(2) == b"F3S_ERR_INVALID_CSR"
    assert f3s._lib.f3s_status_string(0) == b"F3S_OK"


def test_host_argument_validation(f3s):
    # NULL plan is rejected before any CUDA call
    st = f3s._lib.f3s_attention(None, None, None, None, None, 1.0, 1, 64, 0, None)
    assert st == f3s.INVALID_VALUE
    st = f3s._lib.f3s_plan(None, None, 4, None, ctypes.byref(ctypes.c_void_p()))
    assert st == f3s.INVALID_VALUE
    assert b"NULL" in f3s._lib.f3s_last_error()
    assert f3s._lib.f3s_plan_set_split(None, 4) == f3s.INVALID_VALUE
    # the training pair and the backward entry points: NULL plan first
    assert f3s._lib.f3s_attention_fwd(None, None, None, None, None, None, 1.0, 1, 64, 0, None) == f3s.INVALID_VALUE
    for fn in (f3s._lib.f3s_attention_backward_saved, f3s._lib.f3s_attention_backward_saved_lp):
        assert fn(None, None, None, None, None, None, None, None, None, None, 1.0, 1, 64, 0, None) == f3s.INVALID_VALUE
    assert f3s._lib.f3s_attention_backward(None, None, None, None, None, None, None, None, 1.0, 1, 64, 0,
                                           None) == f3s.INVALID_VALUE
    # bad sizes are rejected before any CUDA call too
    assert f3s._lib.f3s_attention_merge(0, None, None, 4, 1, 64, None, None) == f3s.INVALID_VALUE
    assert f3s._lib.f3s_attention_merge(2, None, None, 4, 1, 96, None, None) == f3s.INVALID_VALUE


def nnz_of_range(rp, b, e):
    return int(rp[e] - rp[b])


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_rows_balanced_and_aligned(f3s, parts):
    g = fi.chung_lu(20000, 150000, gamma=2.2, max_deg=2000, seed=2)
    b = f3s.partition_rows(g.row_ptr, parts)
    assert b[0] == 0 and b[-1] == g.n_rows and np.all(np.diff(b) >= 0)
    assert np.all(b[1:-1] % 16 == 0)
    total = g.nnz
    # each cut is the window boundary closest to its target
    for q in range(1, parts):
        target = total * q / parts
        bnd = np.minimum(np.arange(0, g.n_rows + 16, 16), g.n_rows)
        best = np.min(np.abs(g.row_ptr[bnd] - target))
        assert abs(g.row_ptr[b[q]] - target) <= best + 1e-9
    loads = [nnz_of_range(g.row_ptr, b[q], b[q + 1]) for q in range(parts)]
    assert max(loads) <= total / parts + np.diff(g.row_ptr).max() * 16 + 1


def test_partition_at_graph_boundaries(f3s):
    g = fi.molecules(500, seed=3)
    b = f3s.partition_at(g.row_ptr, g.graph_ptr, 4)
    assert set(b.tolist()) <= set(g.graph_ptr.tolist())
    assert b[0] == 0 and b[-1] == g.n_rows


def test_partition_degenerate(f3s):
    rp = np.zeros(1, np.int32)
    assert list(f3s.partition_rows(rp, 3)) == [0, 0, 0, 0]
    rp = np.arange(11, dtype=np.int32)
    b = f3s.partition_rows(rp, 4)
    assert b[0] == 0 and b[-1] == 10 and np.all(np.diff(b) >= 0)
    with pytest.raises(f3s.F3SError):
        f3s.partition_rows(np.array([0, 3, 1], np.int32), 2)
