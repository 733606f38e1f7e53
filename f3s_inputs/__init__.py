"""Seeded synthetic inputs shared by the CUDA path and the oracle.

Holds none of the method's arithmetic: graphs (CSR) shaped like the paper's datasets
(Tab.datasets) and Q/K/V tensors from a counter-based splitmix64 stream
rounded RNE to fp16/bf16 (Tab.mixedp).  The C implementation is
`inputs.c`; this module builds it on demand and wraps it with ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "inputs.c")
_LIB = os.path.join(_HERE, "libf3sinputs.so")
_lib = None

FP16, BF16 = 0, 1
DTYPES = {"fp16": FP16, "bf16": BF16}


def build(force: bool = False) -> str:
    """Compile inputs.c into libf3sinputs.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32, i64, u64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        pp = ctypes.POINTER(ctypes.c_void_p)
        lib.f3si_fill_values.argtypes = [vp, i64, i64, u64, i32, ctypes.c_float]
        lib.f3si_round_f32.argtypes = [vp, vp, i64, i32]
        lib.f3si_chung_lu.argtypes = [i32, i64, i32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, i32, i32, i32, u64, pp, pp, ctypes.POINTER(i64)]
        lib.f3si_dcsbm.argtypes = [i32, i64, i32, ctypes.c_double, ctypes.c_double, ctypes.c_double, u64,
                                   pp, pp, ctypes.POINTER(i64)]
        lib.f3si_dcsbm_w.argtypes = [i32, i64, i32, vp, vp, u64, pp, pp, ctypes.POINTER(i64)]
        lib.f3si_windows.argtypes = [i32, vp, vp, i32, ctypes.c_double, ctypes.c_double, u64, pp, pp, ctypes.POINTER(i64)]
        lib.f3si_molecules.argtypes = [i32, i32, i32, i32, u64, pp, pp, ctypes.POINTER(i64),
                                       ctypes.POINTER(i32), pp]
        lib.f3si_random_csr.argtypes = [i32, i32, i32, i32, i32, i32, u64, pp, pp, ctypes.POINTER(i64)]
        lib.f3si_free.argtypes = [vp]
        _lib = lib
    return _lib


@dataclass
class CSR:
    """Binary sparse matrix A (n_rows x n_cols) in CSR; only the support matters."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # int32[n_rows+1]
    col_idx: np.ndarray  # int32[nnz]
    graph_ptr: np.ndarray | None = None  # batched mode: first node of each graph

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1] - self.row_ptr[0]) if self.n_rows > 0 else 0


def _take(ptr: ctypes.c_void_p, n: int, dtype) -> np.ndarray:
    lib = _load()
    arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(np.ctypeslib.as_ctypes_type(dtype))), shape=(n,)).copy() if n > 0 else np.zeros(0, dtype)
    lib.f3si_free(ptr)
    return arr


def _csr_from(rp, ci, nnz, n_rows, n_cols) -> CSR:
    row_ptr = _take(rp, n_rows + 1, np.int32)
    col_idx = _take(ci, int(nnz.value), np.int32) if nnz.value > 0 else (_load().f3si_free(ci) or np.zeros(0, np.int32))
    return CSR(n_rows, n_cols, row_ptr, col_idx)


def chung_lu(n: int, n_pairs: int, *, directed: bool = False, gamma: float = 2.5, max_deg: float = 100.0,
             gamma_in: float = 2.5, max_deg_in: float = 100.0, symmetrize: bool = True,
             self_loops: bool = False, permute: bool = True, seed: int = 1) -> CSR:
    lib = _load()
    rp, ci, nnz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    rc = lib.f3si_chung_lu(n, n_pairs, int(directed), gamma, max_deg, gamma_in, max_deg_in, int(symmetrize),
                           int(self_loops), int(permute), seed, ctypes.byref(rp), ctypes.byref(ci), ctypes.byref(nnz))
    if rc:
        raise RuntimeError(f"f3si_chung_lu failed ({rc})")
    return _csr_from(rp, ci, nnz, n, n)


def dcsbm(n: int, n_pairs: int, *, comm_size: int, mu: float, gamma: float, max_deg: float, seed: int) -> CSR:
    lib = _load()
    rp, ci, nnz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    rc = lib.f3si_dcsbm(n, n_pairs, comm_size, mu, gamma, max_deg, seed, ctypes.byref(rp), ctypes.byref(ci),
                        ctypes.byref(nnz))
    if rc:
        raise RuntimeError(f"f3si_dcsbm failed ({rc})")
    return _csr_from(rp, ci, nnz, n, n)


def dcsbm_w(n: int, n_pairs: int, *, comm_size: int, mu, weights: np.ndarray, seed: int) -> CSR:
    """Block model with caller-given node weights (expected-degree shape) and local fraction mu
    (a scalar or one value per node)."""
    lib = _load()
    w = np.ascontiguousarray(weights, dtype=np.float64)
    m = np.ascontiguousarray(np.broadcast_to(np.asarray(mu, dtype=np.float64), (n,)))
    assert w.shape == (n,)
    rp, ci, nnz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    rc = lib.f3si_dcsbm_w(n, n_pairs, comm_size, m.ctypes.data, w.ctypes.data, seed, ctypes.byref(rp), ctypes.byref(ci),
                          ctypes.byref(nnz))
    if rc:
        raise RuntimeError(f"f3si_dcsbm_w failed ({rc})")
    return _csr_from(rp, ci, nnz, n, n)


def windows(n: int, tcb: np.ndarray, ratio: np.ndarray, *, comm_size: int, mu: float, gamma: float,
            seed: int) -> CSR:
    """A built row window by row window with given TCB counts (8 * tcb distinct columns per window)
    and mean nnz/TCB ratios (inputs.c: f3si_windows)."""
    lib = _load()
    R = (n + 15) // 16
    t = np.ascontiguousarray(tcb, dtype=np.int32)
    r = np.ascontiguousarray(ratio, dtype=np.float64)
    assert t.shape == (R,) and r.shape == (R,)
    rp, ci, nnz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    rc = lib.f3si_windows(n, t.ctypes.data, r.ctypes.data, comm_size, mu, gamma, seed, ctypes.byref(rp),
                          ctypes.byref(ci), ctypes.byref(nnz))
    if rc:
        raise RuntimeError(f"f3si_windows failed ({rc})")
    return _csr_from(rp, ci, nnz, n, n)


def molecules(n_graphs: int, n_min: int = 25, n_max: int = 150, *, self_loops: bool = False, seed: int = 1) -> CSR:
    lib = _load()
    rp, ci, gp, nnz, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int32()
    rc = lib.f3si_molecules(n_graphs, n_min, n_max, int(self_loops), seed, ctypes.byref(rp), ctypes.byref(ci),
                            ctypes.byref(nnz), ctypes.byref(n), ctypes.byref(gp))
    if rc:
        raise RuntimeError(f"f3si_molecules failed ({rc})")
    csr = _csr_from(rp, ci, nnz, n.value, n.value)
    csr.graph_ptr = _take(gp, n_graphs + 1, np.int32)
    return csr


def random_csr(n_rows: int, n_cols: int, deg_min: int, deg_max: int, *, keep_dups: bool = False,
               unsorted: bool = False, seed: int = 1) -> CSR:
    """Uniform random CSR for tests; `keep_dups`+`unsorted` leaves rows raw (duplicates, draw order)."""
    lib = _load()
    rp, ci, nnz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    rc = lib.f3si_random_csr(n_rows, n_cols, deg_min, deg_max, int(keep_dups), int(unsorted), seed,
                             ctypes.byref(rp), ctypes.byref(ci), ctypes.byref(nnz))
    if rc:
        raise RuntimeError(f"f3si_random_csr failed ({rc})")
    return _csr_from(rp, ci, nnz, n_rows, n_cols)


def values(shape, *, seed: int, dtype: str = "fp16", amp: float = 1.0, offset: int = 0) -> np.ndarray:
    """uint16 bit patterns of fp16/bf16 values on the 2^-23 grid in [-amp, amp), RNE-rounded.

    Element i (flat) is a pure function of (seed, offset + i): any slice can be regenerated alone.
    """
    lib = _load()
    count = int(np.prod(shape))
    out = np.empty(count, np.uint16)
    rc = lib.f3si_fill_values(out.ctypes.data, count, offset, seed, DTYPES[dtype], float(amp))
    if rc:
        raise RuntimeError("f3si_fill_values failed")
    return out.reshape(shape)


def round_f32(x: np.ndarray, dtype: str) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(x.shape, np.uint16)
    _load().f3si_round_f32(x.ctypes.data, out.ctypes.data, x.size, DTYPES[dtype])
    return out


def seed_for(config_index: int, tensor: int) -> int:
    """seed_t = (seed_graph << 8) | t, seed_graph = 1000 + config index; t: Q=1, K=2, V=3."""
    return ((1000 + config_index) << 8) | tensor
