"""CPU oracle for the fused 3S hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import this package.  The product package `paper_2505_08098_b200` never imports it
and shares no code with it (see oracle.c's header for the definitions and citations).

`attention()` is Eq.1 with the max-stabilised softmax of Eq.7
 in fp64; `plan()` is the BSB-equivalent row-window plan of §3.1
 with the RW reordering of PAPER.md:402.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
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
        i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        pp = ctypes.POINTER(ctypes.c_void_p)
        lib.oracle_attention.argtypes = [i32, i32, vp, vp, i32, i32, i32, vp, vp, vp, ctypes.c_double, vp, i32, vp, i32]
        lib.oracle_plan.argtypes = [i32, i32, vp, vp, pp, pp, pp, pp, ctypes.POINTER(i64)]
        lib.oracle_free.argtypes = [vp]
        lib.oracle_attention_backward.argtypes = [i32, i32, vp, vp, i32, i32, vp, vp, vp, vp, ctypes.c_double, vp, vp, vp]
        lib.oracle_attention_f64.argtypes = [i32, i32, vp, vp, i32, i32, vp, vp, vp, ctypes.c_double, vp]
        lib.oracle_num_threads.restype = i32
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def attention(row_ptr, col_idx, Q, K, V, *, scale: float, dtype: str = "fp16", n_cols: int | None = None,
              rows=None, n_threads: int = 0) -> np.ndarray:
    """fp64 O[n, H, d] (or O[len(rows), H, d]) of Eq.1 with Q,K,V given as uint16 bit patterns [N, H, d]."""
    lib = _load()
    row_ptr = _c(row_ptr, np.int32)
    col_idx = _c(col_idx, np.int32) if len(col_idx) else np.zeros(1, np.int32)
    Q, K, V = _c(Q, np.uint16), _c(K, np.uint16), _c(V, np.uint16)
    n_rows = len(row_ptr) - 1
    H, d = Q.shape[1], Q.shape[2]
    n_cols = K.shape[0] if n_cols is None else n_cols
    sel = None if rows is None else _c(rows, np.int32)
    count = n_rows if sel is None else len(sel)
    out = np.empty((count, H, d), np.float64)
    rc = lib.oracle_attention(n_rows, n_cols, row_ptr.ctypes.data, col_idx.ctypes.data, H, d,
                              1 if dtype == "bf16" else 0, Q.ctypes.data, K.ctypes.data, V.ctypes.data,
                              float(scale), None if sel is None else sel.ctypes.data, count,
                              out.ctypes.data, n_threads)
    if rc:
        raise ValueError(f"oracle_attention: invalid input (code {rc})")
    return out


def attention_f64(row_ptr, col_idx, Q, K, V, *, scale: float) -> np.ndarray:
    """Eq.1 on fp64 inputs Q [n, H, d], K, V [n_cols, H, d] (the function differentiated by
    attention_backward)."""
    lib = _load()
    row_ptr = _c(row_ptr, np.int32)
    col_idx = _c(col_idx, np.int32) if len(col_idx) else np.zeros(1, np.int32)
    Q, K, V = _c(Q, np.float64), _c(K, np.float64), _c(V, np.float64)
    n_rows, H, d = Q.shape
    out = np.empty(Q.shape, np.float64)
    rc = lib.oracle_attention_f64(n_rows, K.shape[0], row_ptr.ctypes.data, col_idx.ctypes.data, H, d, Q.ctypes.data,
                                  K.ctypes.data, V.ctypes.data, float(scale), out.ctypes.data)
    if rc:
        raise ValueError(f"oracle_attention_f64: invalid input (code {rc})")
    return out


def attention_backward(row_ptr, col_idx, Q, K, V, dO, *, scale: float):
    """fp64 (dQ, dK, dV) of Eq.1 for the given dO; all inputs fp64 arrays [rows, H, d]."""
    lib = _load()
    row_ptr = _c(row_ptr, np.int32)
    col_idx = _c(col_idx, np.int32) if len(col_idx) else np.zeros(1, np.int32)
    Q, K, V, dO = _c(Q, np.float64), _c(K, np.float64), _c(V, np.float64), _c(dO, np.float64)
    n_rows, H, d = Q.shape
    dQ, dK, dV = np.empty_like(Q), np.empty_like(K), np.empty_like(V)
    rc = lib.oracle_attention_backward(n_rows, K.shape[0], row_ptr.ctypes.data, col_idx.ctypes.data, H, d,
                                       Q.ctypes.data, K.ctypes.data, V.ctypes.data, dO.ctypes.data, float(scale),
                                       dQ.ctypes.data, dK.ctypes.data, dV.ctypes.data)
    if rc:
        raise ValueError(f"oracle_attention_backward: invalid input (code {rc})")
    return dQ, dK, dV


@dataclass
class Plan:
    rw_ptr: np.ndarray    # int32[R+1]
    cols: np.ndarray      # int32[W]
    masks: np.ndarray     # uint16[W]
    rw_order: np.ndarray  # int32[R]

    @property
    def num_rw(self) -> int:
        return len(self.rw_order)

    @property
    def widths(self) -> np.ndarray:
        return np.diff(self.rw_ptr)

    @property
    def tcb8(self) -> np.ndarray:
        return (self.widths + 7) // 8


def _take(lib, ptr, n, dtype):
    arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(np.ctypeslib.as_ctypes_type(dtype))), shape=(max(n, 1),))[:n].copy()
    lib.oracle_free(ptr)
    return arr


def plan(row_ptr, col_idx, n_cols: int) -> Plan:
    lib = _load()
    row_ptr = _c(row_ptr, np.int32)
    col_idx = _c(col_idx, np.int32) if len(col_idx) else np.zeros(1, np.int32)
    n_rows = len(row_ptr) - 1
    a, b, c, e = (ctypes.c_void_p() for _ in range(4))
    W = ctypes.c_int64()
    rc = lib.oracle_plan(n_rows, n_cols, row_ptr.ctypes.data, col_idx.ctypes.data, ctypes.byref(a), ctypes.byref(b),
                         ctypes.byref(c), ctypes.byref(e), ctypes.byref(W))
    if rc:
        raise ValueError(f"oracle_plan: invalid CSR (code {rc})")
    R = (n_rows + 15) // 16
    return Plan(_take(lib, a, R + 1, np.int32), _take(lib, b, W.value, np.int32), _take(lib, c, W.value, np.uint16),
                _take(lib, e, R, np.int32))
