"""Shared helpers for GPU tests: seeded inputs -> device tensors, oracle comparison metrics."""
import numpy as np

import f3s_inputs as fi

TOL_MAX_ABS = 1e-2   # BASELINE.json north_star: max-abs error 1e-2
TOL_REL_FRO = 5e-3   # and relative Frobenius error 5e-3


def make_qkv(n_rows, n_cols, H, d, dtype="fp16", seed=1, amp_qk=1.0, amp_v=1.0):
    Q = fi.values((n_rows, H, d), seed=(seed << 8) | 1, dtype=dtype, amp=amp_qk)
    K = fi.values((n_cols, H, d), seed=(seed << 8) | 2, dtype=dtype, amp=amp_qk)
    V = fi.values((n_cols, H, d), seed=(seed << 8) | 3, dtype=dtype, amp=amp_v)
    return Q, K, V


def to_dev(bits: np.ndarray, dtype: str):
    import torch
    t = torch.from_numpy(bits.view(np.int16)).cuda()
    return t.view(torch.float16 if dtype == "fp16" else torch.bfloat16)


def csr_to_dev(csr):
    import torch
    return torch.from_numpy(csr.row_ptr).cuda(), torch.from_numpy(csr.col_idx if len(csr.col_idx) else np.zeros(1, np.int32)).cuda()


def errors(O_gpu: np.ndarray, O_ref: np.ndarray):
    diff = O_gpu.astype(np.float64) - O_ref
    max_abs = float(np.abs(diff).max()) if diff.size else 0.0
    ref_norm = float(np.linalg.norm(O_ref))
    fro = float(np.linalg.norm(diff))
    rel = fro / ref_norm if ref_norm > 0 else fro
    return max_abs, rel


def assert_close(O_gpu, O_ref, tol_abs=TOL_MAX_ABS, tol_rel=TOL_REL_FRO):
    assert np.all(np.isfinite(O_gpu)), "non-finite output"
    max_abs, rel = errors(O_gpu, O_ref)
    assert max_abs <= tol_abs and rel <= tol_rel, f"max_abs={max_abs:.3e} rel_fro={rel:.3e}"
    return max_abs, rel
