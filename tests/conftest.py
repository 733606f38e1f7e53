import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libf3s.so")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def inputs_mod():
    import f3s_inputs
    f3s_inputs.build()
    return f3s_inputs


def decode(bits: np.ndarray, dtype: str) -> np.ndarray:
    """fp64 values of uint16 fp16/bf16 bit patterns via numpy / bit shifts (library decode,
    independent of the oracle's own decoder)."""
    bits = np.asarray(bits, np.uint16)
    if dtype == "fp16":
        return bits.view(np.float16).astype(np.float64)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def encode(x: np.ndarray, dtype: str) -> np.ndarray:
    """uint16 bit patterns of x rounded RNE (numpy float16 cast / torch bfloat16 cast)."""
    x = np.asarray(x, np.float32)
    if dtype == "fp16":
        return x.astype(np.float16).view(np.uint16)
    import torch
    return torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def csr_from_dense(A: np.ndarray):
    A = np.asarray(A, bool)
    row_ptr = np.concatenate([[0], np.cumsum(A.sum(1))]).astype(np.int32)
    col_idx = np.nonzero(A)[1].astype(np.int32)
    return row_ptr, col_idx


def dense_from_csr(row_ptr, col_idx, n_rows, n_cols):
    A = np.zeros((n_rows, n_cols), bool)
    rows = np.repeat(np.arange(n_rows), np.diff(row_ptr))
    A[rows, col_idx[row_ptr[0]:row_ptr[-1]]] = True
    return A
