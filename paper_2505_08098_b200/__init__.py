"""B200-native fused 3S sparse attention (Fused3S, arXiv 2505.08098).

O = softmax_row((Q K^T) ⊙ A) V computed by libf3s.so (C ABI: include/f3s.h):
  f3s.plan(row_ptr, col_idx, n)                -> device row-window plan (§3.1)
  f3s.attention(plan, Q, K, V, scale=...)       -> fused tcgen05/TMA pass (Alg.1)
  dist.*                                        -> multi-GPU row sharding + K/V all-gather
"""
from ._build import build  # noqa: F401


def __getattr__(name):
    if name in ("f3s", "dist"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
