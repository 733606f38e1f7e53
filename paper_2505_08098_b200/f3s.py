"""Thin Python binding of the C ABI in include/f3s.h (argument marshalling only).

Every step of the hot path runs in libf3s.so's CUDA kernels; torch supplies device memory
and streams.  There is no fallback: if libf3s.so is missing, importing this module raises.
Names follow the C ABI: plan, plan_rows, attention, attention_host, partition_rows.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libf3s.so")
if os.environ.get("F3S_LIB_VARIANT"):  # experiment builds (tools/, _build.py VARIANT ...)
    LIB_PATH = os.path.join(_HERE, f"libf3s_{os.environ['F3S_LIB_VARIANT']}.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)

OK, INVALID_VALUE, INVALID_CSR, UNSUPPORTED, OUT_OF_MEMORY, CUDA, INTERNAL = range(7)
FP16, BF16, E4M3 = 0, 1, 2  # f3s_dtype
VARIANT_DEFAULT, VARIANT_NO_REORDER, VARIANT_SIMT, VARIANT_ONE_HEAD = 0, 1, 2, 3
VARIANTS = {"default": VARIANT_DEFAULT, "no_reorder": VARIANT_NO_REORDER, "simt": VARIANT_SIMT,
            "one_head": VARIANT_ONE_HEAD}


class PlanInfo(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int32), ("n_cols", ctypes.c_int32), ("num_rw", ctypes.c_int32),
                ("max_width", ctypes.c_int32), ("nnz", ctypes.c_int64), ("total_cols", ctypes.c_int64),
                ("total_tcb8", ctypes.c_int64), ("device_bytes", ctypes.c_int64), ("build_ms", ctypes.c_float),
                ("reserved", ctypes.c_float), ("split_chunks", ctypes.c_int32), ("split_groups", ctypes.c_int32),
                ("total_chunks", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


_i32, _i64, _vp, _f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_float
_lib.f3s_plan.argtypes = [_vp, _vp, _i32, _vp, ctypes.POINTER(_vp)]
_lib.f3s_plan_rows.argtypes = [_vp, _vp, _i32, _i32, _vp, ctypes.POINTER(_vp)]
_lib.f3s_plan_destroy.argtypes = [_vp]
_lib.f3s_plan_get_info.argtypes = [_vp, ctypes.POINTER(PlanInfo)]
_lib.f3s_plan_export.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.f3s_plan_set_split.argtypes = [_vp, _i32]
_lib.f3s_attention.argtypes = [_vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_kv.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _f32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_strided.argtypes = [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _f32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_partial.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_merge.argtypes = [_i32, _vp, _vp, _i64, _i32, _i32, _vp, _vp]
_lib.f3s_attention_ex.argtypes = [_vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_trace.argtypes = [_vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp]
_lib.f3s_attention_backward.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_fwd.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_backward_saved.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32,
                                              _i32, _vp]
_lib.f3s_attention_backward_saved_lp.argtypes = _lib.f3s_attention_backward_saved.argtypes
_lib.f3s_attention_backward_ex.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_host.argtypes = [_vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _vp]
_lib.f3s_attention_host_async.argtypes = [_vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _vp]
_lib.f3s_partition_rows.argtypes = [_vp, _i32, _i32, _vp]
_lib.f3s_partition_at.argtypes = [_vp, _i32, _vp, _i32, _i32, _vp]
_lib.f3s_default_split_chunks.argtypes = [_i64, _i32]
_lib.f3s_default_split_chunks.restype = _i32
_lib.f3s_status_string.argtypes = [_i32]
_lib.f3s_status_string.restype = ctypes.c_char_p
_lib.f3s_last_error.restype = ctypes.c_char_p
_lib.f3s_launch_count.restype = _i64
for _name in ("f3s_plan", "f3s_plan_rows", "f3s_plan_destroy", "f3s_plan_get_info", "f3s_plan_export", "f3s_plan_set_split",
              "f3s_attention", "f3s_attention_kv", "f3s_attention_strided", "f3s_attention_partial",
              "f3s_attention_merge", "f3s_attention_ex", "f3s_attention_trace", "f3s_attention_host", "f3s_partition_rows",
              "f3s_partition_at", "f3s_attention_backward", "f3s_attention_backward_ex", "f3s_attention_host_async"):
    getattr(_lib, _name).restype = _i32

EXPORTED = ["f3s_plan", "f3s_plan_rows", "f3s_plan_destroy", "f3s_plan_get_info", "f3s_plan_export", "f3s_plan_set_split",
            "f3s_attention", "f3s_attention_kv", "f3s_attention_strided", "f3s_attention_partial",
            "f3s_attention_merge", "f3s_attention_ex", "f3s_attention_trace", "f3s_attention_host",
            "f3s_partition_rows", "f3s_partition_at",
            "f3s_attention_backward", "f3s_attention_backward_ex", "f3s_attention_fwd", "f3s_attention_backward_saved",
            "f3s_attention_backward_saved_lp", "f3s_attention_host_async", "f3s_default_split_chunks",
            "f3s_status_string", "f3s_last_error", "f3s_launch_count"]


class F3SError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.f3s_last_error().decode()
        super().__init__(f"{where}: {_lib.f3s_status_string(status).decode()}: {detail}")


def _check(status: int, where: str) -> None:
    if status != OK:
        raise F3SError(status, where)


def _stream(stream):
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float16:
        return FP16
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float8_e4m3fn:
        return E4M3
    raise TypeError(f"Q/K/V must be float16, bfloat16 or float8_e4m3fn, got {t.dtype}")


def _check_tensors(p: "Plan", Q, K, V, O=None, *, out_dtype=None, what="f3s_attention", strided_kv=False):
    """The C ABI sees raw pointers only: check here that the tensors match the plan and each
    other (device, contiguity, dtype, [rows, H, d] shapes) before any pointer crosses it."""
    import torch
    inf = p.info()
    for name, t in (("Q", Q), ("K", K), ("V", V)):
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{what}: {name} must be a torch.Tensor")
        if not t.is_cuda:
            raise ValueError(f"{what}: {name} must be a CUDA tensor")
        if not t.is_contiguous() and not (strided_kv and name != "Q"):
            raise ValueError(f"{what}: {name} must be contiguous")
        if t.dim() != 3:
            raise ValueError(f"{what}: {name} must be [rows, heads, d], got shape {tuple(t.shape)}")
    if not (K.dtype == V.dtype == Q.dtype):
        raise ValueError(f"{what}: Q, K, V dtypes differ ({Q.dtype}, {K.dtype}, {V.dtype})")
    if not (K.device == V.device == Q.device):
        raise ValueError(f"{what}: Q, K, V on different devices")
    H, d = Q.shape[1], Q.shape[2]
    if tuple(K.shape[1:]) != (H, d) or tuple(V.shape[1:]) != (H, d):
        raise ValueError(f"{what}: K/V heads and d must match Q's ({H}, {d})")
    if Q.shape[0] != inf["n_rows"]:
        raise ValueError(f"{what}: Q has {Q.shape[0]} rows, the plan {inf['n_rows']}")
    if K.shape[0] < inf["n_cols"] or V.shape[0] < inf["n_cols"]:
        raise ValueError(f"{what}: K/V need at least n_cols = {inf['n_cols']} rows")
    if O is not None:
        if not O.is_cuda or not O.is_contiguous() or O.device != Q.device:
            raise ValueError(f"{what}: O must be a contiguous CUDA tensor on Q's device")
        if O.dtype != (out_dtype or torch.float32) or tuple(O.shape) != tuple(Q.shape):
            raise ValueError(f"{what}: O must be float32 of shape {tuple(Q.shape)}")


def default_split_chunks(total_chunks: int, num_sms: int) -> int:
    """f3s_default_split_chunks: the heavy-window split bound for a problem of total_chunks chunks."""
    return int(_lib.f3s_default_split_chunks(int(total_chunks), int(num_sms)))


class Plan:
    """Owning handle of a device plan (f3s_plan_t)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = PlanInfo()
        _check(_lib.f3s_plan_get_info(self._h, ctypes.byref(inf)), "f3s_plan_get_info")
        return inf.as_dict()

    def export(self):
        """Host copies of the canonical arrays: rw_ptr, cols, masks, rw_order (numpy)."""
        inf = self.info()
        R, W = inf["num_rw"], inf["total_cols"]
        rw_ptr = np.empty(R + 1, np.int32)
        cols = np.empty(max(W, 1), np.int32)
        masks = np.empty(max(W, 1), np.uint16)
        order = np.empty(max(R, 1), np.int32)
        _check(_lib.f3s_plan_export(self._h, rw_ptr.ctypes.data, cols.ctypes.data, masks.ctypes.data,
                                    order.ctypes.data), "f3s_plan_export")
        return rw_ptr, cols[:W], masks[:W], order[:R]

    def set_split(self, max_chunks: int) -> None:
        """f3s_plan_set_split: heavy row windows processed as pieces of <= max_chunks 128-column
        chunks (0: never split)."""
        _check(_lib.f3s_plan_set_split(self._h, int(max_chunks)), "f3s_plan_set_split")

    def destroy(self) -> None:
        if self._h:
            _lib.f3s_plan_destroy(self._h)
            self._h = ctypes.c_void_p(None)

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def plan(row_ptr, col_idx, n: int, stream=None) -> Plan:
    """f3s_plan on device CSR tensors (int32, cuda)."""
    h = ctypes.c_void_p()
    _check(_lib.f3s_plan(row_ptr.data_ptr(), col_idx.data_ptr() if col_idx.numel() else None, n, _stream(stream),
                         ctypes.byref(h)), "f3s_plan")
    return Plan(h.value)


def plan_rows(row_ptr, col_idx, n_rows: int, n_cols: int, stream=None) -> Plan:
    """f3s_plan_rows: row_ptr may be a view into a global row_ptr (non-zero base)."""
    h = ctypes.c_void_p()
    _check(_lib.f3s_plan_rows(row_ptr.data_ptr(), col_idx.data_ptr() if col_idx.numel() else None, n_rows, n_cols,
                              _stream(stream), ctypes.byref(h)), "f3s_plan_rows")
    return Plan(h.value)


def attention(p: Plan, Q, K, V, O=None, *, scale: float = 1.0, variant: str | int = "default", stream=None):
    """f3s_attention(_ex) on device tensors Q [n_rows,H,d], K/V [n_cols,H,d] (fp16/bf16); O float32."""
    import torch
    _check_tensors(p, Q, K, V, O)
    H, d = Q.shape[1], Q.shape[2]
    if O is None:
        O = torch.empty(Q.shape, dtype=torch.float32, device=Q.device)
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    st = _lib.f3s_attention_ex(p.handle, Q.data_ptr(), K.data_ptr(), V.data_ptr(), O.data_ptr(), float(scale), H, d,
                               _dtype_code(Q), v, _stream(stream))
    _check(st, "f3s_attention")
    return O


def attention_kv(p: Plan, Q, KV, O=None, *, scale: float = 1.0, stream=None):
    """f3s_attention_kv on an interleaved [n_cols, 2, H, d] buffer (K = KV[:, 0], V = KV[:, 1]),
    the layout one all-gather of [K || V] shards produces."""
    import torch
    if KV.dim() != 4 or KV.shape[1] != 2 or not KV.is_contiguous():
        raise ValueError("attention_kv: KV must be a contiguous [n_cols, 2, heads, d] tensor")
    _check_tensors(p, Q, KV[:, 0], KV[:, 1], O, what="f3s_attention_kv", strided_kv=True)
    H, d = Q.shape[1], Q.shape[2]
    if O is None:
        O = torch.empty(Q.shape, dtype=torch.float32, device=Q.device)
    es = KV.element_size()
    _check(_lib.f3s_attention_kv(p.handle, Q.data_ptr(), KV.data_ptr(), KV.data_ptr() + H * d * es, 2 * H * d,
                                 O.data_ptr(), float(scale), H, d, _dtype_code(Q), _stream(stream)), "f3s_attention_kv")
    return O


def attention_kv_raw(p: Plan, q_ptr: int, k_ptr: int, v_ptr: int, kv_row_stride: int, o_ptr: int, scale: float,
                     heads: int, d: int, dtype: int, stream: int) -> None:
    """Pointer-level f3s_attention_kv (bench loops)."""
    _check(_lib.f3s_attention_kv(p.handle, q_ptr, k_ptr, v_ptr, int(kv_row_stride), o_ptr, float(scale), heads, d,
                                 dtype, stream), "f3s_attention_kv")


def attention_qkv(p: Plan, QKV, O=None, *, scale: float = 1.0, stream=None):
    """f3s_attention_strided on a packed projection output QKV [n, 3, H, d] (Q, K, V = QKV[:, 0/1/2]):
    the fused pass reads the three row-strided operands in place (no split copies)."""
    import torch
    if QKV.dim() != 4 or QKV.shape[1] != 3 or not QKV.is_contiguous() or not QKV.is_cuda:
        raise ValueError("attention_qkv: QKV must be a contiguous CUDA [n, 3, heads, d] tensor")
    inf = p.info()
    n, _, H, d = QKV.shape
    if n != inf["n_rows"] or n < inf["n_cols"]:
        raise ValueError(f"attention_qkv: {n} rows for a plan of {inf['n_rows']} x {inf['n_cols']}")
    if O is None:
        O = torch.empty((n, H, d), dtype=torch.float32, device=QKV.device)
    elif O.dtype != torch.float32 or tuple(O.shape) != (n, H, d) or not O.is_contiguous():
        raise ValueError("attention_qkv: O must be float32 [n, heads, d]")
    es, base = QKV.element_size(), QKV.data_ptr()
    _check(_lib.f3s_attention_strided(p.handle, base, 3 * H * d, base + H * d * es, base + 2 * H * d * es, 3 * H * d,
                                      O.data_ptr(), float(scale), H, d, _dtype_code(QKV), _stream(stream)),
           "f3s_attention_strided")
    return O


def attention_partial_raw(p: Plan, q_ptr: int, k_ptr: int, v_ptr: int, kv_row_stride: int, o_part_ptr: int,
                          ml_part_ptr: int, scale: float, heads: int, d: int, dtype: int, max_ctas: int,
                          stream: int) -> None:
    """f3s_attention_partial: one column block's unnormalised O and per-row (m, l)."""
    _check(_lib.f3s_attention_partial(p.handle, q_ptr, k_ptr, v_ptr, int(kv_row_stride), o_part_ptr, ml_part_ptr,
                                      float(scale), heads, d, dtype, int(max_ctas), stream), "f3s_attention_partial")


def attention_merge(O_parts, ml_parts, O=None, stream=None):
    """f3s_attention_merge of [parts, n, H, d] partials and [parts, n, H, 2] (m, l) into O [n, H, d]."""
    import torch
    if O_parts.dtype != torch.float32 or ml_parts.dtype != torch.float32 or not O_parts.is_contiguous() \
            or not ml_parts.is_contiguous() or tuple(ml_parts.shape) != tuple(O_parts.shape[:3]) + (2,):
        raise ValueError("attention_merge: float32 contiguous O_parts [P, n, H, d] and ml_parts [P, n, H, 2]")
    P, n, H, d = O_parts.shape
    if O is None:
        O = torch.empty((n, H, d), dtype=torch.float32, device=O_parts.device)
    _check(_lib.f3s_attention_merge(P, O_parts.data_ptr(), ml_parts.data_ptr(), n, H, d, O.data_ptr(), _stream(stream)),
           "f3s_attention_merge")
    return O


def attention_raw(p: Plan, q_ptr: int, k_ptr: int, v_ptr: int, o_ptr: int, scale: float, heads: int, d: int,
                  dtype: int, stream: int, variant: int = VARIANT_DEFAULT) -> None:
    """Pointer-level call (no torch); used by bench loops and CUDA-graph capture."""
    _check(_lib.f3s_attention_ex(p.handle, q_ptr, k_ptr, v_ptr, o_ptr, float(scale), heads, d, dtype, variant, stream),
           "f3s_attention")


BACKWARD_VARIANTS = {"tc": 0, "simt": 1}


def attention_backward(p: Plan, Q, K, V, dO, *, scale: float, stream=None, variant: str = "tc"):
    """f3s_attention_backward(_ex): (dQ, dK, dV) fp32 device tensors for dO = dL/dO (fp32 [N, H, d]);
    variant "tc" (tensor cores, the default) or "simt" (the CUDA-core kernels)."""
    import torch
    _check_tensors(p, Q, K, V, dO, what="f3s_attention_backward")
    H, d = Q.shape[1], Q.shape[2]
    dQ = torch.empty(Q.shape, dtype=torch.float32, device=Q.device)
    dK = torch.empty(K.shape, dtype=torch.float32, device=K.device)
    dV = torch.empty(V.shape, dtype=torch.float32, device=V.device)
    _check(_lib.f3s_attention_backward_ex(p.handle, Q.data_ptr(), K.data_ptr(), V.data_ptr(), dO.data_ptr(),
                                          dQ.data_ptr(), dK.data_ptr(), dV.data_ptr(), float(scale), H, d,
                                          _dtype_code(Q), BACKWARD_VARIANTS[variant], _stream(stream)),
           "f3s_attention_backward")
    return dQ, dK, dV


def attention_fwd(p: Plan, Q, K, V, O=None, ml=None, *, scale: float = 1.0, stream=None):
    """f3s_attention_fwd: O (bitwise as attention()) and the per-row softmax statistics ml
    [N, H, 2] = (m, l) that attention_backward_saved consumes."""
    import torch
    _check_tensors(p, Q, K, V, O, what="f3s_attention_fwd")
    H, d = Q.shape[1], Q.shape[2]
    if O is None:
        O = torch.empty(Q.shape, dtype=torch.float32, device=Q.device)
    if ml is None:
        ml = torch.empty((Q.shape[0], H, 2), dtype=torch.float32, device=Q.device)
    elif ml.dtype != torch.float32 or tuple(ml.shape) != (Q.shape[0], H, 2) or not ml.is_contiguous() \
            or ml.device != Q.device:
        raise ValueError(f"attention_fwd: ml must be a contiguous float32 [{Q.shape[0]}, {H}, 2] tensor on Q's device")
    _check(_lib.f3s_attention_fwd(p.handle, Q.data_ptr(), K.data_ptr(), V.data_ptr(), O.data_ptr(), ml.data_ptr(),
                                  float(scale), H, d, _dtype_code(Q), _stream(stream)), "f3s_attention_fwd")
    return O, ml


def attention_backward_saved(p: Plan, Q, K, V, O, ml, dO, *, scale: float, stream=None):
    """f3s_attention_backward_saved(_lp): (dQ, dK, dV) from the saved outputs (O, ml) of
    attention_fwd; dO float32 (gradients float32), or in Q's dtype (the _lp entry point: dO read in
    place, gradients in Q's dtype)."""
    import torch
    lp = dO.dtype == Q.dtype
    if not lp and dO.dtype != torch.float32:
        raise ValueError(f"attention_backward_saved: dO must be float32 or Q's dtype {Q.dtype}, got {dO.dtype}")
    _check_tensors(p, Q, K, V, dO, out_dtype=Q.dtype if lp else None, what="f3s_attention_backward_saved")
    _check_tensors(p, Q, K, V, O, what="f3s_attention_backward_saved")
    H, d = Q.shape[1], Q.shape[2]
    if ml.dtype != torch.float32 or tuple(ml.shape) != (Q.shape[0], H, 2) or not ml.is_contiguous() \
            or ml.device != Q.device:
        raise ValueError("attention_backward_saved: ml must be attention_fwd's float32 [N, H, 2] statistics")
    gdt = Q.dtype if lp else torch.float32  # _lp: gradients in the input dtype too
    dQ = torch.empty(Q.shape, dtype=gdt, device=Q.device)
    dK = torch.empty(K.shape, dtype=gdt, device=K.device)
    dV = torch.empty(V.shape, dtype=gdt, device=V.device)
    fn = _lib.f3s_attention_backward_saved_lp if lp else _lib.f3s_attention_backward_saved
    _check(fn(p.handle, Q.data_ptr(), K.data_ptr(), V.data_ptr(), O.data_ptr(), ml.data_ptr(), dO.data_ptr(),
              dQ.data_ptr(), dK.data_ptr(), dV.data_ptr(), float(scale), H, d, _dtype_code(Q), _stream(stream)),
           "f3s_attention_backward_saved" + ("_lp" if lp else ""))
    return dQ, dK, dV


class _AttentionFn:
    """torch.autograd.Function over the C ABI (built lazily so that importing this module needs no
    torch): forward = f3s_attention_fwd, backward = f3s_attention_backward_saved on the saved
    (O, ml).  Gradients come back in fp32 and are cast to the inputs' dtypes."""
    fn = None

    @classmethod
    def get(cls):
        if cls.fn is None:
            import torch

            class Fn(torch.autograd.Function):
                @staticmethod
                def forward(ctx, Q, K, V, p, scale, out_dtype):
                    O, ml = attention_fwd(p, Q, K, V, scale=scale)
                    ctx.save_for_backward(Q, K, V, O, ml)
                    ctx.plan, ctx.scale = p, scale
                    return O if out_dtype is None else O.to(out_dtype)

                @staticmethod
                def backward(ctx, dO):
                    Q, K, V, O, ml = ctx.saved_tensors
                    # dO in Q's dtype goes to the _lp entry point as it is; anything else as fp32
                    dO = (dO if dO.dtype == Q.dtype else dO.to(torch.float32)).contiguous()
                    dQ, dK, dV = attention_backward_saved(ctx.plan, Q, K, V, O, ml, dO, scale=ctx.scale)
                    return dQ.to(Q.dtype), dK.to(K.dtype), dV.to(V.dtype), None, None, None

            cls.fn = Fn
        return cls.fn


class _AttentionQKVFn:
    """The same over a packed projection output QKV [n, 3, H, d]: the backward writes dQ, dK, dV
    straight into one packed gradient (three cast copies) instead of autograd's per-slice
    zero-filled buffers and their sum."""
    fn = None

    @classmethod
    def get(cls):
        if cls.fn is None:
            import torch

            class Fn(torch.autograd.Function):
                @staticmethod
                def forward(ctx, QKV, p, scale, out_dtype):
                    Q, K, V = (QKV[:, i].contiguous() for i in range(3))
                    O, ml = attention_fwd(p, Q, K, V, scale=scale)
                    ctx.save_for_backward(Q, K, V, O, ml)
                    ctx.plan, ctx.scale = p, scale
                    return O if out_dtype is None else O.to(out_dtype)

                @staticmethod
                def backward(ctx, dO):
                    Q, K, V, O, ml = ctx.saved_tensors
                    dO = (dO if dO.dtype == Q.dtype else dO.to(torch.float32)).contiguous()
                    grads = attention_backward_saved(ctx.plan, Q, K, V, O, ml, dO, scale=ctx.scale)
                    dQKV = torch.empty((Q.shape[0], 3) + tuple(Q.shape[1:]), dtype=Q.dtype, device=Q.device)
                    for i, g in enumerate(grads):
                        dQKV[:, i].copy_(g)
                    return dQKV, None, None, None

            cls.fn = Fn
        return cls.fn


def attention_autograd_qkv(p: Plan, QKV, *, scale: float = 1.0, out_dtype=None):
    """attention_autograd on a packed [n, 3, H, d] projection output (Q, K, V = QKV[:, 0/1/2]);
    the gradient comes back packed the same way."""
    if QKV.dim() != 4 or QKV.shape[1] != 3:
        raise ValueError("attention_autograd_qkv: QKV must be [n, 3, heads, d]")
    return _AttentionQKVFn.get().apply(QKV, p, float(scale), out_dtype)


def attention_autograd(p: Plan, Q, K, V, *, scale: float = 1.0, out_dtype=None):
    """O = f3s attention with autograd support (training): the forward saves O and the per-row
    softmax statistics; O.backward() runs the tensor-core backward without recomputing the forward.
    Q, K, V: contiguous fp16/bf16 CUDA tensors (gradients in the same dtypes); O: float32, or cast to
    out_dtype (= Q's dtype: its gradient then reaches f3s_attention_backward_saved_lp unconverted)."""
    return _AttentionFn.get().apply(Q, K, V, p, float(scale), out_dtype)


def attention_trace(p: Plan, Q, K, V, O, *, scale: float, trace_chunks: int = 4096, grid: int = 0,
                    variant: str | int = "default", stream=None):
    """Run the default kernel with F3S_TRACE on; returns uint64 [grid, trace_chunks, 16] globaltimer stamps."""
    import torch
    import math
    H, d = Q.shape[1], Q.shape[2]
    g = grid or torch.cuda.get_device_properties(Q.device).multi_processor_count * 2  # upper bound on the grid
    tr = torch.zeros((g, max(trace_chunks, 16), 16), dtype=torch.int64, device=Q.device)
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    _check(_lib.f3s_attention_trace(p.handle, Q.data_ptr(), K.data_ptr(), V.data_ptr(), O.data_ptr(), float(scale), H, d,
                                    _dtype_code(Q), v, tr.data_ptr(), trace_chunks, grid, _stream(stream)),
           "f3s_attention_trace")
    return tr


def attention_host(p: Plan, Q, K, V, O, *, scale: float, heads: int, d: int, dtype: int, stream=None) -> None:
    """f3s_attention_host on HOST buffers (numpy uint16 bit patterns or pinned torch tensors); O float32 host."""
    def ptr(x):
        return x.ctypes.data if isinstance(x, np.ndarray) else x.data_ptr()
    _check(_lib.f3s_attention_host(p.handle, ptr(Q), ptr(K), ptr(V), ptr(O), float(scale), heads, d, dtype,
                                   _stream(stream)), "f3s_attention_host")


def attention_host_async(p: Plan, Q, K, V, O, *, scale: float, heads: int, d: int, dtype: int, stream=None) -> None:
    """f3s_attention_host_async: enqueue on `stream`; O (pinned host) is valid once the stream completes."""
    _check(_lib.f3s_attention_host_async(p.handle, Q.data_ptr(), K.data_ptr(), V.data_ptr(), O.data_ptr(), float(scale),
                                         heads, d, dtype, _stream(stream)), "f3s_attention_host_async")


def partition_rows(row_ptr: np.ndarray, parts: int) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    bounds = np.empty(parts + 1, np.int32)
    _check(_lib.f3s_partition_rows(row_ptr.ctypes.data, len(row_ptr) - 1, parts, bounds.ctypes.data),
           "f3s_partition_rows")
    return bounds


def partition_at(row_ptr: np.ndarray, cuts: np.ndarray, parts: int) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    cuts = np.ascontiguousarray(cuts, np.int32)
    bounds = np.empty(parts + 1, np.int32)
    _check(_lib.f3s_partition_at(row_ptr.ctypes.data, len(row_ptr) - 1, cuts.ctypes.data, len(cuts), parts,
                                 bounds.ctypes.data), "f3s_partition_at")
    return bounds


def launch_count() -> int:
    return int(_lib.f3s_launch_count())
