"""ctypes binding of libb2.so (include/b2.h).

The library is the only compute path: there is no CPU fallback. Loading the
.so works on any host (the CPU test suite checks its exports); the first call
that needs a device raises ``RuntimeError`` when no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import (POINTER, Structure, c_char_p, c_double, c_float, c_int, c_int64,
                    c_size_t, c_uint32, c_uint64, c_void_p)

HERE = os.path.dirname(os.path.abspath(__file__))
# B2_LIB_PATH: an alternative in-tree build of the same library (A/B kernel
# experiments); the product path is always libb2.so next to this file
LIB_PATH = os.environ.get("B2_LIB_PATH") or os.path.join(HERE, "libb2.so")

i64p = POINTER(c_int64)


class GemmDesc(Structure):
    """include/b2.h b2_gemm_desc."""
    _fields_ = [("algo", c_int), ("trans_a", c_int), ("trans_b", c_int), ("M", c_int64),
                ("N", c_int64), ("K", c_int64), ("a", c_void_p * 3), ("lda", c_int64),
                ("b", c_void_p * 3), ("ldb", c_int64), ("C", c_void_p), ("ldc", c_int64),
                ("bias", c_void_p), ("epilogue", c_int), ("mask", c_void_p),
                ("mask_bits", c_void_p), ("c_hi", c_void_p), ("c_lo", c_void_p),
                ("relu_bits_out", c_void_p), ("colsum", c_void_p)]


class OptTensor(Structure):
    _fields_ = [("param", c_void_p), ("grad", c_void_p), ("slot0", c_void_p),
                ("slot1", c_void_p), ("n", c_int64), ("bc1", c_double), ("bc2", c_double)]


# name -> (restype, argtypes); every function returns an int status
_SIGS = {
    "b2_last_error": (c_char_p, []),
    "b2_version": (c_int, [POINTER(c_int), POINTER(c_int)]),
    "b2_init": (c_int, [c_int]),
    "b2_device_count": (c_int, [POINTER(c_int)]),
    "b2_device_info": (c_int, [POINTER(c_int), POINTER(c_int), POINTER(c_int), POINTER(c_size_t)]),
    "b2_default_stream": (c_int, [POINTER(c_void_p)]),
    "b2_stream_create": (c_int, [POINTER(c_void_p)]),
    "b2_stream_create_priority": (c_int, [c_void_p]),
    "b2_stream_destroy": (c_int, [c_void_p]),
    "b2_stream_sync": (c_int, [c_void_p]),
    "b2_device_sync": (c_int, []),
    "b2_event_create": (c_int, [POINTER(c_void_p)]),
    "b2_event_destroy": (c_int, [c_void_p]),
    "b2_event_record": (c_int, [c_void_p, c_void_p]),
    "b2_event_sync": (c_int, [c_void_p]),
    "b2_event_elapsed_ms": (c_int, [c_void_p, c_void_p, POINTER(c_float)]),
    "b2_stream_wait_event": (c_int, [c_void_p, c_void_p]),
    "b2_launch_count": (c_int, [POINTER(c_uint64)]),
    "b2_graph_begin": (c_int, [c_void_p]),
    "b2_graph_end": (c_int, [c_void_p, POINTER(c_int)]),
    "b2_graph_launch": (c_int, [c_int, c_void_p]),
    "b2_graph_destroy": (c_int, [c_int]),
    "b2_alloc": (c_int, [c_size_t, c_void_p, POINTER(c_void_p)]),
    "b2_free": (c_int, [c_void_p, c_void_p]),
    "b2_alloc_stats": (c_int, [POINTER(c_size_t), POINTER(c_size_t), POINTER(c_size_t),
                               POINTER(c_uint64)]),
    "b2_empty_cache": (c_int, []),
    "b2_host_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
    "b2_host_free": (c_int, [c_void_p]),
    "b2_memcpy_h2d": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "b2_memcpy_d2h": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "b2_memcpy_d2h_async": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "b2_memcpy_d2d": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "b2_fill_f32": (c_int, [c_void_p, c_float, c_int64, c_void_p]),
    "b2_binary": (c_int, [c_int, c_void_p, c_int, i64p, c_void_p, i64p, c_void_p, i64p, c_void_p]),
    "b2_binary_scalar": (c_int, [c_int, c_void_p, c_int, i64p, c_void_p, i64p, c_float, c_int,
                                 c_void_p]),
    "b2_unary": (c_int, [c_int, c_void_p, c_int, i64p, c_void_p, i64p, c_double, c_double,
                         c_void_p]),
    "b2_copy_strided": (c_int, [c_void_p, c_int, i64p, c_void_p, i64p, c_void_p]),
    "b2_write_strided": (c_int, [c_void_p, c_int, i64p, i64p, c_void_p, c_void_p]),
    "b2_fused_muladd_relu_fwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                         c_void_p]),
    "b2_fused_muladd_relu_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                                         c_void_p]),
    "b2_muladd_relu_stats": (c_int, [c_void_p] * 13 + [c_float, c_float, c_int64, c_int64, c_void_p]),
    "b2_reduce": (c_int, [c_int, c_void_p, c_void_p, c_int, i64p, c_void_p, i64p, c_uint32,
                          c_void_p]),
    "b2_max_scatter": (c_int, [c_void_p, c_int, i64p, c_uint32, c_void_p, c_void_p, c_void_p]),
    "b2_gemm": (c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                        c_int64, c_void_p, c_int64, c_void_p, c_int, c_int, c_void_p]),
    "b2_gemm_select": (c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_int64, c_int64,
                               POINTER(c_int)]),
    "b2_tf32_split": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "b2_gemm_presplit": (c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int, c_void_p]),
    "b2_bf16x2_split": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "b2_gemm_tf32x": (c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                              c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
                              c_void_p, c_int, c_void_p]),
    "b2_gemm_tf32x_ex": (c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_int64,
                                 c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                 c_void_p, c_int64, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p]),
    "b2_bf16x3_split": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "b2_bf16x3_split2": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64,
                                 c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "b2_bf16x3_join": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "b2_gemm_3xbf16": (c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_int64, c_void_p, c_int, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p]),
    "b2_gemm_fused": (c_int, [c_void_p, c_void_p]),
    "b2_gemm_fused_group": (c_int, [c_void_p, c_int, c_void_p]),
    "b2_gemm_set_sm_reserve": (c_int, [c_int]),
    "b2_gemm_get_sm_reserve": (c_int, [c_void_p]),
    "b2_bf16_cast": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p]),
    "b2_gemm_bf16": (c_int, [c_int, c_int, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                             c_int64, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "b2_im2col": (c_int, [c_void_p, c_void_p] + [c_int64] * 10 + [c_void_p]),
    "b2_col2im": (c_int, [c_void_p, c_void_p] + [c_int64] * 10 + [c_void_p]),
    "b2_xent_fwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_double,
                            c_void_p]),
    "b2_xent_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                            c_double, c_void_p]),
    "b2_xent_bwd_split": (c_int, [c_void_p] * 8 + [c_int64, c_int64, c_double, c_void_p]),
    "b2_softmax_fwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p]),
    "b2_softmax_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                               c_void_p]),
    "b2_softmax_wmean_fwd": (c_int, [c_void_p] * 7 + [c_int64, c_int64, c_void_p]),
    "b2_softmax_wmean_bwd": (c_int, [c_void_p] * 5 + [c_float] + [c_void_p] * 4
                             + [c_int64, c_int64, c_void_p]),
    "b2_sgd_multi": (c_int, [POINTER(OptTensor), c_int, c_double, c_double, c_double, c_void_p]),
    "b2_adam_multi": (c_int, [POINTER(OptTensor), c_int, c_double, c_double, c_double, c_double,
                              c_double, c_void_p]),
    "b2_rmsprop_multi": (c_int, [POINTER(OptTensor), c_int, c_double, c_double, c_double, c_double,
                                 c_void_p]),
    "b2_comm_unique_id": (c_int, [ctypes.c_char_p]),
    "b2_comm_init": (c_int, [c_int, c_int, ctypes.c_char_p]),
    "b2_comm_destroy": (c_int, []),
    "b2_allreduce_f32": (c_int, [c_void_p, c_int64, c_int, c_void_p]),
    "b2_reduce_scatter_f32": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p]),
    "b2_all_gather_f32": (c_int, [c_void_p, c_int64, c_int, c_void_p]),
    "b2_comm_async_error": (c_int, [POINTER(c_int)]),
    "b2_comm_abort": (c_int, []),
    "b2_stream_wait_timeout": (c_int, [c_void_p, c_double]),
}

# enum values (include/b2.h)
ADD, SUB, MUL, DIV, RELU_BWD, SIGN_MUL, SIGMOID_BWD, TANH_BWD, GELU_BWD = range(9)
(NEG, EXP, LOG, SQRT, ABS, RELU, RELU_MASK, COPY, CLAMP, SCALE, DIV_SCALAR, CLAMP_MASK, SIGMOID, TANH,
 GELU) = range(15)
RED_SUM, RED_MEAN, RED_MAX = range(3)
GEMM_AUTO, GEMM_SIMT, GEMM_3XTF32, GEMM_1XTF32, GEMM_TF32X, GEMM_3XBF16 = range(6)
GEMM_BF16 = 6  # host-side selector for b2_gemm_bf16 (bf16 variant; never auto-selected)
GEMM_REF = 7  # reference arithmetic: fp64 sums of exact fp32 products, one f32 rounding (parity mode)
GEMM_REF_BF16 = 8  # the same on bf16-rounded operands (exact-arithmetic control of the bf16 variant)
EPI_NONE, EPI_BIAS, EPI_BIAS_RELU, EPI_RELU = range(4)

_lib = None
_lock = threading.Lock()
_ready = False


class LibraryMissing(ImportError):
    pass


def _nccl_path():
    try:
        import importlib.util

        spec = importlib.util.find_spec("nvidia")
        for base in (spec.submodule_search_locations or []):
            p = os.path.join(base, "nccl", "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except Exception:
        pass
    return None


def lib():
    """The loaded libb2 (raises LibraryMissing if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -m paper_2602_00125_b200.build` "
                "(there is no CPU fallback)")
        if "B2_NCCL_LIB" not in os.environ:
            p = _nccl_path()
            if p:
                os.environ["B2_NCCL_LIB"] = p
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def exported_symbols():
    return list(_SIGS)


def last_error() -> str:
    msg = lib().b2_last_error()
    return msg.decode() if msg else "unknown libb2 error"


def check(rc: int):
    if rc != 0:
        raise RuntimeError(f"libb2: {last_error()}")


def ensure_device(device: int = -1):
    """Initialise libb2 on a CUDA device; fails loudly without one."""
    global _ready
    if _ready:
        return
    L = lib()
    rc = L.b2_init(device)
    if rc != 0:
        raise RuntimeError(f"libb2: {last_error()}")
    _ready = True


def call(name, *args):
    """Invoke a libb2 entry point on an initialised device and check it."""
    if not _ready:
        ensure_device()
    check(getattr(_lib, name)(*args))


def i64s(vals):
    n = len(vals)
    return (c_int64 * max(n, 1))(*vals)


def launch_count() -> int:
    v = c_uint64(0)
    lib().b2_launch_count(ctypes.byref(v))
    return v.value


def alloc_stats():
    a, b, c, d = c_size_t(), c_size_t(), c_size_t(), c_uint64()
    check(lib().b2_alloc_stats(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)))
    return {"in_use": a.value, "cached": b.value, "peak": c.value, "cuda_mallocs": d.value}


def device_info():
    ensure_device()
    sm, ma, mi, tot = c_int(), c_int(), c_int(), c_size_t()
    check(lib().b2_device_info(ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi), ctypes.byref(tot)))
    return {"sm_count": sm.value, "cc": (ma.value, mi.value), "total_mem": tot.value}


def default_stream():
    ensure_device()
    s = c_void_p()
    check(lib().b2_default_stream(ctypes.byref(s)))
    return s.value


class Event:
    """CUDA event on a libb2 stream (device-side timing for bench/tests)."""

    def __init__(self):
        ensure_device()
        h = c_void_p()
        check(lib().b2_event_create(ctypes.byref(h)))
        self.h = h.value

    def record(self, stream=None):
        check(lib().b2_event_record(self.h, stream))

    def synchronize(self):
        check(lib().b2_event_sync(self.h))

    def elapsed_ms(self, end: "Event") -> float:
        ms = c_float()
        check(lib().b2_event_elapsed_ms(self.h, end.h, ctypes.byref(ms)))
        return ms.value

    def __del__(self):
        try:
            if _lib is not None and self.h:
                _lib.b2_event_destroy(self.h)
        except Exception:
            pass


def synchronize(stream=None):
    check(lib().b2_stream_sync(stream))
