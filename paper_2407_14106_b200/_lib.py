"""Loader for the in-tree CUDA library (libgte_b200.so, C ABI in include/gte_b200.h).

There is no fallback: if the library is missing or was built for another
architecture, every entry point raises. Build it with
``make -C paper_2407_14106_b200/csrc`` or ``python -c "import __graft_entry__ as g; g.build()"``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GTE_LIB_PATH") or os.path.join(HERE, "libgte_b200.so")  # override: A/B builds

GTE_OK, GTE_CONFIG, GTE_DATA, GTE_DIVERGENCE, GTE_CUDA, GTE_NCCL = 0, 2, 3, 4, 5, 6
GTE_F64, GTE_F32, GTE_BF16 = 0, 1, 2
GTE_FORBID_EMPTY_ROWS = 1

DTYPES = {"f64": GTE_F64, "f32": GTE_F32, "bf16": GTE_BF16}


class GteError(RuntimeError):
    """Base of the error taxonomy (reference proj/include/gte/types.hpp:13-24)."""


class ConfigError(GteError):
    pass


class DataError(GteError):
    pass


class DivergenceError(GteError):
    pass


class CudaError(GteError):
    pass


class NcclError(GteError):
    pass


_ERRS = {GTE_CONFIG: ConfigError, GTE_DATA: DataError, GTE_DIVERGENCE: DivergenceError, GTE_CUDA: CudaError,
         GTE_NCCL: NcclError}

_lib = None
_lock = threading.Lock()

VP = C.c_void_p
I64 = C.c_int64
I32 = C.c_int


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"gte_b200 CUDA library not built: {LIB_PATH} is missing "
                                  "(run `make -C paper_2407_14106_b200/csrc`)")
            L = C.CDLL(LIB_PATH)
            L.gte_last_error.restype = C.c_char_p
            L.gte_version.restype = C.c_char_p
            L.gte_ctx_launches.restype = I64
            L.gte_ctx_launches.argtypes = [VP]
            L.gte_ctx_create.argtypes = [I32, C.POINTER(VP)]
            L.gte_ctx_destroy.argtypes = [VP]
            L.gte_ctx_set_stream.argtypes = [VP, VP]
            L.gte_ctx_sync.argtypes = [VP]
            L.gte_plan_create_host.argtypes = [VP, I64, I64, VP, VP, C.POINTER(VP)]
            L.gte_plan_create_device.argtypes = [VP, I64, I64, VP, VP, C.POINTER(VP)]
            L.gte_plan_destroy.argtypes = [VP]
            L.gte_plan_shape.argtypes = [VP, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]
            L.gte_plan_device_csr.argtypes = [VP, C.POINTER(VP), C.POINTER(VP)]
            L.gte_community_order.argtypes = [I64, I64, VP, VP, I64, VP, C.POINTER(I64)]
            L.gte_plan_schedule.argtypes = [VP, I64, C.POINTER(I64)]
            L.gte_plan_set_order.argtypes = [VP, VP]
            L.gte_plan_set_output_rows.argtypes = [VP, I64]
            L.gte_plan_set_blocks.argtypes = [VP, I64, VP, I64, C.POINTER(I64)]
            L.gte_plan_blocks.argtypes = [VP, C.POINTER(I64), C.POINTER(I64)]
            L.gte_sparse_attn_fwd.argtypes = [VP, VP, I32, I32, I32, I32, VP, VP, I64, VP, I64, VP, VP, VP, VP, I32]
            L.gte_sparse_attn_bwd.argtypes = [VP, VP, I32, I32, I32, I32, VP, VP, I64, VP, I64, VP, VP, VP, VP, VP,
                                              VP, VP, VP, VP]
            L.gte_sparse_attn_fwd_host.argtypes = [VP, VP, I32, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP, I32]
            L.gte_sparse_attn_bwd_host.argtypes = [VP, VP, I32, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP,
                                                   VP, VP]
            L.gte_sparse_attn_fwd_bwd_host.argtypes = [VP, VP, I32, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP, VP,
                                                       VP, VP]
            L.gte_sparse_attn_fwd_bwd_host_async.argtypes = L.gte_sparse_attn_fwd_bwd_host.argtypes
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != GTE_OK:
        msg = lib().gte_last_error().decode()
        raise _ERRS.get(rc, GteError)(msg)


def exported_symbols_of_header(header: str) -> list[str]:
    """Names of every function declared in a C header of include/ (for the
    symbol-export test)."""
    import re

    text = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(gte_[a-z_0-9]+)\s*\(", text, re.M)))
