"""Host control logic of the path through libgte_b200 (csrc/host_api.cpp):
the ECR tuner, select_k / select_db (reference proj/src/reformation.cpp:
224-296) and the interleave conditions / mode (proj/src/interleave.cpp:
68-106)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check

VP, I64, D = C.c_void_p, C.c_int64, C.c_double


def _bind():
    L = _lib.lib()
    if not getattr(L, "_control_bound", False):
        L.gte_tuner_create.argtypes = [D, I64, C.POINTER(VP)]
        L.gte_tuner_update.argtypes = [VP, D, D, I64]
        L.gte_tuner_state.argtypes = [VP, C.POINTER(D), C.POINTER(I64), VP, C.POINTER(I64), C.POINTER(C.c_int32)]
        L.gte_tuner_destroy.argtypes = [VP]
        L.gte_select_k.argtypes = [I64, I64, I64, C.POINTER(I64)]
        L.gte_select_db.argtypes = [I64, VP, VP, C.POINTER(I64)]
        L.gte_check_conditions.argtypes = [I64, I64, VP, VP, I64, VP, VP]
        L.gte_select_mode.argtypes = [VP, I64, I64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L._control_bound = True
    return L


class Tuner:
    """TunerState (reformation.cpp:224-265): thresholds {0, beta_G, 1.5, 5, 7,
    10 beta_G, 1}; beta_thre() is the current one."""

    def __init__(self, beta_g: float, delta: int = 1):
        h = VP()
        check(_bind().gte_tuner_create(beta_g, delta, C.byref(h)))
        self.h = h

    def update(self, loss: float, epoch_time_s: float, epoch: int):
        check(_bind().gte_tuner_update(self.h, loss, epoch_time_s, epoch))

    def state(self):
        avg, idx, n, has = D(), I64(), I64(), C.c_int32()
        thr = np.zeros(16, np.float64)
        check(_bind().gte_tuner_state(self.h, C.byref(avg), C.byref(idx), thr.ctypes.data, C.byref(n), C.byref(has)))
        return avg.value, idx.value, thr[: n.value].copy(), bool(has.value)

    def beta_thre(self) -> float:
        _, idx, thr, _ = self.state()
        return float(thr[idx])

    def __del__(self):
        try:
            _bind().gte_tuner_destroy(self.h)
        except Exception:
            pass


def select_k(l2_bytes: int, hidden_dim: int, i: int) -> int:
    out = I64()
    check(_bind().gte_select_k(l2_bytes, hidden_dim, i, C.byref(out)))
    return out.value


def select_db(db, thr) -> int:
    a = np.ascontiguousarray(db, np.int64)
    b = np.ascontiguousarray(thr, np.float64)
    out = I64()
    check(_bind().gte_select_db(a.shape[0], a.ctypes.data, b.ctypes.data, C.byref(out)))
    return out.value


def check_conditions(row_offsets, cols, layers: int):
    """-> (flags {c1, c2, c3}, ints {layers, sweep_from, sweep_to, diameter_lb})."""
    ro = np.ascontiguousarray(row_offsets, np.int64)
    co = np.ascontiguousarray(cols, np.int64)
    flags = np.zeros(3, np.int32)
    ints = np.zeros(4, np.int64)
    check(_bind().gte_check_conditions(ro.shape[0] - 1, co.shape[0], ro.ctypes.data, co.ctypes.data, layers,
                                       flags.ctypes.data, ints.ctypes.data))
    return flags, ints


def select_mode(flags, epoch: int, dense_period: int):
    """-> (mode 0 sparse / 1 dense, reason)."""
    f = np.ascontiguousarray(flags, np.int32)
    mode, reason = C.c_int32(), C.c_int32()
    check(_bind().gte_select_mode(f.ctypes.data, epoch, dense_period, C.byref(mode), C.byref(reason)))
    return mode.value, reason.value
