"""One GPH transformer block around the sparse attention on the device
(reference Trainer forward/backward proj/src/model.cpp:533-595,
669-744) through gte_gph_layer (csrc/gph_layer.cu: cuBLAS projections,
LayerNorm / GELU / bias-gradient kernels, the plan's sparse attention)."""
from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import check
from .attention import DevicePlan

VP = C.c_void_p
NAMES = ("ln1_scale", "ln1_shift", "w_q", "b_q", "w_k", "b_k", "w_v", "b_v", "w_o", "b_o",
         "ln2_scale", "ln2_shift", "w_ff1", "b_ff1", "w_ff2", "b_ff2")
WEIGHTS = ("w_q", "w_k", "w_v", "w_o", "w_ff1", "w_ff2")


class _Params(C.Structure):
    _fields_ = [(n, VP) for n in NAMES]


def _bind():
    L = _lib.lib()
    if not getattr(L, "_layer_bound", False):
        L.gte_gph_layer_create.argtypes = [VP, VP, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(VP)]
        L.gte_gph_layer_set_params.argtypes = [VP, C.POINTER(_Params)]
        L.gte_gph_layer_fwd.argtypes = [VP, VP, VP]
        L.gte_gph_layer_bwd.argtypes = [VP, VP, VP, C.POINTER(_Params), VP]
        L.gte_gph_layer_destroy.argtypes = [VP]
        L._layer_bound = True
    return L


def param_shapes(d: int, ffn: int) -> dict:
    sh = {n: (d,) for n in NAMES}
    sh.update(w_q=(d, d), w_k=(d, d), w_v=(d, d), w_o=(d, d), w_ff1=(d, ffn), b_ff1=(ffn,), w_ff2=(ffn, d))
    return sh


class GphLayer:
    """Parameters: dict of CUDA tensors (weights [in, out] of the layer dtype,
    biases / LayerNorm in the accumulate type). forward(h, bias_vals) updates
    h in place; backward(dh, bias_vals, grads) accumulates into `grads` (all
    accumulate type), updates dh in place, returns the attention dbias [E]."""

    def __init__(self, plan: DevicePlan, dtype: str, heads: int, hidden: int, ffn: int, params: dict):
        self.plan, self.dtype, self.H, self.d, self.ffn = plan, dtype, heads, hidden, ffn
        h = VP()
        check(_bind().gte_gph_layer_create(plan.ctx.h, plan.h, _lib.DTYPES[dtype], heads, hidden, ffn, C.byref(h)))
        self.h = h
        self.params = params
        self._p = _Params(*[params[n].data_ptr() for n in NAMES])
        check(_bind().gte_gph_layer_set_params(self.h, C.byref(self._p)))

    def _stream(self):
        import torch

        self.plan.ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def forward(self, h, bias_vals=None):
        self._stream()
        check(_bind().gte_gph_layer_fwd(self.h, h.data_ptr(), None if bias_vals is None else bias_vals.data_ptr()))
        return h

    def backward(self, dh, bias_vals, grads: dict):
        import torch

        self._stream()
        acc = torch.float64 if self.dtype == "f64" else torch.float32
        dbias = torch.empty(max(self.plan.nnz, 1), dtype=acc, device=dh.device)
        gp = _Params(*[grads[n].data_ptr() for n in NAMES])
        check(_bind().gte_gph_layer_bwd(self.h, dh.data_ptr(), None if bias_vals is None else bias_vals.data_ptr(),
                                        C.byref(gp), dbias.data_ptr()))
        return dbias[: self.plan.nnz]

    def close(self):
        if getattr(self, "h", None):
            _bind().gte_gph_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
