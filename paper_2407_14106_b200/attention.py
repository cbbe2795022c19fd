"""Host-side mirror of the reference attention operator API over the CUDA C ABI.

Names, argument meaning and error behaviour follow the reference
``gte::`` attention interface (proj/include/gte/attention.hpp:13-77,
proj/src/attention.cpp): ``sparse_attention``, ``sparse_attention_backward``,
``edge_sparse_attention``, ``pattern_from_graph``, ``dense_pattern``,
``MacCounter``/``AttnResult``/``AttnGrads``. Host entries take numpy arrays and
run through the library's host-pointer twins (synchronous, like the
reference). ``DevicePlan`` / ``DeviceSparseAttention`` are the HBM-resident
multi-head path used by the benchmark and the distributed layer (torch CUDA
tensors as plumbing only).

Every call lands in libgte_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import ConfigError, DataError, check

# --------------------------------------------------------------------------
# pattern / graph containers (reference attention.hpp:13-23, graph.hpp:17-31)
# --------------------------------------------------------------------------


@dataclass
class Graph:
    num_nodes: int
    row_offsets: np.ndarray
    col_indices: np.ndarray

    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    def neighbors(self, u: int) -> np.ndarray:
        return self.col_indices[self.row_offsets[u]:self.row_offsets[u + 1]]


@dataclass
class AttnPattern:
    rows: int
    row_offsets: np.ndarray
    cols: np.ndarray

    def nnz(self) -> int:
        return int(self.cols.shape[0])

    def row_cols(self, r: int) -> np.ndarray:
        return self.cols[self.row_offsets[r]:self.row_offsets[r + 1]]


def pattern_from_graph(g: Graph) -> AttnPattern:
    """reference proj/src/attention.cpp:26-32"""
    return AttnPattern(g.num_nodes, np.asarray(g.row_offsets, np.int64), np.asarray(g.col_indices, np.int64))


def dense_pattern(n: int) -> AttnPattern:
    """reference proj/src/attention.cpp:34-44 (materialises n^2 pairs; small n only)."""
    ro = np.arange(n + 1, dtype=np.int64) * n
    cols = np.tile(np.arange(n, dtype=np.int64), n)
    return AttnPattern(n, ro, cols)


@dataclass
class MacCounter:
    score_macs: int = 0
    weight_macs: int = 0

    def __iadd__(self, o: "MacCounter"):
        self.score_macs += o.score_macs
        self.weight_macs += o.weight_macs
        return self


@dataclass
class AttnResult:
    output: np.ndarray
    macs: MacCounter = field(default_factory=MacCounter)


@dataclass
class AttnGrads:
    dq: np.ndarray
    dk: np.ndarray
    dv: np.ndarray
    dbias: np.ndarray


# --------------------------------------------------------------------------
# context + plans
# --------------------------------------------------------------------------


class Context:
    """gte_ctx for one device (device, stream, workspaces, latched errors)."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int = 0):
        L = _lib.lib()
        h = C.c_void_p()
        check(L.gte_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def get(cls, device: int = 0) -> "Context":
        if device not in cls._by_device:
            cls._by_device[device] = Context(device)
        return cls._by_device[device]

    def set_stream(self, stream_handle: int | None) -> None:
        _lib.lib().gte_ctx_set_stream(self.h, C.c_void_p(stream_handle or 0))

    def sync(self) -> None:
        check(_lib.lib().gte_ctx_sync(self.h))

    @property
    def launches(self) -> int:
        return int(_lib.lib().gte_ctx_launches(self.h))


def community_order(row_offsets, cols, iters: int = 20):
    """Host label-propagation execution order of a CSR pattern
    (gte_community_order); returns (order int64[n], communities)."""
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    co = np.ascontiguousarray(cols, dtype=np.int64)
    n = ro.shape[0] - 1
    out = np.empty(max(n, 1), dtype=np.int64)
    nc = C.c_int64()
    cp = co if co.shape[0] else np.zeros(1, dtype=np.int64)
    check(_lib.lib().gte_community_order(n, co.shape[0], ro.ctypes.data, cp.ctypes.data, iters, out.ctypes.data,
                                         C.byref(nc)))
    return out[:n], nc.value


class DevicePlan:
    """gte_plan: the pattern resident in HBM as int32 CSR + CSC."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.h = handle
        self.ctx = ctx
        rows, nnz, mr, mc = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.lib().gte_plan_shape(handle, C.byref(rows), C.byref(nnz), C.byref(mr), C.byref(mc))
        self.rows, self.nnz = rows.value, nnz.value
        self.max_row_deg, self.max_col_deg = mr.value, mc.value

    @classmethod
    def from_host(cls, row_offsets, cols, ctx: Context | None = None) -> "DevicePlan":
        ctx = ctx or Context.get()
        ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
        co = np.ascontiguousarray(cols, dtype=np.int64)
        if co.shape[0] == 0:
            co = np.zeros(1, dtype=np.int64)
            nnz = 0
        else:
            nnz = co.shape[0]
        h = C.c_void_p()
        check(_lib.lib().gte_plan_create_host(ctx.h, ro.shape[0] - 1, nnz, ro.ctypes.data, co.ctypes.data, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_pattern(cls, pat: AttnPattern, ctx: Context | None = None) -> "DevicePlan":
        return cls.from_host(pat.row_offsets, pat.cols, ctx)

    @classmethod
    def from_device(cls, rows: int, nnz: int, row_ptr_ptr: int, cols_ptr: int, ctx: Context | None = None):
        ctx = ctx or Context.get()
        h = C.c_void_p()
        check(_lib.lib().gte_plan_create_device(ctx.h, rows, nnz, C.c_void_p(row_ptr_ptr), C.c_void_p(cols_ptr),
                                                C.byref(h)))
        return cls(h, ctx)

    def schedule(self, iters: int = 20) -> int:
        """Community execution order (label propagation, csrc/schedule.cpp);
        returns the number of communities. Results are unchanged."""
        n = C.c_int64()
        check(_lib.lib().gte_plan_schedule(self.h, iters, C.byref(n)))
        return n.value

    def set_order(self, order) -> None:
        """Explicit execution order (a permutation of the rows); None clears."""
        if order is None:
            check(_lib.lib().gte_plan_set_order(self.h, None))
            return
        o = np.ascontiguousarray(order, dtype=np.int64)
        if o.shape[0] != self.rows:
            raise ConfigError("plan: order length must equal the row count")
        check(_lib.lib().gte_plan_set_order(self.h, o.ctypes.data))

    def set_output_rows(self, n: int) -> None:
        """Rows >= n (which must have no edges) produce no outputs: the
        forward and the backward's CSR pass skip them (gte_plan_set_output_rows)."""
        check(_lib.lib().gte_plan_set_output_rows(self.h, int(n)))

    def set_blocks(self, origins, d_b: int = 16) -> int:
        """Registers ECR sub-blocks (global (row0, col0) origins, side d_b;
        ClusterSparseLayout.global_blocks()): with d_b == 16, bf16 calls run
        their pairs as dense tiles on the tensor pipe (csrc/ecr_tile.cuh) and
        the rest on the sparse kernels. Returns the number executed as tiles."""
        o = np.ascontiguousarray(np.asarray(origins, dtype=np.int64).reshape(-1, 2))
        used = C.c_int64()
        check(_lib.lib().gte_plan_set_blocks(self.h, o.shape[0], o.ctypes.data if o.size else None, d_b,
                                             C.byref(used)))
        return used.value

    def blocks(self):
        """(registered sub-blocks, remainder nnz)."""
        nb, rn = C.c_int64(), C.c_int64()
        check(_lib.lib().gte_plan_blocks(self.h, C.byref(nb), C.byref(rn)))
        return nb.value, rn.value

    def close(self):
        if self.h:
            _lib.lib().gte_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# reference-shaped host API (one head per call, like the reference)
# --------------------------------------------------------------------------

_NP = {"f64": np.float64, "f32": np.float32}


def _check_shapes(q, k, v):
    # reference proj/src/attention.cpp:12-18
    if q.shape[0] != k.shape[0] or q.shape[0] != v.shape[0]:
        raise ConfigError("attention: Q/K/V row counts differ")
    if q.shape[1] != k.shape[1]:
        raise ConfigError("attention: Q/K column counts differ")
    if q.shape[1] < 1:
        raise ConfigError("attention: d_K must be >= 1")


def _ptr(a):
    return None if a is None else a.ctypes.data


def _prep(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def sparse_attention(q, k, v, pat: AttnPattern, bias=None, weight_mult=None, forbid_empty_rows: bool = False,
                     *, dtype: str = "f64", plan: DevicePlan | None = None, return_lse: bool = False):
    """reference proj/src/attention.cpp:96-162 (fp64 conformance by default)."""
    q, k, v = (np.asarray(x) for x in (q, k, v))
    _check_shapes(q, k, v)
    if pat.rows != q.shape[0]:
        raise ConfigError("sparse_attention: pattern/sequence length mismatch")
    if bias is not None and len(bias) and len(bias) != pat.nnz():
        raise ConfigError("sparse_attention: bias must cover exactly the attended pairs")
    if weight_mult is not None and len(weight_mult) and len(weight_mult) != pat.nnz():
        raise ConfigError("sparse_attention: weight_mult size mismatch")
    bias = None if bias is None or len(bias) == 0 else bias
    weight_mult = None if weight_mult is None or len(weight_mult) == 0 else weight_mult
    dt = _NP[dtype]
    S, dk = q.shape
    dv = v.shape[1]
    qq, kk, vv = _prep(q, dt), _prep(k, dt), _prep(v, dt)
    b, w = _prep(bias, dt), _prep(weight_mult, dt)
    plan = plan or DevicePlan.from_pattern(pat)
    out = np.zeros((S, dv), dtype=dt)
    lse = np.zeros((S, 1), dtype=dt)
    if S > 0:
        check(_lib.lib().gte_sparse_attn_fwd_host(plan.ctx.h, plan.h, _lib.DTYPES[dtype], 1, dk, dv, qq.ctypes.data,
                                                  kk.ctypes.data, vv.ctypes.data, _ptr(b), _ptr(w), out.ctypes.data,
                                                  lse.ctypes.data, _lib.GTE_FORBID_EMPTY_ROWS if forbid_empty_rows else 0))
    res = AttnResult(out, MacCounter(pat.nnz() * dk, pat.nnz() * dv))
    if return_lse:
        return res, lse
    return res


def sparse_attention_backward(q, k, v, pat: AttnPattern, bias, weight_mult, upstream, *, dtype: str = "f64",
                              plan: DevicePlan | None = None) -> AttnGrads:
    """reference proj/src/attention.cpp:241-320"""
    q, k, v, upstream = (np.asarray(x) for x in (q, k, v, upstream))
    _check_shapes(q, k, v)
    S, dk = q.shape
    dv = v.shape[1]
    if pat.rows != S:
        raise ConfigError("sparse_attention_backward: pattern mismatch")
    if upstream.shape != (S, dv):
        raise ConfigError("sparse_attention_backward: upstream shape mismatch")
    bias = None if bias is None or len(bias) == 0 else bias
    weight_mult = None if weight_mult is None or len(weight_mult) == 0 else weight_mult
    dt = _NP[dtype]
    plan = plan or DevicePlan.from_pattern(pat)
    # the softmax statistics come from a forward through the same kernels
    # (the reference recomputes them inside its backward, attention.cpp:275-290)
    fwd, lse = _forward_nocheck(q, k, v, plan, bias, weight_mult, dtype)
    qq, kk, vv, uu = (_prep(x, dt) for x in (q, k, v, upstream))
    b, w = _prep(bias, dt), _prep(weight_mult, dt)
    dq, dkk, dvv = np.zeros((S, dk), dt), np.zeros((S, dk), dt), np.zeros((S, dv), dt)
    db = np.zeros(max(pat.nnz(), 1), dt)
    if S > 0:
        check(_lib.lib().gte_sparse_attn_bwd_host(plan.ctx.h, plan.h, _lib.DTYPES[dtype], 1, dk, dv, qq.ctypes.data,
                                                  kk.ctypes.data, vv.ctypes.data, fwd.ctypes.data, lse.ctypes.data,
                                                  uu.ctypes.data, _ptr(b), _ptr(w), dq.ctypes.data, dkk.ctypes.data,
                                                  dvv.ctypes.data, db.ctypes.data))
    return AttnGrads(dq, dkk, dvv, db[:pat.nnz()])


def _forward_nocheck(q, k, v, plan, bias, wm, dtype):
    dt = _NP[dtype]
    S, dk = q.shape
    dv = v.shape[1]
    qq, kk, vv = _prep(q, dt), _prep(k, dt), _prep(v, dt)
    b, w = _prep(bias, dt), _prep(wm, dt)  # keep the converted copies alive across the call
    out = np.zeros((S, dv), dt)
    lse = np.zeros((S, 1), dt)
    if S > 0:
        rc = _lib.lib().gte_sparse_attn_fwd_host(plan.ctx.h, plan.h, _lib.DTYPES[dtype], 1, dk, dv, qq.ctypes.data,
                                                 kk.ctypes.data, vv.ctypes.data, _ptr(b), _ptr(w),
                                                 out.ctypes.data, lse.ctypes.data, 0)
        if rc == _lib.GTE_DATA:
            # the reference backward performs no finiteness check
            # (attention.cpp:241-320); NaNs simply propagate
            pass
        else:
            check(rc)
    return out, lse


def edge_sparse_attention(q, k, v, g: Graph, bias=None, weight_mult=None, **kw) -> AttnResult:
    """reference proj/src/attention.cpp:164-172"""
    if g.num_nodes != np.asarray(q).shape[0]:
        raise ConfigError("edge_sparse_attention: graph/sequence length mismatch")
    return sparse_attention(q, k, v, pattern_from_graph(g), bias, weight_mult, forbid_empty_rows=True, **kw)


# --------------------------------------------------------------------------
# HBM-resident multi-head path (torch CUDA tensors are plumbing only)
# --------------------------------------------------------------------------

_TORCH_DT = {"f64": "float64", "f32": "float32", "bf16": "bfloat16"}


class DeviceSparseAttention:
    """All heads of one attention sublayer over a DevicePlan.

    q/k: [S, H*dk], v/out/dout: [S, H*dv] CUDA tensors of `dtype`;
    bias [nnz], weight_mult [H, nnz] in the accumulate type (f64 for f64,
    else f32). Launches on torch's current stream.
    """

    def __init__(self, plan: DevicePlan, heads: int, dk: int, dv: int | None = None, dtype: str = "f32"):
        self.plan, self.H, self.dk, self.dv, self.dtype = plan, heads, dk, dv or dk, dtype
        self.code = _lib.DTYPES[dtype]

    def _stream(self):
        import torch

        self.plan.ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def _check(self, qk, vo, acc):
        """The C ABI takes one leading dimension for the Q-shaped tensors
        (q, k, dq, dk) and one for the V-shaped ones (v, out, dout, dv): check
        that they agree, rows are unit-stride, dtypes match this instance and
        everything sits on one CUDA device. `acc` are the accumulate-typed
        tensors (lse, bias, weight_mult, dbias)."""
        import torch

        want = getattr(torch, _TORCH_DT[self.dtype])
        acc_t = torch.float64 if self.dtype == "f64" else torch.float32
        S = self.plan.rows
        dev = None
        for group, width, name in ((qk, self.H * self.dk, "q/k"), (vo, self.H * self.dv, "v/out")):
            ld = None
            for t in group:
                if t is None:
                    continue
                if t.dtype != want:
                    raise ConfigError(f"sparse_attention: {name} tensor dtype {t.dtype} != {want}")
                if t.dim() != 2 or t.shape[0] != S or t.shape[1] != width or t.stride(1) != 1:
                    raise ConfigError(f"sparse_attention: {name} tensors must be [S, {width}] with unit column stride")
                if ld is None:
                    ld = t.stride(0)
                elif t.stride(0) != ld:
                    raise ConfigError(f"sparse_attention: {name} tensors must share one row stride")
                dev = dev or t.device
                if t.device != dev or t.device.type != "cuda":
                    raise ConfigError("sparse_attention: all tensors must be on the plan's CUDA device")
        for t in acc:
            if t is None:
                continue
            if t.dtype != acc_t or not t.is_contiguous():
                raise ConfigError(f"sparse_attention: lse/bias/weight_mult/dbias must be contiguous {acc_t}")
            if t.device != dev:
                raise ConfigError("sparse_attention: all tensors must be on the plan's CUDA device")
        if dev is not None and dev.index is not None and dev.index != self.plan.ctx.device:
            raise ConfigError("sparse_attention: tensors are not on the plan's device")

    def forward(self, q, k, v, bias=None, weight_mult=None, out=None, lse=None, forbid_empty_rows=False):
        import torch

        S = self.plan.rows
        acc = torch.float64 if self.dtype == "f64" else torch.float32
        if out is None:
            out = torch.empty((S, self.H * self.dv), dtype=v.dtype, device=v.device)
        if lse is None:
            lse = torch.empty((S, self.H), dtype=acc, device=v.device)
        self._check((q, k), (v, out), (lse, bias, weight_mult))
        self._stream()
        check(_lib.lib().gte_sparse_attn_fwd(
            self.plan.ctx.h, self.plan.h, self.code, self.H, self.dk, self.dv, q.data_ptr(), k.data_ptr(),
            q.stride(0), v.data_ptr(), v.stride(0), None if bias is None else bias.data_ptr(),
            None if weight_mult is None else weight_mult.data_ptr(), out.data_ptr(), lse.data_ptr(),
            _lib.GTE_FORBID_EMPTY_ROWS if forbid_empty_rows else 0))
        return out, lse

    def backward(self, q, k, v, out, lse, dout, bias=None, weight_mult=None, dq=None, dk=None, dv=None, dbias=None):
        import torch

        acc = torch.float64 if self.dtype == "f64" else torch.float32
        dq = torch.empty_like(q) if dq is None else dq
        dk = torch.empty_like(k) if dk is None else dk
        dv = torch.empty_like(v) if dv is None else dv
        if dbias is None:
            dbias = torch.empty(max(self.plan.nnz, 1), dtype=acc, device=q.device)
        self._check((q, k, dq, dk), (v, out, dout, dv), (lse, bias, weight_mult, dbias))
        self._stream()
        check(_lib.lib().gte_sparse_attn_bwd(
            self.plan.ctx.h, self.plan.h, self.code, self.H, self.dk, self.dv, q.data_ptr(), k.data_ptr(),
            q.stride(0), v.data_ptr(), v.stride(0), out.data_ptr(), lse.data_ptr(), dout.data_ptr(),
            None if bias is None else bias.data_ptr(), None if weight_mult is None else weight_mult.data_ptr(),
            dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), dbias.data_ptr()))
        return dq, dk, dv, dbias

    def fwd_bwd_host(self, q, k, v, dout, bias, out, dq, dk, dv, dbias, sync: bool = True):
        """End-to-end unit with host (ideally pinned) buffers: H2D, fwd, bwd, D2H.
        Arguments are CPU tensors/arrays exposing .data_ptr() or ctypes.
        sync=False enqueues the step and returns (gte_sparse_attn_fwd_bwd_host_async):
        consecutive steps overlap downloads with the next uploads; call
        plan.ctx.sync() before reading the outputs."""
        def p(x):
            if x is None:
                return None
            return x.data_ptr() if hasattr(x, "data_ptr") else x.ctypes.data

        self._stream()
        fn = _lib.lib().gte_sparse_attn_fwd_bwd_host if sync else _lib.lib().gte_sparse_attn_fwd_bwd_host_async
        check(fn(
            self.plan.ctx.h, self.plan.h, self.code, self.H, self.dk, self.dv, p(q), p(k), p(v), p(dout), p(bias),
            p(out), p(dq), p(dk), p(dv), p(dbias)))


# --------------------------------------------------------------------------
# dense (all-pairs) attention, flash-style kernels (csrc/dense.cu)
# --------------------------------------------------------------------------

def _bind_dense():
    L = _lib.lib()
    if not getattr(L, "_dense_bound", False):
        VPt, I64t, I32t = C.c_void_p, C.c_int64, C.c_int
        L.gte_dense_attn_fwd.argtypes = [VPt, I32t, I64t, I64t, I32t, I32t, I32t, VPt, VPt, I64t, VPt, I64t, VPt, VPt,
                                         VPt, VPt]
        L.gte_dense_attn_bwd.argtypes = [VPt, I32t, I64t, I64t, I32t, I32t, I32t, VPt, VPt, I64t, VPt, I64t, VPt, VPt,
                                         VPt, VPt, VPt, VPt, VPt, VPt, VPt]
        L.gte_dense_attn_fwd_host.argtypes = [VPt, I32t, I64t, I64t, I32t, I32t, I32t, VPt, VPt, VPt, VPt, VPt, VPt,
                                              VPt]
        L.gte_dense_attn_bwd_host.argtypes = [VPt, I32t, I64t, I64t, I32t, I32t, I32t, VPt, VPt, VPt, VPt, VPt, VPt,
                                              VPt, VPt, VPt, VPt]
        L.gte_dense_attn_fwd_buckets.argtypes = [VPt, I32t, I64t, I64t, I32t, I32t, I32t, VPt, VPt, I64t, VPt, I64t,
                                                 VPt, VPt, I64t, VPt, VPt, VPt]
        L.gte_dense_attn_bwd_buckets.argtypes = [VPt, I32t, I64t, I64t, I32t, I32t, I32t, VPt, VPt, I64t, VPt, I64t,
                                                 VPt, VPt, VPt, VPt, VPt, I64t, VPt, VPt, VPt, VPt, VPt]
        L._dense_bound = True
    return L


def _dense_checks(q, k, v, bias, weight_mult):
    _check_shapes(q, k, v)
    s = q.shape[0]
    for m, nm in ((q, "Q"), (k, "K"), (v, "V")):  # attention.cpp:20-22
        if not np.all(np.isfinite(m)):
            raise DataError(f"attention: non-finite {nm}")
    if bias is not None:
        if np.shape(bias) != (s, s):
            raise ConfigError("dense_attention: bias shape")
        if not np.all(np.isfinite(bias)):
            raise DataError("attention: non-finite bias")
    if weight_mult is not None and np.shape(weight_mult) != (s, s):
        raise ConfigError("dense_attention: weight_mult shape")


def dense_attention(q, k, v, bias=None, weight_mult=None, *, dtype: str = "f64") -> AttnResult:
    """reference proj/src/attention.cpp:46-94 (bias, weight_mult: S x S or None)."""
    q, k, v = (np.asarray(x) for x in (q, k, v))
    _dense_checks(q, k, v, bias, weight_mult)
    L = _bind_dense()
    dt = _NP[dtype]
    S, dk = q.shape
    dv = v.shape[1]
    qq, kk, vv, b, w = _prep(q, dt), _prep(k, dt), _prep(v, dt), _prep(bias, dt), _prep(weight_mult, dt)
    out = np.zeros((S, dv), dt)
    check(L.gte_dense_attn_fwd_host(Context.get().h, _lib.DTYPES[dtype], S, S, 1, dk, dv, qq.ctypes.data,
                                    kk.ctypes.data, vv.ctypes.data, _ptr(b), _ptr(w), out.ctypes.data, None))
    return AttnResult(out, MacCounter(S * S * dk, S * S * dv))


def dense_attention_backward(q, k, v, bias, weight_mult, upstream, *, dtype: str = "f64") -> AttnGrads:
    """reference proj/src/attention.cpp:174-239; dbias is S x S row-major (flattened)."""
    q, k, v, upstream = (np.asarray(x) for x in (q, k, v, upstream))
    _check_shapes(q, k, v)
    S, dk = q.shape
    dv = v.shape[1]
    if upstream.shape != (S, dv):
        raise ConfigError("dense_attention_backward: upstream shape mismatch")
    L = _bind_dense()
    dt = _NP[dtype]
    qq, kk, vv, uu = (_prep(x, dt) for x in (q, k, v, upstream))
    b, w = _prep(bias, dt), _prep(weight_mult, dt)
    dq, dkk, dvv = np.zeros((S, dk), dt), np.zeros((S, dk), dt), np.zeros((S, dv), dt)
    db = np.zeros(S * S, dt)
    check(L.gte_dense_attn_bwd_host(Context.get().h, _lib.DTYPES[dtype], S, S, 1, dk, dv, qq.ctypes.data,
                                    kk.ctypes.data, vv.ctypes.data, _ptr(b), _ptr(w), uu.ctypes.data, dq.ctypes.data,
                                    dkk.ctypes.data, dvv.ctypes.data, db.ctypes.data))
    return AttnGrads(dq, dkk, dvv, db)


class DeviceDenseAttention:
    """All heads of a dense sublayer on CUDA tensors (q/k [S, H*dk], v [S, H*dv]).
    s_real < S gives the Trainer's dense epoch (model.cpp:395-405): real rows
    attend [0, s_real), pad rows only themselves. bias [S, S] / weight_mult
    [H, S, S] in the accumulate type, optional."""

    def __init__(self, S: int, heads: int, dk: int, dv: int | None = None, dtype: str = "f32",
                 s_real: int | None = None, ctx: Context | None = None):
        self.S, self.H, self.dk, self.dv, self.dtype = S, heads, dk, dv or dk, dtype
        self.s_real = S if s_real is None else s_real
        self.ctx = ctx or Context.get()
        self.code = _lib.DTYPES[dtype]

    def _check(self, qk, vo, acc=()):
        """The C ABI takes one row stride for the Q-shaped tensors (q, k and
        the dq, dk it writes) and one for the V-shaped ones (v, out, dout,
        dv): they must agree, rows must be unit-stride, dtypes must match this
        instance and everything must sit on the context's CUDA device."""
        import torch

        want = getattr(torch, _TORCH_DT[self.dtype])
        acc_t = torch.float64 if self.dtype == "f64" else torch.float32
        for group, width, name in ((qk, self.H * self.dk, "q/k"), (vo, self.H * self.dv, "v/out")):
            ld = None
            for t in group:
                if t.dtype != want:
                    raise ConfigError(f"dense_attention: {name} tensor dtype {t.dtype} != {want}")
                if t.dim() != 2 or t.shape[0] != self.S or t.shape[1] != width or t.stride(1) != 1:
                    raise ConfigError(f"dense_attention: {name} tensors must be [S, {width}] with unit column stride")
                if ld is None:
                    ld = t.stride(0)
                elif t.stride(0) != ld:
                    raise ConfigError(f"dense_attention: {name} tensors must share one row stride")
                if t.device.type != "cuda" or t.device.index != self.ctx.device:
                    raise ConfigError("dense_attention: tensors are not on the context's CUDA device")
        for t in acc:
            if t is None:
                continue
            if t.dtype not in (acc_t, torch.uint8) or not t.is_contiguous():
                raise ConfigError(f"dense_attention: lse/bias/weight_mult/buckets must be contiguous {acc_t}")
            if t.device.type != "cuda" or t.device.index != self.ctx.device:
                raise ConfigError("dense_attention: tensors are not on the context's CUDA device")

    def forward(self, q, k, v, bias=None, weight_mult=None):
        import torch

        self._check((q, k), (v,), (bias, weight_mult))
        L = _bind_dense()
        acc = torch.float64 if self.dtype == "f64" else torch.float32
        out = torch.empty_strided(v.shape, v.stride(), dtype=v.dtype, device=v.device)  # written with v's row stride
        lse = torch.empty((self.S, self.H), dtype=acc, device=v.device)
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        check(L.gte_dense_attn_fwd(self.ctx.h, self.code, self.S, self.s_real, self.H, self.dk, self.dv, q.data_ptr(),
                                   k.data_ptr(), q.stride(0), v.data_ptr(), v.stride(0),
                                   None if bias is None else bias.data_ptr(),
                                   None if weight_mult is None else weight_mult.data_ptr(), out.data_ptr(),
                                   lse.data_ptr()))
        return out, lse

    def backward(self, q, k, v, out, lse, dout, bias=None, weight_mult=None, want_dbias=False):
        import torch

        L = _bind_dense()
        acc = torch.float64 if self.dtype == "f64" else torch.float32
        self._check((q, k), (v, out, dout), (lse, bias, weight_mult))
        dq, dk, dv = (torch.empty_strided(x.shape, x.stride(), dtype=x.dtype, device=x.device) for x in (q, k, v))
        db = torch.empty((self.S, self.S), dtype=acc, device=q.device) if want_dbias else None
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        check(L.gte_dense_attn_bwd(self.ctx.h, self.code, self.S, self.s_real, self.H, self.dk, self.dv, q.data_ptr(),
                                   k.data_ptr(), q.stride(0), v.data_ptr(), v.stride(0), out.data_ptr(),
                                   lse.data_ptr(), dout.data_ptr(), None if bias is None else bias.data_ptr(),
                                   None if weight_mult is None else weight_mult.data_ptr(), dq.data_ptr(),
                                   dk.data_ptr(), dv.data_ptr(), None if db is None else db.data_ptr()))
        return dq, dk, dv, db

    # bucket-bias form of the Trainer's dense epoch (model.cpp:395-423, 520-523):
    # bias[r][c] = table[buckets[r][c]] (uint8 [S, S], glue.dense_buckets); the
    # backward returns the table's gradient instead of an S x S dbias
    def forward_buckets(self, q, k, v, buckets, table, weight_mult=None):
        import torch

        self._check((q, k), (v,), (buckets, table, weight_mult))
        L = _bind_dense()
        acc = torch.float64 if self.dtype == "f64" else torch.float32
        out = torch.empty_strided(v.shape, v.stride(), dtype=v.dtype, device=v.device)
        lse = torch.empty((self.S, self.H), dtype=acc, device=v.device)
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        check(L.gte_dense_attn_fwd_buckets(self.ctx.h, self.code, self.S, self.s_real, self.H, self.dk, self.dv,
                                           q.data_ptr(), k.data_ptr(), q.stride(0), v.data_ptr(), v.stride(0),
                                           buckets.data_ptr(), table.data_ptr(), table.numel(),
                                           None if weight_mult is None else weight_mult.data_ptr(), out.data_ptr(),
                                           lse.data_ptr()))
        return out, lse

    def backward_buckets(self, q, k, v, out, lse, dout, buckets, table, weight_mult=None):
        import torch

        self._check((q, k), (v, out, dout), (lse, buckets, table, weight_mult))
        L = _bind_dense()
        dq, dk, dv = (torch.empty_strided(x.shape, x.stride(), dtype=x.dtype, device=x.device) for x in (q, k, v))
        dtable = torch.empty_like(table)
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        check(L.gte_dense_attn_bwd_buckets(self.ctx.h, self.code, self.S, self.s_real, self.H, self.dk, self.dv,
                                           q.data_ptr(), k.data_ptr(), q.stride(0), v.data_ptr(), v.stride(0),
                                           out.data_ptr(), lse.data_ptr(), dout.data_ptr(), buckets.data_ptr(),
                                           table.data_ptr(), table.numel(),
                                           None if weight_mult is None else weight_mult.data_ptr(), dq.data_ptr(),
                                           dk.data_ptr(), dv.data_ptr(), dtable.data_ptr()))
        return dq, dk, dv, dtable
