"""Trainer glue around the attention kernels (reference
proj/src/model.cpp:76-83, 407-423, 447-463, 520-523): pad loops on the
pattern, SPD bias buckets per attended pair, the per-pair bias gathered from
the layer's bucket table and the table's gradient. All computation in
libgte_b200.so (csrc/glue.cu); torch tensors are device-memory plumbing."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check
from .attention import Context

VP, I64 = C.c_void_p, C.c_int64


def _bind():
    L = _lib.lib()
    if not getattr(L, "_glue_bound", False):
        L.gte_extend_with_pad_loops_host.argtypes = [I64, I64, VP, VP, I64, VP, VP]
        L.gte_pattern_buckets.argtypes = [VP, I64, I64, VP, VP, VP, I64, I64, VP, VP, VP, I64, VP]
        L.gte_bias_from_table.argtypes = [VP, I64, VP, VP, I64, VP]
        L.gte_dbias_to_table.argtypes = [VP, I64, VP, VP, I64, VP, VP]
        L.gte_spd_table.argtypes = [VP, I64, I64, VP, VP, I64, C.POINTER(VP)]
        L.gte_spd_info.argtypes = [VP, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]
        L.gte_spd_copy_host.argtypes = [VP, VP, VP, VP]
        L.gte_spd_destroy.argtypes = [VP]
        L.gte_spd_pairs.argtypes = [VP, I64, I64, VP, VP, I64, I64, VP, VP, VP]
        L.gte_pattern_buckets_graph.argtypes = [VP, I64, I64, VP, VP, VP, I64, I64, I64, VP, VP, I64, VP]
        L.gte_dense_buckets.argtypes = [VP, I64, I64, VP, VP, I64, I64, I64, VP, VP, I64, VP]
        L._glue_bound = True
    return L


def extend_with_pad_loops(row_offsets, cols, s_pad: int):
    """model.cpp:76-83 -> (row_offsets, cols) with one self-loop per pad row."""
    ro = np.ascontiguousarray(row_offsets, dtype=np.int64)
    co = np.ascontiguousarray(cols, dtype=np.int64)
    rows = ro.shape[0] - 1
    extra = max(0, s_pad - rows)
    oro = np.zeros(rows + extra + 1, dtype=np.int64)
    oco = np.zeros(max(co.shape[0] + extra, 1), dtype=np.int64)
    check(_bind().gte_extend_with_pad_loops_host(rows, co.shape[0], ro.ctypes.data,
                                                 co.ctypes.data if co.shape[0] else None, s_pad, oro.ctypes.data,
                                                 oco.ctypes.data))
    return oro, oco[: co.shape[0] + extra]


def pattern_buckets(row_offsets, cols, perm_inverse, global_index: int, spd, max_dist: int, ctx: Context | None = None):
    """Bucket per attended pair (model.cpp:447-463). spd = (row_off, cols, dist
    uint16, num_nodes) — the reference SpdTable. Returns an int32 CUDA tensor."""
    import torch

    ctx = ctx or Context.get(0)
    dev = torch.device("cuda", ctx.device)
    ro = torch.tensor(np.asarray(row_offsets, dtype=np.int32), device=dev)
    co = torch.tensor(np.asarray(cols, dtype=np.int32), device=dev)
    inv = torch.tensor(np.asarray(perm_inverse, dtype=np.int64), device=dev)
    sro, sco, sdi, sn = spd
    t_sro = torch.tensor(np.asarray(sro, dtype=np.int64), device=dev)
    t_sco = torch.tensor(np.asarray(sco, dtype=np.int64) if len(sco) else np.zeros(1, np.int64), device=dev)
    t_sdi = torch.tensor(np.asarray(sdi, dtype=np.int16).view(np.int16) if len(sdi) else np.zeros(1, np.int16),
                         device=dev)
    out = torch.empty(max(co.numel(), 1), dtype=torch.int32, device=dev)
    check(_bind().gte_pattern_buckets(ctx.h, ro.numel() - 1, co.numel(), ro.data_ptr(), co.data_ptr(),
                                      inv.data_ptr(), global_index, sn, t_sro.data_ptr(), t_sco.data_ptr(),
                                      t_sdi.data_ptr(), max_dist, out.data_ptr()))
    return out[: co.numel()]


def bias_from_table(buckets, table, ctx: Context | None = None):
    """bias[e] = spd_bias[bucket[e]] (model.cpp:520-523); CUDA tensors."""
    import torch

    ctx = ctx or Context.get(0)
    bias = torch.empty(buckets.numel(), dtype=torch.float32, device=buckets.device)
    check(_bind().gte_bias_from_table(ctx.h, buckets.numel(), buckets.data_ptr(), table.data_ptr(), table.numel(),
                                      bias.data_ptr()))
    return bias


def dbias_to_table(buckets, dbias, n_buckets: int, ctx: Context | None = None):
    """Gradient of the bucket table: sum of dbias per bucket (fixed order)."""
    import torch

    ctx = ctx or Context.get(0)
    out = torch.empty(n_buckets, dtype=torch.float32, device=buckets.device)
    ws = torch.empty(296 * n_buckets, dtype=torch.float32, device=buckets.device)
    check(_bind().gte_dbias_to_table(ctx.h, buckets.numel(), buckets.data_ptr(), dbias.data_ptr(), n_buckets,
                                     out.data_ptr(), ws.data_ptr()))
    return out


def _dev_csr(row_offsets, cols, dev):
    import torch

    ro = torch.tensor(np.asarray(row_offsets, dtype=np.int32), device=dev)
    co = np.asarray(cols, dtype=np.int32)
    co = torch.tensor(co if co.shape[0] else np.zeros(1, np.int32), device=dev)
    return ro, co, int(np.asarray(cols).shape[0])


def spd_table(row_offsets, cols, max_dist: int, ctx: Context | None = None):
    """The reference SpdTable (graph.cpp:216-262) built on the GPU, any size
    whose table fits: (row_off int64, cols int64, dist uint16, num_nodes)."""
    ctx = ctx or Context.get(0)
    import torch

    dev = torch.device("cuda", ctx.device)
    ro, co, m = _dev_csr(row_offsets, cols, dev)
    n = ro.numel() - 1
    h = VP()
    L = _bind()
    check(L.gte_spd_table(ctx.h, n, m, ro.data_ptr(), co.data_ptr(), max_dist, C.byref(h)))
    try:
        nn, md, tot = I64(), I64(), I64()
        L.gte_spd_info(h, C.byref(nn), C.byref(md), C.byref(tot))
        sro = np.zeros(n + 1, np.int64)
        sco = np.zeros(max(tot.value, 1), np.int64)
        sdi = np.zeros(max(tot.value, 1), np.uint16)
        check(L.gte_spd_copy_host(h, sro.ctypes.data, sco.ctypes.data, sdi.ctypes.data))
        return sro, sco[: tot.value], sdi[: tot.value], n
    finally:
        L.gte_spd_destroy(h)


def spd_pairs(row_offsets, cols, max_dist: int, src, dst, ctx: Context | None = None):
    """Capped shortest-path distance of each (src, dst) pair on the GPU,
    without the table (max_dist + 1 beyond the cap); int32 numpy."""
    ctx = ctx or Context.get(0)
    import torch

    dev = torch.device("cuda", ctx.device)
    ro, co, m = _dev_csr(row_offsets, cols, dev)
    s = torch.tensor(np.asarray(src, np.int32), device=dev)
    d = torch.tensor(np.asarray(dst, np.int32), device=dev)
    out = torch.empty(max(s.numel(), 1), dtype=torch.int32, device=dev)
    check(_bind().gte_spd_pairs(ctx.h, ro.numel() - 1, m, ro.data_ptr(), co.data_ptr(), max_dist, s.numel(),
                                s.data_ptr(), d.data_ptr(), out.data_ptr()))
    return out[: s.numel()].cpu().numpy()


def pattern_buckets_graph(row_offsets, cols, perm_inverse, global_index: int, graph_row_offsets, graph_cols,
                          max_dist: int, ctx: Context | None = None):
    """Bucket per attended pair (model.cpp:447-463) with the SPD computed from
    the graph on the GPU (no N <= 20000 table guard). int32 CUDA tensor."""
    ctx = ctx or Context.get(0)
    import torch

    dev = torch.device("cuda", ctx.device)
    ro, co, m = _dev_csr(row_offsets, cols, dev)
    gro, gco, gm = _dev_csr(graph_row_offsets, graph_cols, dev)
    inv = torch.tensor(np.asarray(perm_inverse, dtype=np.int64), device=dev)
    out = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    check(_bind().gte_pattern_buckets_graph(ctx.h, ro.numel() - 1, m, ro.data_ptr(), co.data_ptr(), inv.data_ptr(),
                                            global_index, gro.numel() - 1, gm, gro.data_ptr(), gco.data_ptr(),
                                            max_dist, out.data_ptr()))
    return out[:m]


def dense_buckets(S: int, s_real: int, perm_forward, perm_inverse, global_index: int, graph_row_offsets, graph_cols,
                  max_dist: int, ctx: Context | None = None):
    """Bucket matrix of the Trainer's dense epoch (model.cpp:407-423) in
    execution coordinates: uint8 CUDA tensor [S, S], rows/columns < s_real set
    (0 self, 1 global token, capped SPD else), one device BFS per row."""
    ctx = ctx or Context.get(0)
    import torch

    dev = torch.device("cuda", ctx.device)
    gro, gco, gm = _dev_csr(graph_row_offsets, graph_cols, dev)
    fwd = torch.tensor(np.asarray(perm_forward, dtype=np.int64), device=dev)
    inv = torch.tensor(np.asarray(perm_inverse, dtype=np.int64), device=dev)
    out = torch.empty((S, S), dtype=torch.uint8, device=dev)
    check(_bind().gte_dense_buckets(ctx.h, S, s_real, fwd.data_ptr(), inv.data_ptr(), global_index, gro.numel() - 1,
                                    gm, gro.data_ptr(), gco.data_ptr(), max_dist, out.data_ptr()))
    return out
