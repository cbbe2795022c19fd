"""Host mirror of the reference partition / reformation operator API over the
C ABI (reference proj/include/gte/partition.hpp, reformation.hpp).

``reorder`` runs the exact host reorder (csrc/reorder.cpp); the CSR
transforms (``graph_from_edges``, ``add_self_loops``, ``permute_graph``), the
cluster grid and the layout materialisation run on the GPU; results come back
as numpy arrays shaped like the reference structs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import ConfigError, DataError, check
from .attention import AttnPattern, Context, DevicePlan, Graph

I64P = C.POINTER(C.c_int64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


@dataclass
class Permutation:
    forward: np.ndarray  # old id -> new position
    inverse: np.ndarray  # new position -> old id

    def size(self) -> int:
        return int(self.forward.shape[0])

    @staticmethod
    def identity(n: int) -> "Permutation":
        a = np.arange(n, dtype=np.int64)
        return Permutation(a, a.copy())

    def valid(self) -> bool:
        n = self.size()
        if self.inverse.shape[0] != n:
            return False
        f = self.forward
        if n and (f.min() < 0 or f.max() >= n):
            return False
        return bool(np.array_equal(self.inverse[f], np.arange(n)))


@dataclass
class ClusterGrid:
    k: int
    boundaries: np.ndarray
    cell_nnz: np.ndarray
    cell_density: np.ndarray

    def range_size(self, a: int) -> int:
        return int(self.boundaries[a + 1] - self.boundaries[a])

    def cluster_of(self, pos: int) -> int:
        n = int(self.boundaries[-1])
        base, rem = n // self.k, n % self.k
        cut = rem * (base + 1)
        return pos // (base + 1) if pos < cut else rem + (pos - cut) // base

    def total_nnz(self) -> int:
        return int(self.cell_nnz.sum())


@dataclass
class ClusterSparseLayout:
    seq_len: int
    k: int
    d_b: int
    boundaries: np.ndarray
    cell_state: np.ndarray  # 0 untouched, 1 transferred
    block_off: np.ndarray
    blocks: np.ndarray  # [n_blocks, 2] cell-local (row, col)
    dropped_edges: int
    pattern: AttnPattern
    device_plan: DevicePlan | None = field(default=None, repr=False)

    def transferred_cells(self) -> int:
        return int(self.cell_state.sum())

    def subblock_count(self) -> int:
        return int(self.blocks.shape[0])

    def global_blocks(self) -> np.ndarray:
        """Sub-block origins in sequence coordinates, [n_blocks, 2] (row0, col0),
        cell by cell (reformation.cpp:176-189 places tile (r, c) of cell (a, b)
        at (boundaries[a] + r, boundaries[b] + c))."""
        out = np.zeros((int(self.block_off[-1]), 2), dtype=np.int64)
        for cell in range(self.k * self.k):
            b0, b1 = int(self.block_off[cell]), int(self.block_off[cell + 1])
            if b1 > b0:
                a, b = divmod(cell, self.k)
                out[b0:b1, 0] = self.blocks[b0:b1, 0] + self.boundaries[a]
                out[b0:b1, 1] = self.blocks[b0:b1, 1] + self.boundaries[b]
        return out

    def cell_blocks(self, cell: int) -> np.ndarray:
        return self.blocks[self.block_off[cell]:self.block_off[cell + 1]]


# ------------------------------------------------------------------ device CSR helpers

class DeviceCSR:
    """int32 CSR resident on the GPU (torch tensors as plumbing)."""

    def __init__(self, n: int, row_ptr, cols, nnz: int):
        self.n, self.row_ptr, self.cols, self.nnz = n, row_ptr, cols, nnz

    @classmethod
    def from_graph(cls, g: Graph, device=None):
        import torch

        dev = device or torch.device("cuda", torch.cuda.current_device())
        rp = torch.as_tensor(np.asarray(g.row_offsets, dtype=np.int32), device=dev)
        co = torch.as_tensor(np.asarray(g.col_indices, dtype=np.int32), device=dev)
        return cls(g.num_nodes, rp, co, g.nnz())

    def to_graph(self) -> Graph:
        ro = self.row_ptr[: self.n + 1].cpu().numpy().astype(np.int64)
        co = self.cols[: self.nnz].cpu().numpy().astype(np.int64)
        return Graph(self.n, ro, co)


def _ctx() -> Context:
    import torch

    ctx = Context.get(torch.cuda.current_device())
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    return ctx


def graph_from_edges(n: int, src, dst) -> Graph:
    """reference proj/src/graph.cpp:49-66 (GPU sort + unique)."""
    import torch

    ctx = _ctx()
    dev = torch.device("cuda", ctx.device)
    s = torch.as_tensor(np.asarray(src, dtype=np.int64), device=dev)
    d = torch.as_tensor(np.asarray(dst, dtype=np.int64), device=dev)
    if n < 0:
        raise DataError("graph_from_edges: negative node count")
    bad = ((s < 0) | (s >= n) | (d < 0) | (d >= n)).nonzero()
    if bad.numel():
        e = int(bad[0, 0])
        u, v = int(s[e]), int(d[e])
        badv = u if (u < 0 or u >= n) else v
        raise DataError(f"graph_from_edges: node id {badv} out of range [0, {n})")
    s32, d32 = s.to(torch.int32), d.to(torch.int32)
    m = s32.numel()
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    co = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    nnz = C.c_int64()
    check(_lib.lib().gte_graph_from_edges(ctx.h, C.c_int64(n), C.c_int64(m), C.c_void_p(s32.data_ptr()),
                                          C.c_void_p(d32.data_ptr()), C.c_void_p(rp.data_ptr()),
                                          C.c_void_p(co.data_ptr()), C.byref(nnz)))
    return DeviceCSR(n, rp, co, nnz.value).to_graph()


def add_self_loops(g: Graph) -> Graph:
    """reference proj/src/graph.cpp:127-149."""
    import torch

    ctx = _ctx()
    dc = DeviceCSR.from_graph(g, torch.device("cuda", ctx.device))
    rp = torch.empty(g.num_nodes + 1, dtype=torch.int32, device=dc.row_ptr.device)
    co = torch.empty(max(g.nnz() + g.num_nodes, 1), dtype=torch.int32, device=dc.row_ptr.device)
    nnz = C.c_int64()
    check(_lib.lib().gte_add_self_loops(ctx.h, C.c_int64(g.num_nodes), C.c_int64(g.nnz()),
                                        C.c_void_p(dc.row_ptr.data_ptr()), C.c_void_p(dc.cols.data_ptr()),
                                        C.c_void_p(rp.data_ptr()), C.c_void_p(co.data_ptr()), C.byref(nnz)))
    return DeviceCSR(g.num_nodes, rp, co, nnz.value).to_graph()


def density(g: Graph) -> float:
    """reference proj/src/graph.cpp:151-155."""
    if g.num_nodes < 1:
        raise DataError("density: empty graph")
    return float(g.nnz()) / (float(g.num_nodes) * float(g.num_nodes))


def reorder(g: Graph, k: int, seed: int) -> Permutation:
    """reference proj/src/partition.cpp:413-433 (exact, host)."""
    n = g.num_nodes
    ro, co = _i64(g.row_offsets), _i64(g.col_indices)
    if co.shape[0] == 0:
        co = np.zeros(1, dtype=np.int64)
    fwd = np.zeros(max(n, 1), dtype=np.int64)
    inv = np.zeros(max(n, 1), dtype=np.int64)
    check(_lib.lib().gte_reorder(C.c_int64(n), C.c_int64(g.nnz()), ro.ctypes.data_as(I64P), co.ctypes.data_as(I64P),
                                 C.c_int64(k), C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), fwd.ctypes.data_as(I64P),
                                 inv.ctypes.data_as(I64P)))
    return Permutation(fwd[:n], inv[:n])


def cluster_boundaries(n: int, k: int) -> np.ndarray:
    b = np.zeros(k + 1, dtype=np.int64)
    check(_lib.lib().gte_cluster_boundaries(C.c_int64(n), C.c_int64(k), b.ctypes.data_as(I64P)))
    return b


def permute_graph(g: Graph, p: Permutation) -> Graph:
    """reference proj/src/partition.cpp:435-456."""
    import torch

    if p.size() != g.num_nodes or not p.valid():
        raise ConfigError("permute_graph: bad permutation")
    ctx = _ctx()
    dc = DeviceCSR.from_graph(g, torch.device("cuda", ctx.device))
    rp = torch.empty(g.num_nodes + 1, dtype=torch.int32, device=dc.row_ptr.device)
    co = torch.empty(max(g.nnz(), 1), dtype=torch.int32, device=dc.row_ptr.device)
    f = _i64(p.forward)
    check(_lib.lib().gte_permute_graph(ctx.h, C.c_int64(g.num_nodes), C.c_int64(g.nnz()),
                                       C.c_void_p(dc.row_ptr.data_ptr()), C.c_void_p(dc.cols.data_ptr()),
                                       f.ctypes.data_as(I64P), C.c_void_p(rp.data_ptr()), C.c_void_p(co.data_ptr())))
    return DeviceCSR(g.num_nodes, rp, co, g.nnz()).to_graph()


def build_cluster_grid(g: Graph, p: Permutation | None, k: int) -> ClusterGrid:
    """reference proj/src/partition.cpp:514-539 (p=None: graph already ordered)."""
    import torch

    if k < 1 or k > g.num_nodes:
        raise ConfigError("build_cluster_grid: invalid k")
    if p is not None and (p.size() != g.num_nodes or not p.valid()):
        raise ConfigError("build_cluster_grid: permutation does not match graph")
    ctx = _ctx()
    dc = DeviceCSR.from_graph(g, torch.device("cuda", ctx.device))
    bnd = np.zeros(k + 1, dtype=np.int64)
    nnz = np.zeros(k * k, dtype=np.int64)
    den = np.zeros(k * k, dtype=np.float64)
    f = None if p is None else _i64(p.forward)
    check(_lib.lib().gte_build_cluster_grid(ctx.h, C.c_int64(g.num_nodes), C.c_int64(g.nnz()),
                                            C.c_void_p(dc.row_ptr.data_ptr()), C.c_void_p(dc.cols.data_ptr()),
                                            None if f is None else f.ctypes.data_as(I64P), C.c_int64(k),
                                            bnd.ctypes.data_as(I64P), nnz.ctypes.data_as(I64P),
                                            den.ctypes.data_as(C.POINTER(C.c_double))))
    return ClusterGrid(k, bnd, nnz, den)


def diagonal_edge_fraction(grid: ClusterGrid) -> float:
    out = C.c_double()
    cn = _i64(grid.cell_nnz)
    check(_lib.lib().gte_diagonal_edge_fraction(C.c_int64(grid.k), cn.ctypes.data_as(I64P), C.byref(out)))
    return out.value


INDOLENT, ELASTIC = 0, 1


def pack_subblocks(cell_edges, n_rows: int, n_cols: int, d_b: int) -> np.ndarray:
    """reference proj/src/reformation.cpp:56-109; returns [n_tiles, 2] origins."""
    e = np.asarray(cell_edges, dtype=np.int64).reshape(-1, 2)
    er, ec = _i64(e[:, 0]), _i64(e[:, 1])
    m = e.shape[0]
    cap = max(1, (m + d_b * d_b - 1) // (d_b * d_b)) if d_b >= 1 else 1
    out = np.zeros(2 * cap + 2, dtype=np.int64)
    nt = C.c_int64()
    if m == 0:
        er = ec = np.zeros(1, dtype=np.int64)
    check(_lib.lib().gte_pack_subblocks(C.c_int64(m), er.ctypes.data_as(I64P), ec.ctypes.data_as(I64P),
                                        C.c_int64(n_rows), C.c_int64(n_cols), C.c_int64(d_b),
                                        out.ctypes.data_as(I64P), C.byref(nt)))
    return out[: 2 * nt.value].reshape(-1, 2)


def build_layout(grid: ClusterGrid, g_perm: Graph, strategy: int, beta_thre: float, beta_g: float, d_b: int,
                 keep_device_plan: bool = False) -> ClusterSparseLayout:
    """reference proj/src/reformation.cpp:111-195."""
    import torch

    ctx = _ctx()
    dc = DeviceCSR.from_graph(g_perm, torch.device("cuda", ctx.device))
    k = grid.k
    bnd, cn, cd = _i64(grid.boundaries), _i64(grid.cell_nnz), np.ascontiguousarray(grid.cell_density, np.float64)
    h = C.c_void_p()
    check(_lib.lib().gte_build_layout(ctx.h, C.c_int64(g_perm.num_nodes), C.c_int64(g_perm.nnz()),
                                      C.c_void_p(dc.row_ptr.data_ptr()), C.c_void_p(dc.cols.data_ptr()), C.c_int64(k),
                                      bnd.ctypes.data_as(I64P), cn.ctypes.data_as(I64P),
                                      cd.ctypes.data_as(C.POINTER(C.c_double)), C.c_int(strategy),
                                      C.c_double(beta_thre), C.c_double(beta_g), C.c_int64(d_b), C.byref(h)))
    L = _lib.lib()
    try:
        tr, nb, dr, pn = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        L.gte_layout_info(h, C.byref(tr), C.byref(nb), C.byref(dr), C.byref(pn))
        state = np.zeros(k * k, dtype=np.int32)
        boff = np.zeros(k * k + 1, dtype=np.int64)
        blocks = np.zeros(2 * nb.value + 2, dtype=np.int64)
        L.gte_layout_cells(h, state.ctypes.data_as(C.POINTER(C.c_int32)), boff.ctypes.data_as(I64P),
                           blocks.ctypes.data_as(I64P))
        n = g_perm.num_nodes
        ro = np.zeros(n + 1, dtype=np.int64)
        co = np.zeros(max(pn.value, 1), dtype=np.int64)
        check(L.gte_layout_pattern_host(h, ro.ctypes.data_as(I64P), co.ctypes.data_as(I64P)))
        plan = None
        if keep_device_plan:
            rp, cl = C.c_void_p(), C.c_void_p()
            L.gte_layout_pattern_device(h, C.byref(rp), C.byref(cl))
            plan = DevicePlan.from_device(n, pn.value, rp.value, cl.value or 0, ctx)
        return ClusterSparseLayout(n, k, d_b, bnd.copy(), state, boff, blocks[: 2 * nb.value].reshape(-1, 2),
                                   dr.value, AttnPattern(n, ro, co[: pn.value]), plan)
    finally:
        L.gte_layout_destroy(h)
