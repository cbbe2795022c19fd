"""Cluster-halo sequence parallelism ("Mode H") for the
sparse attention layer.

The reference parallelises a layer by splitting heads (the Ulysses
all-to-all of parallel.cpp, mirrored in parallel.py). For the *sparse* layer
that moves ~S·d·e bytes per GPU per exchange — as much as the kernel itself
reads. After the cluster-aware reorder (partition.cpp:413-433) the pattern is
near block-diagonal over the k clusters, so here each GPU owns a contiguous
range of rows (a cluster when P = k) with *all* heads and exchanges only the
rows its edges reach in other ranges:

  forward   gather own K/V rows each peer needs -> all_to_allv straight into
            the halo tail of the local K/V buffers [own | halo] -> the same
            sparse kernels on the local plan (own rows' edges, columns
            renumbered into [own | halo]; halo rows have no edges)
  backward  same kernels: dQ of own rows and dbias of own edges are complete;
            dK/dV of halo rows are partial sums of this rank's edges -> sent
            back to their owners (all_to_allv) and added to the owners' rows
            in rank order (gte_rows_scatter_add; unique rows per source, no
            atomics)

Overlap (opt-in `overlap=True`): each rank's own rows split into *interior* rows
(every column local) and *boundary* rows (some column in the halo), each with
its own device plan over the same [own | halo] index space. The forward runs
the interior rows while the K|V halo exchange is in flight on a second
stream, then the boundary rows; the backward runs the boundary rows first
(their dK|dV halo partials are complete then), sends those back on the
second stream while the interior rows' backward runs, and adds the two
plans' dQ / dK / dV (disjoint rows; own-column partial sums) before the
owners' ordered scatter-add. Measured on the C3 pattern (profiles/r2w): the
halo exchange is small (~10K rows of 2 x 128 B per rank at P = 8, a few us
over NVLink) while the second plan per rank costs +30-60 % of the kernel
time, so the default is one plan per rank; the step is then one stream of
work that bench.py replays as a CUDA graph.

The math per pair is the reference's (sparse_attention / _backward, the
attention.cpp:96-320 semantics); only the summation order of dK/dV over
ranks (and over the interior / boundary split) differs from a single GPU.
The bias/dbias of a rank are the contiguous slice of the global pattern's
edges that its rows own.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ConfigError, check
from .attention import Context, DevicePlan, DeviceSparseAttention

VP, I64, I32 = C.c_void_p, C.c_int64, C.c_int


def _bind():
    L = _lib.lib()
    if not getattr(L, "_halo_bound", False):
        L.gte_rows_gather.argtypes = [VP, I32, I64, VP, VP, I64, I64, VP]
        L.gte_rows_scatter_add.argtypes = [VP, I32, I64, VP, VP, I64, VP, I64]
        L.gte_comm_all_to_allv.argtypes = [VP, VP, VP, VP, VP, VP, VP, VP]
        L.gte_rows_scatter_add_seq.argtypes = [VP, I32, I64, VP, VP, VP, VP, I64, I64, VP, I64]
        L._halo_bound = True
    return L


def row_ranges(S: int, P: int) -> np.ndarray:
    """Near-equal contiguous ranges, first S % P get one more
    (cluster_boundaries, partition.cpp:495-500)."""
    base, extra = divmod(S, P)
    sizes = np.full(P, base, dtype=np.int64)
    sizes[:extra] += 1
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


@dataclass
class RankHalo:
    """One rank's share of the pattern and its exchange lists."""
    rank: int
    lo: int
    hi: int
    n_own: int
    halo_ids: np.ndarray     # global ids of halo rows (sorted: by owner, then id)
    recv_counts: np.ndarray  # [P] halo rows received from each peer
    send_idx: list           # [P] local own-row indices each peer needs (ascending global id)
    local_ro: np.ndarray     # CSR over [own | halo] rows (halo rows empty)
    local_co: np.ndarray
    e_lo: int                # own rows' edges are [e_lo, e_hi) of the global CSR
    e_hi: int
    # interior / boundary split: the same CSR with only one kind of own row
    # keeping its edges; eidx_* = those edges' positions in the local CSR
    boundary: np.ndarray = None  # [n_ext] bool, own rows with a halo column
    ro_i: np.ndarray = None
    co_i: np.ndarray = None
    eidx_i: np.ndarray = None
    ro_b: np.ndarray = None
    co_b: np.ndarray = None
    eidx_b: np.ndarray = None

    @property
    def n_ext(self) -> int:
        return self.n_own + int(self.halo_ids.shape[0])

    def boundary_rows(self) -> tuple[int, int]:
        """(rows received, rows sent) per exchange: the Mode H ledger."""
        return int(self.recv_counts.sum()), int(sum(len(s) for s in self.send_idx))


def build_halo_plan(row_offsets, cols, P: int) -> list[RankHalo]:
    """Host planner (numpy, O(E)) for all P ranks; every rank can run it on the
    replicated pattern, so no index lists travel."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    co = np.asarray(cols, dtype=np.int64)
    S = ro.shape[0] - 1
    if P < 1 or P > S:
        raise ConfigError("halo: worker count must lie in [1, S]")
    b = row_ranges(S, P)
    owner_of = np.repeat(np.arange(P), np.diff(b))
    halos = []
    for p in range(P):
        lo, hi = int(b[p]), int(b[p + 1])
        e_lo, e_hi = int(ro[lo]), int(ro[hi])
        c = co[e_lo:e_hi]
        remote = np.unique(c[(c < lo) | (c >= hi)])  # sorted by id == by owner then id
        halos.append((lo, hi, e_lo, e_hi, remote))
    plans = []
    for p in range(P):
        lo, hi, e_lo, e_hi, remote = halos[p]
        n_own = hi - lo
        recv_counts = np.bincount(owner_of[remote], minlength=P).astype(np.int64) if remote.size else np.zeros(P, np.int64)
        send_idx = []
        for q in range(P):
            rq = halos[q][4]
            mine = rq[(rq >= lo) & (rq < hi)] if q != p else rq[:0]
            send_idx.append((mine - lo).astype(np.int32))
        c = co[e_lo:e_hi]
        own = (c >= lo) & (c < hi)
        lc = np.empty_like(c)
        lc[own] = c[own] - lo
        lc[~own] = n_own + np.searchsorted(remote, c[~own])
        n_ext = n_own + remote.shape[0]
        lro = np.empty(n_ext + 1, dtype=np.int64)
        lro[: n_own + 1] = ro[lo:hi + 1] - e_lo
        lro[n_own + 1:] = e_hi - e_lo
        r = RankHalo(p, lo, hi, n_own, remote, recv_counts, send_idx, lro, lc, e_lo, e_hi)
        _split_rows(r)
        plans.append(r)
    return plans


def _split_rows(r: RankHalo) -> None:
    """Interior / boundary sub-patterns of a rank's local CSR (same row space)."""
    n_ext, ro, co = r.n_ext, r.local_ro, r.local_co
    deg = np.diff(ro)
    row_of = np.repeat(np.arange(n_ext), deg)
    halo_edge = co >= r.n_own
    boundary = np.zeros(n_ext, dtype=bool)
    boundary[row_of[halo_edge]] = True
    r.boundary = boundary
    for tag, keep_rows in (("i", ~boundary), ("b", boundary)):
        keep = keep_rows[row_of]
        d = np.where(keep_rows, deg, 0)
        sub_ro = np.concatenate([[0], np.cumsum(d)]).astype(np.int64)
        setattr(r, "ro_" + tag, sub_ro)
        setattr(r, "co_" + tag, co[keep])
        setattr(r, "eidx_" + tag, np.nonzero(keep)[0].astype(np.int64))


class HaloLoopback:
    """All P ranks in one process on one GPU: the all_to_allv is a set of
    device copies between the ranks' buffers (the reference's own execution
    model of logical workers)."""

    def __init__(self, P: int):
        self.P = P

    def exchange(self, sends: dict, recvs: dict, send_counts: dict, recv_counts: dict, row_elems: int):
        """sends[p]: [sum_q send_counts[p][q], w] blocks in peer order; recvs[p]: destination
        [sum_q recv_counts[p][q], w] in peer order. Copies block (p -> q)."""
        for q in range(self.P):
            off_q = 0
            for p in range(self.P):
                n = int(recv_counts[q][p])
                if n:
                    off_p = int(np.sum(send_counts[p][:q]))
                    recvs[q][off_q:off_q + n].copy_(sends[p][off_p:off_p + n])
                off_q += n


class HaloNccl:
    """One rank per GPU: gte_comm_all_to_allv over the NCCL communicator of a
    parallel.NcclExchange (which owns the id broadcast)."""

    def __init__(self, comm_exchange, rank: int, ctx: Context):
        self.cx, self.rank, self.ctx = comm_exchange, rank, ctx

    def exchange(self, sends: dict, recvs: dict, send_counts: dict, recv_counts: dict, row_elems: int):
        import torch

        p = self.rank
        x, y = sends[p], recvs[p]
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)  # the exchange stream under HaloAttention
        es = x.element_size() * row_elems
        sc = np.asarray(send_counts[p], dtype=np.int64) * es
        rc = np.asarray(recv_counts[p], dtype=np.int64) * es
        so = np.concatenate([[0], np.cumsum(sc)[:-1]]).astype(np.int64)
        ro_ = np.concatenate([[0], np.cumsum(rc)[:-1]]).astype(np.int64)
        check(_bind().gte_comm_all_to_allv(self.cx.h, self.ctx.h, x.data_ptr(), so.ctypes.data, sc.ctypes.data,
                                           y.data_ptr(), ro_.ctypes.data, rc.ctypes.data))


class TorchDistHalo:
    """all_to_allv over an existing torch.distributed group (gloo on CPU for
    the multi-process tests; one rank per process)."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange(self, sends: dict, recvs: dict, send_counts: dict, recv_counts: dict, row_elems: int):
        import torch.distributed as dist

        p = self.rank
        sc = [int(x) for x in send_counts[p]]
        rc = [int(x) for x in recv_counts[p]]
        x = sends[p][: sum(sc)].contiguous()
        y = recvs[p]
        out = y.new_empty((sum(rc),) + tuple(y.shape[1:]))
        dist.all_to_all_single(out, x, output_split_sizes=rc, input_split_sizes=sc, group=self.group)
        if sum(rc):
            y[: sum(rc)].copy_(out)


class DeviceHaloOps:
    """The device half of HaloAttention: local plans + the sparse attention
    kernels, row gather and ordered scatter-add (csrc/sp.cu), and a second
    CUDA stream for the exchanges."""

    def __init__(self, heads: int, dh: int, dtype: str, ctx=None, schedule: bool = True):
        self.H, self.dh, self.dtype, self.d = heads, dh, dtype, heads * dh
        self.ctx = ctx or Context.get(0)
        self.schedule = schedule
        self.att = {}
        self._comm = None

    def setup(self, key, n: int, ro: np.ndarray, co: np.ndarray, n_out: int | None = None):
        plan = DevicePlan.from_host(ro, co, self.ctx)
        if self.schedule:
            plan.schedule()
        if n_out is not None and n_out < n:  # halo rows exist only as columns: no tiles for them
            plan.set_output_rows(n_out)
        self.att[key] = DeviceSparseAttention(plan, self.H, self.dh, self.dh, self.dtype)

    def index(self, idx: np.ndarray):
        import torch

        return torch.tensor(idx.astype(np.int32), device=torch.device("cuda", self.ctx.device))

    def _stream_here(self):
        import torch

        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)

    def gather(self, ext, idx, n: int):
        import torch

        buf = torch.empty((max(n, 1), self.d), dtype=ext.dtype, device=ext.device)
        if n:
            self._stream_here()
            check(_bind().gte_rows_gather(self.ctx.h, _lib.DTYPES[self.dtype], n, idx.data_ptr(), ext.data_ptr(),
                                          self.d, self.d, buf.data_ptr()))
        return buf

    def scatter_add(self, dst, idx, src, n: int):
        self._stream_here()
        check(_bind().gte_rows_scatter_add(self.ctx.h, _lib.DTYPES[self.dtype], n, idx.data_ptr(), src.data_ptr(),
                                           self.d, dst.data_ptr(), self.d))

    def scatter_add_seq(self, dst, seq, src, col0: int):
        """dst[rows[u]] += src[pos[j], col0:col0+d] for j in [ptr[u], ptr[u+1])
        in order: every peer's partials in one launch (gte_rows_scatter_add_seq)."""
        rows, ptr, pos = seq
        n = int(rows.numel())
        if n:
            self._stream_here()
            check(_bind().gte_rows_scatter_add_seq(self.ctx.h, _lib.DTYPES[self.dtype], n, rows.data_ptr(),
                                                   ptr.data_ptr(), pos.data_ptr(),
                                                   src.data_ptr() + col0 * src.element_size(), src.stride(0),
                                                   self.d, dst.data_ptr(), dst.stride(0)))

    def attn_fwd(self, key, q, k, v, b):
        return self.att[key].forward(q, k, v, b)

    def attn_bwd(self, key, q, k, v, o, lse, do, b):
        return self.att[key].backward(q, k, v, o, lse, do, b)

    # ---- the exchange stream: work under `comm()` is ordered after the
    # current stream's work so far; `join()` orders the current stream after it
    def comm(self):
        import torch

        if self._comm is None:
            self._comm = torch.cuda.Stream(device=torch.device("cuda", self.ctx.device))
        self._comm.wait_stream(torch.cuda.current_stream())
        return torch.cuda.stream(self._comm)

    def join(self):
        import torch

        if self._comm is not None:
            torch.cuda.current_stream().wait_stream(self._comm)


class _Serial:
    """Exchange "stream" of ops without one (CPU checkers): run in place."""

    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class HaloAttention:
    """The sparse attention layer over P ranks with a cluster-halo exchange.
    `ranks` are the RankHalo plans this process holds (all P for the loopback,
    one for NCCL / torch.distributed). Shards: own rows [n_own, H*dh] per
    rank. `ops` supplies the kernels (DeviceHaloOps unless given). With
    `overlap` the interior / boundary rows run on their own plans so the
    exchanges overlap the interior rows' kernels (module docstring)."""

    def __init__(self, ranks: list[RankHalo], P: int, heads: int, dh: int, dtype: str, exchange, ctx=None,
                 schedule: bool = True, ops=None, overlap: bool = False):
        self.ranks, self.P, self.H, self.dh, self.dtype, self.x = ranks, P, heads, dh, dtype, exchange
        self.d = heads * dh
        self.ops = ops or DeviceHaloOps(heads, dh, dtype, ctx, schedule)
        self.overlap = overlap
        import torch

        dev = torch.device("cuda", self.ops.ctx.device) if hasattr(self.ops, "ctx") else torch.device("cpu")
        self.idx = {}
        self.parts = {}  # rank -> [(tag, local edge positions)] of the plans that run
        self._bmask = {}
        self._seq = {}
        for r in ranks:
            if overlap and r.boundary is not None and r.n_ext > r.n_own:
                parts = []
                for tag in ("i", "b"):
                    ro_, co_, ei = getattr(r, "ro_" + tag), getattr(r, "co_" + tag), getattr(r, "eidx_" + tag)
                    if co_.shape[0]:
                        self.ops.setup((r.rank, tag), r.n_ext, ro_, co_, r.n_own)
                        parts.append((tag, torch.tensor(ei, dtype=torch.int64, device=dev)))
                self.parts[r.rank] = parts
                self._bmask[r.rank] = torch.tensor(r.boundary, device=dev)
            else:
                self.ops.setup((r.rank, "all"), r.n_ext, r.local_ro, r.local_co, r.n_own)
                self.parts[r.rank] = [("all", None)]
            cat = np.concatenate(r.send_idx) if r.send_idx else np.zeros(0, np.int32)
            self.idx[r.rank] = self.ops.index(cat)
            if hasattr(self.ops, "scatter_add_seq"):  # the peers' partials per own row, in peer order
                order = np.argsort(cat, kind="stable")
                rows_u, first, cnt = np.unique(cat[order], return_index=True, return_counts=True)
                ptr = np.concatenate([[0], np.cumsum(cnt)])
                self._seq[r.rank] = tuple(self.ops.index(x) for x in (rows_u, ptr, order))
        self._send_counts = {r.rank: [len(s) for s in r.send_idx] for r in ranks}
        self._recv_counts = {r.rank: list(r.recv_counts) for r in ranks}
        if len(ranks) == P:  # loopback: every rank's counts are local
            self._all_send = self._send_counts
            self._all_recv = self._recv_counts
        self.cache = {}
        self._bufs = {}

    def _comm(self):
        return self.ops.comm() if hasattr(self.ops, "comm") else _Serial()

    def _join(self):
        if hasattr(self.ops, "join"):
            self.ops.join()

    def _ext(self, r: RankHalo, own, name: str, zero_tail: bool = False):
        """[own | halo] buffer, persistent per (rank, tensor): allocated once,
        own rows copied in each step. Tails are zeroed once: the kernels'
        padding slots may read any row of the local index space, and with the
        overlap the interior plan's own-row checks read the K / V tails while
        the exchange rewrites them (always finite values)."""
        if r.n_ext == r.n_own:
            return own.contiguous()
        key = (r.rank, name)
        t = self._bufs.get(key)
        if t is None or t.dtype != own.dtype or t.device != own.device:
            t = own.new_empty((r.n_ext, self.d))
            if zero_tail:
                t[r.n_own:].zero_()
            self._bufs[key] = t
        if own.data_ptr() != t.data_ptr() or own.stride() != t.stride():  # not written in place (own_view)
            t[: r.n_own].copy_(own)
        return t

    def own_view(self, rank: int, name: str, dtype, device):
        """The own rows of the persistent [own | halo] buffer of tensor `name`
        ("q", "k", "v", "do"): a caller that writes a step's shard here saves
        the per-step copy into the buffer (bench.py's ranks do)."""
        r = next(x for x in self.ranks if x.rank == rank)
        key = (rank, name)
        t = self._bufs.get(key)
        if t is None or t.dtype != dtype or t.device != device:
            import torch

            t = torch.zeros((r.n_ext, self.d), dtype=dtype, device=device)
            self._bufs[key] = t
        return t[: r.n_own]

    def _halo_in_kv(self, kx: dict, vx: dict):
        """Fill the halo tails of the K and V ext buffers with the owners' rows:
        one all_to_allv of [K row | V row] pairs (2d wide) instead of two."""
        import torch

        sends, recvs = {}, {}
        for r in self.ranks:
            n = int(self.idx[r.rank].numel())
            m = r.n_ext - r.n_own
            if n:
                sends[r.rank] = torch.cat([self.ops.gather(kx[r.rank], self.idx[r.rank], n),
                                           self.ops.gather(vx[r.rank], self.idx[r.rank], n)], dim=1)
            else:
                sends[r.rank] = kx[r.rank].new_zeros((1, 2 * self.d))
            recvs[r.rank] = kx[r.rank].new_empty((max(m, 1), 2 * self.d))
        self.x.exchange(sends, recvs, self._all_send_counts(), self._all_recv_counts(), 2 * self.d)
        for r in self.ranks:
            m = r.n_ext - r.n_own
            if m:
                kx[r.rank][r.n_own:].copy_(recvs[r.rank][:m, : self.d])
                vx[r.rank][r.n_own:].copy_(recvs[r.rank][:m, self.d:])

    def _halo_back_send(self, gk: dict, gv: dict) -> dict:
        """Send the halo rows' dK | dV partial sums to their owners in one
        all_to_allv; returns the received blocks per rank."""
        import torch

        sends, recvs = {}, {}
        for r in self.ranks:
            m = r.n_ext - r.n_own
            n = int(self.idx[r.rank].numel())
            if m:
                sends[r.rank] = torch.cat([gk[r.rank][r.n_own:], gv[r.rank][r.n_own:]], dim=1)
            else:
                sends[r.rank] = gk[r.rank].new_zeros((1, 2 * self.d))
            recvs[r.rank] = gk[r.rank].new_empty((max(n, 1), 2 * self.d))
        self.x.exchange(sends, recvs, self._all_recv_counts(), self._all_send_counts(), 2 * self.d)
        return recvs

    def _halo_back_add(self, gk: dict, gv: dict, recvs: dict):
        """Add the received partials to the owners' rows, source by source in
        rank order (unique rows per source: no atomics, fixed order) — on the
        device as one ordered launch per tensor."""
        for r in self.ranks:
            if r.rank in self._seq:
                self.ops.scatter_add_seq(gk[r.rank], self._seq[r.rank], recvs[r.rank], 0)
                self.ops.scatter_add_seq(gv[r.rank], self._seq[r.rank], recvs[r.rank], self.d)
                continue
            off = 0
            idx, rv = self.idx[r.rank], recvs[r.rank]
            for n in self._send_counts[r.rank]:
                if n:
                    blk = rv[off:off + n]
                    self.ops.scatter_add(gk[r.rank], idx[off:off + n], blk[:, : self.d].contiguous(), n)
                    self.ops.scatter_add(gv[r.rank], idx[off:off + n], blk[:, self.d:].contiguous(), n)
                off += n

    def _all_send_counts(self):
        return getattr(self, "_all_send", self._send_counts)

    def _all_recv_counts(self):
        return getattr(self, "_all_recv", self._recv_counts)

    @staticmethod
    def _take(b, ei):
        return None if b is None or ei is None else b[ei]

    def _merge_rows(self, r: RankHalo, a, b):
        """Rows of the boundary plan's result over the interior plan's."""
        if a is None or b is None:
            return a if b is None else b
        m = self._bmask[r.rank]
        return a.where(~m.view(-1, *([1] * (a.dim() - 1))), b)

    def forward(self, q: dict, k: dict, v: dict, bias=None):
        """bias: the global pattern's [E] (each rank uses its edges' slice)."""
        kx = {r.rank: self._ext(r, k[r.rank], "k", zero_tail=True) for r in self.ranks}
        vx = {r.rank: self._ext(r, v[r.rank], "v", zero_tail=True) for r in self.ranks}
        qx = {r.rank: self._ext(r, q[r.rank], "q", zero_tail=True) for r in self.ranks}
        bl = {r.rank: None if bias is None else bias[r.e_lo:r.e_hi] for r in self.ranks}
        res = {r.rank: {} for r in self.ranks}
        with self._comm():  # halo rows in, on the exchange stream
            self._halo_in_kv(kx, vx)
        for r in self.ranks:  # interior rows (no halo column) meanwhile
            for tag, ei in self.parts[r.rank]:
                if tag == "i":
                    res[r.rank][tag] = self.ops.attn_fwd((r.rank, tag), qx[r.rank], kx[r.rank], vx[r.rank],
                                                         self._take(bl[r.rank], ei))
        self._join()
        out = {}
        for r in self.ranks:
            for tag, ei in self.parts[r.rank]:
                if tag != "i":
                    b = bl[r.rank] if tag == "all" else self._take(bl[r.rank], ei)
                    res[r.rank][tag] = self.ops.attn_fwd((r.rank, tag), qx[r.rank], kx[r.rank], vx[r.rank], b)
            got = res[r.rank]
            if "all" in got:
                o, lse = got["all"]
            else:
                oi, li = got.get("i", (None, None))
                ob, lb = got.get("b", (None, None))
                o, lse = self._merge_rows(r, oi, ob), self._merge_rows(r, li, lb)
            self.cache[r.rank] = (qx[r.rank], kx[r.rank], vx[r.rank], o, lse, bl[r.rank])
            out[r.rank] = o[: r.n_own]
        return out

    def backward(self, dout: dict):
        """Returns {rank: (dq_own, dk_own, dv_own, dbias_own_edges)}."""
        import torch

        got, dox = {}, {}
        for r in self.ranks:  # boundary rows first: the halo partials are complete after them
            qx, kx, vx, o, lse, b = self.cache[r.rank]
            dox[r.rank] = self._ext(r, dout[r.rank], "do", zero_tail=True)
            got[r.rank] = {}
            for tag, ei in self.parts[r.rank]:
                if tag != "i":
                    bb = b if tag == "all" else self._take(b, ei)
                    got[r.rank][tag] = self.ops.attn_bwd((r.rank, tag), qx, kx, vx, o, lse, dox[r.rank], bb)
        first = {r.rank: next(iter(got[r.rank].values())) if got[r.rank] else None for r in self.ranks}
        send_k = {p: (g[1] if g is not None else None) for p, g in first.items()}
        send_v = {p: (g[2] if g is not None else None) for p, g in first.items()}
        for r in self.ranks:  # a rank without boundary rows sends zeros
            if send_k[r.rank] is None:
                qx = self.cache[r.rank][0]
                send_k[r.rank] = qx.new_zeros((r.n_ext, self.d))
                send_v[r.rank] = qx.new_zeros((r.n_ext, self.d))
        with self._comm():  # halo dK | dV partials back, on the exchange stream
            recvs = self._halo_back_send(send_k, send_v)
        for r in self.ranks:  # interior rows meanwhile
            qx, kx, vx, o, lse, b = self.cache[r.rank]
            for tag, ei in self.parts[r.rank]:
                if tag == "i":
                    got[r.rank][tag] = self.ops.attn_bwd((r.rank, tag), qx, kx, vx, o, lse, dox[r.rank],
                                                         self._take(b, ei))
        gq, gk, gv, gb = {}, {}, {}, {}
        for r in self.ranks:
            parts = got[r.rank]
            if "all" in parts:
                gq[r.rank], gk[r.rank], gv[r.rank], gb[r.rank] = parts["all"]
                continue
            dq = dk = dv = None
            db = None
            for tag, ei in self.parts[r.rank]:
                a_q, a_k, a_v, a_b = parts[tag]
                # disjoint rows for dQ; own-column partial sums for dK / dV
                dq = a_q if dq is None else dq + a_q
                dk = a_k if dk is None else dk + a_k
                dv = a_v if dv is None else dv + a_v
                if a_b is not None:
                    if db is None:
                        db = a_b.new_zeros(r.e_hi - r.e_lo)
                    db[ei] = a_b[: ei.shape[0]]
            gq[r.rank], gk[r.rank], gv[r.rank], gb[r.rank] = dq, dk, dv, db
        self._join()
        self._halo_back_add(gk, gv, recvs)
        return {r.rank: (gq[r.rank][: r.n_own], gk[r.rank][: r.n_own], gv[r.rank][: r.n_own],
                         gb[r.rank][: r.e_hi - r.e_lo]) for r in self.ranks}
