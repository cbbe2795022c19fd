"""Sequence parallelism on B200: the reference's distributed attention layer
(proj/include/gte/parallel.hpp, proj/src/parallel.cpp) with the Ulysses
all-to-all on the device.

The reference runs P *logical* workers in one process: each owns a shard of
token rows (partition_sequence, parallel.cpp:96-113); Q/K/V are gathered over
the sequence and split over heads by one all-to-all (seq->head, :115-155),
every worker runs its H/P heads over the whole (cluster-permuted) pattern, and
the output goes back by the inverse all-to-all (head->seq, :157-188). Here the
same layer runs with

* ``Loopback`` — P logical workers in one process on one GPU (the reference's
  own execution model; run_distributed_layer / _backward below mirror its API
  and semantics, ledger included), or
* ``NcclExchange`` — one rank per GPU, NCCL send/recv all-to-all over NVLink
  (gte_comm_* in csrc/sp.cu), or
* any object with the same ``all_to_all`` / ``gather_parts`` contract (the
  CPU tests plug in torch.distributed over gloo).

Per exchange: pack (one kernel) -> all-to-all of P equal chunks -> unpack
(one kernel); the cluster permutation is folded into the unpack/pack of the
head-sliced side (csrc/sp.cu). Everything computes through libgte_b200.so;
torch tensors are device-memory plumbing only.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import ConfigError, check
from .attention import Context, DevicePlan, DeviceSparseAttention, MacCounter

VP, I64, I32 = C.c_void_p, C.c_int64, C.c_int


def _bind():
    L = _lib.lib()
    if getattr(L, "_sp_bound", False):
        return L
    L.gte_partition_sequence.argtypes = [I64, I64, C.c_uint64, VP, C.POINTER(I64)]
    L.gte_sp_create.argtypes = [VP, I64, I64, VP, VP, C.POINTER(VP)]
    L.gte_sp_destroy.argtypes = [VP]
    for nm in ("gte_sp_pack_seq", "gte_sp_unpack_head", "gte_sp_pack_head", "gte_sp_unpack_seq"):
        getattr(L, nm).argtypes = [VP, VP, I32, I64, I64, VP, VP]
    L.gte_sp_loopback.argtypes = [VP, VP, I32, I64, VP, VP]
    L.gte_sp_ordered_sum.argtypes = [VP, I32, I64, I64, VP, VP]
    L.gte_nccl_unique_id.argtypes = [VP]
    L.gte_comm_create.argtypes = [VP, I32, I32, VP, C.POINTER(VP)]
    L.gte_comm_destroy.argtypes = [VP]
    L.gte_comm_all_to_all.argtypes = [VP, VP, VP, VP, I64]
    L.gte_comm_all_gather.argtypes = [VP, VP, VP, VP, I64]
    L._sp_bound = True
    return L


# --------------------------------------------------------------------------
# reference types (parallel.hpp:15-44, :70-91)
# --------------------------------------------------------------------------

@dataclass
class LedgerEntry:
    qkv_gather: int = 0
    qkv_gather_cross: int = 0
    output_scatter: int = 0
    output_scatter_cross: int = 0
    bias_exchange: int = 0


class CommLedger:
    """Exact per-worker element counts of the two collectives (parallel.hpp:23-44)."""

    def __init__(self, num_workers: int = 0):
        self.workers = [LedgerEntry() for _ in range(num_workers)]

    def reset(self):
        self.workers = [LedgerEntry() for _ in self.workers]

    def accumulate(self, other: "CommLedger"):
        """parallel.cpp:83-94"""
        if len(self.workers) != len(other.workers):
            raise ConfigError("ledger: worker count mismatch")
        for a, b in zip(self.workers, other.workers):
            a.qkv_gather += b.qkv_gather
            a.qkv_gather_cross += b.qkv_gather_cross
            a.output_scatter += b.output_scatter
            a.output_scatter_cross += b.output_scatter_cross
            a.bias_exchange += b.bias_exchange

    def transport_elements(self, w: int) -> int:
        return self.workers[w].qkv_gather + self.workers[w].output_scatter

    def tally(self, P: int, rows: int, slice_: int, as_qkv: bool):
        """One all-to-all of P x P chunks of rows x slice elements: every
        worker sends P chunks, P-1 of them cross (parallel.cpp:134-146,
        :171-185; both directions count per *source* worker)."""
        elems = rows * slice_
        for e in self.workers:
            if as_qkv:
                e.qkv_gather += P * elems
                e.qkv_gather_cross += (P - 1) * elems
            else:
                e.output_scatter += P * elems
                e.output_scatter_cross += (P - 1) * elems


@dataclass
class WorkerShard:
    worker_id: int
    token_ids: np.ndarray
    q_sub: object = None
    k_sub: object = None
    v_sub: object = None


@dataclass
class DistAttnResult:
    out_shards: list
    macs: MacCounter = field(default_factory=MacCounter)


@dataclass
class DistAttnGrads:
    dq_sub: list
    dk_sub: list
    dv_sub: list
    dbias: object


def partition_sequence(seq_len: int, num_workers: int, seed: int) -> list[WorkerShard]:
    """parallel.cpp:96-113: pad to a multiple of P, shuffle with
    mt19937_64(seed), split contiguously (C ABI gte_partition_sequence)."""
    L = _bind()
    if num_workers < 1:
        raise ConfigError("partition_sequence: worker count must be >= 1")
    if seq_len < 1:
        raise ConfigError("partition_sequence: empty sequence")
    padded = ((seq_len + num_workers - 1) // num_workers) * num_workers
    ids = np.zeros(padded, dtype=np.int64)
    pad = I64()
    check(L.gte_partition_sequence(seq_len, num_workers, C.c_uint64(seed), ids.ctypes.data, C.byref(pad)))
    per = padded // num_workers
    return [WorkerShard(w, ids[w * per:(w + 1) * per].copy()) for w in range(num_workers)]


# --------------------------------------------------------------------------
# device exchange plan + exchanges
# --------------------------------------------------------------------------

class SequenceParallelPlan:
    """gte_sp: token ids per worker + the cluster permutation's forward map."""

    def __init__(self, token_ids: list, perm_forward=None, ctx: Context | None = None):
        L = _bind()
        self.ctx = ctx or Context.get(0)
        self.P = len(token_ids)
        self.rows = int(len(token_ids[0]))
        if any(len(t) != self.rows for t in token_ids):
            raise ConfigError("all_to_all: token ids misaligned with shard rows")
        self.total = self.P * self.rows
        tok = np.ascontiguousarray(np.concatenate([np.asarray(t, dtype=np.int64) for t in token_ids]))
        fwd = None if perm_forward is None else np.ascontiguousarray(np.asarray(perm_forward, dtype=np.int64))
        if fwd is not None and fwd.shape[0] != self.total:
            raise ConfigError("run_distributed_layer: permutation size mismatch")
        h = VP()
        check(L.gte_sp_create(self.ctx.h, self.P, self.rows, tok.ctypes.data,
                              None if fwd is None else fwd.ctypes.data, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            _lib.lib().gte_sp_destroy(self.h)
        except Exception:
            pass


class Loopback:
    """All P workers in this process (one GPU): send_all [src][dst] -> recv_all [dst][src]."""

    def __init__(self, sp: SequenceParallelPlan):
        self.sp = sp
        self.local = list(range(sp.P))

    def all_to_all(self, send: dict, dtype: str, d: int) -> dict:
        import torch

        P = self.sp.P
        src = torch.stack([send[w] for w in range(P)])  # [P, P*chunk]
        dst = torch.empty_like(src)
        check(_bind().gte_sp_loopback(self.sp.ctx.h, self.sp.h, _lib.DTYPES[dtype], d, src.data_ptr(),
                                      dst.data_ptr()))
        return {w: dst[w] for w in range(P)}

    def gather_parts(self, parts: dict):
        import torch

        return torch.stack([parts[w] for w in range(self.sp.P)])


class NcclExchange:
    """One rank per GPU: rank r is worker r. The 128-byte NCCL id travels over
    an existing torch.distributed group (plumbing); the data path is NCCL."""

    def __init__(self, sp: SequenceParallelPlan | None, rank: int, world: int, group=None, ctx: Context | None = None):
        import torch
        import torch.distributed as dist

        L = _bind()
        if sp is not None and sp.P != world:
            raise ConfigError("comm: worker count must equal the world size")
        self.sp, self.rank, self.local = sp, rank, [rank]
        self.ctx = sp.ctx if sp is not None else (ctx or Context.get(0))
        idb = (C.c_uint8 * 128)()
        if rank == 0:
            check(L.gte_nccl_unique_id(C.cast(idb, VP)))
        t = torch.tensor(list(bytes(idb)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0, group=group)
        raw = bytes(t.cpu().tolist())
        idb = (C.c_uint8 * 128).from_buffer_copy(raw)
        h = VP()
        check(L.gte_comm_create(self.ctx.h, world, rank, C.cast(idb, VP), C.byref(h)))
        self.h = h

    def all_to_all(self, send: dict, dtype: str, d: int) -> dict:
        import torch

        x = send[self.rank]
        y = torch.empty_like(x)
        nbytes = x.numel() * x.element_size() // self.sp.P
        check(_bind().gte_comm_all_to_all(self.h, self.sp.ctx.h, x.data_ptr(), y.data_ptr(), nbytes))
        return {self.rank: y}

    def gather_parts(self, parts: dict):
        import torch

        x = parts[self.rank]
        y = torch.empty((self.sp.P,) + tuple(x.shape), dtype=x.dtype, device=x.device)
        check(_bind().gte_comm_all_gather(self.h, self.sp.ctx.h, x.data_ptr(), y.data_ptr(),
                                          x.numel() * x.element_size()))
        return y

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().gte_comm_destroy(self.h)
            self.h = None


# --------------------------------------------------------------------------
# the distributed attention sublayer
# --------------------------------------------------------------------------

class DeviceOps:
    """The device half of the layer: pack/unpack kernels (csrc/sp.cu), the
    sparse attention kernels over the execution-coordinate pattern, the
    worker-ordered dbias sum. All through libgte_b200.so."""

    def __init__(self, plan: DevicePlan, sp: SequenceParallelPlan, heads: int, d: int, dtype: str):
        self.plan, self.sp, self.H, self.d, self.dtype = plan, sp, heads, d, dtype
        self.code = _lib.DTYPES[dtype]
        self.slice = d // sp.P
        self.hpw = heads // sp.P
        self.att = DeviceSparseAttention(plan, self.hpw, d // heads, d // heads, dtype)

    def _run(self, fn, x, shape):
        import torch

        y = torch.empty(shape, dtype=x.dtype, device=x.device)
        check(getattr(_bind(), fn)(self.sp.ctx.h, self.sp.h, self.code, self.d, self.H, x.data_ptr(), y.data_ptr()))
        return y

    def pack_seq(self, shard):
        return self._run("gte_sp_pack_seq", shard, (self.sp.P * self.sp.rows * self.slice,))

    def unpack_head(self, buf):
        return self._run("gte_sp_unpack_head", buf, (self.sp.total, self.slice))

    def pack_head(self, sl):
        return self._run("gte_sp_pack_head", sl, (self.sp.P * self.sp.rows * self.slice,))

    def unpack_seq(self, buf):
        return self._run("gte_sp_unpack_seq", buf, (self.sp.rows, self.d))

    def attn_fwd(self, q, k, v, bias, wm):
        return self.att.forward(q, k, v, bias, wm)

    def attn_bwd(self, q, k, v, o, lse, up, bias, wm):
        import torch

        acc = torch.float64 if self.dtype == "f64" else torch.float32
        db = torch.empty(max(self.plan.nnz, 1), dtype=acc, device=q.device)
        dq, dk, dv, _ = self.att.backward(q, k, v, o, lse, up, bias, wm, dbias=db)
        return dq, dk, dv, db[: self.plan.nnz]

    def ordered_sum(self, stacked):
        import torch

        P, n = stacked.shape[0], stacked.shape[1]
        out = torch.empty(max(n, 1), dtype=stacked.dtype, device=stacked.device)
        code = _lib.GTE_F64 if stacked.dtype == torch.float64 else _lib.GTE_F32
        check(_bind().gte_sp_ordered_sum(self.sp.ctx.h, code, P, n, stacked.data_ptr(), out.data_ptr()))
        return out[:n]


class TorchDistExchange:
    """Exchange over an existing torch.distributed group (gloo on CPU for the
    multi-process tests; NCCL through torch works the same way). Rank r is
    worker r."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group, self.local = rank, world, group, [rank]

    def all_to_all(self, send: dict, dtype: str, d: int) -> dict:
        import torch
        import torch.distributed as dist

        x = send[self.rank].contiguous()
        y = torch.empty_like(x)
        dist.all_to_all_single(y, x, group=self.group)
        return {self.rank: y}

    def gather_parts(self, parts: dict):
        import torch
        import torch.distributed as dist

        x = parts[self.rank].contiguous()
        out = [torch.empty_like(x) for _ in range(self.world)]
        dist.all_gather(out, x, group=self.group)
        return torch.stack(out)


class UlyssesAttention:
    """run_distributed_layer / run_distributed_layer_backward (parallel.cpp:
    190-332) for the workers this process holds (`exchange.local`).

    Shards are tensors [rows, d]; the pattern is in execution coordinates
    with S_pad rows; bias [E] is replicated (ledger bias_exchange = E per
    worker, :222-224); weight_mult [H, E] head-major (worker w uses heads
    w*H/P .. (w+1)*H/P, :233-243). The forward caches the head-sliced
    Q/K/V/O and LSE for the backward (the reference re-gathers Q/K/V,
    :291-293 — same values, three exchanges fewer)."""

    def __init__(self, ops, P: int, rows: int, heads: int, d: int, nnz: int, exchange):
        if heads % P != 0:
            raise ConfigError("all_to_all: head count not divisible by worker count")
        if d % heads != 0:
            raise ConfigError("all_to_all: hidden dim not divisible by head count")
        self.ops, self.P, self.rows, self.H, self.d, self.E, self.x = ops, P, rows, heads, d, nnz, exchange
        self.hpw, self.dh, self.slice = heads // P, d // heads, d // P
        self.dtype = ops.dtype
        self.cache = {}

    @classmethod
    def on_device(cls, plan: DevicePlan, sp: SequenceParallelPlan, heads: int, d: int, dtype: str, exchange):
        if plan.rows != sp.total:
            raise ConfigError("run_distributed_layer: pattern/sequence mismatch")
        return cls(DeviceOps(plan, sp, heads, d, dtype), sp.P, sp.rows, heads, d, plan.nnz, exchange)

    def _seq_to_head(self, shards: dict) -> dict:
        recv = self.x.all_to_all({w: self.ops.pack_seq(x) for w, x in shards.items()}, self.dtype, self.d)
        return {w: self.ops.unpack_head(b) for w, b in recv.items()}

    def _head_to_seq(self, slices: dict) -> dict:
        recv = self.x.all_to_all({w: self.ops.pack_head(x) for w, x in slices.items()}, self.dtype, self.d)
        return {w: self.ops.unpack_seq(b) for w, b in recv.items()}

    def _wm(self, weight_mult, w):
        if weight_mult is None:
            return None
        return weight_mult[w * self.hpw:(w + 1) * self.hpw].contiguous()

    def forward(self, q: dict, k: dict, v: dict, bias=None, weight_mult=None, ledger: CommLedger | None = None):
        qs, ks, vs = self._seq_to_head(q), self._seq_to_head(k), self._seq_to_head(v)
        if ledger is not None:
            for _ in range(3):
                ledger.tally(self.P, self.rows, self.slice, True)
            if bias is not None:
                for e in ledger.workers:
                    e.bias_exchange += int(bias.numel())
        outs = {}
        for w in self.x.local:
            o, lse = self.ops.attn_fwd(qs[w], ks[w], vs[w], bias, self._wm(weight_mult, w))
            outs[w] = o
            self.cache[w] = (qs[w], ks[w], vs[w], o, lse)
        macs = MacCounter(self.H * self.E * self.dh, self.H * self.E * self.dh)  # attention.cpp:159-160 per head
        res = self._head_to_seq(outs)
        if ledger is not None:
            ledger.tally(self.P, self.rows, self.slice, False)
        return res, macs

    def backward(self, dout: dict, bias=None, weight_mult=None):
        ups = self._seq_to_head(dout)  # backward of the output scatter is the forward gather (:294)
        dqs, dks, dvs, parts = {}, {}, {}, {}
        for w in self.x.local:
            q, k, v, o, lse = self.cache[w]
            dqs[w], dks[w], dvs[w], parts[w] = self.ops.attn_bwd(q, k, v, o, lse, ups[w], bias,
                                                                 self._wm(weight_mult, w))
        dq, dk, dv = self._head_to_seq(dqs), self._head_to_seq(dks), self._head_to_seq(dvs)
        dbias = self.ops.ordered_sum(self.x.gather_parts(parts))  # [P, E] in worker order (:319)
        return dq, dk, dv, dbias


# --------------------------------------------------------------------------
# reference API mirror: P logical workers in one process (parallel.cpp:190-332)
# --------------------------------------------------------------------------

def _as_dev(x, dtype):
    import torch

    td = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=td).contiguous()
    return torch.tensor(np.asarray(x), dtype=td, device="cuda")


def run_distributed_layer(shards: list[WorkerShard], pattern, perm, num_heads: int, bias=None, weight_mult=None,
                          ledger: CommLedger | None = None, dtype: str = "f64", _keep=None) -> DistAttnResult:
    """parallel.cpp:190-252. `pattern` is an AttnPattern/Graph-like object with
    row_offsets/cols (execution coordinates), `perm` a Permutation (forward
    old -> new). Returns host (numpy) shards like the reference."""
    if not shards:
        raise ConfigError("run_distributed_layer: no shards")
    P = len(shards)
    if ledger is not None and len(ledger.workers) != P:
        raise ConfigError("run_distributed_layer: ledger sized for wrong worker count")
    d = np.asarray(shards[0].q_sub).shape[1]
    total = np.asarray(shards[0].q_sub).shape[0] * P
    rows = _rows_of(pattern)
    if rows != total:
        raise ConfigError("run_distributed_layer: pattern/sequence mismatch")
    if perm is not None and perm.size() != total:
        raise ConfigError("run_distributed_layer: permutation size mismatch")
    if num_heads % P != 0:
        raise ConfigError("all_to_all: head count not divisible by worker count")
    if d % num_heads != 0:
        raise ConfigError("all_to_all: hidden dim not divisible by head count")
    E = _nnz_of(pattern)
    if weight_mult is not None and np.asarray(weight_mult).size != num_heads * E:
        raise ConfigError("run_distributed_layer: weight_mult size mismatch")
    layer = _layer(shards, pattern, perm, num_heads, d, dtype)
    acc = "f64" if dtype == "f64" else "f32"
    b = None if bias is None or np.asarray(bias).size == 0 else _as_dev(np.asarray(bias).reshape(-1), acc)
    wm = None if weight_mult is None else _as_dev(np.asarray(weight_mult).reshape(num_heads, E), acc)
    q = {s.worker_id: _as_dev(s.q_sub, dtype) for s in shards}
    k = {s.worker_id: _as_dev(s.k_sub, dtype) for s in shards}
    v = {s.worker_id: _as_dev(s.v_sub, dtype) for s in shards}
    out, macs = layer.forward(q, k, v, b, wm, ledger)
    layer.plan.ctx.sync()
    if _keep is not None:
        _keep.append((layer, b, wm))
    return DistAttnResult([out[w].double().cpu().numpy() for w in range(P)], macs)


def run_distributed_layer_backward(shards: list[WorkerShard], pattern, perm, num_heads: int, bias, weight_mult,
                                   upstream_shards: list, dtype: str = "f64") -> DistAttnGrads:
    """parallel.cpp:271-332 (the forward is re-run for its cached slices; the
    reference re-gathers Q/K/V the same way)."""
    keep = []
    run_distributed_layer(shards, pattern, perm, num_heads, bias, weight_mult, None, dtype, _keep=keep)
    layer, b, wm = keep[0]
    up = {s.worker_id: _as_dev(u, dtype) for s, u in zip(shards, upstream_shards)}
    dq, dk, dv, db = layer.backward(up, b, wm)
    layer.plan.ctx.sync()
    P = len(shards)
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    return DistAttnGrads([f(dq[w]) for w in range(P)], [f(dk[w]) for w in range(P)], [f(dv[w]) for w in range(P)],
                         f(db))


def _rows_of(pattern) -> int:
    for nm in ("rows", "num_nodes", "n"):
        if hasattr(pattern, nm):
            return int(getattr(pattern, nm))
    return int(np.asarray(pattern.row_offsets).shape[0] - 1)


def _nnz_of(pattern) -> int:
    cols = getattr(pattern, "cols", None)
    if cols is None:
        cols = pattern.col_indices
    return int(np.asarray(cols).shape[0])


def _layer(shards, pattern, perm, num_heads, d, dtype) -> UlyssesAttention:
    ro = np.asarray(pattern.row_offsets, dtype=np.int64)
    cols = getattr(pattern, "cols", None)
    if cols is None:
        cols = pattern.col_indices
    plan = DevicePlan.from_host(ro, np.asarray(cols, dtype=np.int64))
    sp = SequenceParallelPlan([s.token_ids for s in shards], None if perm is None else perm.forward, plan.ctx)
    layer = UlyssesAttention.on_device(plan, sp, num_heads, d, dtype, Loopback(sp))
    layer.plan = plan
    return layer
