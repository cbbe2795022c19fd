"""TEST INFRASTRUCTURE — ctypes front-end for the CPU checkers.

Two libraries are wrapped with the same Python surface:

* ``Oracle()``  -> ``oracle/liboracle.so``: the plain-C fp64 restatement of the
  reference hot path (oracle/*.c, each function cites reference file:line).
* ``RefOracle()`` -> ``oracle/_ref/libgteref_capi.so``: the compiled reference
  itself (built from /root/reference by ``make -C oracle ref``); present only
  where it was built. Used to generate/pin golden fixtures.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may
import this module, and only as the checker — never as the measured path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ConfigError(OracleError):
    pass


class DataError(OracleError):
    pass


def _raise(code: int, msg: str):
    if code == 2:
        raise ConfigError(code, msg)
    if code == 3:
        raise DataError(code, msg)
    raise OracleError(code, msg)


class _CCsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("row_off", I64P), ("cols", I64P)]


@dataclass
class CSR:
    n: int
    row_off: np.ndarray  # int64 [n+1]
    cols: np.ndarray  # int64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.cols.shape[0])

    def to_c(self) -> _CCsr:
        ro = np.ascontiguousarray(self.row_off, dtype=np.int64)
        co = np.ascontiguousarray(self.cols, dtype=np.int64)
        c = _CCsr(self.n, co.shape[0], ro.ctypes.data_as(I64P), co.ctypes.data_as(I64P))
        c._keep = (ro, co)  # type: ignore[attr-defined]
        return c


def _ptr(a, t=F64P):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class _Base:
    lib: C.CDLL
    prefix: str

    def _err(self) -> str:
        f = getattr(self.lib, self.prefix + "last_error")
        f.restype = C.c_char_p
        return f().decode()

    def _call(self, name, *args):
        rc = getattr(self.lib, self.prefix + name)(*args)
        if rc:
            _raise(rc, self._err())

    def _take_csr(self, c: _CCsr) -> CSR:
        n, nnz = c.n, c.nnz
        ro = np.ctypeslib.as_array(c.row_off, shape=(n + 1,)).copy()
        co = np.ctypeslib.as_array(c.cols, shape=(max(nnz, 1),))[:nnz].copy()
        self._free_csr(c)
        return CSR(n, ro, co)


class Oracle(_Base):
    """The C restatement (oracle/liboracle.so)."""

    prefix = "orc_"

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.lib.orc_cluster_of.restype = C.c_int64

    def _free_csr(self, c):
        self.lib.orc_csr_free(C.byref(c))

    # ---- graph ----
    def graph_from_edges(self, n, src, dst) -> CSR:
        s, d = _i64(src), _i64(dst)
        out = _CCsr()
        self._call("graph_from_edges", C.c_int64(n), C.c_int64(s.shape[0]), _ptr(s, I64P), _ptr(d, I64P), C.byref(out))
        return self._take_csr(out)

    def add_self_loops(self, g: CSR) -> CSR:
        out = _CCsr()
        gc = g.to_c()
        self._call("add_self_loops", C.byref(gc), C.byref(out))
        return self._take_csr(out)

    def density(self, g: CSR) -> float:
        out = C.c_double()
        gc = g.to_c()
        self._call("density", C.byref(gc), C.byref(out))
        return out.value

    # ---- attention (one head) ----
    def sparse_fwd(self, q, k, v, pat: CSR, bias=None, wmult=None, forbid_empty=False):
        q, k, v, bias, wmult = map(_f64, (q, k, v, bias, wmult))
        S, dk = q.shape
        dv = v.shape[1]
        out = np.zeros((S, dv))
        self._call("sparse_attn_fwd", C.c_int64(S), C.c_int64(dk), C.c_int64(dv), _ptr(q), _ptr(k), _ptr(v),
                   _ptr(_i64(pat.row_off), I64P), _ptr(_i64(pat.cols), I64P), _ptr(bias), _ptr(wmult),
                   C.c_int(int(forbid_empty)), _ptr(out))
        return out

    def sparse_bwd(self, q, k, v, pat: CSR, bias, wmult, up):
        q, k, v, bias, wmult, up = map(_f64, (q, k, v, bias, wmult, up))
        S, dk = q.shape
        dv = v.shape[1]
        dq, dkk, dvv = np.zeros((S, dk)), np.zeros((S, dk)), np.zeros((S, dv))
        db = np.zeros(max(pat.nnz, 1))
        self._call("sparse_attn_bwd", C.c_int64(S), C.c_int64(dk), C.c_int64(dv), _ptr(q), _ptr(k), _ptr(v),
                   _ptr(_i64(pat.row_off), I64P), _ptr(_i64(pat.cols), I64P), _ptr(bias), _ptr(wmult), _ptr(up),
                   _ptr(dq), _ptr(dkk), _ptr(dvv), _ptr(db))
        return dq, dkk, dvv, db[: pat.nnz]

    def dense_fwd(self, q, k, v, bias=None, wmult=None):
        q, k, v, bias, wmult = map(_f64, (q, k, v, bias, wmult))
        S, dk = q.shape
        out = np.zeros((S, v.shape[1]))
        self._call("dense_attn_fwd", C.c_int64(S), C.c_int64(dk), C.c_int64(v.shape[1]), _ptr(q), _ptr(k), _ptr(v),
                   _ptr(bias), _ptr(wmult), _ptr(out))
        return out

    def dense_bwd(self, q, k, v, bias, wmult, up):
        q, k, v, bias, wmult, up = map(_f64, (q, k, v, bias, wmult, up))
        S, dk = q.shape
        dv = v.shape[1]
        dq, dkk, dvv, db = np.zeros((S, dk)), np.zeros((S, dk)), np.zeros((S, dv)), np.zeros((S, S))
        self._call("dense_attn_bwd", C.c_int64(S), C.c_int64(dk), C.c_int64(dv), _ptr(q), _ptr(k), _ptr(v),
                   _ptr(bias), _ptr(wmult), _ptr(up), _ptr(dq), _ptr(dkk), _ptr(dvv), _ptr(db))
        return dq, dkk, dvv, db

    # ---- partition ----
    def cluster_boundaries(self, n, k):
        b = np.zeros(k + 1, dtype=np.int64)
        self.lib.orc_cluster_boundaries(C.c_int64(n), C.c_int64(k), _ptr(b, I64P))
        return b

    def reorder(self, g: CSR, k: int, seed: int):
        fwd = np.zeros(g.n, dtype=np.int64)
        inv = np.zeros(g.n, dtype=np.int64)
        gc = g.to_c()
        self._call("reorder", C.byref(gc), C.c_int64(k), C.c_uint64(seed), _ptr(fwd, I64P), _ptr(inv, I64P))
        return fwd, inv

    def permute_graph(self, g: CSR, fwd) -> CSR:
        out = _CCsr()
        gc = g.to_c()
        self._call("permute_graph", C.byref(gc), _ptr(_i64(fwd), I64P), C.byref(out))
        return self._take_csr(out)

    def build_cluster_grid(self, g: CSR, fwd, k):
        bnd = np.zeros(k + 1, dtype=np.int64)
        nnz = np.zeros(k * k, dtype=np.int64)
        den = np.zeros(k * k)
        gc = g.to_c()
        self._call("build_cluster_grid", C.byref(gc), _ptr(_i64(fwd), I64P), C.c_int64(k), _ptr(bnd, I64P),
                   _ptr(nnz, I64P), _ptr(den))
        return bnd, nnz, den

    def diagonal_edge_fraction(self, k, cell_nnz):
        out = C.c_double()
        self._call("diagonal_edge_fraction", C.c_int64(k), _ptr(_i64(cell_nnz), I64P), C.byref(out))
        return out.value

    # ---- reformation ----
    def pack_subblocks(self, er, ec, n_rows, n_cols, d_b):
        er, ec = _i64(er), _i64(ec)
        m = er.shape[0]
        cap = max(1, (m + d_b * d_b - 1) // (d_b * d_b)) if d_b >= 1 else 1
        tiles = np.zeros(2 * cap + 2, dtype=np.int64)
        nt = C.c_int64()
        self._call("pack_subblocks", C.c_int64(m), _ptr(er, I64P), _ptr(ec, I64P), C.c_int64(n_rows),
                   C.c_int64(n_cols), C.c_int64(d_b), _ptr(tiles, I64P), C.c_int64(cap), C.byref(nt))
        return tiles[: 2 * nt.value].reshape(-1, 2)

    def pack_subblocks_sparse(self, er, ec, n_rows, n_cols, d_b):
        """The same greedy over candidate origins (orc_pack_sparse.cpp)."""
        er, ec = _i64(er), _i64(ec)
        m = er.shape[0]
        cap = max(1, (m + d_b * d_b - 1) // (d_b * d_b)) if d_b >= 1 else 1
        tiles = np.zeros(2 * cap + 2, dtype=np.int64)
        nt = C.c_int64()
        self._call("pack_subblocks_sparse", C.c_int64(m), _ptr(er, I64P), _ptr(ec, I64P), C.c_int64(n_rows),
                   C.c_int64(n_cols), C.c_int64(d_b), _ptr(tiles, I64P), C.c_int64(cap), C.byref(nt))
        return tiles[: 2 * nt.value].reshape(-1, 2)

    def set_pack_mode(self, mode: int):
        """orc_build_layout's packer: 0 auto, 1 coverage field, 2 candidate origins."""
        self.lib.orc_set_pack_mode(C.c_int(mode))

    def build_layout(self, k, bnd, cell_nnz, cell_density, g_perm: CSR, strategy, beta_thre, beta_g, d_b):
        L = _OrcLayout()
        gc = g_perm.to_c()
        self._call("build_layout", C.c_int64(k), _ptr(_i64(bnd), I64P), _ptr(_i64(cell_nnz), I64P),
                   _ptr(_f64(cell_density)), C.byref(gc), C.c_int(strategy), C.c_double(beta_thre),
                   C.c_double(beta_g), C.c_int64(d_b), C.byref(L))
        kk = k * k
        state = np.ctypeslib.as_array(L.cell_state, shape=(kk,)).copy()
        boff = np.ctypeslib.as_array(L.block_off, shape=(kk + 1,)).copy()
        nb = int(boff[-1])
        blocks = np.ctypeslib.as_array(L.blocks, shape=(2 * nb + 2,))[: 2 * nb].copy().reshape(-1, 2)
        pat = CSR(L.pattern.n, np.ctypeslib.as_array(L.pattern.row_off, shape=(L.pattern.n + 1,)).copy(),
                  np.ctypeslib.as_array(L.pattern.cols, shape=(L.pattern.nnz + 1,))[: L.pattern.nnz].copy())
        dropped = L.dropped_edges
        self.lib.orc_layout_free(C.byref(L))
        return Layout(state, boff, blocks, dropped, pat)

    def tuner_run(self, beta_g, delta, losses, times):
        st = _OrcTuner()
        self._call("make_tuner", C.c_double(beta_g), C.c_int64(delta), C.byref(st))
        idx, avg = [], []
        for e, (l, t) in enumerate(zip(losses, times)):
            self._call("tuner_update", C.byref(st), C.c_double(l), C.c_double(t), C.c_int64(e))
            idx.append(st.idx)
            avg.append(st.avg_loss)
        thr = [st.thresholds[i] for i in range(st.n_thr)]
        self.lib.orc_tuner_free(C.byref(st))
        return np.array(idx), np.array(avg), np.array(thr)

    def select_k(self, l2, d, i):
        out = C.c_int64()
        self._call("select_k", C.c_int64(l2), C.c_int64(d), C.c_int64(i), C.byref(out))
        return out.value

    def select_db(self, db, thr):
        db, thr = _i64(db), _f64(thr)
        out = C.c_int64()
        self._call("select_db", C.c_int64(db.shape[0]), _ptr(db, I64P), _ptr(thr), C.byref(out))
        return out.value

    def pattern_buckets(self, pat: CSR, perm_inv, global_index, spd, max_dist):
        """model.cpp:447-463 bucket fill; spd = (row_off, cols, dist uint16, n)."""
        ro, co, dist, n = spd
        out = np.zeros(max(pat.nnz, 1), dtype=np.int32)
        pc = pat.to_c()
        d16 = np.ascontiguousarray(dist, dtype=np.uint16)
        self._call("pattern_buckets", C.byref(pc), _ptr(_i64(perm_inv), I64P), C.c_int64(global_index),
                   C.c_int64(n), _ptr(_i64(ro), I64P), _ptr(_i64(co), I64P),
                   d16.ctypes.data_as(C.POINTER(C.c_uint16)), C.c_int64(max_dist), _ptr(out, I32P))
        return out[: pat.nnz]

    def extend_with_pad_loops(self, pat: CSR, s_pad) -> CSR:
        out = _CCsr()
        pc = pat.to_c()
        self._call("extend_with_pad_loops", C.byref(pc), C.c_int64(s_pad), C.byref(out))
        return self._take_csr(out)

    def check_conditions(self, g: CSR, layers):
        r = _OrcCond()
        gc = g.to_c()
        self._call("check_conditions", C.byref(gc), C.c_int64(layers), C.byref(r))
        return dict(c1=bool(r.c1), c2=bool(r.c2), c3=bool(r.c3), layers=r.layers, sweep_from=r.sf,
                    sweep_to=r.st, diameter_lower_bound=r.dlb)

    # ---- parallel ----
    def partition_sequence(self, S, P, seed):
        pad = ((S + P - 1) // P) * P
        ids = np.zeros(max(pad, 1), dtype=np.int64)
        padded = C.c_int64()
        self._call("partition_sequence", C.c_int64(S), C.c_int64(P), C.c_uint64(seed), _ptr(ids, I64P),
                   C.byref(padded))
        return ids[:pad].reshape(P, -1)

    def dist_fwd(self, P, ids, q, k, v, pat: CSR, fwd, inv, H, bias=None, wmult=None):
        q, k, v, bias, wmult = map(_f64, (q, k, v, bias, wmult))
        S, d = q.shape
        out = np.zeros((S, d))
        ledger = np.zeros((P, 5), dtype=np.int64)
        macs = C.c_int64()
        self._call("dist_layer_fwd", C.c_int64(P), C.c_int64(S), C.c_int64(d), C.c_int64(H),
                   _ptr(_i64(ids), I64P), _ptr(q), _ptr(k), _ptr(v), _ptr(_i64(pat.row_off), I64P),
                   _ptr(_i64(pat.cols), I64P), _ptr(_i64(fwd), I64P), _ptr(_i64(inv), I64P), _ptr(bias),
                   C.c_int64(0 if bias is None else bias.shape[0]), _ptr(wmult), _ptr(out), _ptr(ledger, I64P),
                   C.byref(macs))
        return out, ledger, macs.value

    def dist_bwd(self, P, ids, q, k, v, pat: CSR, fwd, inv, H, bias, wmult, up):
        q, k, v, bias, wmult, up = map(_f64, (q, k, v, bias, wmult, up))
        S, d = q.shape
        dq, dk, dv = np.zeros((S, d)), np.zeros((S, d)), np.zeros((S, d))
        db = np.zeros(max(pat.nnz, 1))
        self._call("dist_layer_bwd", C.c_int64(P), C.c_int64(S), C.c_int64(d), C.c_int64(H),
                   _ptr(_i64(ids), I64P), _ptr(q), _ptr(k), _ptr(v), _ptr(_i64(pat.row_off), I64P),
                   _ptr(_i64(pat.cols), I64P), _ptr(_i64(fwd), I64P), _ptr(_i64(inv), I64P), _ptr(bias),
                   _ptr(wmult), _ptr(up), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(db))
        return dq, dk, dv, db[: pat.nnz]


class _OrcLayout(C.Structure):
    _fields_ = [("seq_len", C.c_int64), ("k", C.c_int64), ("d_b", C.c_int64), ("boundaries", I64P),
                ("cell_state", I32P), ("block_off", I64P), ("blocks", I64P), ("dropped_edges", C.c_int64),
                ("pattern", _CCsr)]


class _OrcTuner(C.Structure):
    _fields_ = [("avg_loss", C.c_double), ("ldr_epoch", I64P), ("ldr_val", F64P), ("n_ldr", C.c_int64),
                ("cap_ldr", C.c_int64), ("thresholds", C.c_double * 7), ("n_thr", C.c_int64), ("idx", C.c_int64),
                ("delta", C.c_int64), ("has_loss", C.c_int)]


class _OrcCond(C.Structure):
    _fields_ = [("c1", C.c_int32), ("c2", C.c_int32), ("c3", C.c_int32), ("layers", C.c_int64), ("sf", C.c_int64),
                ("st", C.c_int64), ("dlb", C.c_int64)]


@dataclass
class Layout:
    cell_state: np.ndarray
    block_off: np.ndarray
    blocks: np.ndarray
    dropped_edges: int
    pattern: CSR


class RefOracle(_Base):
    """The compiled reference (oracle/_ref/libgteref_capi.so)."""

    prefix = "refc_"

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libgteref_capi.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)

    def _free_csr(self, c):
        self.lib.refc_free(c.row_off)
        self.lib.refc_free(c.cols)

    def graph_from_edges(self, n, src, dst) -> CSR:
        s, d = _i64(src), _i64(dst)
        out = _CCsr()
        self._call("graph_from_edges", C.c_int64(n), C.c_int64(s.shape[0]), _ptr(s, I64P), _ptr(d, I64P), C.byref(out))
        return self._take_csr(out)

    def add_self_loops(self, g: CSR) -> CSR:
        out = _CCsr()
        gc = g.to_c()
        self._call("add_self_loops", C.byref(gc), C.byref(out))
        return self._take_csr(out)

    def reorder(self, g: CSR, k, seed):
        fwd = np.zeros(g.n, dtype=np.int64)
        inv = np.zeros(g.n, dtype=np.int64)
        gc = g.to_c()
        self._call("reorder", C.byref(gc), C.c_int64(k), C.c_uint64(seed), _ptr(fwd, I64P), _ptr(inv, I64P))
        return fwd, inv

    def permute_graph(self, g: CSR, fwd, inv) -> CSR:
        out = _CCsr()
        gc = g.to_c()
        self._call("permute_graph", C.byref(gc), _ptr(_i64(fwd), I64P), _ptr(_i64(inv), I64P), C.byref(out))
        return self._take_csr(out)

    def build_cluster_grid(self, g: CSR, fwd, inv, k):
        bnd = np.zeros(k + 1, dtype=np.int64)
        nnz = np.zeros(k * k, dtype=np.int64)
        den = np.zeros(k * k)
        gc = g.to_c()
        self._call("build_cluster_grid", C.byref(gc), _ptr(_i64(fwd), I64P), _ptr(_i64(inv), I64P), C.c_int64(k),
                   _ptr(bnd, I64P), _ptr(nnz, I64P), _ptr(den))
        return bnd, nnz, den

    def pack_subblocks(self, er, ec, n_rows, n_cols, d_b):
        er, ec = _i64(er), _i64(ec)
        tiles = I64P()
        nt = C.c_int64()
        self._call("pack_subblocks", C.c_int64(er.shape[0]), _ptr(er, I64P), _ptr(ec, I64P), C.c_int64(n_rows),
                   C.c_int64(n_cols), C.c_int64(d_b), C.byref(tiles), C.byref(nt))
        arr = np.ctypeslib.as_array(tiles, shape=(2 * nt.value + 2,))[: 2 * nt.value].copy().reshape(-1, 2)
        self.lib.refc_free(tiles)
        return arr

    def build_layout(self, g_orig: CSR, fwd, inv, k, strategy, thre, bg, d_b):
        state = np.zeros(k * k, dtype=np.int32)
        boff = np.zeros(k * k + 1, dtype=np.int64)
        blocks = I64P()
        dropped = C.c_int64()
        pat = _CCsr()
        gc = g_orig.to_c()
        self._call("build_layout", C.byref(gc), _ptr(_i64(fwd), I64P), _ptr(_i64(inv), I64P), C.c_int64(k),
                   C.c_int(strategy), C.c_double(thre), C.c_double(bg), C.c_int64(d_b), _ptr(state, I32P),
                   _ptr(boff, I64P), C.byref(blocks), C.byref(dropped), C.byref(pat))
        nb = int(boff[-1])
        bl = np.ctypeslib.as_array(blocks, shape=(2 * nb + 1,))[: 2 * nb].copy().reshape(-1, 2)
        self.lib.refc_free(blocks)
        return Layout(state, boff, bl, dropped.value, self._take_csr(pat))

    def sparse_fwd(self, q, k, v, pat: CSR, bias=None, wmult=None, forbid_empty=False):
        q, k, v, bias, wmult = map(_f64, (q, k, v, bias, wmult))
        S, dk = q.shape
        out = np.zeros((S, v.shape[1]))
        macs = np.zeros(2, dtype=np.int64)
        pc = pat.to_c()
        self._call("sparse_fwd", C.c_int64(S), C.c_int64(dk), C.c_int64(v.shape[1]), _ptr(q), _ptr(k), _ptr(v),
                   C.byref(pc), _ptr(bias), _ptr(wmult), C.c_int(int(forbid_empty)), _ptr(out), _ptr(macs, I64P))
        return out

    def sparse_bwd(self, q, k, v, pat: CSR, bias, wmult, up):
        q, k, v, bias, wmult, up = map(_f64, (q, k, v, bias, wmult, up))
        S, dk = q.shape
        dv = v.shape[1]
        dq, dkk, dvv = np.zeros((S, dk)), np.zeros((S, dk)), np.zeros((S, dv))
        db = np.zeros(max(pat.nnz, 1))
        pc = pat.to_c()
        self._call("sparse_bwd", C.c_int64(S), C.c_int64(dk), C.c_int64(dv), _ptr(q), _ptr(k), _ptr(v), C.byref(pc),
                   _ptr(bias), _ptr(wmult), _ptr(up), _ptr(dq), _ptr(dkk), _ptr(dvv), _ptr(db))
        return dq, dkk, dvv, db[: pat.nnz]

    def dense_fwd(self, q, k, v, bias=None, wmult=None):
        q, k, v, bias, wmult = map(_f64, (q, k, v, bias, wmult))
        S, dk = q.shape
        out = np.zeros((S, v.shape[1]))
        self._call("dense_fwd", C.c_int64(S), C.c_int64(dk), C.c_int64(v.shape[1]), _ptr(q), _ptr(k), _ptr(v),
                   _ptr(bias), _ptr(wmult), _ptr(out))
        return out

    def dense_bwd(self, q, k, v, bias, wmult, up):
        q, k, v, bias, wmult, up = map(_f64, (q, k, v, bias, wmult, up))
        S, dk = q.shape
        dv = v.shape[1]
        dq, dkk, dvv, db = np.zeros((S, dk)), np.zeros((S, dk)), np.zeros((S, dv)), np.zeros((S, S))
        self._call("dense_bwd", C.c_int64(S), C.c_int64(dk), C.c_int64(dv), _ptr(q), _ptr(k), _ptr(v), _ptr(bias),
                   _ptr(wmult), _ptr(up), _ptr(dq), _ptr(dkk), _ptr(dvv), _ptr(db))
        return dq, dkk, dvv, db

    def partition_sequence(self, S, P, seed):
        pad = ((S + P - 1) // P) * P
        ids = np.zeros(pad, dtype=np.int64)
        self._call("partition_sequence", C.c_int64(S), C.c_int64(P), C.c_uint64(seed), _ptr(ids, I64P))
        return ids.reshape(P, -1)

    def dist_fwd(self, P, ids, q, k, v, pat: CSR, fwd, inv, H, bias=None, wmult=None):
        q, k, v, bias, wmult = map(_f64, (q, k, v, bias, wmult))
        S, d = q.shape
        out = np.zeros((S, d))
        ledger = np.zeros((P, 5), dtype=np.int64)
        macs = C.c_int64()
        pc = pat.to_c()
        self._call("dist_fwd", C.c_int64(P), C.c_int64(S), C.c_int64(d), C.c_int64(H), _ptr(_i64(ids), I64P),
                   _ptr(q), _ptr(k), _ptr(v), C.byref(pc), _ptr(_i64(fwd), I64P), _ptr(_i64(inv), I64P), _ptr(bias),
                   _ptr(wmult), _ptr(out), _ptr(ledger, I64P), C.byref(macs))
        return out, ledger, macs.value

    def dist_bwd(self, P, ids, q, k, v, pat: CSR, fwd, inv, H, bias, wmult, up):
        q, k, v, bias, wmult, up = map(_f64, (q, k, v, bias, wmult, up))
        S, d = q.shape
        dq, dk, dv = np.zeros((S, d)), np.zeros((S, d)), np.zeros((S, d))
        db = np.zeros(max(pat.nnz, 1))
        pc = pat.to_c()
        self._call("dist_bwd", C.c_int64(P), C.c_int64(S), C.c_int64(d), C.c_int64(H), _ptr(_i64(ids), I64P),
                   _ptr(q), _ptr(k), _ptr(v), C.byref(pc), _ptr(_i64(fwd), I64P), _ptr(_i64(inv), I64P), _ptr(bias),
                   _ptr(wmult), _ptr(up), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(db))
        return dq, dk, dv, db[: pat.nnz]

    def check_conditions(self, g: CSR, layers):
        flags = np.zeros(3, dtype=np.int32)
        ints = np.zeros(4, dtype=np.int64)
        gc = g.to_c()
        self._call("check_conditions", C.byref(gc), C.c_int64(layers), _ptr(flags, I32P), _ptr(ints, I64P))
        return dict(c1=bool(flags[0]), c2=bool(flags[1]), c3=bool(flags[2]), layers=int(ints[0]),
                    sweep_from=int(ints[1]), sweep_to=int(ints[2]), diameter_lower_bound=int(ints[3]))

    def spd_table(self, g: CSR, max_dist):
        """The compiled reference's gte::spd_table (graph.cpp:216-262)."""
        ro, co, di = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.POINTER(C.c_uint16)()
        nnz = C.c_int64()
        gc = g.to_c()
        self._call("spd_table", C.byref(gc), C.c_int64(max_dist), C.byref(ro), C.byref(co), C.byref(di), C.byref(nnz))
        n, m = g.n, nnz.value
        out = (np.ctypeslib.as_array(ro, (n + 1,)).copy(), np.ctypeslib.as_array(co, (max(m, 1),))[:m].copy(),
               np.ctypeslib.as_array(di, (max(m, 1),))[:m].copy(), n)
        for p_ in (ro, co, di):
            self.lib.refc_free(C.cast(p_, C.c_void_p))
        return out

    def generate_sbm(self, n, blocks, pin, pout, seed, noise=0.0):
        out = _CCsr()
        labels = np.zeros(n, dtype=np.int32)
        self._call("generate_sbm", C.c_int64(n), C.c_int64(blocks), C.c_double(pin), C.c_double(pout),
                   C.c_uint64(seed), C.c_double(noise), C.byref(out), _ptr(labels, I32P))
        return self._take_csr(out), labels

    def random_graph(self, n, p, seed, loops=True) -> CSR:
        out = _CCsr()
        self._call("random_graph", C.c_int64(n), C.c_double(p), C.c_uint64(seed), C.c_int(int(loops)), C.byref(out))
        return self._take_csr(out)

    def tuner_run(self, beta_g, delta, losses, times):
        losses, times = _f64(losses), _f64(times)
        n = losses.shape[0]
        idx = np.zeros(n, dtype=np.int64)
        avg = np.zeros(n)
        thr = np.zeros(7)
        nthr = C.c_int64()
        self._call("tuner_run", C.c_double(beta_g), C.c_int64(delta), C.c_int64(n), _ptr(losses), _ptr(times),
                   _ptr(idx, I64P), _ptr(avg), _ptr(thr), C.byref(nthr))
        return idx, avg, thr[: nthr.value]

    def select_k(self, l2, d, i):
        out = C.c_int64()
        self._call("select_k", C.c_int64(l2), C.c_int64(d), C.c_int64(i), C.byref(out))
        return out.value

    def select_db(self, db, thr):
        db, thr = _i64(db), _f64(thr)
        out = C.c_int64()
        self._call("select_db", C.c_int64(db.shape[0]), _ptr(db, I64P), _ptr(thr), C.byref(out))
        return out.value


def fnv1a64(arr: np.ndarray) -> str:
    """FNV-1a-64 over the raw little-endian bytes (SURVEY.md §8(c6) checksum)."""
    h = 1469598103934665603
    for b in np.ascontiguousarray(arr).tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def fnv1a64_fast(arr: np.ndarray) -> str:
    """Vectorised-enough FNV-1a-64 (same result as fnv1a64) for multi-MB arrays."""
    data = np.frombuffer(np.ascontiguousarray(arr).tobytes(), dtype=np.uint8)
    h = 1469598103934665603
    prime = 1099511628211
    mask = 0xFFFFFFFFFFFFFFFF
    for b in data.tolist():
        h = ((h ^ b) * prime) & mask
    return f"{h:016x}"
