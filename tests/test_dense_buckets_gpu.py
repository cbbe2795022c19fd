"""Dense epochs with the SPD bucket bias (reference Trainer
model.cpp:395-423 dense_pattern_exec + dense_buckets, :520-523 bias gather):
bias[r][c] = table[bucket[r][c]] over the uint8 bucket matrix built on the GPU
(glue.dense_buckets), the table's gradient reduced per bucket — never an S x S
float bias or dbias.

Pinned by: the bucket matrix == the Trainer rule over the product spd_table
(itself == the compiled reference's, tests/test_spd_gpu.py); attention ==
the fp64 oracle over the explicit execution pattern with the gathered biases;
dtable == the oracle's per-pair dbias summed per bucket. Sizes: a graph task
with a global token and pad rows (S = 304), C1 (S = 4096, all rows) and a
community graph at S = 32,768 (sampled rows, forward)."""
import numpy as np
import pytest

from oracle import CSR

from paper_2407_14106_b200 import attention as A
from paper_2407_14106_b200 import glue
from paper_2407_14106_b200 import partition as P
from paper_2407_14106_b200.datagen import c1_edges, community_graph

pytestmark = pytest.mark.gpu
TOL = {"f64": (1e-12, 1e-12), "f32": (1e-5, 1e-5), "bf16": (2e-2, 1e-2)}


def close(got, want, dtype, what):
    scale = max(np.abs(want).max(), 1e-300)
    e_max = np.abs(got - want).max() / scale
    e_nrm = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
    assert e_max <= TOL[dtype][0] and e_nrm <= TOL[dtype][1], f"{what} [{dtype}] {e_max:.3g} {e_nrm:.3g}"


def trainer_case(n, src, dst, with_global, s_pad_extra, k=4, cap=8):
    """Graph task (model.cpp:349-365): attention graph = graph + global token,
    self loops; reorder; s_pad = s_real + s_pad_extra. Returns the pieces."""
    g0 = P.graph_from_edges(n, src, dst)
    glob = n if with_global else -1
    if with_global:
        s2 = np.r_[src, np.arange(n), np.full(n, n)]
        d2 = np.r_[dst, np.full(n, n), np.arange(n)]
        attn = P.add_self_loops(P.graph_from_edges(n + 1, s2, d2))
    else:
        attn = P.add_self_loops(g0)
    s_real = attn.num_nodes
    perm = P.reorder(attn, k, 1)
    S = s_real + s_pad_extra
    inv = np.r_[np.asarray(perm.inverse, np.int64), np.arange(s_real, S)]
    fwd = np.asarray(perm.forward, np.int64)
    return g0, glob, s_real, S, fwd, inv, cap


def host_buckets(g0, glob, s_real, inv, cap):
    ro, co = np.asarray(g0.row_offsets), np.asarray(g0.col_indices)
    sro, scol, sdist, sn = glue.spd_table(ro, co, cap)
    full = np.full((s_real, s_real), cap + 1, np.int32)
    for r in range(s_real):
        i = inv[r]
        for c in range(s_real):
            j = inv[c]
            if i == j:
                full[r, c] = 0
            elif i == glob or j == glob:
                full[r, c] = 1
            elif i < sn and j < sn:
                row = scol[sro[i]:sro[i + 1]]
                p = np.searchsorted(row, j)
                if p < row.shape[0] and row[p] == j:
                    full[r, c] = sdist[sro[i] + p]
    return full


def planted(seed, n=300):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, 700)
    dst = (src // 30) * 30 + rng.integers(0, 30, 700)
    dst[:40] = rng.integers(0, n, 40)
    return n, src, dst


@pytest.mark.parametrize("with_global,cap", [(True, 8), (False, 3)])
def test_bucket_matrix_is_the_trainer_rule(cuda, with_global, cap):
    n, src, dst = planted(12)
    g0, glob, s_real, S, fwd, inv, cap = trainer_case(n, src, dst, with_global, 3, cap=cap)
    b = glue.dense_buckets(S, s_real, fwd, inv, glob, g0.row_offsets, g0.col_indices, cap).cpu().numpy()
    want = host_buckets(g0, glob, s_real, inv, cap)
    assert np.array_equal(b[:s_real, :s_real].astype(np.int32), want)


def run_dense(S, s_real, H, dh, dtype, buckets, table, seed):
    import torch

    td = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    acc = torch.float64 if dtype == "f64" else torch.float32
    rng = np.random.default_rng(seed)
    q, k, v, up = (torch.tensor(rng.standard_normal((S, H * dh)), dtype=td, device="cuda") for _ in range(4))
    tb = torch.tensor(table, dtype=acc, device="cuda")
    att = A.DeviceDenseAttention(S, H, dh, dh, dtype, s_real=s_real)
    out, lse = att.forward_buckets(q, k, v, buckets, tb)
    dq, dk, dv, dt = att.backward_buckets(q, k, v, out, lse, up, buckets, tb)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    return dict(q=f(q), k=f(k), v=f(v), up=f(up), out=f(out), dq=f(dq), dk=f(dk), dv=f(dv), dt=f(dt))


def oracle_dense(orc, S, s_real, H, dh, r, bfull, table):
    ro, co = [0], []
    for i in range(S):
        co.extend(range(s_real) if i < s_real else [i])
        ro.append(len(co))
    g = CSR(S, np.array(ro, np.int64), np.array(co, np.int64))
    rows = np.repeat(np.arange(S), np.diff(g.row_off))
    bk = np.zeros(g.nnz, np.int64)
    real = rows < s_real
    bk[real] = bfull[rows[real], g.cols[real]]
    b_e = np.asarray(table)[bk]
    want = {x: np.zeros((S, H * dh)) for x in ("out", "dq", "dk", "dv")}
    db = np.zeros(g.nnz)
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        want["out"][:, sl] = orc.sparse_fwd(r["q"][:, sl], r["k"][:, sl], r["v"][:, sl], g, b_e)
        a, b, c, e = orc.sparse_bwd(r["q"][:, sl], r["k"][:, sl], r["v"][:, sl], g, b_e, None, r["up"][:, sl])
        want["dq"][:, sl], want["dk"][:, sl], want["dv"][:, sl] = a, b, c
        db += e
    want["dt"] = np.bincount(bk[real], weights=db[real], minlength=len(table))
    return want


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_dense_bucket_bias_global_token_and_pads(cuda, orc, dtype):
    import torch

    n, src, dst = planted(12)
    g0, glob, s_real, S, fwd, inv, cap = trainer_case(n, src, dst, True, 3)
    bm = glue.dense_buckets(S, s_real, fwd, inv, glob, g0.row_offsets, g0.col_indices, cap)
    table = np.random.default_rng(1).normal(0, 0.3, cap + 2)
    r = run_dense(S, s_real, 4, 8, dtype, bm, table, seed=3)
    bfull = bm.cpu().numpy().astype(np.int64)
    want = oracle_dense(orc, S, s_real, 4, 8, r, bfull, table)
    for x in ("out", "dq", "dk", "dv", "dt"):
        close(r[x], want[x], dtype, x)
    if dtype != "bf16":  # deterministic table gradient
        r2 = run_dense(S, s_real, 4, 8, dtype, bm, table, seed=3)
        assert np.array_equal(r["dt"], r2["dt"])
    assert torch.cuda.is_available()


def test_dense_bucket_bias_c1_full(cuda, orc):
    """C1 (BASELINE configs[0]: N = 4096, E = 69,497), node task, cap 8, two
    heads of GPH-slim (dh = 8), f32, every row against the oracle."""
    s, t = c1_edges()
    g0 = P.graph_from_edges(4096, s, t)
    attn = P.add_self_loops(g0)
    perm = P.reorder(attn, 8, 1)
    fwd, inv = np.asarray(perm.forward, np.int64), np.asarray(perm.inverse, np.int64)
    bm = glue.dense_buckets(4096, 4096, fwd, inv, -1, g0.row_offsets, g0.col_indices, 8)
    b = bm.cpu().numpy()
    assert b.max() <= 9 and (np.diag(b) == 0).all()
    table = np.random.default_rng(2).normal(0, 0.3, 10)
    r = run_dense(4096, 4096, 2, 8, "f32", bm, table, seed=4)
    want = oracle_dense(orc, 4096, 4096, 2, 8, r, b.astype(np.int64), table)
    for x in ("out", "dq", "dk", "dv", "dt"):
        close(r[x], want[x], "f32", f"C1 {x}")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dense_bucket_bias_32k_sampled_rows(cuda, dtype):
    """S = 32,768 community graph (products density), all 8 heads: 16 sampled
    rows of the output against a numpy fp64 softmax over all real columns with
    the gathered bucket biases; those rows' buckets against a host BFS."""
    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg
    import torch

    n = 32768
    ro, co = community_graph(n, 61859140 / 2449029, community=256, seed=5, shuffle=True)
    g0 = A.Graph(n, np.asarray(ro, np.int64), np.asarray(co, np.int64))
    attn = P.add_self_loops(g0)
    perm = P.reorder(attn, 8, 1)
    fwd, inv = np.asarray(perm.forward, np.int64), np.asarray(perm.inverse, np.int64)
    bm = glue.dense_buckets(n, n, fwd, inv, -1, ro, co, 8)
    rows = np.random.default_rng(0).choice(n, 16, replace=False)
    b = bm[torch.tensor(rows, device="cuda")].cpu().numpy().astype(np.int64)
    Adj = sp.csr_matrix((np.ones(co.shape[0]), co, ro), shape=(n, n))
    Adj = ((Adj + Adj.T) > 0).astype(np.int8)
    D = cg.shortest_path(Adj, unweighted=True, indices=inv[rows])
    for k_, r in enumerate(rows):
        d = D[k_][inv]
        want = np.where(np.isfinite(d) & (d <= 8), d, 9).astype(np.int64)
        assert np.array_equal(b[k_], want), r
    H, dh = 8, 8
    table = np.random.default_rng(3).normal(0, 0.3, 10)
    td = torch.float32 if dtype == "f32" else torch.bfloat16
    rng = np.random.default_rng(6)
    q, k, v = (torch.tensor(rng.standard_normal((n, H * dh)), dtype=td, device="cuda") for _ in range(3))
    att = A.DeviceDenseAttention(n, H, dh, dh, dtype)
    out, _ = att.forward_buckets(q, k, v, bm, torch.tensor(table, dtype=torch.float32, device="cuda"))
    torch.cuda.synchronize()
    qn, kn, vn, on = (x.double().cpu().numpy() for x in (q, k, v, out))
    for k_, r in enumerate(rows):
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            s = kn[:, sl] @ qn[r, sl] / np.sqrt(dh) + table[b[k_]]
            p = np.exp(s - s.max())
            w = p / p.sum()
            want = w @ vn[:, sl]
            # a 32K-term weighted sum cancels to ~1/sqrt(S) of its terms: bound
            # the error by the sum's condition scale sum_j w_j |v_j|
            cond = (w @ np.abs(vn[:, sl])).max()
            tol = 1e-5 if dtype == "f32" else 2e-2
            assert np.abs(on[r, sl] - want).max() <= tol * cond, (r, h)
