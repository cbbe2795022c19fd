"""Parity of the sm_100a sparse graph-attention kernels (through the C ABI)
against the CPU oracle (oracle/liboracle.so, itself pinned to the compiled
reference by tests/test_oracle_golden.py).

Tolerances (BASELINE.md "Parity definition"), per tensor:
  f64: max|a-b| <= 1e-12*max|ref|
  f32: max|a-b| <= 1e-5*max|ref|  and  ||a-b||/||ref|| <= 1e-5
  bf16 (inputs rounded to bf16, fp32 accumulate, bf16 outputs):
       max|a-b| <= 2e-2*max|ref|  and  ||a-b||/||ref|| <= 1e-2
The oracle always runs in fp64 on the *same* (dtype-rounded) inputs.
"""
import numpy as np
import pytest

from conftest import rel_err
from oracle import CSR

from paper_2407_14106_b200 import attention as A
from paper_2407_14106_b200._lib import ConfigError, DataError
from paper_2407_14106_b200.datagen import arxiv_c2, c1_edges, malnet_c4, papers_c5, community_graph, csr_from_pairs

pytestmark = pytest.mark.gpu

TOL = {"f64": (1e-12, 1e-12), "f32": (1e-5, 1e-5), "bf16": (2e-2, 1e-2)}


def assert_close(got, want, dtype, what=""):
    e_max, e_nrm = rel_err(got, want)
    tmax, tnrm = TOL[dtype]
    assert e_max <= tmax and e_nrm <= tnrm, f"{what} [{dtype}] max-norm {e_max:.3g} l2 {e_nrm:.3g}"


def pat_of(g: CSR) -> A.AttnPattern:
    return A.AttnPattern(g.n, g.row_off, g.cols)


# ---------------------------------------------------------------- golden, reference-shaped API

@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_golden_cases_per_head(cuda, golden, orc, dtype):
    d = golden("attention_small.npz")
    for ci in range(int(d["ncases"])):
        p = f"a{ci}_"
        g = CSR(int(d[p + "g_n"]), d[p + "g_ro"], d[p + "g_cols"])
        bias = d[p + "bias"] if p + "bias" in d else None
        wm = d[p + "wm"] if p + "wm" in d else None
        q, k, v, up = (d[p + n] for n in ("q", "k", "v", "up"))
        if dtype == "f32":  # oracle on the fp32-rounded inputs
            q, k, v, up = (x.astype(np.float32).astype(np.float64) for x in (q, k, v, up))
            bias = None if bias is None else bias.astype(np.float32).astype(np.float64)
            want = orc.sparse_fwd(q, k, v, g, bias, wm)
            wq, wk, wv, wb = orc.sparse_bwd(q, k, v, g, bias, wm, up)
        else:
            want = d[p + "out"]
            wq, wk, wv, wb = (d[p + n] for n in ("dq", "dk", "dv", "db"))
        res = A.sparse_attention(q, k, v, pat_of(g), bias, wm, dtype=dtype)
        assert_close(res.output, want, dtype, f"case {ci} out")
        assert res.macs.score_macs == g.nnz * q.shape[1]
        gr = A.sparse_attention_backward(q, k, v, pat_of(g), bias, wm, up, dtype=dtype)
        for got, w, nm in ((gr.dq, wq, "dq"), (gr.dk, wk, "dk"), (gr.dv, wv, "dv"), (gr.dbias, wb, "dbias")):
            assert_close(got, w, dtype, f"case {ci} {nm}")


# ---------------------------------------------------------------- multi-head device path

def _torch_dtype(dtype):
    import torch

    return {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]


def run_device(row_off, cols, H, dh, dtype, seed=0, with_bias=True, with_wm=False, S=None, order=None, blocks=None):
    """Runs fwd+bwd through DeviceSparseAttention; returns the dtype-rounded fp64
    inputs and the outputs, as numpy fp64."""
    import torch

    S = row_off.shape[0] - 1
    E = cols.shape[0]
    rng = np.random.default_rng(seed)
    td = _torch_dtype(dtype)
    acc = torch.float64 if dtype == "f64" else torch.float32
    dev = torch.device("cuda:0")
    q, k, v, do = (torch.tensor(rng.standard_normal((S, H * dh)), dtype=td, device=dev) for _ in range(4))
    bias = torch.tensor(rng.normal(0, 0.3, E), dtype=acc, device=dev) if with_bias else None
    wm = torch.tensor((rng.random((H, E)) < 0.7) / 0.7, dtype=acc, device=dev) if with_wm else None
    plan = A.DevicePlan.from_host(row_off, cols)
    if isinstance(order, str) and order == "schedule":
        plan.schedule()
    elif order is not None:
        plan.set_order(order)
    tiles = plan.set_blocks(blocks, 16) if blocks is not None else 0
    att = A.DeviceSparseAttention(plan, H, dh, dh, dtype)
    out, lse = att.forward(q, k, v, bias, wm)
    dq, dk, dv, db = att.backward(q, k, v, out, lse, do, bias, wm)
    plan.ctx.sync()
    f = lambda t: None if t is None else t.double().cpu().numpy()  # noqa: E731
    return dict(q=f(q), k=f(k), v=f(v), do=f(do), bias=f(bias), wm=f(wm), out=f(out), dq=f(dq), dk=f(dk), dv=f(dv),
                db=f(db)[:E], lse=f(lse), tiles=tiles)


def oracle_multihead(orc, g: CSR, r, H, dh):
    S = g.n
    out = np.zeros((S, H * dh))
    dq, dk, dv = np.zeros_like(out), np.zeros_like(out), np.zeros_like(out)
    db = np.zeros(g.nnz)
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        wm = None if r["wm"] is None else r["wm"][h]
        out[:, sl] = orc.sparse_fwd(r["q"][:, sl], r["k"][:, sl], r["v"][:, sl], g, r["bias"], wm)
        a, b, c, e = orc.sparse_bwd(r["q"][:, sl], r["k"][:, sl], r["v"][:, sl], g, r["bias"], wm, r["do"][:, sl])
        dq[:, sl], dk[:, sl], dv[:, sl] = a, b, c
        db += e  # head order 0..H-1 as parallel.cpp:319
    return out, dq, dk, dv, db


def check_sampled_rows(r, ro, co, rows, H, dh, dtype, what):
    """All heads of sampled rows against a float64 numpy restatement of
    attention.cpp:96-162 / 241-320: the output row, the dQ row and the
    head-summed dbias of the row's edges (parallel.cpp:319). `r`: fp64 numpy
    q, k, v, do, bias (the dtype-rounded device inputs) and out, dq, db."""
    scale = 1.0 / np.sqrt(dh)
    got_o, want_o, got_q, want_q, got_b, want_b = [], [], [], [], [], []
    for i in rows:
        e0, e1 = int(ro[i]), int(ro[i + 1])
        if e1 == e0:
            continue
        cols = co[e0:e1]
        b = r["bias"][e0:e1]
        dbs = np.zeros(e1 - e0)
        o_row = np.zeros(H * dh)
        q_row = np.zeros(H * dh)
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            kc, vc = r["k"][cols, sl], r["v"][cols, sl]
            sc = kc @ r["q"][i, sl] * scale + b
            p = np.exp(sc - sc.max())
            p /= p.sum()
            o_row[sl] = p @ vc
            dw = vc @ r["do"][i, sl]
            ds = np.zeros_like(p) if e1 - e0 == 1 else p * (dw - p @ dw)
            q_row[sl] = scale * (ds @ kc)
            dbs += ds
        got_o.append(r["out"][i]); want_o.append(o_row)
        got_q.append(r["dq"][i]); want_q.append(q_row)
        got_b.append(r["db"][e0:e1]); want_b.append(dbs)
    assert_close(np.concatenate(got_o), np.concatenate(want_o), dtype, f"{what} sampled rows out")
    assert_close(np.concatenate(got_q), np.concatenate(want_q), dtype, f"{what} sampled rows dq")
    assert_close(np.concatenate(got_b), np.concatenate(want_b), dtype, f"{what} sampled rows dbias (all heads)")


@pytest.fixture(scope="module")
def c1_graph():
    s, t = c1_edges()
    ro, co = csr_from_pairs(4096, s, t)
    return CSR(4096, ro, co)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
def test_c1_multihead(cuda, orc, c1_graph, dtype):
    g = c1_graph
    assert g.nnz == 69497
    r = run_device(g.row_off, g.cols, 8, 8, dtype, seed=1)
    want = oracle_multihead(orc, g, r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, dtype, f"C1 {nm}")


@pytest.fixture(scope="module")
def c2_graph():
    ro, co = arxiv_c2()
    return CSR(169343, ro, co)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c2_arxiv_shape_multihead(cuda, orc, c2_graph, dtype):
    """C2 (BASELINE configs[1]: ogbn-arxiv shape, 169,343 nodes, E = 1,335,586
    with loops; GT H = 8, dh = 16) at full size against the fp64 oracle, in the
    community execution order the bench uses."""
    g = c2_graph
    assert g.nnz == 1335586
    r = run_device(g.row_off, g.cols, 8, 16, dtype, seed=5, order="schedule")
    want = oracle_multihead(orc, g, r, 8, 16)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, dtype, f"C2 {nm}")


@pytest.fixture(scope="module")
def c4_graph():
    return malnet_c4()


@pytest.mark.parametrize("H,dh", [(32, 24), (8, 8)])
def test_c4_malnet_shape_global_token(cuda, orc, c4_graph, H, dh):
    """C4 (BASELINE configs[3] shape: 524,288 nodes + a global token attending
    to / attended by every node, E = 2.84M; GPH-large H = 32, dh = 24) at full
    size in f32: the degree-524,289 row and column go through the generic
    kernels' two-level sums (dh = 24) or the tile path's hub kernels (H = 8,
    dh = 8, the GPH-slim geometry). Heads 0, H/2 and H-1 against the fp64
    oracle over the whole graph (~2.5 s per head); every head, incl. the
    head-summed dbias, on 96 sampled rows and the global token's row."""
    import torch

    ro, co = c4_graph
    S, E = ro.shape[0] - 1, co.shape[0]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(9)
    q, k, v, do = (torch.randn((S, H * dh), generator=g, device=dev) for _ in range(4))
    bias = 0.3 * torch.randn(E, generator=g, device=dev)
    plan = A.DevicePlan.from_host(ro, co)
    plan.schedule()
    att = A.DeviceSparseAttention(plan, H, dh, dh, "f32")
    out, lse = att.forward(q, k, v, bias, None)
    dq, dk, dv, db = att.backward(q, k, v, out, lse, do, bias, None)
    plan.ctx.sync()
    G = CSR(S, ro, co)
    b64 = bias.double().cpu().numpy()
    for h in (0, H // 2, H - 1):
        sl = slice(h * dh, (h + 1) * dh)
        f = lambda t: t[:, sl].double().cpu().numpy()  # noqa: E731
        qh, kh, vh, doh = f(q), f(k), f(v), f(do)
        assert_close(f(out), orc.sparse_fwd(qh, kh, vh, G, b64, None), "f32", f"C4 head {h} out")
        wq, wk, wv, _ = orc.sparse_bwd(qh, kh, vh, G, b64, None, doh)
        for got, w, nm in ((dq, wq, "dq"), (dk, wk, "dk"), (dv, wv, "dv")):
            assert_close(f(got), w, "f32", f"C4 head {h} {nm}")
    # every head, sampled rows incl. the global token (degree 524,289):
    # output, dQ and the head-summed dbias of their edges
    deg = np.diff(ro)
    rows = np.r_[np.random.default_rng(1).choice(S, 96, replace=False), np.argmax(deg)]
    fn = lambda t: t.double().cpu().numpy()  # noqa: E731
    rr = dict(q=fn(q), k=fn(k), v=fn(v), do=fn(do), bias=b64, out=fn(out), dq=fn(dq), db=fn(db)[:E])
    check_sampled_rows(rr, ro, co, rows, H, dh, "f32", f"C4 H={H}")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c3_bench_pattern_full_size(cuda, orc, dtype):
    """C3, the bench's own workload (BASELINE configs[2]: products shape,
    S = 262,144, cluster reorder k = 8 + Elastic layout at 5 beta_G, d_b = 16,
    E = 6.39M; GPH-slim H = 8, dh = 8) at full size in community order: all
    heads and the head-summed dbias against the fp64 oracle."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    ro, co = bench.cached_workload("ecr", {})
    g = CSR(ro.shape[0] - 1, ro.astype(np.int64), co.astype(np.int64))
    assert g.n == 262144
    r = run_device(g.row_off, g.cols, 8, 8, dtype, seed=4, order="schedule")
    want = oracle_multihead(orc, g, r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, dtype, f"C3 {nm}")


@pytest.fixture(scope="module")
def c5_graph():
    return papers_c5()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c5_papers_shape_heads(cuda, orc, c5_graph, dtype):
    """C5 (BASELINE configs[4] shape on one GPU: S = 1,048,576, E ~ 16M,
    GPH-slim H = 8, dh = 8) at full size through the tile kernels in community
    order; heads 0 and 5 against the fp64 oracle (~5 s per head)."""
    import torch

    ro, co = c5_graph
    S, E, H, dh = ro.shape[0] - 1, co.shape[0], 8, 8
    dev = torch.device("cuda:0")
    td = _torch_dtype(dtype)
    g = torch.Generator(device=dev).manual_seed(21)
    q, k, v, do = (torch.randn((S, H * dh), generator=g, device=dev).to(td) for _ in range(4))
    bias = 0.3 * torch.randn(E, generator=g, device=dev)
    plan = A.DevicePlan.from_host(ro, co)
    plan.schedule()
    att = A.DeviceSparseAttention(plan, H, dh, dh, dtype)
    out, lse = att.forward(q, k, v, bias, None)
    dq, dk, dv, db = att.backward(q, k, v, out, lse, do, bias, None)
    plan.ctx.sync()
    G = CSR(S, ro, co)
    b64 = bias.double().cpu().numpy()
    for h in (0, 5):
        sl = slice(h * dh, (h + 1) * dh)
        f = lambda t: t[:, sl].double().cpu().numpy()  # noqa: E731
        qh, kh, vh, doh = f(q), f(k), f(v), f(do)
        assert_close(f(out), orc.sparse_fwd(qh, kh, vh, G, b64, None), dtype, f"C5 head {h} out")
        wq, wk, wv, _ = orc.sparse_bwd(qh, kh, vh, G, b64, None, doh)
        for got, w, nm in ((dq, wq, "dq"), (dk, wk, "dk"), (dv, wv, "dv")):
            assert_close(f(got), w, dtype, f"C5 head {h} {nm}")
    # every head, 256 sampled rows: output, dQ, head-summed dbias
    rows = np.random.default_rng(2).choice(S, 256, replace=False)
    fn = lambda t: t.double().cpu().numpy()  # noqa: E731
    rr = dict(q=fn(q), k=fn(k), v=fn(v), do=fn(do), bias=b64, out=fn(out), dq=fn(dq), db=fn(db)[:E])
    check_sampled_rows(rr, ro, co, rows, H, dh, dtype, "C5")


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_c1_with_dropout_mask(cuda, orc, c1_graph, dtype):
    r = run_device(c1_graph.row_off, c1_graph.cols, 8, 8, dtype, seed=2, with_wm=True)
    want = oracle_multihead(orc, c1_graph, r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, dtype, f"C1+mask {nm}")


@pytest.mark.parametrize("H,dh", [(1, 8), (2, 16), (4, 4), (3, 5), (16, 8), (32, 24), (8, 64)])
def test_head_geometries_f32(cuda, orc, H, dh):
    ro, co = community_graph(1500, 9.0, community=64, seed=H * 100 + dh)
    g = CSR(1500, ro, co)
    r = run_device(ro, co, H, dh, "f32", seed=H + dh)
    want = oracle_multihead(orc, g, r, H, dh)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, "f32", f"H={H} dh={dh} {nm}")


def test_hub_rows_and_columns_f32(cuda, orc):
    # a global token attending / attended by every node (proj/src/model.cpp:349-357)
    n = 5000
    s, t = c1_edges(n - 1, 6, 9)
    glob = n - 1
    src = np.r_[s, np.arange(n - 1), np.full(n - 1, glob)]
    dst = np.r_[t, np.full(n - 1, glob), np.arange(n - 1)]
    ro, co = csr_from_pairs(n, src, dst)
    g = CSR(n, ro, co)
    r = run_device(ro, co, 8, 8, "f32", seed=5)
    want = oracle_multihead(orc, g, r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, "f32", f"hub {nm}")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [1100, 2048, 1038])
def test_hub_degree_slot_trip_counts(cuda, orc, dtype, n):
    """Hub rows / columns whose degree leaves the slots of one warp with
    different trip counts (degree mod (slots x EPL) odd): the hub kernels keep
    a warp-uniform loop (their head sums shuffle across the warp's slots)."""
    s = np.arange(n)
    src = np.r_[s, s, np.full(n, n)]
    dst = np.r_[(s + 1) % n, np.full(n, n), s]
    ro, co = csr_from_pairs(n + 1, src, dst)
    g = CSR(n + 1, ro, co)
    r = run_device(ro, co, 8, 8, dtype, seed=8)
    want = oracle_multihead(orc, g, r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, dtype, f"hub d={n + 1} {nm}")


@pytest.mark.parametrize("dtype,wm", [("f32", False), ("bf16", False), ("f32", True)])
def test_hub_rows_bf16_and_schedule(cuda, orc, dtype, wm):
    # hub row/column longer than a tile's staging capacity (global-memory ids)
    n = 3000
    s, t = c1_edges(n - 1, 5, 11)
    glob = n - 1
    src = np.r_[s, np.arange(n - 1), np.full(n - 1, glob)]
    dst = np.r_[t, np.full(n - 1, glob), np.arange(n - 1)]
    ro, co = csr_from_pairs(n, src, dst)
    g = CSR(n, ro, co)
    r = run_device(ro, co, 8, 8, dtype, seed=6, order="schedule", with_wm=wm)
    want = oracle_multihead(orc, g, r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, dtype, f"hub+schedule {nm}")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_execution_order_is_bit_identical(cuda, dtype):
    # the community schedule / any execution order changes nothing (each row
    # is computed by one slot with the same arithmetic, written in place)
    ro, co = community_graph(20000, 12.0, community=128, seed=3, shuffle=True)
    base = run_device(ro, co, 8, 8, dtype, seed=4, with_wm=(dtype == "f32"))
    rnd = np.random.default_rng(0).permutation(20000)
    for order in ("schedule", rnd):
        r = run_device(ro, co, 8, 8, dtype, seed=4, with_wm=(dtype == "f32"), order=order)
        for nm in ("out", "lse", "dq", "dk", "dv", "db"):
            assert np.array_equal(r[nm], base[nm]), f"{nm} differs under execution order"


# ---------------------------------------------------------------- edge semantics

def test_empty_and_singleton_rows_exact(cuda):
    # row 0 -> {1}; row 1 -> {} ; row 2 -> {0,1,2}; row 3 -> {3}
    ro = np.array([0, 1, 1, 4, 5], dtype=np.int64)
    co = np.array([1, 0, 1, 2, 3], dtype=np.int64)
    pat = A.AttnPattern(4, ro, co)
    rng = np.random.default_rng(0)
    q, k, v, up = (rng.standard_normal((4, 3)) for _ in range(4))
    wm = np.array([2.0, 1.0, 0.0, 1.5, 0.5])
    for dtype in ("f64", "f32"):
        res = A.sparse_attention(q, k, v, pat, None, wm, dtype=dtype)
        vv = v.astype(np.float32) if dtype == "f32" else v
        assert np.array_equal(res.output[0], (2.0 * vv[1]).astype(res.output.dtype))  # deg 1: m * v_j exactly
        assert np.all(res.output[1] == 0)  # deg 0: zero row
        assert np.array_equal(res.output[3], (0.5 * vv[3]).astype(res.output.dtype))
        gr = A.sparse_attention_backward(q, k, v, pat, None, wm, up, dtype=dtype)
        assert np.all(gr.dq[0] == 0) and np.all(gr.dq[1] == 0) and np.all(gr.dq[3] == 0)
        assert gr.dbias[0] == 0 and gr.dbias[4] == 0
    with pytest.raises(DataError, match=r"row 1 attends to nothing; run add_self_loops"):
        A.edge_sparse_attention(q, k, v, A.Graph(4, ro, co))


def test_non_finite_inputs_raise(cuda):
    ro = np.array([0, 1, 2, 3], dtype=np.int64)
    co = np.array([0, 1, 1], dtype=np.int64)  # row 2 never referenced as a column
    pat = A.AttnPattern(3, ro, co)
    base = np.ones((3, 2))
    for which, name in ((0, "Q"), (1, "K"), (2, "V")):
        args = [base.copy(), base.copy(), base.copy()]
        args[which][2, 1] = np.inf if which != 1 else np.nan
        with pytest.raises(DataError, match=f"non-finite {name}"):
            A.sparse_attention(*args, pat)
    ok = A.sparse_attention(base, base, base, pat)
    assert np.allclose(ok.output, 1.0)


def test_shape_errors(cuda):
    pat = A.AttnPattern(2, np.array([0, 1, 2]), np.array([0, 1]))
    with pytest.raises(ConfigError, match="row counts differ"):
        A.sparse_attention(np.zeros((2, 2)), np.zeros((3, 2)), np.zeros((2, 2)), pat)
    with pytest.raises(ConfigError, match="bias must cover"):
        A.sparse_attention(np.zeros((2, 2)), np.zeros((2, 2)), np.zeros((2, 2)), pat, bias=np.zeros(3))
    with pytest.raises(ConfigError, match="pattern/sequence length mismatch"):
        A.sparse_attention(np.zeros((3, 2)), np.zeros((3, 2)), np.zeros((3, 2)), pat)


def test_complete_graph_equals_dense(cuda, orc):
    # reference proj/tests/test_attention.cpp:75-87 / acceptance C1
    rng = np.random.default_rng(100)
    for s in (4, 7, 10, 13, 16):
        ro, co = csr_from_pairs(s, np.repeat(np.arange(s), s), np.tile(np.arange(s), s), self_loops=False)
        q, k, v = (rng.standard_normal((s, 4)) for _ in range(3))
        dense = orc.dense_fwd(q, k, v)
        got = A.edge_sparse_attention(q, k, v, A.Graph(s, ro, co)).output
        assert np.abs(got - dense).max() <= 1e-12


# ---------------------------------------------------------------- wide (32-byte lane) tile kernels

def _mixed_degree_graph(n=3000, seed=21):
    """Rows of every degree 0..9 plus a community bulk: exercises the per-row
    padding of the wide kernels (pads = first neighbour, bias -inf)."""
    rng = np.random.default_rng(seed)
    src, dst = [], []
    for u in range(n):
        d = u % 10 if u < 600 else int(rng.integers(5, 40))
        if d:
            nb = rng.choice(n, size=d, replace=False)
            src += [u] * d
            dst += list(nb)
    return csr_from_pairs(n, np.array(src), np.array(dst), self_loops=False)


@pytest.mark.parametrize("dtype,H,dh,wm", [("f32", 8, 8, False), ("bf16", 8, 8, False), ("bf16", 8, 8, True),
                                           ("bf16", 8, 16, False), ("f32", 4, 16, True), ("bf16", 16, 8, False)])
def test_mixed_degrees_empty_and_singleton_rows(cuda, orc, dtype, H, dh, wm):
    ro, co = _mixed_degree_graph()
    g = CSR(ro.shape[0] - 1, ro, co)
    r = run_device(ro, co, H, dh, dtype, seed=H * dh + wm, with_wm=wm, order="schedule")
    want = oracle_multihead(orc, g, r, H, dh)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, dtype, f"mixed H={H} dh={dh} wm={wm} {nm}")
    deg = np.diff(ro)
    one = np.nonzero(deg == 1)[0]
    zero = np.nonzero(deg == 0)[0]
    # degree-1 rows: out = m * v_j exactly, dq = 0 and dbias = 0 exactly (attention.cpp:128-135, 265-272)
    j = co[ro[one]]
    if not wm:
        assert np.array_equal(r["out"][one], r["v"][j])
    assert np.all(r["dq"][one] == 0) and np.all(r["db"][ro[one]] == 0)
    assert np.all(r["out"][zero] == 0) and np.all(r["dq"][zero] == 0)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_fwd_bwd_host_matches_device_path(cuda, dtype):
    """gte_sparse_attn_fwd_bwd_host (pinned host buffers, copies on a second
    stream overlapped with the kernels) == the device-resident path, bit for
    bit, over repeated calls (the bench's e2e leg)."""
    import torch

    ro, co = community_graph(6000, 10.0, community=64, seed=8)
    r = run_device(ro, co, 8, 8, dtype, seed=9)
    td = _torch_dtype(dtype)
    pin = lambda a, t: torch.tensor(a, dtype=t).pin_memory()  # noqa: E731
    hq, hk, hv, hdo = (pin(r[n], td) for n in ("q", "k", "v", "do"))
    hb = pin(r["bias"], torch.float32)
    plan = A.DevicePlan.from_host(ro, co)
    att = A.DeviceSparseAttention(plan, 8, 8, 8, dtype)
    outs = [torch.empty(hv.shape, dtype=td).pin_memory() for _ in range(4)]
    hdb = torch.empty(co.shape[0], dtype=torch.float32).pin_memory()
    for _ in range(3):
        att.fwd_bwd_host(hq, hk, hv, hdo, hb, *outs, hdb)
    for got, nm in zip(outs + [hdb], ("out", "dq", "dk", "dv", "db")):
        assert np.array_equal(got.double().numpy(), r[nm]), nm
    # asynchronous steps back to back (uploads of one overlap downloads of the previous)
    for t in outs + [hdb]:
        t.zero_()
    for _ in range(4):
        att.fwd_bwd_host(hq, hk, hv, hdo, hb, *outs, hdb, sync=False)
    plan.ctx.sync()
    for got, nm in zip(outs + [hdb], ("out", "dq", "dk", "dv", "db")):
        assert np.array_equal(got.double().numpy(), r[nm]), nm


@pytest.mark.parametrize("dtype,which", [("f32", 0), ("bf16", 0), ("f32", 1), ("bf16", 2)])
def test_non_finite_multihead_tile_path(cuda, dtype, which):
    """attention.cpp:20-22 on the tile kernels: a NaN/inf anywhere in Q, K or V
    (here in a row that is some tile's own row) raises DataError at sync."""
    import torch

    ro, co = community_graph(3000, 8.0, community=64, seed=2)
    td = _torch_dtype(dtype)
    q, k, v = (torch.randn((3000, 64), device="cuda").to(td) for _ in range(3))
    [q, k, v][which][1234, 17] = float("nan") if which != 1 else float("inf")
    plan = A.DevicePlan.from_host(ro, co)
    att = A.DeviceSparseAttention(plan, 8, 8, 8, dtype)
    att.forward(q, k, v)
    with pytest.raises(DataError, match=f"non-finite {'QKV'[which]}"):
        plan.ctx.sync()
    att.forward(*(torch.randn((3000, 64), device="cuda").to(td) for _ in range(3)))
    plan.ctx.sync()  # the error latch was reset
