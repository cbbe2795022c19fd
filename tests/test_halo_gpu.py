"""Cluster-halo sequence parallelism on the device (halo.py + csrc/sp.cu
gather / scatter-add / all_to_allv): P logical ranks on one GPU (loopback
exchange) against the single-GPU layer and the oracle; the NCCL all_to_allv
on a one-rank communicator."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import CSR

from paper_2407_14106_b200 import attention as A
from paper_2407_14106_b200.datagen import community_graph
from paper_2407_14106_b200.halo import HaloAttention, HaloLoopback, build_halo_plan

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5, "bf16": 1e-2}


def _run(ro, co, P, H, dh, dtype, seed=0, overlap=False):
    import torch

    td = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    acc = torch.float64 if dtype == "f64" else torch.float32
    S, E = ro.shape[0] - 1, co.shape[0]
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(td) for _ in range(4))
    bias = (0.3 * torch.randn(E, generator=g, device="cuda")).to(acc)
    plans = build_halo_plan(ro, co, P)
    layer = HaloAttention(plans, P, H, dh, dtype, HaloLoopback(P), overlap=overlap)
    sl = lambda t, r: t[r.lo:r.hi].contiguous()  # noqa: E731
    out = layer.forward({r.rank: sl(q, r) for r in plans}, {r.rank: sl(k, r) for r in plans},
                        {r.rank: sl(v, r) for r in plans}, bias)
    grads = layer.backward({r.rank: sl(up, r) for r in plans})
    torch.cuda.synchronize()
    cat = lambda d: torch.cat([d[r.rank] for r in plans]).double().cpu().numpy()  # noqa: E731
    res = dict(out=cat(out), dq=cat({p: grads[p][0] for p in grads}), dk=cat({p: grads[p][1] for p in grads}),
               dv=cat({p: grads[p][2] for p in grads}), db=cat({p: grads[p][3] for p in grads}))
    # single-GPU reference path
    plan = A.DevicePlan.from_host(ro, co)
    att = A.DeviceSparseAttention(plan, H, dh, dh, dtype)
    o1, lse1 = att.forward(q, k, v, bias)
    dq1, dk1, dv1, db1 = att.backward(q, k, v, o1, lse1, up, bias)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()  # noqa: E731
    one = dict(out=f(o1), dq=f(dq1), dk=f(dk1), dv=f(dv1), db=f(db1)[:E])
    inputs = dict(q=f(q), k=f(k), v=f(v), up=f(up), bias=f(bias))
    return res, one, inputs, plans


@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_halo_matches_single_gpu(cuda, dtype, P, overlap):
    """P logical ranks on one GPU against the single-GPU layer; with
    `overlap` the interior / boundary plans and the exchange stream."""
    ro, co = community_graph(20000, 12.0, community=256, seed=P, shuffle=False)
    res, one, _, plans = _run(ro, co, P, 8, 8, dtype, seed=P, overlap=overlap)
    for nm in ("out", "dq", "dk", "dv", "db"):
        e = rel_err(res[nm], one[nm])
        assert max(e) <= TOL[dtype], (nm, e)
    if dtype == "f32":  # rows whose columns are all local: identical arithmetic
        assert np.array_equal(res["out"][:10], res["out"][:10])
    recv = sum(r.boundary_rows()[0] for r in plans)
    assert recv > 0


def test_halo_f64_vs_oracle(cuda, orc):
    ro, co = community_graph(3000, 9.0, community=64, seed=11, shuffle=True)
    res, _, x, _ = _run(ro, co, 3, 2, 4, "f64", seed=3)
    g = CSR(3000, ro, co)
    db = np.zeros(co.shape[0])
    for h in range(2):
        sl = slice(h * 4, (h + 1) * 4)
        w = orc.sparse_fwd(x["q"][:, sl], x["k"][:, sl], x["v"][:, sl], g, x["bias"])
        assert max(rel_err(res["out"][:, sl], w)) <= 1e-12
        a, b, c, e = orc.sparse_bwd(x["q"][:, sl], x["k"][:, sl], x["v"][:, sl], g, x["bias"], None, x["up"][:, sl])
        for got, want in ((res["dq"][:, sl], a), (res["dk"][:, sl], b), (res["dv"][:, sl], c)):
            assert max(rel_err(got, want)) <= 1e-12
        db += e
    assert max(rel_err(res["db"], db)) <= 1e-12


def test_all_to_allv_single_rank(cuda):
    """gte_comm_all_to_allv on a one-rank NCCL communicator: a local copy."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2407_14106_b200 import parallel as SP
    from paper_2407_14106_b200.halo import HaloNccl

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29563")
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
    ctx = A.Context.get(0)
    sp = SP.SequenceParallelPlan([np.arange(8, dtype=np.int64)], None, ctx)
    nx = SP.NcclExchange(sp, 0, 1)
    hx = HaloNccl(nx, 0, ctx)
    x = torch.arange(40, dtype=torch.float32, device="cuda").reshape(10, 4)
    y = torch.zeros_like(x)
    hx.exchange({0: x}, {0: y}, {0: [10]}, {0: [10]}, 4)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    nx.close()


@pytest.mark.parametrize("overlap", [False, True])
def test_halo_step_graph_capture_matches_eager(cuda, overlap):
    """The Mode H step captured as one CUDA graph (what bench.py replays per
    rank) gives the eager step's results bit for bit: every op of the path is
    stream-ordered on the capturing stream (or forked / joined from it)."""
    import torch

    P, H, dh = 4, 8, 8
    ro, co = community_graph(12000, 10.0, community=256, seed=11, shuffle=False)
    S, E = ro.shape[0] - 1, co.shape[0]
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    bias = (0.3 * torch.randn(E, generator=g, device="cuda")).float()
    plans = build_halo_plan(ro, co, P)
    layer = HaloAttention(plans, P, H, dh, "bf16", HaloLoopback(P), overlap=overlap)
    sl = lambda t, r: t[r.lo:r.hi]  # noqa: E731

    def step():
        o = layer.forward({r.rank: sl(q, r) for r in plans}, {r.rank: sl(k, r) for r in plans},
                          {r.rank: sl(v, r) for r in plans}, bias)
        gr = layer.backward({r.rank: sl(up, r) for r in plans})
        return [o[r.rank] for r in plans] + [x for r in plans for x in gr[r.rank]]

    eager = [x.clone() for x in step()]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = step()
    for t_ in out:
        t_.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for a_, b_ in zip(eager, out):
        assert torch.equal(a_, b_)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f64"])
def test_scatter_add_seq_equals_per_peer_adds(cuda, dtype):
    """gte_rows_scatter_add_seq (all peers' partials in one launch, peer order
    per row) is bit-identical to one gte_rows_scatter_add per peer, including
    rows that several peers send partials for and a strided source."""
    import torch

    from paper_2407_14106_b200.halo import DeviceHaloOps

    td = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    H, dh, n_own, P = 4, 8, 500, 5
    d = H * dh
    rng = np.random.default_rng(3)
    send = [np.sort(rng.choice(n_own, size=int(rng.integers(0, 200)), replace=False)).astype(np.int32)
            for _ in range(P)]
    cat = np.concatenate(send)
    g = torch.Generator(device="cuda").manual_seed(1)
    src = torch.randn((cat.shape[0], 2 * d), generator=g, device="cuda").to(td)  # [K | V] rows
    base = torch.randn((n_own, d), generator=g, device="cuda").to(td)
    ops = DeviceHaloOps(H, dh, dtype)
    want = base.clone()
    off = 0
    for s in send:
        if s.shape[0]:
            ops.scatter_add(want, ops.index(s), src[off:off + s.shape[0], d:].contiguous(), s.shape[0])
        off += s.shape[0]
    order = np.argsort(cat, kind="stable")
    rows_u, cnt = np.unique(cat[order], return_counts=True)
    seq = tuple(ops.index(x) for x in (rows_u, np.concatenate([[0], np.cumsum(cnt)]), order))
    got = base.clone()
    ops.scatter_add_seq(got, seq, src, d)  # the V half of the strided [K | V] rows
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert (cnt > 1).any()


def test_own_view_inputs_match_copied_inputs(cuda):
    """Shards written straight into the layer's [own | halo] buffers
    (HaloAttention.own_view, what bench.py's ranks do) give the results of
    shards passed as separate tensors, bit for bit."""
    import torch

    P, H, dh = 3, 8, 8
    ro, co = community_graph(6000, 10.0, community=128, seed=2, shuffle=False)
    S, E = ro.shape[0] - 1, co.shape[0]
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    bias = (0.3 * torch.randn(E, generator=g, device="cuda")).float()
    plans = build_halo_plan(ro, co, P)
    res = []
    for in_place in (False, True):
        layer = HaloAttention(plans, P, H, dh, "bf16", HaloLoopback(P))
        sh = {}
        for nm, t in (("q", q), ("k", k), ("v", v), ("do", up)):
            sh[nm] = {}
            for r in plans:
                if in_place:
                    view = layer.own_view(r.rank, nm, t.dtype, t.device)
                    view.copy_(t[r.lo:r.hi])
                    sh[nm][r.rank] = view
                else:
                    sh[nm][r.rank] = t[r.lo:r.hi].clone()
        o = layer.forward(sh["q"], sh["k"], sh["v"], bias)
        gr = layer.backward(sh["do"])
        torch.cuda.synchronize()
        res.append([o[r.rank].clone() for r in plans] + [x.clone() for r in plans for x in gr[r.rank]])
    for a_, b_ in zip(*res):
        assert torch.equal(a_, b_)


def test_plan_output_rows(cuda):
    """gte_plan_set_output_rows: rows >= n (edge-free) get no forward / CSR-pass
    work; rows < n and every dK / dV column equal the full plan's bit for bit.
    Rows >= n with edges are refused (ConfigError)."""
    import torch

    from paper_2407_14106_b200._lib import ConfigError

    H, dh, n_own, n_halo = 8, 8, 3000, 700
    rng = np.random.default_rng(4)
    deg = rng.integers(1, 12, n_own)
    ro = np.concatenate([[0], np.cumsum(deg), np.full(n_halo, deg.sum())]).astype(np.int64)
    co = np.concatenate([np.sort(rng.choice(n_own + n_halo, int(d), replace=False)) for d in deg]).astype(np.int64)
    S, E = n_own + n_halo, co.shape[0]
    g = torch.Generator(device="cuda").manual_seed(4)
    q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    bias = (0.3 * torch.randn(E, generator=g, device="cuda")).float()
    res = []
    for limit in (False, True):
        plan = A.DevicePlan.from_host(ro, co)
        plan.schedule()
        if limit:
            plan.set_output_rows(n_own)
        att = A.DeviceSparseAttention(plan, H, dh, dh, "bf16")
        o, lse = att.forward(q, k, v, bias)
        dq, dk, dv, db = att.backward(q, k, v, o, lse, up, bias)
        torch.cuda.synchronize()
        res.append((o[:n_own].clone(), lse[:n_own].clone(), dq[:n_own].clone(), dk.clone(), dv.clone(), db[:E].clone()))
    for a_, b_ in zip(*res):
        assert torch.equal(a_, b_)
    plan = A.DevicePlan.from_host(ro, co)
    with pytest.raises(ConfigError):
        plan.set_output_rows(n_own - 1)
