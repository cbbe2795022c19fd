"""Sequence-parallel attention layer on the device (csrc/sp.cu +
paper_2407_14106_b200/parallel.py) against the compiled reference's
run_distributed_layer(_backward) golden outputs (tests/golden/
parallel_interleave_small.npz, made by tests/golden/make_golden.py) and the
C oracle at larger sizes: outputs, ledger (4Sd/P contract, halving), MACs,
P-invariance; the NCCL exchange on a one-rank communicator against the
loopback exchange."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import CSR

from paper_2407_14106_b200 import parallel as SP
from paper_2407_14106_b200.attention import AttnPattern, DevicePlan
from paper_2407_14106_b200.datagen import community_graph
from paper_2407_14106_b200.partition import Permutation

pytestmark = pytest.mark.gpu


def _shards(ids, q, k, v):
    P = ids.shape[0]
    return [SP.WorkerShard(w, ids[w], q[ids[w]], k[ids[w]], v[ids[w]]) for w in range(P)]


def _full(shards_out, ids, S, d):
    out = np.zeros((S, d))
    for w in range(ids.shape[0]):
        out[ids[w]] = shards_out[w]
    return out


def _ledger_arr(L):
    return np.array([[e.qkv_gather, e.qkv_gather_cross, e.output_scatter, e.output_scatter_cross, e.bias_exchange]
                     for e in L.workers], dtype=np.int64)


def test_distributed_layer_golden(cuda, golden):
    d = golden("parallel_interleave_small.npz")
    ro, co = d["dl_g_ro"], d["dl_g_cols"]
    S = int(d["dl_g_n"])
    pat = AttnPattern(S, ro, co)
    perm = Permutation(d["dl_fwd"], d["dl_inv"])
    q, k, v, up = (d["dl_" + n] for n in ("q", "k", "v", "up"))
    for P in (1, 2, 4):
        ids = d[f"dl{P}_ids"]
        shards = _shards(ids, q, k, v)
        ledger = SP.CommLedger(P)
        res = SP.run_distributed_layer(shards, pat, perm, 4, d["dl_bias"], d["dl_wm"], ledger)
        out = _full(res.out_shards, ids, S, q.shape[1])
        assert np.abs(out - d[f"dl{P}_out"]).max() <= 1e-12, P
        assert np.array_equal(_ledger_arr(ledger), d[f"dl{P}_ledger"]), P
        assert res.macs.score_macs == int(d[f"dl{P}_macs"]), P
        g = SP.run_distributed_layer_backward(shards, pat, perm, 4, d["dl_bias"], d["dl_wm"],
                                              [up[ids[w]] for w in range(P)])
        for got, nm in ((g.dq_sub, "dq"), (g.dk_sub, "dk"), (g.dv_sub, "dv")):
            assert np.abs(_full(got, ids, S, q.shape[1]) - d[f"dl{P}_{nm}"]).max() <= 1e-12, (P, nm)
        assert np.abs(g.dbias - d[f"dl{P}_db"]).max() <= 1e-12, P


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_distributed_layer_vs_oracle(cuda, orc, dtype):
    S, H, dh = 4096, 8, 8
    ro, co = community_graph(S, 12.0, community=64, seed=3)
    g = CSR(S, ro, co)
    rng = np.random.default_rng(7)
    fwd = rng.permutation(S).astype(np.int64)
    inv = np.argsort(fwd).astype(np.int64)
    q, k, v, up = (rng.standard_normal((S, H * dh)) for _ in range(4))
    if dtype == "f32":
        q, k, v, up = (x.astype(np.float32).astype(np.float64) for x in (q, k, v, up))
    bias = rng.normal(0, 0.3, co.shape[0])
    tol = 1e-12 if dtype == "f64" else 1e-5
    for P in (2, 8):
        ids = orc.partition_sequence(S, P, 11 + P)
        want, wl, wm_ = orc.dist_fwd(P, ids, q, k, v, g, fwd, inv, H, bias)
        shards = _shards(ids, q, k, v)
        ledger = SP.CommLedger(P)
        res = SP.run_distributed_layer(shards, AttnPattern(S, ro, co), Permutation(fwd, inv), H, bias, None, ledger,
                                       dtype=dtype)
        e = rel_err(_full(res.out_shards, ids, S, H * dh), want)
        assert max(e) <= tol, (P, e)
        assert np.array_equal(_ledger_arr(ledger), wl)
        # 4Sd/P per worker (acceptance_main.cpp:127) and halving with P
        assert all(ledger.transport_elements(w) == 4 * S * H * dh // P for w in range(P))
        gq, gk, gv, gb = orc.dist_bwd(P, ids, q, k, v, g, fwd, inv, H, bias, None, up)
        gr = SP.run_distributed_layer_backward(shards, AttnPattern(S, ro, co), Permutation(fwd, inv), H, bias, None,
                                               [up[ids[w]] for w in range(P)], dtype=dtype)
        for got, w_, nm in ((gr.dq_sub, gq, "dq"), (gr.dk_sub, gk, "dk"), (gr.dv_sub, gv, "dv")):
            e = rel_err(_full(got, ids, S, H * dh), w_)
            assert max(e) <= tol, (P, nm, e)
        assert max(rel_err(gr.dbias, gb)) <= tol


def test_nccl_single_rank_matches_loopback(cuda):
    """The NCCL exchange (gte_comm_*) on a one-rank communicator: same bits as
    the loopback exchange (P = 1, all chunks local)."""
    import os

    import torch
    import torch.distributed as dist

    S, H, dh = 2048, 8, 8
    ro, co = community_graph(S, 10.0, community=64, seed=5)
    rng = np.random.default_rng(1)
    q, k, v, up = (torch.tensor(rng.standard_normal((S, H * dh)), dtype=torch.float32, device="cuda") for _ in range(4))
    fwd = rng.permutation(S).astype(np.int64)
    plan = DevicePlan.from_host(ro, co)
    ids = [np.arange(S, dtype=np.int64)]
    sp = SP.SequenceParallelPlan(ids, fwd, plan.ctx)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    if not dist.is_initialized():
        dist.init_process_group("gloo", rank=0, world_size=1)
    nx = SP.NcclExchange(sp, 0, 1)
    outs = []
    for ex in (nx, SP.Loopback(sp)):
        layer = SP.UlyssesAttention.on_device(plan, sp, H, H * dh, "f32", ex)
        o, _ = layer.forward({0: q}, {0: k}, {0: v})
        dq, dk, dv, db = layer.backward({0: up})
        torch.cuda.synchronize()
        outs.append([t[0].cpu() if isinstance(t, dict) else t.cpu() for t in (o, dq, dk, dv, db)])
    nx.close()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_config_errors(cuda):
    S = 16
    ro = np.arange(S + 1, dtype=np.int64)
    co = np.arange(S, dtype=np.int64)
    pat = AttnPattern(S, ro, co)
    sh = SP.partition_sequence(S, 4, 1)
    rng = np.random.default_rng(0)
    for s in sh:
        s.q_sub, s.k_sub, s.v_sub = (rng.standard_normal((4, 12)) for _ in range(3))
    with pytest.raises(SP.ConfigError, match="head count not divisible by worker count"):
        SP.run_distributed_layer(sh, pat, Permutation.identity(S), 6, None, None, SP.CommLedger(4))
    with pytest.raises(SP.ConfigError, match="ledger sized for wrong worker count"):
        SP.run_distributed_layer(sh, pat, Permutation.identity(S), 4, None, None, SP.CommLedger(3))
