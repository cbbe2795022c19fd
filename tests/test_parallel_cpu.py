"""Multi-process sequence parallelism on CPU (gloo, world_size 2): the
UlyssesAttention orchestration (exchange order, chunk layout, ledger, cached
slices, worker-ordered dbias) with TorchDistExchange, against the C oracle's
run_distributed_layer(_backward) (oracle/orc_parallel.c, pinned to the
compiled reference by tests/test_oracle_golden.py::test_parallel_golden).

The device halves (pack/unpack kernels, attention kernels) are GPU-only; here
they are replaced by `CpuOps`, a test-local restatement of the reference's
row copies (parallel.cpp:48-79, 115-188) with the oracle's per-head
attention — the checker, not the product. The product's device halves are
tested on the GPU (tests/test_parallel_gpu.py)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class CpuOps:
    def __init__(self, orc, P, ids, fwd, heads, d, ro, co):
        import torch

        from oracle import CSR

        self.orc, self.P, self.ids, self.fwd, self.H, self.d = orc, P, ids, fwd, heads, d
        self.rows, self.S = ids.shape[1], ids.size
        self.slice, self.hpw, self.dh = d // P, heads // P, d // heads
        self.g = CSR(self.S, ro, co)
        self.pos = torch.tensor(fwd[ids.reshape(-1)])  # execution position of (worker, row)
        self.dtype = "f64"

    def pack_seq(self, shard):
        return shard.reshape(self.rows, self.P, self.slice).permute(1, 0, 2).reshape(-1).contiguous()

    def unpack_head(self, buf):
        import torch

        out = torch.zeros((self.S, self.slice), dtype=buf.dtype)
        out[self.pos] = buf.reshape(-1, self.slice)
        return out

    def pack_head(self, sl):
        return sl[self.pos].reshape(-1).contiguous()

    def unpack_seq(self, buf):
        return buf.reshape(self.P, self.rows, self.slice).permute(1, 0, 2).reshape(self.rows, self.d).contiguous()

    def _heads(self, x, t):
        return x[:, t * self.dh:(t + 1) * self.dh].numpy()

    def attn_fwd(self, q, k, v, bias, wm):
        import torch

        o = np.zeros((self.S, self.slice))
        b = None if bias is None else bias.numpy()
        for t in range(self.hpw):
            o[:, t * self.dh:(t + 1) * self.dh] = self.orc.sparse_fwd(self._heads(q, t), self._heads(k, t),
                                                                      self._heads(v, t), self.g, b,
                                                                      None if wm is None else wm[t].numpy())
        return torch.tensor(o), None

    def attn_bwd(self, q, k, v, o, lse, up, bias, wm):
        import torch

        dq, dk, dv = (np.zeros((self.S, self.slice)) for _ in range(3))
        db = np.zeros(self.g.nnz)
        b = None if bias is None else bias.numpy()
        for t in range(self.hpw):
            sl = slice(t * self.dh, (t + 1) * self.dh)
            a, c, e, f = self.orc.sparse_bwd(self._heads(q, t), self._heads(k, t), self._heads(v, t), self.g, b,
                                             None if wm is None else wm[t].numpy(), self._heads(up, t))
            dq[:, sl], dk[:, sl], dv[:, sl] = a, c, e
            db += f
        return torch.tensor(dq), torch.tensor(dk), torch.tensor(dv), torch.tensor(db)

    def ordered_sum(self, stacked):
        out = stacked[0].clone()
        for w in range(1, stacked.shape[0]):
            out += stacked[w]
        return out


def _worker(rank, world, port, path):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle

    from paper_2407_14106_b200 import parallel as SP

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = np.load(path)
    orc = Oracle()
    ids, fwd = d["ids"], d["fwd"]
    H, dm = int(d["H"]), d["q"].shape[1]
    ops = CpuOps(orc, world, ids, fwd, H, dm, d["ro"], d["co"])
    layer = SP.UlyssesAttention(ops, world, ids.shape[1], H, dm, d["co"].shape[0], SP.TorchDistExchange(rank, world))
    t = lambda a: torch.tensor(a[ids[rank]])  # noqa: E731
    ledger = SP.CommLedger(world)
    bias = torch.tensor(d["bias"])
    wm = torch.tensor(d["wm"])
    out, macs = layer.forward({rank: t(d["q"])}, {rank: t(d["k"])}, {rank: t(d["v"])}, bias, wm, ledger)
    dq, dk, dv, db = layer.backward({rank: t(d["up"])}, bias, wm)
    np.savez(path + f".rank{rank}.npz", out=out[rank].numpy(), dq=dq[rank].numpy(), dk=dk[rank].numpy(),
             dv=dv[rank].numpy(), db=db.numpy(), macs=macs.score_macs,
             ledger=np.array([[e.qkv_gather, e.qkv_gather_cross, e.output_scatter, e.output_scatter_cross,
                               e.bias_exchange] for e in ledger.workers]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_match_oracle(orc, tmp_path):
    import torch.multiprocessing as mp

    from paper_2407_14106_b200.datagen import community_graph

    world, S, H, dh = 2, 512, 4, 4
    ro, co = community_graph(S, 8.0, community=32, seed=9)
    rng = np.random.default_rng(3)
    q, k, v, up = (rng.standard_normal((S, H * dh)) for _ in range(4))
    bias = rng.normal(0, 0.3, co.shape[0])
    wm = (rng.random((H, co.shape[0])) < 0.8) / 0.8
    fwd = rng.permutation(S).astype(np.int64)
    inv = np.argsort(fwd).astype(np.int64)
    ids = orc.partition_sequence(S, world, 5)
    path = str(tmp_path / "case.npz")
    np.savez(path, ids=ids, fwd=fwd, H=H, q=q, k=k, v=v, up=up, bias=bias, wm=wm, ro=ro, co=co)
    mp.start_processes(_worker, args=(world, 29000 + os.getpid() % 1000, path), nprocs=world, start_method="spawn")

    from oracle import CSR

    g = CSR(S, ro, co)
    want, wl, wmacs = orc.dist_fwd(world, ids, q, k, v, g, fwd, inv, H, bias, wm.reshape(-1))
    gq, gk, gv, gb = orc.dist_bwd(world, ids, q, k, v, g, fwd, inv, H, bias, wm.reshape(-1), up)
    for r in range(world):
        got = np.load(path + f".rank{r}.npz")
        rows = ids[r]
        assert np.abs(got["out"] - want[rows]).max() <= 1e-12
        assert np.abs(got["dq"] - gq[rows]).max() <= 1e-12
        assert np.abs(got["dk"] - gk[rows]).max() <= 1e-12
        assert np.abs(got["dv"] - gv[rows]).max() <= 1e-12
        assert np.abs(got["db"] - gb).max() <= 1e-12
        assert np.array_equal(got["ledger"], wl) and int(got["macs"]) == wmacs


def test_ledger_arithmetic(orc):
    """CommLedger.tally == the reference's per-(src, dst) loop (parallel.cpp:134-146)."""
    from paper_2407_14106_b200 import parallel as SP

    for P, rows, sl in ((1, 7, 3), (4, 5, 2), (8, 32, 8)):
        L = SP.CommLedger(P)
        L.tally(P, rows, sl, True)
        L.tally(P, rows, sl, False)
        for e in L.workers:
            assert e.qkv_gather == P * rows * sl and e.qkv_gather_cross == (P - 1) * rows * sl
            assert e.output_scatter == P * rows * sl and e.output_scatter_cross == (P - 1) * rows * sl
        M = SP.CommLedger(P)
        M.accumulate(L)
        M.accumulate(L)
        assert M.transport_elements(0) == 2 * L.transport_elements(0)
    with pytest.raises(SP.ConfigError, match="worker count mismatch"):
        SP.CommLedger(2).accumulate(SP.CommLedger(3))


def test_partition_sequence_matches_oracle(orc):
    from paper_2407_14106_b200 import parallel as SP

    for S, P, seed in ((16, 4, 1), (17, 4, 2), (1000, 8, 42), (5, 8, 3)):
        sh = SP.partition_sequence(S, P, seed)
        assert np.array_equal(np.stack([s.token_ids for s in sh]), orc.partition_sequence(S, P, seed))
