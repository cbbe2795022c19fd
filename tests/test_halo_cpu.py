"""Host planner of the cluster-halo sequence parallelism (paper_2407_14106_b200/
halo.py): the local plans and exchange lists of all ranks
reassemble the global pattern exactly, and a 2-rank gloo run of the exchange
protocol (numpy attention from the oracle per rank) reproduces the oracle's
single-process results."""
import numpy as np
import pytest

from paper_2407_14106_b200.datagen import community_graph
from paper_2407_14106_b200.halo import build_halo_plan, row_ranges


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_plans_reassemble_pattern(P):
    ro, co = community_graph(3000, 9.0, community=64, seed=P, shuffle=True)
    S = ro.shape[0] - 1
    plans = build_halo_plan(ro, co, P)
    b = row_ranges(S, P)
    assert b[0] == 0 and b[-1] == S and np.all(np.diff(b) >= S // P)
    for r in plans:
        ext_ids = np.concatenate([np.arange(r.lo, r.hi), r.halo_ids])
        # local CSR maps back to the global rows' edges, in order
        for i in range(r.n_own):
            g = co[ro[r.lo + i]:ro[r.lo + i + 1]]
            l = r.local_co[r.local_ro[i]:r.local_ro[i + 1]]
            assert np.array_equal(ext_ids[l], g)
        assert np.all(np.diff(r.local_ro[r.n_own:]) == 0)  # halo rows have no edges
        assert r.e_hi - r.e_lo == r.local_ro[-1]
        assert np.all((r.halo_ids < r.lo) | (r.halo_ids >= r.hi)) and np.all(np.diff(r.halo_ids) > 0)
        # what p receives from q is exactly what q sends to p, in the same order
        for q in plans:
            sent = q.send_idx[r.rank] + q.lo
            owner = (r.halo_ids >= q.lo) & (r.halo_ids < q.hi)
            assert np.array_equal(r.halo_ids[owner], sent)
            assert r.recv_counts[q.rank] == sent.shape[0]


def test_exchange_protocol_matches_oracle(orc):
    """Single process, 3 logical ranks, numpy buffers: the halo-in / halo-back
    protocol of HaloAttention with the oracle as the per-rank kernel."""
    from oracle import CSR

    P, H, dh = 3, 2, 4
    ro, co = community_graph(900, 7.0, community=50, seed=4, shuffle=True)
    S = ro.shape[0] - 1
    rng = np.random.default_rng(0)
    q, k, v, up = (rng.standard_normal((S, H * dh)) for _ in range(4))
    bias = rng.normal(0, 0.3, co.shape[0])
    plans = build_halo_plan(ro, co, P)
    out = np.zeros((S, H * dh))
    dq, dk, dv = (np.zeros((S, H * dh)) for _ in range(3))
    db = np.zeros(co.shape[0])
    partial_k, partial_v = {}, {}
    for r in plans:
        ext = np.concatenate([np.arange(r.lo, r.hi), r.halo_ids])
        g = CSR(r.n_ext, r.local_ro, r.local_co)
        qx = np.zeros((r.n_ext, H * dh))
        qx[: r.n_own] = q[r.lo:r.hi]
        kx, vx = k[ext], v[ext]  # halo-in: owners' rows
        upx = np.zeros((r.n_ext, H * dh))
        upx[: r.n_own] = up[r.lo:r.hi]
        b = bias[r.e_lo:r.e_hi]
        gk, gv = np.zeros_like(kx), np.zeros_like(vx)
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            out[r.lo:r.hi, sl] = orc.sparse_fwd(qx[:, sl], kx[:, sl], vx[:, sl], g, b)[: r.n_own]
            a, c, e, f = orc.sparse_bwd(qx[:, sl], kx[:, sl], vx[:, sl], g, b, None, upx[:, sl])
            dq[r.lo:r.hi, sl] = a[: r.n_own]
            gk[:, sl], gv[:, sl] = c, e
            db[r.e_lo:r.e_hi] += f
        dk[r.lo:r.hi] += gk[: r.n_own]
        dv[r.lo:r.hi] += gv[: r.n_own]
        partial_k[r.rank], partial_v[r.rank] = gk[r.n_own:], gv[r.n_own:]
    for r in plans:  # halo-back: add every peer's partials to the owner rows
        for p in plans:
            own = (p.halo_ids >= r.lo) & (p.halo_ids < r.hi)
            rows = p.halo_ids[own]
            assert np.array_equal(rows - r.lo, r.send_idx[p.rank])
            dk[rows] += partial_k[p.rank][own]
            dv[rows] += partial_v[p.rank][own]
    g = CSR(S, ro, co)
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        assert np.abs(out[:, sl] - orc.sparse_fwd(q[:, sl], k[:, sl], v[:, sl], g, bias)).max() < 1e-12
        a, c, e, f = orc.sparse_bwd(q[:, sl], k[:, sl], v[:, sl], g, bias, None, up[:, sl])
        for x, y in ((dq[:, sl], a), (dk[:, sl], c), (dv[:, sl], e)):
            assert np.abs(x - y).max() < 1e-12
        db -= f
    assert np.abs(db).max() < 1e-12


class CpuHaloOps:
    """Test-local kernels for HaloAttention on CPU tensors: the oracle's per-head
    attention on each rank's local plan, numpy-equivalent gather / scatter-add
    (the checker; the product's device ops are tested in test_halo_gpu.py)."""

    def __init__(self, orc, H, dh):
        self.orc, self.H, self.dh, self.g = orc, H, dh, {}

    def setup(self, key, n, ro, co, n_out=None):
        from oracle import CSR

        self.g[key] = CSR(n, ro, co)

    def index(self, idx):
        import torch

        return torch.tensor(idx.astype(np.int64))

    def gather(self, ext, idx, n):
        return ext[idx] if n else ext.new_zeros((1, ext.shape[1]))

    def scatter_add(self, dst, idx, src, n):
        dst[idx] += src

    def _heads(self, x, h):
        return x[:, h * self.dh:(h + 1) * self.dh].numpy()

    def attn_fwd(self, key, q, k, v, b):
        import torch

        o = np.zeros(q.shape)
        for h in range(self.H):
            o[:, h * self.dh:(h + 1) * self.dh] = self.orc.sparse_fwd(
                self._heads(q, h), self._heads(k, h), self._heads(v, h), self.g[key], None if b is None else b.numpy())
        return torch.tensor(o), None

    def attn_bwd(self, key, q, k, v, o, lse, do, b):
        import torch

        dq, dk, dv = (np.zeros(q.shape) for _ in range(3))
        db = np.zeros(self.g[key].nnz)
        for h in range(self.H):
            sl = slice(h * self.dh, (h + 1) * self.dh)
            a, c, e, f = self.orc.sparse_bwd(self._heads(q, h), self._heads(k, h), self._heads(v, h), self.g[key],
                                             None if b is None else b.numpy(), None, self._heads(do, h))
            dq[:, sl], dk[:, sl], dv[:, sl] = a, c, e
            db += f
        return torch.tensor(dq), torch.tensor(dk), torch.tensor(dv), torch.tensor(db)


def _halo_worker(rank, world, port, path):
    import os
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    from oracle import Oracle
    from test_halo_cpu import CpuHaloOps

    from paper_2407_14106_b200.halo import HaloAttention, TorchDistHalo, build_halo_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = np.load(path)
    plans = build_halo_plan(d["ro"], d["co"], world)
    r = plans[rank]
    H, dh = int(d["H"]), int(d["dh"])
    layer = HaloAttention([r], world, H, dh, "f64", TorchDistHalo(rank, world), ops=CpuHaloOps(Oracle(), H, dh))
    t = lambda a: torch.tensor(a[r.lo:r.hi])  # noqa: E731
    out = layer.forward({rank: t(d["q"])}, {rank: t(d["k"])}, {rank: t(d["v"])}, torch.tensor(d["bias"]))
    gq, gk, gv, gb = layer.backward({rank: t(d["up"])})[rank]
    np.savez(path + f".rank{rank}.npz", out=out[rank].numpy(), dq=gq.numpy(), dk=gk.numpy(), dv=gv.numpy(),
             db=gb.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_halo_protocol_matches_oracle(orc, tmp_path, world):
    """HaloAttention with one rank per process over gloo (TorchDistHalo
    all_to_allv), the oracle as the per-rank kernel: assembled outputs and
    gradients equal the oracle's single-process layer."""
    import os

    import torch.multiprocessing as mp

    from oracle import CSR

    H, dh, S = 2, 4, 600
    ro, co = community_graph(S, 7.0, community=40, seed=world, shuffle=True)
    rng = np.random.default_rng(world)
    q, k, v, up = (rng.standard_normal((S, H * dh)) for _ in range(4))
    bias = rng.normal(0, 0.3, co.shape[0])
    path = str(tmp_path / "halo.npz")
    np.savez(path, ro=ro, co=co, q=q, k=k, v=v, up=up, bias=bias, H=H, dh=dh)
    mp.start_processes(_halo_worker, args=(world, 29300 + os.getpid() % 500 + world, path), nprocs=world,
                       start_method="spawn")
    plans = build_halo_plan(ro, co, world)
    g = CSR(S, ro, co)
    got = {n: np.zeros((S, H * dh)) for n in ("out", "dq", "dk", "dv")}
    db = np.zeros(co.shape[0])
    for r in plans:
        x = np.load(path + f".rank{r.rank}.npz")
        for n in got:
            got[n][r.lo:r.hi] = x[n]
        db[r.e_lo:r.e_hi] = x["db"]
    dbw = np.zeros(co.shape[0])
    for h in range(H):
        sl = slice(h * dh, (h + 1) * dh)
        assert np.abs(got["out"][:, sl] - orc.sparse_fwd(q[:, sl], k[:, sl], v[:, sl], g, bias)).max() < 1e-12
        a, b, c, e = orc.sparse_bwd(q[:, sl], k[:, sl], v[:, sl], g, bias, None, up[:, sl])
        for n, w in (("dq", a), ("dk", b), ("dv", c)):
            assert np.abs(got[n][:, sl] - w).max() < 1e-12, n
        dbw += e
    assert np.abs(db - dbw).max() < 1e-12


@pytest.mark.parametrize("P", [2, 3, 8])
def test_interior_boundary_split_partitions_local_csr(P):
    """The overlap's two sub-plans: boundary rows are exactly the own rows with
    a halo column; each sub-CSR keeps its rows' edges in local order and the
    two edge position lists partition the local CSR."""
    ro, co = community_graph(3000, 9.0, community=64, seed=P, shuffle=True)
    for r in build_halo_plan(ro, co, P):
        want_b = np.zeros(r.n_ext, dtype=bool)
        for i in range(r.n_own):
            want_b[i] = np.any(r.local_co[r.local_ro[i]:r.local_ro[i + 1]] >= r.n_own)
        assert np.array_equal(r.boundary, want_b)
        both = np.sort(np.concatenate([r.eidx_i, r.eidx_b]))
        assert np.array_equal(both, np.arange(r.local_co.shape[0]))
        for tag, rows in (("i", ~r.boundary), ("b", r.boundary)):
            sro, sco, ei = getattr(r, "ro_" + tag), getattr(r, "co_" + tag), getattr(r, "eidx_" + tag)
            assert sro.shape[0] == r.n_ext + 1 and sro[-1] == sco.shape[0] == ei.shape[0]
            assert np.array_equal(sco, r.local_co[ei])
            for i in range(r.n_ext):
                n = sro[i + 1] - sro[i]
                assert n == (r.local_ro[i + 1] - r.local_ro[i] if rows[i] else 0)
        assert np.all(r.co_i < r.n_own)  # interior rows never touch the halo


def test_overlapped_protocol_matches_serial(orc):
    """HaloAttention with the interior / boundary split (overlap) against the
    single-plan protocol, 3 logical ranks in one process with the oracle as
    the kernel (f64): outputs, dQ, dK, dV and dbias agree to 1e-12."""
    import torch

    from oracle import Oracle

    from paper_2407_14106_b200.halo import HaloAttention, HaloLoopback

    P, H, dh = 3, 2, 4
    ro, co = community_graph(900, 7.0, community=50, seed=5, shuffle=True)
    S = ro.shape[0] - 1
    rng = np.random.default_rng(1)
    q, k, v, up = (torch.tensor(rng.standard_normal((S, H * dh))) for _ in range(4))
    bias = torch.tensor(rng.normal(0, 0.3, co.shape[0]))
    plans = build_halo_plan(ro, co, P)
    assert all(r.boundary[: r.n_own].any() and (~r.boundary[: r.n_own]).any() for r in plans)
    res = {}
    for overlap in (False, True):
        layer = HaloAttention(plans, P, H, dh, "f64", HaloLoopback(P), ops=CpuHaloOps(Oracle(), H, dh),
                              overlap=overlap)
        sl = lambda t, r: t[r.lo:r.hi].clone()  # noqa: E731
        out = layer.forward({r.rank: sl(q, r) for r in plans}, {r.rank: sl(k, r) for r in plans},
                            {r.rank: sl(v, r) for r in plans}, bias)
        grads = layer.backward({r.rank: sl(up, r) for r in plans})
        res[overlap] = [torch.cat([out[r.rank] for r in plans]).numpy()] + [
            torch.cat([grads[r.rank][j] for r in plans]).numpy() for j in range(4)]
    for a, b in zip(res[False], res[True]):
        assert np.abs(a - b).max() <= 1e-12 * max(1.0, np.abs(a).max())
