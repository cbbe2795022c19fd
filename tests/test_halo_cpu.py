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
