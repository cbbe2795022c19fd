"""SPD buckets on the GPU (reference spd_table, graph.cpp:208-261,
and the Trainer's bucket rule, model.cpp:447-463), without the reference's
N <= 20000 guard.

Pinned to the compiled reference: tests/golden/glue_small.npz holds
gte::spd_table of three planted graphs (caps 8, 3, 8; one with a global token)
and the bucket fill of reordered + ECR layout patterns over them."""
import numpy as np
import pytest

from paper_2407_14106_b200 import glue
from paper_2407_14106_b200 import partition as P

pytestmark = pytest.mark.gpu
CASES = (0, 1, 2)
SEEDS = {0: (True, 8, 12), 1: (False, 3, 13), 2: (False, 8, 14)}


def _case(golden, ci):
    d = golden("glue_small.npz")
    return {k[len(f"c{ci}_"):]: d[k] for k in d.files if k.startswith(f"c{ci}_")}


def graph_of(ci):
    """tests/golden/make_glue_golden.py case(): the same planted graph, built by
    the product's graph_from_edges + add_self_loops (bit-exact with the
    reference's, tests/test_graph_layout_gpu.py)."""
    with_global, cap, seed = SEEDS[ci]
    n = 300
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, 700)
    dst = (src // 30) * 30 + rng.integers(0, 30, 700)
    dst[:40] = rng.integers(0, n, 40)
    nn = n
    if with_global:
        glob = n
        nn = n + 1
        src = np.r_[src, np.arange(n), np.full(n, glob)]
        dst = np.r_[dst, np.full(n, glob), np.arange(n)]
    g = P.add_self_loops(P.graph_from_edges(nn, src, dst))
    return np.asarray(g.row_offsets, np.int64), np.asarray(g.col_indices, np.int64), cap


@pytest.mark.parametrize("ci", CASES)
def test_spd_table_matches_reference(cuda, golden, ci):
    c = _case(golden, ci)
    ro, co, cap = graph_of(ci)
    sro, sco, sdi, n = glue.spd_table(ro, co, cap)
    assert n == int(c["spd_n"])
    assert np.array_equal(sro, c["spd_ro"]) and np.array_equal(sco, c["spd_cols"])
    assert np.array_equal(sdi, c["spd_dist"])


def _lookup(c, i, j):
    sro, scol, sdist = c["spd_ro"], c["spd_cols"], c["spd_dist"]
    row = scol[sro[i]:sro[i + 1]]
    p = np.searchsorted(row, j)
    return int(sdist[sro[i] + p]) if p < row.shape[0] and row[p] == j else int(c["cap"]) + 1


@pytest.mark.parametrize("ci", CASES)
@pytest.mark.parametrize("cap", [None, 1, 2, 4, 5])
def test_spd_pairs_all_pairs(cuda, golden, ci, cap):
    """Every ordered pair: the table-free resolver (radius-2 balls, meet in the
    middle, early-exit BFS) == SpdTable::lookup, at the golden cap and at caps
    around the meet-in-the-middle limits (lookups recomputed from the cap-8
    table for the other caps)."""
    c = _case(golden, ci)
    ro, co, gcap = graph_of(ci)
    n = ro.shape[0] - 1
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i, j = i.ravel(), j.ravel()
    k = gcap if cap is None else cap
    got = glue.spd_pairs(ro, co, k, i, j)
    if cap is None:
        want = np.array([_lookup(c, a, b) for a, b in zip(i, j)], np.int32)
    else:
        full = glue.spd_table(ro, co, 255)
        cc = {"spd_ro": full[0], "spd_cols": full[1], "spd_dist": full[2], "cap": 255}
        d = np.array([_lookup(cc, a, b) for a, b in zip(i, j)], np.int32)
        want = np.where(d > k, k + 1, d).astype(np.int32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("ci", CASES)
def test_pattern_buckets_from_graph(cuda, golden, ci):
    """The Trainer's per-pair buckets with the SPD taken from the graph on the
    device == the golden fill from the reference's table."""
    c = _case(golden, ci)
    ro, co, cap = graph_of(ci)
    b = glue.pattern_buckets_graph(c["pat_ro"], c["pat_cols"], c["inv_pad"], int(c["glob"]), ro, co, cap)
    assert np.array_equal(b.cpu().numpy(), c["buckets"])


def test_spd_errors(cuda):
    from paper_2407_14106_b200._lib import ConfigError

    ro, co, _ = graph_of(1)
    with pytest.raises(ConfigError, match="max_dist"):
        glue.spd_table(ro, co, -1)


def test_c3_pattern_buckets_sampled(cuda):
    """C3 (S = 262,144, the bench's ECR pattern in reordered coordinates, cap 8,
    far beyond the reference's 20,000-node guard): the buckets of 64 sampled
    rows == a host BFS over the original graph (scipy)."""
    import os
    import sys

    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2407_14106_b200.datagen import community_graph

    info = {}
    pro, pco = bench.cached_workload("ecr", info)
    fwd = np.asarray(info["_perm_forward"], np.int64)
    inv = np.empty_like(fwd)
    inv[fwd] = np.arange(fwd.shape[0])
    ro, co = community_graph(262144, 61859140 / 2449029, community=256, intra=0.8, sigma=1.0, seed=7, shuffle=True)
    g = P.add_self_loops(P.Graph(262144, np.asarray(ro, np.int64), np.asarray(co, np.int64)))
    gro, gco = np.asarray(g.row_offsets), np.asarray(g.col_indices)
    b = glue.pattern_buckets_graph(pro, pco, inv, -1, gro, gco, 8).cpu().numpy()
    n = 262144
    A = sp.csr_matrix((np.ones(gco.shape[0]), gco, gro), shape=(n, n))
    A = ((A + A.T) > 0).astype(np.int8)
    rows = np.random.default_rng(0).choice(n, 64, replace=False)
    D = cg.shortest_path(A, unweighted=True, indices=inv[rows])
    for k, r in enumerate(rows):
        cols = pco[pro[r]:pro[r + 1]]
        d = D[k, inv[cols]]
        want = np.where(np.isfinite(d) & (d <= 8), d, 9).astype(np.int32)
        want[inv[cols] == inv[r]] = 0
        assert np.array_equal(b[pro[r]:pro[r + 1]], want), r
