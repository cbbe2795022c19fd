"""Bit-exact parity of the GPU graph/CSR builders, cluster grid and ECR layout
against the compiled reference's golden fixtures and the C oracle."""
import numpy as np
import pytest

from oracle import CSR, DataError as OrcDataError

from paper_2407_14106_b200 import attention as A
from paper_2407_14106_b200 import partition as P
from paper_2407_14106_b200._lib import ConfigError, DataError
from paper_2407_14106_b200.attention import Graph
from paper_2407_14106_b200.datagen import c1_edges, community_graph, csr_from_pairs

pytestmark = pytest.mark.gpu


def G(ro, co):
    return Graph(len(ro) - 1, np.asarray(ro, np.int64), np.asarray(co, np.int64))


def same(g: Graph, o: CSR):
    return np.array_equal(g.row_offsets, o.row_off) and np.array_equal(g.col_indices, o.cols)


def test_graph_from_edges_and_loops(cuda, orc):
    rng = np.random.default_rng(0)
    for n, m in ((1, 0), (5, 12), (300, 5000), (40000, 300000)):
        s = rng.integers(0, n, m)
        d = rng.integers(0, n, m)
        got = P.graph_from_edges(n, s, d)
        want = orc.graph_from_edges(n, s, d)
        assert same(got, want), (n, m)
        loops = P.add_self_loops(got)
        assert same(loops, orc.add_self_loops(want))
        assert same(P.add_self_loops(loops), orc.add_self_loops(want))  # idempotent (graph.cpp:127-149)
    with pytest.raises(DataError, match=r"node id 7 out of range \[0, 5\)"):
        P.graph_from_edges(5, [0, 1, 7], [1, 2, 0])
    with pytest.raises(OrcDataError, match=r"node id 7 out of range"):
        orc.graph_from_edges(5, [0, 1, 7], [1, 2, 0])


def test_c1_pipeline_golden(cuda, golden):
    d = golden("c1.npz")
    s, t = c1_edges()
    g = P.add_self_loops(P.graph_from_edges(4096, s, t))
    assert g.nnz() == 69497
    perm = P.reorder(g, 8, 1)
    assert np.array_equal(perm.forward, d["reorder_fwd"])
    grid = P.build_cluster_grid(g, perm, 8)
    assert np.array_equal(grid.boundaries, d["grid_bnd"]) and np.array_equal(grid.cell_nnz, d["grid_nnz"])
    assert np.array_equal(grid.cell_density, d["grid_den"])
    assert P.diagonal_edge_fraction(grid) == 0.32631624386664171
    gp = P.permute_graph(g, perm)
    from oracle import fnv1a64_fast

    assert fnv1a64_fast(gp.col_indices) == str(d["gperm_cols_fnv"])
    bg = P.density(g)
    for tag, th in (("bg", bg), ("5bg", 5 * bg)):
        L = P.build_layout(grid, gp, P.ELASTIC, th, bg, 16)
        assert np.array_equal(L.cell_state, d[f"L{tag}_state"])
        assert np.array_equal(L.block_off, d[f"L{tag}_boff"])
        assert np.array_equal(L.blocks, d[f"L{tag}_blocks"])
        assert L.dropped_edges == int(d[f"L{tag}_dropped"])
        assert L.pattern.nnz() == int(d[f"L{tag}_pnnz"])
        assert fnv1a64_fast(L.pattern.cols) == str(d[f"L{tag}_pcols_fnv"])
        assert fnv1a64_fast(L.pattern.row_offsets) == str(d[f"L{tag}_pro_fnv"])


def test_layout_golden_cases(cuda, golden):
    d = golden("reformation_small.npz")
    for ci in range(int(d["nlcases"])):
        pre = f"l{ci}_"
        g = G(d[pre + "g_ro"], d[pre + "g_cols"])
        k, dbk = (int(x) for x in d[pre + "params"])
        thre, bg = (float(x) for x in d[pre + "thre"])
        perm = P.Permutation(d[pre + "fwd"], d[pre + "inv"])
        grid = P.build_cluster_grid(g, perm, k)
        gp = P.permute_graph(g, perm)
        for strat in (0, 1):
            sp = f"{pre}s{strat}_"
            L = P.build_layout(grid, gp, strat, thre, bg, dbk)
            assert np.array_equal(L.cell_state, d[sp + "state"]), (ci, strat)
            assert np.array_equal(L.block_off, d[sp + "boff"])
            assert np.array_equal(L.blocks, d[sp + "blocks"])
            assert L.dropped_edges == int(d[sp + "dropped"])
            assert np.array_equal(L.pattern.cols, d[sp + "pat_cols"])
            assert np.array_equal(L.pattern.row_offsets, d[sp + "pat_ro"])


@pytest.mark.parametrize("n,k,db,mult", [(8192, 8, 16, 5.0), (3000, 4, 8, 1.0), (2000, 8, 4, 3.0)])
def test_community_pipeline_vs_oracle(cuda, orc, n, k, db, mult):
    ro, co = community_graph(n, 12.0, community=128, seed=n)
    g = G(ro, co)
    perm = P.reorder(g, k, 3)
    ofwd, _ = orc.reorder(CSR(n, ro, co), k, 3)
    assert np.array_equal(perm.forward, ofwd)
    grid = P.build_cluster_grid(g, perm, k)
    obnd, onnz, oden = orc.build_cluster_grid(CSR(n, ro, co), ofwd, k)
    assert np.array_equal(grid.cell_nnz, onnz) and np.array_equal(grid.cell_density, oden)
    gp = P.permute_graph(g, perm)
    ogp = orc.permute_graph(CSR(n, ro, co), ofwd)
    assert same(gp, ogp)
    bg = P.density(g)
    L = P.build_layout(grid, gp, P.ELASTIC, mult * bg, bg, db)
    OL = orc.build_layout(k, obnd, onnz, oden, ogp, 1, mult * bg, bg, db)
    assert np.array_equal(L.cell_state, OL.cell_state)
    assert np.array_equal(L.blocks, OL.blocks) and L.dropped_edges == OL.dropped_edges
    assert np.array_equal(L.pattern.row_offsets, OL.pattern.row_off)
    assert np.array_equal(L.pattern.cols, OL.pattern.cols)


def test_cluster_sparse_attention_on_layout(cuda, orc):
    # attention over an ECR layout pattern (reformation.cpp:197-204), empty rows allowed
    n = 4096
    ro, co = community_graph(n, 10.0, community=64, seed=11)
    g = G(ro, co)
    perm = P.reorder(g, 8, 1)
    grid = P.build_cluster_grid(g, perm, 8)
    gp = P.permute_graph(g, perm)
    bg = P.density(g)
    L = P.build_layout(grid, gp, P.ELASTIC, 5 * bg, bg, 16)
    pat = L.pattern
    rng = np.random.default_rng(1)
    q, k, v, up = (rng.standard_normal((n, 8)).astype(np.float32).astype(np.float64) for _ in range(4))
    bias = rng.normal(0, 0.3, pat.nnz()).astype(np.float32).astype(np.float64)
    want = orc.sparse_fwd(q, k, v, CSR(n, pat.row_offsets, pat.cols), bias)
    got = A.sparse_attention(q, k, v, pat, bias, dtype="f32").output
    e = np.abs(got - want).max() / np.abs(want).max()
    assert e <= 1e-5, e
    gq, gk, gv, gb = orc.sparse_bwd(q, k, v, CSR(n, pat.row_offsets, pat.cols), bias, None, up)
    gr = A.sparse_attention_backward(q, k, v, pat, bias, None, up, dtype="f32")
    for a, b in ((gr.dq, gq), (gr.dk, gk), (gr.dv, gv), (gr.dbias, gb)):
        assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()


def test_errors(cuda):
    g = G(*csr_from_pairs(16, np.arange(15), np.arange(1, 16)))
    with pytest.raises(ConfigError, match="invalid k"):
        P.build_cluster_grid(g, None, 17)
    with pytest.raises(ConfigError, match="permutation"):
        P.permute_graph(g, P.Permutation(np.zeros(16, np.int64), np.zeros(16, np.int64)))
    grid = P.build_cluster_grid(g, None, 4)
    with pytest.raises(ConfigError, match="too large"):
        P.build_layout(grid, g, P.ELASTIC, 1.0, 0.1, 5)
