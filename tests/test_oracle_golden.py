"""Pins the C restatement (oracle/liboracle.so) against golden fixtures produced
by the compiled reference (tests/golden/make_golden.py) and against the
reference tests' known answers. CPU only."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import CSR, ConfigError, DataError, fnv1a64_fast

from paper_2407_14106_b200.datagen import c1_edges


def csr(d, pre):
    return CSR(int(d[pre + "_n"]), d[pre + "_ro"], d[pre + "_cols"])


# ---------------- C1 ----------------

@pytest.fixture(scope="module")
def c1(orc):
    s, t = c1_edges()
    g = orc.add_self_loops(orc.graph_from_edges(4096, s, t))
    return g


def test_c1_graph_checksums(orc, c1, golden):
    d = golden("c1.npz")
    assert c1.nnz == int(d["nnz"]) == 69497
    assert fnv1a64_fast(c1.row_off) == str(d["ro_fnv"]) == "ff1dfa4d3c69368a"
    assert fnv1a64_fast(c1.cols) == str(d["cols_fnv"]) == "6a9bd13d19ef57ef"
    assert orc.density(c1) == 0.0041423439979553223


def test_c1_reorder_grid_layout(orc, c1, golden):
    d = golden("c1.npz")
    fwd, inv = orc.reorder(c1, 8, 1)
    assert np.array_equal(fwd, d["reorder_fwd"])
    assert fnv1a64_fast(fwd) == "5f380573048daa0b"
    assert list(fwd[:8]) == [3072, 1024, 0, 1536, 512, 1025, 3073, 2560]
    assert np.array_equal(inv[fwd], np.arange(4096))
    bnd, cn, cd = orc.build_cluster_grid(c1, fwd, 8)
    assert np.array_equal(bnd, d["grid_bnd"]) and np.array_equal(cn, d["grid_nnz"])
    assert np.array_equal(cd, d["grid_den"])  # fp64 bit-exact
    assert orc.diagonal_edge_fraction(8, cn) == 0.32631624386664171
    gp = orc.permute_graph(c1, fwd)
    assert fnv1a64_fast(gp.cols) == str(d["gperm_cols_fnv"])
    bg = orc.density(c1)
    for tag, th in (("bg", bg), ("5bg", 5 * bg)):
        L = orc.build_layout(8, bnd, cn, cd, gp, 1, th, bg, 16)
        assert np.array_equal(L.cell_state, d[f"L{tag}_state"])
        assert np.array_equal(L.block_off, d[f"L{tag}_boff"])
        assert np.array_equal(L.blocks, d[f"L{tag}_blocks"])
        assert L.dropped_edges == int(d[f"L{tag}_dropped"])
        assert L.pattern.nnz == int(d[f"L{tag}_pnnz"])
        assert fnv1a64_fast(L.pattern.cols) == str(d[f"L{tag}_pcols_fnv"])
        assert fnv1a64_fast(L.pattern.row_off) == str(d[f"L{tag}_pro_fnv"])
    # SURVEY §8(c6) counts
    L = orc.build_layout(8, bnd, cn, cd, gp, 1, bg, bg, 16)
    assert (int(L.cell_state.sum()), L.blocks.shape[0], L.pattern.nnz, L.dropped_edges) == (55, 208, 77017, 44529)


# ---------------- attention ----------------

def test_attention_small_cases(orc, golden):
    d = golden("attention_small.npz")
    for ci in range(int(d["ncases"])):
        p = f"a{ci}_"
        g = csr(d, p + "g")
        bias = d[p + "bias"] if p + "bias" in d else None
        wm = d[p + "wm"] if p + "wm" in d else None
        out = orc.sparse_fwd(d[p + "q"], d[p + "k"], d[p + "v"], g, bias, wm)
        assert np.abs(out - d[p + "out"]).max() <= 1e-14, ci
        dq, dk, dv, db = orc.sparse_bwd(d[p + "q"], d[p + "k"], d[p + "v"], g, bias, wm, d[p + "up"])
        for got, nm in ((dq, "dq"), (dk, "dk"), (dv, "dv"), (db, "db")):
            assert np.abs(got - d[p + nm]).max() <= 1e-14, (ci, nm)
        if p + "dense_out" in d:
            B = d[p + "dbias_in"]
            o = orc.dense_fwd(d[p + "q"], d[p + "k"], d[p + "v"], B)
            assert np.abs(o - d[p + "dense_out"]).max() <= 1e-14
            gq, gk, gv, gb = orc.dense_bwd(d[p + "q"], d[p + "k"], d[p + "v"], B, None, d[p + "up"])
            for got, nm in ((gq, "dense_dq"), (gk, "dense_dk"), (gv, "dense_dv"), (gb, "dense_db")):
                assert np.abs(got - d[p + nm]).max() <= 1e-14, (ci, nm)


def test_attention_known_answers(orc):
    # reference proj/tests/test_attention.cpp:61-73 — singleton rows copy V
    g = orc.graph_from_edges(2, [0, 1], [1, 1])
    rng = np.random.default_rng(3)
    q, k, v = (rng.standard_normal((2, 3)) for _ in range(3))
    out = orc.sparse_fwd(q, k, v, g, forbid_empty=True)
    assert np.array_equal(out[0], v[1]) and np.array_equal(out[1], v[1])
    # empty-row error (test_attention.cpp:89-94)
    g2 = orc.graph_from_edges(2, [0], [1])
    with pytest.raises(DataError, match="add_self_loops"):
        orc.sparse_fwd(np.zeros((2, 2)), np.zeros((2, 2)), np.zeros((2, 2)), g2, forbid_empty=True)
    # non-finite input (attention.cpp:20-22)
    qn = np.zeros((2, 2))
    qn[0, 0] = np.nan
    with pytest.raises(DataError, match="non-finite Q"):
        orc.sparse_fwd(qn, np.zeros((2, 2)), np.zeros((2, 2)), g)
    # ring S=6 -> 18 pairs (test_attention.cpp:96-120)
    s = np.arange(6)
    ring = orc.add_self_loops(orc.graph_from_edges(6, np.r_[s, (s + 1) % 6], np.r_[(s + 1) % 6, s]))
    assert ring.nnz == 18
    assert orc.density(ring) == 18 / 36


# ---------------- partition ----------------

def test_partition_golden(orc, golden):
    d = golden("partition_small.npz")
    for ci in range(int(d["npcases"])):
        p = f"p{ci}_"
        g = csr(d, p + "g")
        k = int(d[p + "k"])
        fwd, inv = orc.reorder(g, k, int(d[p + "seed"]))
        assert np.array_equal(fwd, d[p + "fwd"]) and np.array_equal(inv, d[p + "inv"]), ci
        bnd, cn, cd = orc.build_cluster_grid(g, fwd, k)
        assert np.array_equal(bnd, d[p + "bnd"]) and np.array_equal(cn, d[p + "cnnz"])
        assert np.array_equal(cd, d[p + "cden"])
        gp = orc.permute_graph(g, fwd)
        assert np.array_equal(gp.cols, d[p + "gp_cols"]) and np.array_equal(gp.row_off, d[p + "gp_ro"])
    fwd, _ = orc.reorder(csr(d, "rand24_g"), 4, 3)
    assert np.array_equal(fwd, d["rand24_fwd"])


def test_partition_known_answers(orc):
    assert list(orc.cluster_boundaries(10, 4)) == [0, 3, 6, 8, 10]
    assert list(orc.cluster_boundaries(8, 2)) == [0, 4, 8]
    g = orc.graph_from_edges(10, [0, 1], [1, 0])
    for bad_k in (3, 16, 0):
        with pytest.raises(ConfigError):
            orc.reorder(g, bad_k, 0)
    path = orc.graph_from_edges(4, [0, 1, 1, 2, 2, 3], [1, 0, 2, 1, 3, 2])
    fwd, inv = orc.reorder(path, 2, 11)
    assert {int(inv[0]), int(inv[1])} in ({0, 1}, {2, 3})
    empty = orc.graph_from_edges(4, [], [])
    _, cn, _ = orc.build_cluster_grid(empty, np.arange(4), 2)
    with pytest.raises(DataError):
        orc.diagonal_edge_fraction(2, cn)


# ---------------- reformation ----------------

def test_pack_and_layout_golden(orc, golden):
    d = golden("reformation_small.npz")
    for ci in range(int(d["nkcases"])):
        p = f"k{ci}_"
        rows, cols, db = (int(x) for x in d[p + "shape"])
        tiles = orc.pack_subblocks(d[p + "er"], d[p + "ec"], rows, cols, db)
        assert np.array_equal(tiles, d[p + "tiles"]), ci
    for ci in range(int(d["nlcases"])):
        p = f"l{ci}_"
        g = csr(d, p + "g")
        k, dbk = (int(x) for x in d[p + "params"])
        thre, bg = (float(x) for x in d[p + "thre"])
        fwd = d[p + "fwd"]
        bnd, cn, cd = orc.build_cluster_grid(g, fwd, k)
        gp = orc.permute_graph(g, fwd)
        for strat in (0, 1):
            sp = f"{p}s{strat}_"
            L = orc.build_layout(k, bnd, cn, cd, gp, strat, thre, bg, dbk)
            assert np.array_equal(L.cell_state, d[sp + "state"]), (ci, strat)
            assert np.array_equal(L.block_off, d[sp + "boff"])
            assert np.array_equal(L.blocks, d[sp + "blocks"])
            assert L.dropped_edges == int(d[sp + "dropped"])
            assert np.array_equal(L.pattern.cols, d[sp + "pat_cols"])
            assert np.array_equal(L.pattern.row_off, d[sp + "pat_ro"])


def test_pack_known_answers(orc):
    # reference proj/tests/test_reformation.cpp:93-117
    t = orc.pack_subblocks([0, 0, 1], [0, 1, 0], 4, 4, 2)
    assert t.tolist() == [[0, 0]]
    full = np.array([(r, c) for r in range(4) for c in range(4)])
    assert orc.pack_subblocks(full[:, 0], full[:, 1], 4, 4, 2).shape[0] == 4
    with pytest.raises(ConfigError):
        orc.pack_subblocks([0], [0], 2, 2, 3)
    assert orc.pack_subblocks([], [], 4, 4, 2).shape[0] == 0


def test_tuner_and_selectors_golden(orc, golden):
    d = golden("reformation_small.npz")
    for ci in range(8):
        p = f"t{ci}_"
        losses, times = d[p + "in"]
        idx, avg, thr = orc.tuner_run(float(d[p + "bg"]), int(d[p + "delta"]), losses, times)
        assert np.array_equal(idx, d[p + "idx"]) and np.array_equal(avg, d[p + "avg"]) and np.array_equal(thr, d[p + "thr"])
    for l2, dd, i, want in d["select_k"]:
        assert orc.select_k(int(l2), int(dd), int(i)) == int(want)
    assert orc.select_db([2, 8, 16, 32, 128], [1.0, 2.0, 2.4, 2.1, 1.2]) == int(d["select_db"][0]) == 16
    assert orc.select_db([16], [1.0]) == int(d["select_db"][1])
    assert orc.select_db([2, 8, 16, 32], [1.0, 2.0, 2.0, 1.5]) == int(d["select_db"][2]) == 16
    assert orc.select_db([1, 2, 4, 8], [3.0] * 4) == int(d["select_db"][3])


# ---------------- parallel / interleave ----------------

def test_parallel_golden(orc, golden):
    d = golden("parallel_interleave_small.npz")
    for ci in range(6):
        S, P, seed = (int(x) for x in d[f"ps{ci}_args"])
        assert np.array_equal(orc.partition_sequence(S, P, seed), d[f"ps{ci}"]), ci
    g = csr(d, "dl_g")
    q, k, v, up = (d["dl_" + n] for n in ("q", "k", "v", "up"))
    for P in (1, 2, 4):
        ids = d[f"dl{P}_ids"]
        out, ledger, macs = orc.dist_fwd(P, ids, q, k, v, g, d["dl_fwd"], d["dl_inv"], 4, d["dl_bias"], d["dl_wm"])
        assert np.abs(out - d[f"dl{P}_out"]).max() <= 1e-14
        assert np.array_equal(ledger, d[f"dl{P}_ledger"]) and macs == int(d[f"dl{P}_macs"])
        gq, gk, gv, gb = orc.dist_bwd(P, ids, q, k, v, g, d["dl_fwd"], d["dl_inv"], 4, d["dl_bias"], d["dl_wm"], up)
        for got, nm in ((gq, "dq"), (gk, "dk"), (gv, "dv"), (gb, "db")):
            assert np.abs(got - d[f"dl{P}_{nm}"]).max() <= 1e-13, (P, nm)
        # 4Sd/P transport contract (test_parallel.cpp:199-203)
        assert all(ledger[w, 0] + ledger[w, 2] == 4 * 16 * 8 // P for w in range(P))


def test_interleave_golden(orc, golden):
    d = golden("parallel_interleave_small.npz")
    for ci, row in enumerate(d["cc"]):
        L = int(row[0])
        r = orc.check_conditions(csr(d, f"cc{ci}_g"), L)
        got = [L, r["c1"], r["c2"], r["c3"], r["sweep_from"], r["sweep_to"], r["diameter_lower_bound"]]
        assert got == [int(x) for x in row], ci


def test_rel_err_helper():
    a = np.array([1.0, 2.0])
    assert rel_err(a, a) == (0.0, 0.0)
