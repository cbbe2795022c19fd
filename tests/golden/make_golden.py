"""Generate the golden fixtures in tests/golden/ from the COMPILED REFERENCE.

Run here (where /root/reference exists) after `make -C oracle ref`:
    python tests/golden/make_golden.py
Every array in the .npz files is an output of the reference's own functions
(oracle/_ref/libgteref_capi.so forwards to gte:: in /root/reference/proj/src),
on inputs drawn by the seeded recipes below. The fixtures pin the C
restatement in oracle/ (tests/test_oracle_golden.py) and travel to the GPU box,
where /root/reference does not exist.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import CSR, RefOracle, fnv1a64_fast  # noqa: E402

from paper_2407_14106_b200.datagen import c1_edges  # noqa: E402


def save(name, d):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **d)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(d)} arrays)")


def csr_arrays(prefix, g: CSR, d):
    d[prefix + "_n"] = np.int64(g.n)
    d[prefix + "_ro"] = g.row_off
    d[prefix + "_cols"] = g.cols


def main():
    R = RefOracle()

    # ---------------- C1 graph: CSR, reorder, grid, layouts ----------------
    d = {}
    s, t = c1_edges()
    g = R.add_self_loops(R.graph_from_edges(4096, s, t))
    d["nnz"] = np.int64(g.nnz)
    d["ro_fnv"] = np.array(fnv1a64_fast(g.row_off))
    d["cols_fnv"] = np.array(fnv1a64_fast(g.cols))
    fwd, inv = R.reorder(g, 8, 1)
    d["reorder_fwd"] = fwd
    bnd, cn, cd = R.build_cluster_grid(g, fwd, inv, 8)
    d["grid_bnd"], d["grid_nnz"], d["grid_den"] = bnd, cn, cd
    gp = R.permute_graph(g, fwd, inv)
    d["gperm_cols_fnv"] = np.array(fnv1a64_fast(gp.cols))
    bg = g.nnz / (4096.0 * 4096.0)
    for tag, th in (("bg", bg), ("5bg", 5 * bg)):
        L = R.build_layout(g, fwd, inv, 8, 1, th, bg, 16)
        d[f"L{tag}_state"] = L.cell_state
        d[f"L{tag}_boff"] = L.block_off
        d[f"L{tag}_blocks"] = L.blocks
        d[f"L{tag}_dropped"] = np.int64(L.dropped_edges)
        d[f"L{tag}_pnnz"] = np.int64(L.pattern.nnz)
        d[f"L{tag}_pcols_fnv"] = np.array(fnv1a64_fast(L.pattern.cols))
        d[f"L{tag}_pro_fnv"] = np.array(fnv1a64_fast(L.pattern.row_off))
    save("c1.npz", d)

    # ---------------- attention: small cases, full arrays ----------------
    d = {}
    rng = np.random.default_rng(2024)
    cases = [(1, 3, 2, 0.5), (2, 3, 3, 0.5), (7, 3, 1, 0.4), (16, 4, 4, 0.3), (33, 8, 8, 0.2), (64, 8, 8, 0.1),
             (40, 5, 3, 0.15), (48, 16, 16, 0.2)]
    for ci, (S, dk, dv, p) in enumerate(cases):
        g = R.random_graph(S, p, 100 + ci, loops=(ci % 3 != 2))  # some cases keep empty rows
        q, k = rng.standard_normal((S, dk)), rng.standard_normal((S, dk))
        v, up = rng.standard_normal((S, dv)), rng.standard_normal((S, dv))
        bias = rng.normal(0, 0.5, g.nnz) if ci % 2 == 0 else None
        wm = ((rng.random(g.nnz) < 0.7) / 0.7) if ci % 4 == 0 else None
        out = R.sparse_fwd(q, k, v, g, bias, wm)
        dq, dk_, dv_, db = R.sparse_bwd(q, k, v, g, bias, wm, up)
        pre = f"a{ci}_"
        csr_arrays(pre + "g", g, d)
        for nm, arr in (("q", q), ("k", k), ("v", v), ("up", up), ("out", out), ("dq", dq), ("dk", dk_), ("dv", dv_),
                        ("db", db)):
            d[pre + nm] = arr
        if bias is not None:
            d[pre + "bias"] = bias
        if wm is not None:
            d[pre + "wm"] = wm
        if S <= 16:
            B = rng.normal(0, 0.3, (S, S))
            d[pre + "dbias_in"] = B
            d[pre + "dense_out"] = R.dense_fwd(q, k, v, B)
            gq, gk, gv, gb = R.dense_bwd(q, k, v, B, None, up)
            d[pre + "dense_dq"], d[pre + "dense_dk"], d[pre + "dense_dv"], d[pre + "dense_db"] = gq, gk, gv, gb
    d["ncases"] = np.int64(len(cases))
    save("attention_small.npz", d)

    # ---------------- partition: SBM + path graphs ----------------
    d = {}
    pcases = [(16, 2, 0.9, 0.05, 3, 4, 1), (32, 4, 0.6, 0.05, 7, 4, 1), (40, 2, 0.5, 0.01, 42, 2, 5),
              (60, 4, 0.4, 0.02, 9, 4, 17), (160, 8, 0.3, 0.005, 1, 8, 1), (160, 8, 0.3, 0.005, 4, 8, 21),
              (300, 6, 0.1, 0.01, 11, 8, 3), (12, 2, 0.7, 0.1, 3, 2, 13)]
    for ci, (n, b, pin, pout, seed, k, rseed) in enumerate(pcases):
        g, labels = R.generate_sbm(n, b, pin, pout, seed)
        if ci % 2 == 0:
            g = R.add_self_loops(g)
        fwd, inv = R.reorder(g, k, rseed)
        bnd, cn, cd = R.build_cluster_grid(g, fwd, inv, k)
        gp = R.permute_graph(g, fwd, inv)
        pre = f"p{ci}_"
        csr_arrays(pre + "g", g, d)
        d[pre + "k"], d[pre + "seed"] = np.int64(k), np.uint64(rseed)
        d[pre + "fwd"], d[pre + "inv"] = fwd, inv
        d[pre + "bnd"], d[pre + "cnnz"], d[pre + "cden"] = bnd, cn, cd
        csr_arrays(pre + "gp", gp, d)
    rg = R.random_graph(24, 0.2, 7, True)
    fwd, inv = R.reorder(rg, 4, 3)
    csr_arrays("rand24_g", rg, d)
    d["rand24_fwd"] = fwd
    d["npcases"] = np.int64(len(pcases))
    save("partition_small.npz", d)

    # ---------------- reformation: packing + layouts + tuner ----------------
    d = {}
    rng = np.random.default_rng(77)
    for ci in range(24):
        rows = 3 + ci % 5
        cols = 3 + (ci // 5) % 5
        db = 1 + ci % 3
        db = min(db, rows, cols)
        m = 1 + (ci * 7) % (rows * cols)
        cells = rng.choice(rows * cols, size=m, replace=False)
        er, ec = cells // cols, cells % cols
        tiles = R.pack_subblocks(er, ec, rows, cols, db)
        pre = f"k{ci}_"
        d[pre + "shape"] = np.array([rows, cols, db], dtype=np.int64)
        d[pre + "er"], d[pre + "ec"], d[pre + "tiles"] = er.astype(np.int64), ec.astype(np.int64), tiles
    lcases = [(32, 4, 0.6, 0.05, 7, 4, 1, 2, 0.5), (64, 4, 0.5, 0.02, 3, 4, 2, 4, 0.05), (96, 8, 0.4, 0.01, 5, 8, 3, 2, 0.02),
              (128, 4, 0.3, 0.01, 9, 4, 4, 4, 0.03), (200, 8, 0.25, 0.004, 2, 8, 5, 3, 0.01)]
    for ci, (n, b, pin, pout, seed, k, rseed, dbk, thre) in enumerate(lcases):
        g, _ = R.generate_sbm(n, b, pin, pout, seed)
        g = R.add_self_loops(g)
        fwd, inv = R.reorder(g, k, rseed)
        bg = g.nnz / float(n * n)
        pre = f"l{ci}_"
        csr_arrays(pre + "g", g, d)
        d[pre + "params"] = np.array([k, dbk], dtype=np.int64)
        d[pre + "thre"] = np.array([thre, bg])
        d[pre + "fwd"], d[pre + "inv"] = fwd, inv
        for strat in (0, 1):
            L = R.build_layout(g, fwd, inv, k, strat, thre, bg, dbk)
            sp = f"{pre}s{strat}_"
            d[sp + "state"], d[sp + "boff"], d[sp + "blocks"] = L.cell_state, L.block_off, L.blocks
            d[sp + "dropped"] = np.int64(L.dropped_edges)
            csr_arrays(sp + "pat", L.pattern, d)
    for ci in range(8):
        rng2 = np.random.default_rng(500 + ci)
        n = 60
        losses = np.maximum(0.01, np.cumsum(rng2.uniform(-0.2, 0.18, n)) + 2.0)
        times = rng2.uniform(0.5, 2.0, n)
        bg = 0.01 + 0.02 * ci
        delta = 3 if ci % 2 == 0 else 10
        idx, avg, thr = R.tuner_run(bg, delta, losses, times)
        pre = f"t{ci}_"
        d[pre + "in"] = np.stack([losses, times])
        d[pre + "bg"], d[pre + "delta"] = np.float64(bg), np.int64(delta)
        d[pre + "idx"], d[pre + "avg"], d[pre + "thr"] = idx, avg, thr
    d["select_k"] = np.array([[6291456, 64, 1536, R.select_k(6291456, 64, 1536)], [64, 64, 1, R.select_k(64, 64, 1)],
                              [6291456, 64, 100, R.select_k(6291456, 64, 100)],
                              [126 * 2 ** 20, 64, 1536, R.select_k(126 * 2 ** 20, 64, 1536)]], dtype=np.int64)
    d["select_db"] = np.array([R.select_db([2, 8, 16, 32, 128], [1.0, 2.0, 2.4, 2.1, 1.2]),
                               R.select_db([16], [1.0]), R.select_db([2, 8, 16, 32], [1.0, 2.0, 2.0, 1.5]),
                               R.select_db([1, 2, 4, 8], [3.0, 3.0, 3.0, 3.0])], dtype=np.int64)
    d["nkcases"], d["nlcases"] = np.int64(24), np.int64(len(lcases))
    save("reformation_small.npz", d)

    # ---------------- parallel + interleave ----------------
    d = {}
    for ci, (S, P, seed) in enumerate([(8, 2, 1), (7, 2, 1), (5, 1, 9), (16, 4, 104), (1000, 8, 3), (4097, 8, 11)]):
        d[f"ps{ci}"] = R.partition_sequence(S, P, seed)
        d[f"ps{ci}_args"] = np.array([S, P, seed], dtype=np.int64)
    rng = np.random.default_rng(31)
    S, dmod, H = 16, 8, 4
    q, k, v, up = (rng.standard_normal((S, dmod)) for _ in range(4))
    g = R.random_graph(S, 0.3, 5, True)
    fwd, inv = R.reorder(g, 4, 3)
    bias = rng.normal(0, 0.2, g.nnz)
    wm = (rng.random(H * g.nnz) < 0.8) / 0.8
    csr_arrays("dl_g", g, d)
    for nm, arr in (("q", q), ("k", k), ("v", v), ("up", up), ("fwd", fwd), ("inv", inv), ("bias", bias), ("wm", wm)):
        d["dl_" + nm] = arr
    for P in (1, 2, 4):
        ids = R.partition_sequence(S, P, 100 + P)
        out, ledger, macs = R.dist_fwd(P, ids, q, k, v, g, fwd, inv, H, bias, wm)
        gq, gk, gv, gb = R.dist_bwd(P, ids, q, k, v, g, fwd, inv, H, bias, wm, up)
        d[f"dl{P}_ids"], d[f"dl{P}_out"], d[f"dl{P}_ledger"], d[f"dl{P}_macs"] = ids, out, ledger, np.int64(macs)
        d[f"dl{P}_dq"], d[f"dl{P}_dk"], d[f"dl{P}_dv"], d[f"dl{P}_db"] = gq, gk, gv, gb
    conds = []
    for ci, (n, p, seed, loops, L) in enumerate([(8, 0.9, 1, True, 2), (30, 0.1, 2, True, 3), (12, 0.6, 3, False, 1),
                                                 (20, 0.3, 4, True, 5), (6, 0.0, 5, True, 2)]):
        g = R.random_graph(n, p, seed, loops)
        r = R.check_conditions(g, L)
        csr_arrays(f"cc{ci}_g", g, d)
        conds.append([L, r["c1"], r["c2"], r["c3"], r["sweep_from"], r["sweep_to"], r["diameter_lower_bound"]])
    d["cc"] = np.array(conds, dtype=np.int64)
    save("parallel_interleave_small.npz", d)


if __name__ == "__main__":
    main()
