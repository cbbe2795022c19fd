"""Golden fixture for the Trainer glue: the compiled
reference's gte::spd_table (graph.cpp:216-262, via oracle/_ref) on a small
planted graph with a global token, a reordered + ECR layout pattern with pad
loops, and the bucket fill restated by oracle/orc_parallel.c
(model.cpp:447-463). Run in the build container (needs /root/reference):

    python tests/golden/make_glue_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import CSR, Oracle, RefOracle  # noqa: E402


def case(ref, orc, with_global, cap, seed):
    n, k = 300, 4
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, 700)
    dst = (src // 30) * 30 + rng.integers(0, 30, 700)  # planted communities of 30
    dst[:40] = rng.integers(0, n, 40)  # a few long-range arcs
    glob = -1
    nn = n
    if with_global:  # global token (model.cpp:349-357)
        glob = n
        nn = n + 1
        src = np.r_[src, np.arange(n), np.full(n, glob)]
        dst = np.r_[dst, np.full(n, glob), np.arange(n)]
    g = ref.add_self_loops(ref.graph_from_edges(nn, src, dst))
    spd = ref.spd_table(g, cap)
    fwd, inv = ref.reorder(g, k, 1)
    gp = ref.permute_graph(g, fwd, inv)
    L = ref.build_layout(g, fwd, inv, k, 1, 5 * orc.density(g), orc.density(g), 4)
    s_pad = g.n + 3  # three pad tokens past the real ones
    pat = orc.extend_with_pad_loops(L.pattern, s_pad)
    inv_pad = np.r_[inv, np.arange(g.n, s_pad)]
    b = orc.pattern_buckets(pat, inv_pad, glob, spd, cap)
    print("pairs", pat.nnz, "bucket histogram", np.bincount(b, minlength=cap + 2))
    return dict(spd_ro=spd[0], spd_cols=spd[1], spd_dist=spd[2], spd_n=spd[3], cap=cap, glob=glob,
                pat_ro=pat.row_off, pat_cols=pat.cols, layout_ro=L.pattern.row_off, layout_cols=L.pattern.cols,
                s_pad=s_pad, inv_pad=inv_pad, buckets=b)


def main():
    ref, orc = RefOracle(), Oracle()
    d = {}
    for ci, (glob, cap, seed) in enumerate(((True, 8, 12), (False, 3, 13), (False, 8, 14))):
        for key, val in case(ref, orc, glob, cap, seed).items():
            d[f"c{ci}_{key}"] = val
    out = os.path.join(ROOT, "tests", "golden", "glue_small.npz")
    np.savez_compressed(out, **d)
    print("wrote", out)


if __name__ == "__main__":
    main()
