"""Golden fixtures for the community-structured graphs (the C3 recipe), made by
the COMPILED REFERENCE (oracle/_ref/libgteref_capi.so -> gte:: in
/root/reference/proj/src). TEST INFRASTRUCTURE: run here, never on the GPU box.

    python tests/golden/make_community_golden.py comm16k   # ~1 min
    python tests/golden/make_community_golden.py comm32k   # reorder ~3 min, layout longer
    python tests/golden/make_community_golden.py c3        # offline: reorder of the bench graph, hours

Each stage writes tests/golden/<name>.npz. The graphs come from
paper_2407_14106_b200.datagen.community_graph (pure numpy, the bench's own
generator, SURVEY.md §8(d2) C3 recipe); reorder(g, k=8, seed=1) is what the
Trainer calls (proj/src/model.cpp:378); build_layout(Elastic, 5*beta_G,
d_b=16) is the bench's ECR layout (proj/src/reformation.cpp:111-195).

The reference's build_layout is run only where it finishes (<= 32K nodes): at
C3 its pack_subblocks rebuilds a 32768 x 32768 coverage field per tile and
scans every origin against every placed tile (reformation.cpp:79-99), i.e.
~1e12-1e13 operations per cell and ~10 GB per field, so the C3 layout is
pinned by the independent sparse-candidate restatement in oracle/
(orc_pack_subblocks_sparse), itself checked against the reference here at
16K/32K and on the random cases of make_golden.py.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import CSR, RefOracle, fnv1a64_fast  # noqa: E402

from paper_2407_14106_b200.datagen import community_graph  # noqa: E402

ARCS = 61859140 / 2449029  # ogbn-products arcs per node
RECIPES = {
    # name: (n, seed, run_layout)
    "comm16k": (16384, 21, True),
    "comm32k": (32768, 22, True),
    "comm64k": (65536, 23, True),
    "c3": (262144, 7, False),  # bench.py make_workload: community_graph(262144, ..., seed=7)
}


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def main(name):
    n, seed, run_layout = RECIPES[name]
    R = RefOracle()
    ro, co = community_graph(n, ARCS, community=256, intra=0.8, sigma=1.0, seed=seed, shuffle=True)
    g = CSR(n, ro.astype(np.int64), co.astype(np.int64))
    d = {"n": np.int64(n), "seed": np.int64(seed), "nnz": np.int64(g.nnz),
         "ro_fnv": np.array(fnv1a64_fast(g.row_off)), "cols_fnv": np.array(fnv1a64_fast(g.cols))}
    out = os.path.join(HERE, f"{name}.npz")
    log(f"{name}: n={n} E={g.nnz}; reference reorder(k=8, seed=1) ...")
    t0 = time.time()
    fwd, inv = R.reorder(g, 8, 1)
    d["reorder_s"] = np.float64(time.time() - t0)
    log(f"reorder done in {d['reorder_s']:.1f} s")
    d["reorder_fwd"] = fwd.astype(np.int32)
    d["reorder_fwd_fnv"] = np.array(fnv1a64_fast(fwd))
    bnd, cn, cd = R.build_cluster_grid(g, fwd, inv, 8)
    d["grid_bnd"], d["grid_nnz"], d["grid_den"] = bnd, cn, cd
    gp = R.permute_graph(g, fwd, inv)
    d["gperm_cols_fnv"] = np.array(fnv1a64_fast(gp.cols))
    np.savez_compressed(out, **d)
    log(f"wrote {out} (reorder + grid)")
    if run_layout:
        bg = g.nnz / (float(n) * float(n))
        t0 = time.time()
        L = R.build_layout(g, fwd, inv, 8, 1, 5 * bg, bg, 16)
        d["layout_s"] = np.float64(time.time() - t0)
        d["L5bg_state"] = L.cell_state
        d["L5bg_boff"] = L.block_off
        d["L5bg_blocks"] = L.blocks
        d["L5bg_dropped"] = np.int64(L.dropped_edges)
        d["L5bg_pnnz"] = np.int64(L.pattern.nnz)
        d["L5bg_pcols_fnv"] = np.array(fnv1a64_fast(L.pattern.cols))
        d["L5bg_pro_fnv"] = np.array(fnv1a64_fast(L.pattern.row_off))
        log(f"layout done in {d['layout_s']:.1f} s: {int(L.block_off[-1])} sub-blocks, dropped {L.dropped_edges}")
        np.savez_compressed(out, **d)
        log(f"wrote {out} (+ layout)")
    print(json.dumps({k: (v.item() if hasattr(v, "item") and np.ndim(v) == 0 else None) for k, v in d.items()
                      if np.ndim(v) == 0}))


def sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def c3_layout():
    """C3 layout from the reference's own C3 permutation (c3.npz): the oracle's
    grid (asserted equal to the reference's grid in c3.npz), permute_graph and
    build_layout with the candidate-origin packer (orc_pack_sparse.cpp — the
    reference's packer cannot run at this size, see the module docstring).
    Large arrays are pinned by sha256 (FNV-1a in Python is too slow here)."""
    from oracle import Oracle

    out = os.path.join(HERE, "c3.npz")
    d = dict(np.load(out))
    n, seed = int(d["n"]), int(d["seed"])
    ro, co = community_graph(n, ARCS, community=256, intra=0.8, sigma=1.0, seed=seed, shuffle=True)
    O = Oracle()
    g = CSR(n, ro.astype(np.int64), co.astype(np.int64))
    fwd = d["reorder_fwd"].astype(np.int64)
    bnd, cn, cd = O.build_cluster_grid(g, fwd, 8)
    assert np.array_equal(cn, d["grid_nnz"]) and np.array_equal(cd, d["grid_den"]), "oracle grid != reference grid"
    gp = O.permute_graph(g, fwd)
    d["gperm_cols_sha"] = np.array(sha(gp.cols))
    bg = g.nnz / (float(n) * float(n))
    O.set_pack_mode(2)
    t0 = time.time()
    L = O.build_layout(8, bnd, cn, cd, gp, 1, 5 * bg, bg, 16)
    d["layout_oracle_s"] = np.float64(time.time() - t0)
    d["L5bg_state"] = L.cell_state
    d["L5bg_boff"] = L.block_off
    d["L5bg_blocks"] = L.blocks
    d["L5bg_dropped"] = np.int64(L.dropped_edges)
    d["L5bg_pnnz"] = np.int64(L.pattern.nnz)
    d["L5bg_pcols_sha"] = np.array(sha(L.pattern.cols))
    d["L5bg_pro_sha"] = np.array(sha(L.pattern.row_off))
    np.savez_compressed(out, **d)
    log(f"c3 layout (oracle, candidate packer) in {d['layout_oracle_s']:.1f} s: {int(L.block_off[-1])} sub-blocks, "
        f"dropped {L.dropped_edges}, pattern nnz {L.pattern.nnz}; wrote {out}")


if __name__ == "__main__":
    if sys.argv[1] == "c3layout":
        c3_layout()
    else:
        main(sys.argv[1])
