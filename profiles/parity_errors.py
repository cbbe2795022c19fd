"""Measured parity errors (the two per-tensor norms of the parity definition,
BASELINE.md / SURVEY §8(c5)) of the f32 and bf16 sparse paths against the fp64
oracle: C1 (all heads) and the bench's C3 pattern (all heads)."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import bench
from conftest import rel_err, _ensure_oracle
from oracle import CSR, Oracle
from test_sparse_attention_gpu import run_device, oracle_multihead
from paper_2407_14106_b200.datagen import c1_edges, csr_from_pairs

_ensure_oracle()
orc = Oracle()
s, t = c1_edges()
ro1, co1 = csr_from_pairs(4096, s, t)
ro3, co3 = bench.cached_workload("ecr", {})
print("config dtype tensor max_norm_err l2_rel_err")
for name, ro, co, order in (("C1", ro1, co1, None), ("C3", ro3.astype(np.int64), co3.astype(np.int64), "schedule")):
    g = CSR(ro.shape[0] - 1, ro, co)
    for dt in ("f32", "bf16"):
        r = run_device(g.row_off, g.cols, 8, 8, dt, seed=11, order=order)
        want = oracle_multihead(orc, g, r, 8, 8)
        for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
            a, b = rel_err(got, w)
            print(f"{name} {dt} {nm} {a:.3e} {b:.3e}", flush=True)
