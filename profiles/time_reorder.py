"""Times the product reorder on the bench's C3 graph (S = 262,144, k = 8,
seed 1) and checks its permutation: against the compiled reference's
(tests/golden/c3.npz) when that offline fixture exists, and against the FNV-1a
of the round-1 host implementation's permutation (bit-exact with the
reference at 16K/32K/64K), bcca96b9cf017777."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2407_14106_b200 import partition as P
from paper_2407_14106_b200.attention import Graph
from paper_2407_14106_b200.datagen import community_graph


def fnv(a):
    h = 1469598103934665603
    for b in np.ascontiguousarray(a, "<i8").tobytes():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


ro, co = community_graph(262144, 61859140 / 2449029, community=256, intra=0.8, sigma=1.0, seed=7, shuffle=True)
g = Graph(262144, np.asarray(ro, np.int64), np.asarray(co, np.int64))
small = Graph(64, np.arange(65, dtype=np.int64), np.arange(64, dtype=np.int64))
P.reorder(small, 8, 1)  # CUDA context up before timing
t0 = time.perf_counter()
p = P.reorder(g, 8, 1)
dt = time.perf_counter() - t0
print(f"C3 reorder {dt:.2f} s, fnv {fnv(p.forward)} (round-1 host: bcca96b9cf017777)")
path = os.path.join("tests", "golden", "c3.npz")
if os.path.exists(path):
    print("matches the compiled reference:", np.array_equal(p.forward, np.load(path)["reorder_fwd"].astype(np.int64)))
