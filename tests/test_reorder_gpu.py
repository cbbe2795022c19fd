"""Bit-exactness of the product reorder (csrc/bisection.cpp host greedy passes
+ csrc/partition_gpu.cu device coarsening/splitting) against the golden
fixtures of the compiled reference and against the C oracle (reference
proj/src/partition.cpp:413-433)."""
import numpy as np
import pytest

from oracle import CSR

from paper_2407_14106_b200 import partition as P
from paper_2407_14106_b200._lib import ConfigError
from paper_2407_14106_b200.attention import Graph
from paper_2407_14106_b200.datagen import c1_edges, community_graph, csr_from_pairs

pytestmark = pytest.mark.gpu


def G(ro, co):
    return Graph(len(ro) - 1, np.asarray(ro, np.int64), np.asarray(co, np.int64))


def test_reorder_c1_golden(golden):
    d = golden("c1.npz")
    s, t = c1_edges()
    ro, co = csr_from_pairs(4096, s, t)
    p = P.reorder(G(ro, co), 8, 1)
    assert np.array_equal(p.forward, d["reorder_fwd"])
    assert p.valid()


def test_reorder_golden_cases(golden):
    d = golden("partition_small.npz")
    for ci in range(int(d["npcases"])):
        pre = f"p{ci}_"
        g = G(d[pre + "g_ro"], d[pre + "g_cols"])
        p = P.reorder(g, int(d[pre + "k"]), int(d[pre + "seed"]))
        assert np.array_equal(p.forward, d[pre + "fwd"]), ci
        assert np.array_equal(p.inverse, d[pre + "inv"]), ci
    p = P.reorder(G(d["rand24_g_ro"], d["rand24_g_cols"]), 4, 3)
    assert np.array_equal(p.forward, d["rand24_fwd"])


@pytest.mark.parametrize("n,deg,comm,seed,k", [(3000, 8.0, 64, 1, 8), (2048, 14.0, 128, 2, 4), (5000, 5.0, 32, 3, 16),
                                               (1500, 30.0, 256, 4, 2)])
def test_reorder_matches_oracle(orc, n, deg, comm, seed, k):
    ro, co = community_graph(n, deg, community=comm, seed=seed)
    for rseed in (1, 12345678901234567):
        want_f, want_i = orc.reorder(CSR(n, ro, co), k, rseed)
        p = P.reorder(G(ro, co), k, rseed)
        assert np.array_equal(p.forward, want_f) and np.array_equal(p.inverse, want_i), (n, rseed)


def test_reorder_disconnected_and_tiny(orc):
    # isolated nodes, a star, a path and directed arcs only one way
    src = [0, 0, 0, 0, 5, 6, 7, 20, 21]
    dst = [1, 2, 3, 4, 6, 7, 8, 21, 22]
    ro, co = csr_from_pairs(30, np.array(src), np.array(dst), self_loops=False)
    for k in (1, 2, 4, 8, 16):
        want_f, _ = orc.reorder(CSR(30, ro, co), k, 99)
        assert np.array_equal(P.reorder(G(ro, co), k, 99).forward, want_f), k
    with pytest.raises(ConfigError, match="power of two"):
        P.reorder(G(ro, co), 3, 0)
    with pytest.raises(ConfigError, match="exceeds node count"):
        P.reorder(G(ro, co), 32, 0)
