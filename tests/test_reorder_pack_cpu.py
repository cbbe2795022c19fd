"""Bit-exactness of the product's host-side sub-block packer (exact fast
packer in libgte_b200.so) against the golden fixtures of the compiled
reference and against the C oracle. No GPU needed. (The reorder's coarsening
runs on the GPU: tests/test_reorder_gpu.py.)"""
import numpy as np
import pytest

from oracle import CSR

from paper_2407_14106_b200 import partition as P
from paper_2407_14106_b200._lib import ConfigError
from paper_2407_14106_b200.attention import Graph
from paper_2407_14106_b200.datagen import c1_edges, community_graph, csr_from_pairs


def G(ro, co):
    return Graph(len(ro) - 1, np.asarray(ro, np.int64), np.asarray(co, np.int64))


def test_pack_golden(golden):
    d = golden("reformation_small.npz")
    for ci in range(int(d["nkcases"])):
        pre = f"k{ci}_"
        rows, cols, db = (int(x) for x in d[pre + "shape"])
        t = P.pack_subblocks(np.stack([d[pre + "er"], d[pre + "ec"]], 1), rows, cols, db)
        assert np.array_equal(t, d[pre + "tiles"]), ci


def test_pack_matches_oracle_random(orc):
    rng = np.random.default_rng(5)
    for trial in range(60):
        rows, cols = int(rng.integers(4, 90)), int(rng.integers(4, 90))
        db = int(rng.integers(1, min(rows, cols, 9) + 1))
        m = int(rng.integers(1, min(rows * cols, 400) + 1))
        if trial % 3 == 0:  # clustered edges
            cells = rng.choice(min(rows, 20) * min(cols, 20), size=min(m, min(rows, 20) * min(cols, 20)), replace=False)
            er, ec = cells // min(cols, 20), cells % min(cols, 20)
        else:
            cells = rng.choice(rows * cols, size=m, replace=False)
            er, ec = cells // cols, cells % cols
        want = orc.pack_subblocks(er, ec, rows, cols, db)
        got = P.pack_subblocks(np.stack([er, ec], 1), rows, cols, db)
        assert np.array_equal(got, want), (trial, rows, cols, db, m)


def test_pack_known_answers():
    # reference proj/tests/test_reformation.cpp:93-117
    assert P.pack_subblocks([(0, 0), (0, 1), (1, 0)], 4, 4, 2).tolist() == [[0, 0]]
    full = [(r, c) for r in range(4) for c in range(4)]
    assert P.pack_subblocks(full, 4, 4, 2).shape[0] == 4
    with pytest.raises(ConfigError, match="too large"):
        P.pack_subblocks([(0, 0)], 2, 2, 3)
    assert P.pack_subblocks([], 4, 4, 2).shape[0] == 0
