"""ECR sub-blocks on the tensor pipe (csrc/ecr_tile.cuh, north_star
part 3): the dense 16 x 16 sub-blocks of an Elastic layout run as mma.sync
tiles, the rest of the pattern on the sparse kernels, merged as online-softmax
partials (forward) and fixed-order partial sums (backward).

Parity is against the fp64 oracle on the layout's pattern (the reference's
cluster_sparse_attention, reformation.cpp:197-204), bf16 tolerance of
test_sparse_attention_gpu.py; plus split == unsplit within the same bound, the
registration errors, and the bench's own C3 pattern at full size.
"""
import numpy as np
import pytest

from oracle import CSR
from test_sparse_attention_gpu import assert_close, oracle_multihead, run_device

from paper_2407_14106_b200 import attention as A
from paper_2407_14106_b200 import partition as P
from paper_2407_14106_b200._lib import ConfigError
from paper_2407_14106_b200.datagen import community_graph

pytestmark = pytest.mark.gpu


def layout_of(n, deg, community, seed, mult=5.0):
    ro, co = community_graph(n, deg, community=community, seed=seed)
    g = A.Graph(n, np.asarray(ro, np.int64), np.asarray(co, np.int64))
    perm = P.reorder(g, 8, 1)
    grid = P.build_cluster_grid(g, perm, 8)
    gp = P.permute_graph(g, perm)
    bg = P.density(g)
    return P.build_layout(grid, gp, P.ELASTIC, mult * bg, bg, 16)


@pytest.fixture(scope="module")
def lay4k():
    return layout_of(4096, 12.0, 64, 11)


def split_run(L, H, dh, wm=False, seed=3):
    pat = L.pattern
    blocks = L.global_blocks()
    return run_device(pat.row_offsets, pat.cols, H, dh, "bf16", seed=seed, with_wm=wm, blocks=blocks)


@pytest.mark.parametrize("H,dh", [(8, 8), (4, 16), (8, 16), (16, 8)])
@pytest.mark.parametrize("wm", [False, True])
def test_layout_tiles_vs_oracle(cuda, orc, lay4k, H, dh, wm):
    L = lay4k
    assert L.subblock_count() > 0
    r = split_run(L, H, dh, wm)
    assert r["tiles"] == L.subblock_count()
    g = CSR(L.seq_len, L.pattern.row_offsets, L.pattern.cols)
    want = oracle_multihead(orc, g, r, H, dh)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, "bf16", f"ECR H={H} dh={dh} wm={wm} {nm}")


def test_split_equals_unsplit(cuda, lay4k):
    L = lay4k
    pat = L.pattern
    a = run_device(pat.row_offsets, pat.cols, 8, 8, "bf16", seed=5, blocks=L.global_blocks())
    b = run_device(pat.row_offsets, pat.cols, 8, 8, "bf16", seed=5)
    for nm in ("out", "dq", "dk", "dv", "db"):
        assert_close(a[nm], b[nm], "bf16", f"split vs unsplit {nm}")


def test_rows_made_only_of_tiles_and_empty_rows(cuda, orc):
    """A pattern whose tile rows have no other entries, plus empty rows and
    degree-1 rows (exact shortcut, attention.cpp:128-135)."""
    n = 64
    rows = {i: set() for i in range(n)}
    for r0, c0 in ((0, 16), (16, 40), (20, 0)):  # rows 20..31 carry two sub-blocks (disjoint columns)
        for r in range(r0, r0 + 16):
            rows[r].update(range(c0, c0 + 16))
    for i in (40, 41, 50):
        rows[i].add(i)  # degree-1 rows; 42..49, 51.. empty
    ro = np.zeros(n + 1, np.int64)
    co = []
    for i in range(n):
        co += sorted(rows[i])
        ro[i + 1] = len(co)
    co = np.asarray(co, np.int64)
    blocks = np.array([[0, 16], [16, 40], [20, 0]], np.int64)
    r = run_device(ro, co, 8, 8, "bf16", seed=7, blocks=blocks)
    assert r["tiles"] == 3
    want = oracle_multihead(orc, CSR(n, ro, co), r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, "bf16", f"tile-only rows {nm}")
    for i in (40, 41, 50):  # degree-1: out = v exactly, no score gradient
        assert np.array_equal(r["out"][i], r["v"][i])
        assert not r["dq"][i].any()


def test_registration_errors(cuda, lay4k):
    pat = lay4k.pattern
    plan = A.DevicePlan.from_host(pat.row_offsets, pat.cols)
    b = lay4k.global_blocks()
    with pytest.raises(ConfigError, match="overlap"):
        plan.set_blocks(np.concatenate([b[:1], b[:1]]), 16)
    with pytest.raises(ConfigError, match="not inside the pattern"):
        plan.set_blocks(np.array([[b[0, 0], (b[0, 1] + 5) % (lay4k.seq_len - 16)]]), 16)
    with pytest.raises(ConfigError, match="outside"):
        plan.set_blocks(np.array([[lay4k.seq_len - 8, 0]]), 16)
    assert plan.set_blocks(b, 8) == 0  # other d_b: nothing registered
    assert plan.blocks() == (0, pat.nnz())
    assert plan.set_blocks(b, 16) == b.shape[0]
    nb, rem = plan.blocks()
    assert nb == b.shape[0] and rem == pat.nnz() - 256 * nb


def test_c3_bench_pattern_tiles_full_size(cuda, orc):
    """The bench's C3 workload (S = 262,144, E = 6.39M, 5453 sub-blocks) with
    the sub-blocks on the tensor pipe, community order: all heads + dbias."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    info = {}
    ro, co = bench.cached_workload("ecr", info)
    blocks = info["_blocks"]
    assert blocks.shape[0] == 5453
    g = CSR(ro.shape[0] - 1, ro.astype(np.int64), co.astype(np.int64))
    r = run_device(g.row_off, g.cols, 8, 8, "bf16", seed=4, order="schedule", blocks=blocks)
    assert r["tiles"] == 5453
    want = oracle_multihead(orc, g, r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, "bf16", f"C3 ECR {nm}")


def test_f32_with_blocks_registered_keeps_full_pattern(cuda, orc, lay4k):
    """Registered sub-blocks only change bf16 execution; f32 (the 1e-5 parity
    mode) keeps running every pair on the sparse kernels."""
    L = lay4k
    pat = L.pattern
    r = run_device(pat.row_offsets, pat.cols, 8, 8, "f32", seed=9, blocks=L.global_blocks())
    want = oracle_multihead(orc, CSR(L.seq_len, pat.row_offsets, pat.cols), r, 8, 8)
    for got, w, nm in zip((r["out"], r["dq"], r["dk"], r["dv"], r["db"]), want, ("out", "dq", "dk", "dv", "dbias")):
        assert_close(got, w, "f32", f"f32 with blocks {nm}")
