"""Device-resident Trainer epochs (reference model.cpp:339-468,
806-883): build_plans, the interleave policy, the tuner-driven beta_thre and
its layout cache, SPD buckets on the GPU, GPH blocks on the device, the
bucket table's gradient, SGD. Each piece is pinned elsewhere (reorder, grid,
layout, buckets, block, tuner); here the integration: the policy and the
cache behave as the reference's, and training on a learnable synthetic task
converges."""
import numpy as np
import pytest

from paper_2407_14106_b200 import control
from paper_2407_14106_b200.datagen import community_graph
from paper_2407_14106_b200.trainer import DeviceTrainer, EpochStats

pytestmark = pytest.mark.gpu


def task(n=1024, seed=3):
    ro, co = community_graph(n, 8.0, community=64, seed=seed)
    comm = np.arange(n) // 64  # planted communities (ids not shuffled)
    rng = np.random.default_rng(seed)
    feats = np.eye(16)[comm % 16] + 0.8 * rng.standard_normal((n, 16))
    return ro, co, feats, comm % 4


def test_reference_policy_and_training(cuda):
    ro, co, x, y = task()
    tr = DeviceTrainer(ro, co, x, y, layers=2, heads=4, hidden=32, ffn=64, dense_period=3, lr=0.1)
    # a sparse community graph fails C2 (2 min degree >= n): every epoch is dense
    assert not tr.flags.all()
    stats = [tr.train_epoch() for _ in range(4)]
    assert all(s.mode == "dense" for s in stats)
    assert [s.reason for s in stats] == [0, 0, 1, 0]  # epoch 3 = the period (interleave.cpp:101-106)
    assert stats[0].pattern_nnz == 1024 * 1024 and not stats[0].layout_cached and stats[1].layout_cached
    # forced cluster-sparse epochs: theta from the tuner, one layout per distinct theta
    cl = [tr.train_epoch("cluster") for _ in range(8)]
    thetas = {round(s.beta_thre, 15) for s in cl}
    built = sum(1 for s in cl if not s.layout_cached)
    assert built == len(thetas)
    assert all(s.dropped_edges >= 0 and s.pattern_nnz > 0 for s in cl)
    losses = [s.loss for s in stats + cl]
    assert np.isfinite(losses).all()
    assert min(losses[-3:]) < losses[0]  # learns the planted task
    # the tuner saw the epoch losses in order (reformation.cpp:240-265)
    t = control.Tuner(tr.beta_g, 1)
    for e, l in enumerate(losses):
        t.update(l, 1.0, e)
    assert t.state()[1] == tr.tuner.state()[1]
    assert EpochStats.CSV.count(",") == cl[0].csv().count(",")


def test_edge_pattern_epochs(cuda):
    ro, co, x, y = task(512, seed=5)
    tr = DeviceTrainer(ro, co, x, y, layers=1, heads=4, hidden=32, ffn=64, strategy="none", lr=0.1)
    s = [tr.train_epoch("edge") for _ in range(3)]
    assert s[0].pattern_nnz == tr.g_exec.nnz() and s[1].layout_cached
