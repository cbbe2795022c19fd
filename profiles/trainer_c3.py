"""Device Trainer epochs at C3 (S = 262,144, products-shaped community graph,
GPH-slim: 2 blocks, H = 8, dh = 8, ffn 128, cluster-sparse epochs with the
tuner's beta_thre): build_plans time and the per-epoch metrics CSV."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2407_14106_b200.datagen import community_graph
from paper_2407_14106_b200.trainer import DeviceTrainer, EpochStats

n = 262144
ro, co = community_graph(n, 61859140 / 2449029, community=256, intra=0.8, sigma=1.0, seed=7, shuffle=True)
rng = np.random.default_rng(0)
x = rng.standard_normal((n, 32)).astype(np.float32)
y = rng.integers(0, 8, n)
t0 = time.perf_counter()
tr = DeviceTrainer(ro, co, x, y, layers=2, heads=8, hidden=64, ffn=128, lr=0.05)
print(f"build_plans {time.perf_counter() - t0:.2f} s (reorder + grid + permute on the device, k = 8)")
print(EpochStats.CSV)
for e in range(6):
    print(tr.train_epoch("cluster").csv(), flush=True)
