"""One eager Mode H step of the C3 pattern with P = 8 loopback ranks on one
GPU (bf16), for an ncu launch list: which kernels a rank's step is made of.
    ncu --metrics gpu__time_duration.sum --csv python profiles/halo_p8_launches.py
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_14106_b200 import halo as HL  # noqa: E402

info = {}
ro, co = bench.cached_workload("ecr", info)
S, E = ro.shape[0] - 1, co.shape[0]
H, dh, P = 8, 8, int(os.environ.get("P", 8))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
q, k, v, up = (torch.randn((S, H * dh), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
bias = (0.3 * torch.randn(E, generator=g, device=dev)).float()
plans = HL.build_halo_plan(ro, co, P)
layer = HL.HaloAttention(plans, P, H, dh, "bf16", HL.HaloLoopback(P))
sl = lambda t, r: t[r.lo:r.hi]  # noqa: E731
for it in range(3):
    if it == 2:
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("step")
    layer.forward({r.rank: sl(q, r) for r in plans}, {r.rank: sl(k, r) for r in plans},
                  {r.rank: sl(v, r) for r in plans}, bias)
    layer.backward({r.rank: sl(up, r) for r in plans})
    torch.cuda.synchronize()
print("ok")
