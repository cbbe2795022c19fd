"""Measured row-gather ceiling for the sparse kernels (run on the GPU box from
the repo root): profiles/micro/libgather_bw.so gathers, per edge, one 128-byte
K row and one 128-byte V row (bf16, H*dh = 64) with 8 lanes x 16 bytes, 4
edges per slot per step, from two L2-resident 32 MB tables, for three index
streams: sequential rows, the C3 bench pattern in the tile kernels'
community order, and uniform random rows. Reports requested bytes / time
(bench.py's l2_gather quantity) for several grid sizes."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench
from paper_2407_14106_b200.attention import community_order

lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgather_bw.so"))
lib.gather_bw.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int,
                          C.POINTER(C.c_float), C.c_int]
info = {}
ro, co = bench.cached_workload("ecr", info)
ro, co = np.asarray(ro, np.int64), np.asarray(co, np.int64)
S, E = ro.shape[0] - 1, co.shape[0]
order, _ = community_order(ro, co)
deg = np.diff(ro)
starts = np.repeat(ro[order], deg[order])
within = np.arange(E) - np.repeat(np.cumsum(deg[order]) - deg[order], deg[order])
c3 = co[starts + within].astype(np.int32)
rng = np.random.default_rng(0)
streams = {"sequential": (np.arange(E) % S).astype(np.int32), "c3_community_order": c3,
           "uniform_random": rng.integers(0, S, E).astype(np.int32)}
dev = torch.device("cuda", 0)
sink = torch.zeros(4096, dtype=torch.int32, device=dev)
res = {"S": S, "E": E}
for dt, rb in (("bf16", 128), ("f32", 256)):
    td = torch.bfloat16 if dt == "bf16" else torch.float32
    K = torch.randn((S, 64), device=dev).to(td)
    V = torch.randn((S, 64), device=dev).to(td)
    for name, ix in streams.items():
        t = torch.from_numpy(ix).to(dev)
        best = None
        for mult in (4, 8, 16, 32):
            ms = C.c_float()
            rc = lib.gather_bw(K.data_ptr(), V.data_ptr(), t.data_ptr(), E, sink.data_ptr(), 148 * mult, 10,
                               C.byref(ms), rb)
            assert rc == 0, rc
            gbs = E * 2 * rb / (ms.value * 1e-3) / 1e9
            res[f"{dt}_{name}_blocks{148 * mult}_gbs"] = round(gbs, 1)
            best = max(best or 0, gbs)
        res[f"{dt}_{name}_best_gbs"] = round(best, 1)
print(json.dumps(res))
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "gpurun_out", "gather_bw.json")
with open(out, "w") as f:
    json.dump(res, f, indent=1)
