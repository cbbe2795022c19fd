"""Mode H on one GPU: the cost of the interior / boundary split.

All P ranks of the C3 bench pattern run in one process on one GPU (loopback
exchange = device copies on the exchange stream), bf16, H = 8, dh = 8. For
each P the whole P-rank fwd+bwd step is timed with CUDA events (min of 5 after
warm-up), with the split + overlap and with one plan per rank, launched
eagerly from Python and replayed as one captured CUDA graph. On
one GPU the exchange and the kernels share the same SMs / HBM, so this
measures what the split costs (two plans, result merges, dK/dV adds), not
what the overlap hides over NVLink.
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_14106_b200 import halo as HL  # noqa: E402

info = {}
ro, co = bench.cached_workload("ecr", info)
S, E = ro.shape[0] - 1, co.shape[0]
H, dh = 8, 8
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
q, k, v, up = (torch.randn((S, H * dh), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
bias = (0.3 * torch.randn(E, generator=g, device=dev)).float()
out = {"S": S, "E": E, "dtype": "bf16", "results": []}
for P in (2, 4, 8):
    plans = HL.build_halo_plan(ro, co, P)
    bnd = [int(r.boundary[: r.n_own].sum()) for r in plans]
    for overlap in (False, True):
        layer = HL.HaloAttention(plans, P, H, dh, "bf16", HL.HaloLoopback(P), overlap=overlap)
        sl = lambda t, r: t[r.lo:r.hi]  # noqa: E731
        inp = ({r.rank: sl(q, r) for r in plans}, {r.rank: sl(k, r) for r in plans},
               {r.rank: sl(v, r) for r in plans})
        dd = {r.rank: sl(up, r) for r in plans}
        def step():
            layer.forward(*inp, bias)
            layer.backward(dd)

        def timed(fn):
            ts = []
            for it in range(8):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if it >= 3:
                    ts.append(e0.elapsed_time(e1))
            return min(ts)

        eager = timed(step)
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            step()
        torch.cuda.current_stream().wait_stream(s_)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        replay = timed(graph.replay)
        out["results"].append({"P": P, "overlap": overlap, "ms_per_step_all_ranks": eager,
                               "graph_ms_per_step_all_ranks": replay,
                               "boundary_rows_per_rank": bnd, "own_rows_per_rank": [r.n_own for r in plans],
                               "halo_rows_per_rank": [r.n_ext - r.n_own for r in plans]})
        print(json.dumps(out["results"][-1]), flush=True)
print(json.dumps(out))
