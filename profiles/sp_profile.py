"""Where the time of the N = 1 sequence-parallel step goes: host wall time
per step phase (synchronised) and a cProfile of the step."""
import cProfile, os, pstats, sys, time
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29591")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch.distributed as dist
import bench
from paper_2407_14106_b200 import attention as A, parallel as SP, halo as HL

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0), rank=0, world_size=1)
info = {}
ro, co = bench.cached_workload("ecr", info)
S, E = ro.shape[0] - 1, co.shape[0]
ctx = A.Context.get(0)
hp = HL.build_halo_plan(ro, co, 1)
ex = SP.NcclExchange(None, 0, 1, ctx=ctx)
layer = HL.HaloAttention([hp[0]], 1, 8, 8, "bf16", HL.HaloNccl(ex, 0, ctx), ctx)
q, k, v, do = (torch.randn((S, 64), device="cuda").to(torch.bfloat16) for _ in range(4))
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
def step():
    layer.forward({0: q}, {0: k}, {0: v})
    return layer.backward({0: do})
for _ in range(3): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"enqueue {1e3*(t1-t0)/10:.3f} ms/step, enqueue+drain {1e3*(t2-t0)/10:.3f} ms/step")
flush = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.float32, device="cuda")
stream = torch.cuda.current_stream()
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(10)]
torch.cuda.synchronize()
for i in range(10):
    flush.zero_()
    evs[i][0].record(stream)
    step()
    evs[i][1].record(stream)
torch.cuda.synchronize()
print("event ms per step (with L2 flush):", [round(a.elapsed_time(b), 3) for a, b in evs])
pr = cProfile.Profile(); pr.enable()
for _ in range(5): step()
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
ex.close(); dist.destroy_process_group()
