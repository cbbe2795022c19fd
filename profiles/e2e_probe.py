"""Where the end-to-end step (host buffers through the C ABI) loses time
against the PCIe bound: copy-only pipelines with torch streams vs the API's
asynchronous fwd_bwd_host steps, same bytes (run on the GPU box)."""
import json, sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2407_14106_b200 import attention as A

info = {}
ro, co = bench.cached_workload("ecr", info)
S, E = ro.shape[0] - 1, co.shape[0]
H, DH = bench.H, bench.DH
dev = torch.device("cuda", 0)
td = torch.bfloat16
res = {}
g = torch.Generator(device=dev).manual_seed(1)
q, k, v, do = (torch.randn((S, H * DH), generator=g, device=dev).to(td) for _ in range(4))
bias = (0.3 * torch.randn(E, generator=g, device=dev)).float()
pin = lambda x: x.cpu().pin_memory()
hin = [pin(x) for x in (q, k, v, bias, do)]
hout = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (q, k, v, bias, do)]
dsets = [[torch.empty_like(x) for x in (q, k, v, bias, do)] for _ in range(2)]
up, dn = torch.cuda.Stream(), torch.cuda.Stream()

def timeit(fn, steps):
    fn(2); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(steps); torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e3

def h2d_only(n):
    with torch.cuda.stream(up):
        for i in range(n):
            for d, h in zip(dsets[i % 2], hin): d.copy_(h, non_blocking=True)
def d2h_only(n):
    with torch.cuda.stream(dn):
        for i in range(n):
            for d, h in zip(dsets[i % 2], hout): h.copy_(d, non_blocking=True)
def both(n):
    h2d_only(n); d2h_only(n)

for name, fn in (("h2d_only", h2d_only), ("d2h_only", d2h_only), ("both_concurrent", both)):
    res[name + "_ms"] = timeit(fn, 20)

ctx = A.Context.get(0)
plan = A.DevicePlan.from_host(ro, co, ctx); plan.schedule()
att = A.DeviceSparseAttention(plan, H, DH, DH, "bf16")
ho, hdq, hdk, hdv = (torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in (v, q, k, v))
hdb = torch.empty(E, dtype=torch.float32).pin_memory()
hq, hk, hv, hb, hdo = hin
def api(n):
    for _ in range(n):
        att.fwd_bwd_host(hq, hk, hv, hdo, hb, ho, hdq, hdk, hdv, hdb, sync=False)
    ctx.sync()
def api_sync(n):
    for _ in range(n):
        att.fwd_bwd_host(hq, hk, hv, hdo, hb, ho, hdq, hdk, hdv, hdb, sync=True)
for steps in (20, 60):
    res[f"api_async_{steps}_ms"] = timeit(api, steps)
res["api_sync_20_ms"] = timeit(api_sync, 20)
# host enqueue cost of one async step
t0 = time.perf_counter(); att.fwd_bwd_host(hq, hk, hv, hdo, hb, ho, hdq, hdk, hdv, hdb, sync=False)
res["enqueue_ms"] = (time.perf_counter() - t0) * 1e3; ctx.sync()
res["bytes_per_dir"] = int(sum(x.numel() * x.element_size() for x in hin))
print(json.dumps(res))
