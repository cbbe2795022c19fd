"""Time the dense bf16 (tcgen05) forward and backward at S = 32768, H = 8,
dh = 8 with CUDA events (library from GTE_LIB_PATH for A/B builds)."""
import json, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2407_14106_b200 import attention as A
S, H, dh = int(os.environ.get("S", 32768)), 8, 8
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
att = A.DeviceDenseAttention(S, H, dh, dh, "bf16")
def ev():
    return torch.cuda.Event(enable_timing=True)
f, b = [], []
for i in range(7):
    e0, e1, e2 = ev(), ev(), ev()
    e0.record(); o, lse = att.forward(q, k, v); e1.record()
    att.backward(q, k, v, o, lse, up); e2.record(); torch.cuda.synchronize()
    if i >= 2:
        f.append(e0.elapsed_time(e1)); b.append(e1.elapsed_time(e2))
pairs = S * S * H
print(json.dumps({"lib": os.environ.get("GTE_LIB_PATH", "default"), "S": S, "fwd_ms": min(f), "bwd_ms": min(b),
                  "fwd_pairheads_per_s": pairs / (min(f) * 1e-3)}))
