import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2407_14106_b200 import attention as A
S, H, dh = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
att = A.DeviceDenseAttention(S, H, dh, dh, "bf16")
o, lse = att.forward(q, k, v); torch.cuda.synchronize(); print("fwd ok", flush=True)
r = att.backward(q, k, v, o, lse, up); torch.cuda.synchronize(); print("bwd ok", flush=True)
