import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2407_14106_b200 import attention as A
import os
CASES = ((300, 300, 8, 8), (300, 257, 8, 8), (1024, 1024, 8, 16), (4096, 4096, 8, 8), (32768, 32768, 8, 8), (32768, 32768, 8, 16))
if os.environ.get('DENSE_CASE'):
    CASES = (CASES[int(os.environ['DENSE_CASE'])],)
for (S, s_real, H, dh) in CASES:
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    att = A.DeviceDenseAttention(S, H, dh, dh, "bf16", s_real=s_real)
    o, lse = att.forward(q, k, v); torch.cuda.synchronize()
    att32 = A.DeviceDenseAttention(S, H, dh, dh, "f32", s_real=s_real)
    o32, lse32 = att32.forward(q.float(), k.float(), v.float()); torch.cuda.synchronize()
    e = (o.float() - o32).abs().max().item() / o32.abs().max().item()
    el = (lse[:s_real] - lse32[:s_real]).abs().max().item()
    # timing
    for _ in range(3): att.forward(q, k, v)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): att.forward(q, k, v)
    torch.cuda.synchronize(); t = (time.perf_counter() - t0) / 10
    for _ in range(3): att32.forward(q.float(), k.float(), v.float())
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(10): att32.forward(q.float(), k.float(), v.float())
    torch.cuda.synchronize(); t32 = (time.perf_counter() - t0) / 10
    pairs = s_real * s_real * H
    exps_bound = pairs / (148 * 16 * 1.965e9)  # MUFU ex2: 16 / clk / SM
    print(f"S={S} s_real={s_real} H={H} dh={dh}: tc-vs-f32 max-norm err {e:.3e}, lse err {el:.3e}; tc fwd {t*1e3:.3f} ms "
          f"({pairs / t / 1e12:.2f} T pair-heads/s, {exps_bound / t * 100:.1f}% of the MUFU exp bound, "
          f"{4 * dh * pairs / t / 1e12:.1f} TFLOP/s algorithmic), cuda-core f32 fwd {t32*1e3:.3f} ms", flush=True)

# backward (tcgen05 for bf16 without weight_mult / dbias) vs the CUDA-core f32 backward
for (S, H, dh) in ((4096, 8, 8), (32768, 8, 8)):
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    att = A.DeviceDenseAttention(S, H, dh, dh, "bf16")
    o, lse = att.forward(q, k, v)
    res = att.backward(q, k, v, o, lse, up)
    att32 = A.DeviceDenseAttention(S, H, dh, dh, "f32")
    o32, l32 = att32.forward(q.float(), k.float(), v.float())
    r32 = att32.backward(q.float(), k.float(), v.float(), o32, l32, up.float())
    torch.cuda.synchronize()
    errs = [((a.float() - b).abs().max() / b.abs().max()).item() for a, b in zip(res[:3], r32[:3])]
    def tm(fn, n=5):
        fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(n): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / n
    t = tm(lambda: att.backward(q, k, v, o, lse, up))
    t32 = tm(lambda: att32.backward(q.float(), k.float(), v.float(), o32, l32, up.float()), 2)
    print(f"bwd S={S} H={H} dh={dh}: tc-vs-f32 max-norm err dq/dk/dv {errs[0]:.2e}/{errs[1]:.2e}/{errs[2]:.2e}; "
          f"tc bwd {t*1e3:.3f} ms, cuda-core f32 bwd {t32*1e3:.3f} ms", flush=True)
