"""Host<->device copy rates on the box (pinned, 160 MB, the e2e step's bytes
per direction): H2D alone, D2H alone, both at once on two streams. Bounds
bench.py's e2e leg (PCIe-bound)."""
import json
import torch

N = 160 * 2**20
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_a = torch.empty(N, dtype=torch.uint8, device="cuda")
d_b = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = t(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_b, non_blocking=True))
bi = t(both)
print(json.dumps({"bytes": N, "h2d_ms": h2d, "h2d_gbs": N / h2d / 1e6, "d2h_ms": d2h, "d2h_gbs": N / d2h / 1e6,
                  "both_ms": bi, "both_gbs_per_dir": N / bi / 1e6}))
