#!/bin/bash
# ncu evidence for the tcgen05 dense kernels (run under gpurun, one GPU):
# tensor-pipe, MUFU (XU), issue and DRAM counters of the forward and the two
# backward kernels at S = 32768, H = 8, dh = 8, bf16.
O=gpurun_out
mkdir -p $O
cat > /tmp/dense_one.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2407_14106_b200 import attention as A
S, H, dh = 32768, 8, 8
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, up = (torch.randn((S, H * dh), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
att = A.DeviceDenseAttention(S, H, dh, dh, "bf16")
o, lse = att.forward(q, k, v)
att.backward(q, k, v, o, lse, up)
torch.cuda.synchronize()
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dense_tc" -c 3 -o /tmp/prof_dense -f python /tmp/dense_one.py > /dev/null 2>&1
ncu -i /tmp/prof_dense.ncu-rep --page source --csv --print-source sass > $O/ncu_source_dense_tc.csv 2>/dev/null; gzip -f $O/ncu_source_dense_tc.csv
ncu -i /tmp/prof_dense.ncu-rep --page raw --csv > $O/ncu_raw_dense_tc.csv
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ncu_raw_dense_tc.csv")))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread"]
for r in rows[2:]:
    name = r[idx["Kernel Name"]].split("(")[0]
    print(name + ": " + ", ".join(f"{w.split('.')[0]}={r[idx[w]]}{units[idx[w]]}" for w in want if w in idx))
PY
