#!/bin/bash
# Captures the ncu evidence for one dtype (run under gpurun on ONE GPU):
#   launch list (gpu__time_duration per launch, cold-cache, serialised) and
#   one `--set full` capture of the three sparse attention kernels of the
#   first timed step (3 warm-up steps x 3 kernels skipped), exported to CSV
#   on the box (raw metrics + per-line source counters).
set -e
DT=${1:-f32}
TAG=${2:-r1}
O=gpurun_out
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_${DT}_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --dtype $DT --no-cpu-baseline --no-e2e > /dev/null
ncu --set full --clock-control none --import-source on -k regex:"sparse_|fast_|slot_|tile_" -s 9 -c 3 \
    -o /tmp/prof_${DT}_${TAG} -f \
    python bench.py --steps 1 --warmup 3 --dtype $DT --no-cpu-baseline --no-e2e > /dev/null
ncu -i /tmp/prof_${DT}_${TAG}.ncu-rep --page raw --csv > $O/ncu_raw_${DT}_${TAG}.csv
ncu -i /tmp/prof_${DT}_${TAG}.ncu-rep --page details --csv > $O/ncu_details_${DT}_${TAG}.csv
ncu -i /tmp/prof_${DT}_${TAG}.ncu-rep --page source --csv --print-source sass > $O/ncu_source_${DT}_${TAG}.csv 2>/dev/null || true
gzip -f $O/ncu_source_${DT}_${TAG}.csv || true
SZ=$(stat -c %s /tmp/prof_${DT}_${TAG}.ncu-rep)
if [ "$SZ" -lt 25000000 ]; then cp /tmp/prof_${DT}_${TAG}.ncu-rep $O/; fi
