#!/bin/bash
# Captures the ncu evidence for one dtype (run under gpurun on ONE GPU):
#   launch list (gpu__time_duration per launch, cold-cache, serialised) and
#   one `--set full` capture of the three sparse attention kernels of the
#   first timed step (3 warm-up steps x 3 kernels skipped).
set -e
DT=${1:-f32}
TAG=${2:-r1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${DT}_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --dtype $DT --no-cpu-baseline --no-e2e > /dev/null
ncu --set full --clock-control none --import-source on -k regex:sparse -s 9 -c 3 \
    -o gpurun_out/prof_${DT}_${TAG} -f \
    python bench.py --steps 1 --warmup 3 --dtype $DT --no-cpu-baseline --no-e2e > /dev/null
