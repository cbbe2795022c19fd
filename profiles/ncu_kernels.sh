#!/bin/bash
# ncu --set full of the three sparse-attention kernels of one bench step
# (run under gpurun on ONE GPU):  bash profiles/ncu_kernels.sh TAG REGEX [bench args...]
TAG=$1; RX=$2; shift 2
O=gpurun_out; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 9 -c 3 \
    -o /tmp/prof_${TAG} -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-alt "$@" > $O/ncu_${TAG}.log 2>&1
ncu -i /tmp/prof_${TAG}.ncu-rep --page raw --csv > $O/ncu_raw_${TAG}.csv
ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source sass > $O/ncu_source_${TAG}.csv 2>/dev/null
gzip -f $O/ncu_source_${TAG}.csv
python profiles/ncu_summary.py $O/ncu_raw_${TAG}.csv > $O/ncu_summary_${TAG}.txt 2>&1
cat $O/ncu_summary_${TAG}.txt
