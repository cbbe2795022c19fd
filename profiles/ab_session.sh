#!/bin/bash
# A/B session for kernel work: GPU parity tests (bounded), bench of several
# kernel variants (env), one ncu --set full capture of the default path's
# attention kernels. Usage (under gpurun):
#   bash profiles/ab_session.sh TAG [dtype] [variants...]
# variant syntax: name=ENV=VAL[,ENV=VAL]
TAG=${1:-ab}
DT=${2:-bf16}
shift 2
O=gpurun_out
mkdir -p $O
timeout 420 python -m pytest tests/test_sparse_attention_gpu.py -x -q > $O/pytest_${TAG}.log 2>&1; echo "rc=$?" >> $O/pytest_${TAG}.log
tail -3 $O/pytest_${TAG}.log
python bench.py --dtype bf16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1  # warm the workload cache
for dt in bf16 f32; do
  timeout 240 python bench.py --dtype $dt --no-cpu-baseline --no-e2e > $O/bench_${TAG}_${dt}_default.log 2>&1
  for v in "$@"; do
    name=${v%%=*}; envs=${v#*=}
    env $(echo $envs | tr ',' ' ') timeout 240 python bench.py --dtype $dt --no-cpu-baseline --no-e2e > $O/bench_${TAG}_${dt}_${name}.log 2>&1
  done
done
for f in $O/bench_${TAG}_*.log; do echo "$f $(tail -n1 $f | cut -c1-200)"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"wide_|tile_|hub_" -s 9 -c 3 \
    -o /tmp/prof_${TAG} -f python bench.py --steps 1 --warmup 3 --dtype $DT --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i /tmp/prof_${TAG}.ncu-rep --page raw --csv > $O/ncu_raw_${TAG}.csv
ncu -i /tmp/prof_${TAG}.ncu-rep --page source --csv --print-source sass > $O/ncu_source_${TAG}.csv 2>/dev/null; gzip -f $O/ncu_source_${TAG}.csv
python profiles/ncu_summary.py $O/ncu_raw_${TAG}.csv; python profiles/ncu_stalls.py $O/ncu_raw_${TAG}.csv
exit 0
