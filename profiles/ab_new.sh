#!/bin/bash
# A/B of the working-tree library (default) against a base build, one gpurun
# session: sparse + ECR parity tests on the default build, then the bench
# alternating default / base.
#   gpurun -- 'bash profiles/ab_new.sh TAG paper_2407_14106_b200/alt/base/libgte_b200.so "bf16 f32" REPS'
TAG=$1; BASE=$2; DTS=${3:-bf16}; REPS=${4:-2}
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_sparse_attention_gpu.py tests/test_ecr_tiles_gpu.py -x -q \
  > $O/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> $O/pytest_${TAG}.log; tail -3 $O/pytest_${TAG}.log
for rep in $(seq $REPS); do
  for dt in $DTS; do
    for arm in default base; do
      if [[ $arm == base ]]; then export GTE_LIB_PATH=$BASE; else unset GTE_LIB_PATH; fi
      f=$O/bench_${TAG}_${arm}_${dt}_${rep}.log
      timeout 600 python bench.py --dtype $dt --no-cpu-baseline --no-alt --no-e2e > $f 2>&1
      echo "== $arm $dt $rep"; tail -c 1500 $f | grep -o '"ms_per_step": [0-9.]*\|"kernels_ms": {[^}]*}'
    done
  done
done
unset GTE_LIB_PATH
exit 0
