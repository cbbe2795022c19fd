#!/bin/bash
# A/B of an alternative library build against the default one in one gpurun
# session: sparse parity tests on the alt build, then the bench (bf16, f32)
# alternating default / alt twice.
#   gpurun -- 'bash profiles/ab_lib.sh TAG paper_2407_14106_b200/alt/X/libgte_b200.so'
TAG=$1; ALT=$2
O=gpurun_out; mkdir -p $O
GTE_LIB_PATH=$ALT timeout 900 python -m pytest tests/test_sparse_attention_gpu.py tests/test_ecr_tiles_gpu.py -x -q \
  > $O/pytest_${TAG}_alt.log 2>&1
echo "pytest rc=$?" >> $O/pytest_${TAG}_alt.log; tail -3 $O/pytest_${TAG}_alt.log
for rep in 1 2; do
  for dt in bf16 f32; do
    for arm in default alt; do
      if [[ $arm == alt ]]; then export GTE_LIB_PATH=$ALT; else unset GTE_LIB_PATH; fi
      f=$O/bench_${TAG}_${arm}_${dt}_${rep}.log
      timeout 600 python bench.py --dtype $dt --no-cpu-baseline --no-alt --no-e2e > $f 2>&1
      echo "== $arm $dt $rep"; tail -c 1500 $f | grep -o '"ms_per_step": [0-9.]*\|"kernels_ms": {[^}]*}'
    done
  done
done
unset GTE_LIB_PATH
exit 0
