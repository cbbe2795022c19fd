#!/bin/bash
# Three-arm bench A/B in one gpurun session (sparse + ECR parity tests on the
# working-tree build first): default, then each GTE_LIB_PATH given, twice.
#   gpurun -- 'bash profiles/ab3.sh TAG libA.so libB.so'
TAG=$1; shift
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_sparse_attention_gpu.py tests/test_ecr_tiles_gpu.py -x -q > $O/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> $O/pytest_${TAG}.log; tail -2 $O/pytest_${TAG}.log
for rep in 1 2; do
  for arm in default "$@"; do
    if [[ $arm == default ]]; then unset GTE_LIB_PATH; else export GTE_LIB_PATH=$arm; fi
    f=$O/bench_${TAG}_$(basename $(dirname $arm))_${rep}.log
    timeout 600 python bench.py --no-cpu-baseline --no-alt --no-e2e > $f 2>&1
    echo "== $arm $rep $(tail -c 1500 $f | grep -o '"ms_per_step": [0-9.]*\|"kernels_ms": {[^}]*}' | tr '\n' ' ')"
  done
done
unset GTE_LIB_PATH
