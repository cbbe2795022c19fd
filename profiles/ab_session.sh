#!/bin/bash
# A/B one gpurun session: sparse GPU tests, then the bench with the default
# build and with env variants listed as VAR=VAL arguments.
#   gpurun -- 'bash profiles/ab_session.sh TAG [tests] [GTE_NO_MMA=1 ...]'
TAG=$1; shift
O=gpurun_out; mkdir -p $O
if [[ $1 == tests ]]; then
  shift
  timeout 900 python -m pytest tests/test_sparse_attention_gpu.py -x -q > $O/pytest_sparse_${TAG}.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_sparse_${TAG}.log; tail -3 $O/pytest_sparse_${TAG}.log
fi
timeout 600 python bench.py --no-cpu-baseline --no-alt --no-e2e > $O/bench_${TAG}_default.log 2>&1
tail -c 1500 $O/bench_${TAG}_default.log | grep -o '"ms_per_step": [0-9.]*\|"kernels_ms": {[^}]*}\|"frac": [0-9.]*'
for v in "$@"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --no-alt --no-e2e > $O/bench_${TAG}_${v}.log 2>&1
  echo "== $v"; tail -c 1500 $O/bench_${TAG}_${v}.log | grep -o '"ms_per_step": [0-9.]*\|"kernels_ms": {[^}]*}\|"frac": [0-9.]*'
done
exit 0
