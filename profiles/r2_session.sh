#!/bin/bash
# r2 GPU session: selected GPU tests, then bench variants (env or flags).
#   gpurun -- 'bash profiles/r2_session.sh TAG "tests/a.py tests/b.py" "--flag" ...'
TAG=$1; TESTS=$2; shift 2
O=gpurun_out; mkdir -p $O
if [[ -n $TESTS ]]; then
  timeout 1500 python -m pytest $TESTS -x -q > $O/pytest_${TAG}.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_${TAG}.log; tail -5 $O/pytest_${TAG}.log
fi
i=0
for v in "$@"; do
  i=$((i+1))
  timeout 600 python bench.py --no-cpu-baseline --no-alt --no-e2e $v > $O/bench_${TAG}_$i.log 2>&1
  echo "== bench $v"; tail -c 3000 $O/bench_${TAG}_$i.log | grep -o '"ms_per_step": [0-9.]*\|"kernels_ms": {[^}]*}\|"ecr_tiles": [0-9]*\|Error.*\|error.*' | head -5
done
exit 0
