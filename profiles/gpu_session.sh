#!/bin/bash
# One gpurun session: GPU tests, smoke, bench (f32 + bf16), ncu evidence.
#   gpurun --timeout 2400 -- 'bash profiles/gpu_session.sh r1 [tests|bench|ncu|all]'
TAG=${1:-r1}
WHAT=${2:-all}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/nvidia_smi_${TAG}.txt 2>&1
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_${TAG}.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> $O/smoke_${TAG}.log
  tail -3 $O/pytest_gpu_${TAG}.log
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py > $O/bench_default_${TAG}.log 2>&1; echo "rc=$?" >> $O/bench_default_${TAG}.log
  timeout 600 python bench.py --dtype f32 --no-cpu-baseline > $O/bench_f32_${TAG}.log 2>&1; echo "rc=$?" >> $O/bench_f32_${TAG}.log
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_${TAG}.log 2>&1; echo "rc=$?" >> $O/bench_ref_${TAG}.log
  tail -n 2 $O/bench_default_${TAG}.log
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 900 bash profiles/ncu_capture.sh f32 $TAG > $O/ncu_f32_${TAG}.log 2>&1
  timeout 900 bash profiles/ncu_capture.sh bf16 $TAG > $O/ncu_bf16_${TAG}.log 2>&1
fi
exit 0
