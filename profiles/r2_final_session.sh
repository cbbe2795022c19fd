#!/bin/bash
# End-of-round HEAD session: full GPU suite, smoke, bench (bf16 default, f32,
# reference arm, Mode H path on one NCCL rank), measured parity errors, ncu of
# the dense tcgen05 kernels.
TAG=${1:-r2z}
O=gpurun_out; mkdir -p $O
bash profiles/gpu_session.sh $TAG tests
bash profiles/gpu_session.sh $TAG bench
timeout 600 python bench.py --sp --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_sp1_${TAG}.log 2>&1; echo "rc=$?" >> $O/bench_sp1_${TAG}.log
timeout 900 python profiles/parity_errors.py > $O/parity_errors_${TAG}.txt 2>&1; echo "rc=$?" >> $O/parity_errors_${TAG}.txt
timeout 1200 bash profiles/dense_ncu.sh > $O/dense_ncu_${TAG}.txt 2>&1
cuobjdump -sass paper_2407_14106_b200/libgte_b200.so 2>/dev/null | grep -o 'UTMALDG[.A-Z0-9]*\|UTCHMMA[.A-Z0-9]*\|UTCBAR[.A-Z0-9]*\|LDTM[.A-Z0-9]*\|FHFMA[.A-Z0-9]*' | sort | uniq -c > $O/sass_evidence_${TAG}.txt
exit 0
