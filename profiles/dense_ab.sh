# Dense tcgen05 A/B in one gpurun session: the dense parity tests on the
# working-tree build, then fwd/bwd timings (S = 32,768, H = 8, dh = 8, bf16)
# alternating the working tree and a base library.
#   gpurun -- 'bash profiles/dense_ab.sh [paper_2407_14106_b200/alt/X/libgte_b200.so]'
BASE=${1:-paper_2407_14106_b200/alt/base/libgte_b200.so}
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_dense_attention_gpu.py -x -q > $O/pytest_dense_ab.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_dense_ab.log
for r in 1 2; do
python profiles/dense_time.py
GTE_LIB_PATH=$BASE python profiles/dense_time.py
done
