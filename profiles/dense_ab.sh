O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_dense_attention_gpu.py -x -q > $O/pytest_dense_ab.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_dense_ab.log
for r in 1 2; do
python profiles/dense_time.py
GTE_LIB_PATH=paper_2407_14106_b200/alt/base/libgte_b200.so python profiles/dense_time.py
done
