# A/B of the bf16-weight products (GTE_BF16_W=1): GPU parity tests on the alt build, then bench default vs alt
O=gpurun_out; mkdir -p $O
# alt build: make -C paper_2407_14106_b200/csrc OUT=../alt/libgte_b200.so BUILD=build_alt EXTRA=-DGTE_BF16_W=1
ALT=/root/repo/paper_2407_14106_b200/alt/libgte_b200.so
GTE_LIB_PATH=$ALT timeout 900 python -m pytest tests/test_sparse_attention_gpu.py tests/test_halo_gpu.py tests/test_parallel_gpu.py -x -q > $O/pytest_w1.log 2>&1; echo "rc=$?" >> $O/pytest_w1.log
tail -3 $O/pytest_w1.log
bash profiles/ab_session.sh w1 bf16 bf16w=GTE_LIB_PATH=$ALT > $O/ab_w1.log 2>&1
grep bench_w1 $O/ab_w1.log
