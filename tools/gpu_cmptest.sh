# iterate comparison (tensor level) against libprgd_base.so, then the parity subset
mkdir -p gpurun_out
for c in "1 0 5" "2 0 5" "4 0 5" "6 0 5" "5 200000 3" "3 0 3"; do
  timeout 300 python tools/cmp_variant.py paper_2501_13385_b200/libprgd_base.so paper_2501_13385_b200/libprgd.so $c 2>&1 | grep cfg
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
tail -4 gpurun_out/pytest_iter.log
