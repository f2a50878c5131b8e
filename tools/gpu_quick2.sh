mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "one_step or bucketing or deterministic or byte_indices" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --rank 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_r1.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
