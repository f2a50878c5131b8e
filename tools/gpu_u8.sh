# byte-index entry point: its tests, the end-to-end breakdown with int32 / byte indices, default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "byte_indices or edge or bucketing" > gpurun_out/u8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/u8_tests.log
E2E_IDX=i32 PRGD_TIMING=1 timeout 600 python tools/e2e_breakdown.py 5 > gpurun_out/e2e_i32.log 2>&1
E2E_IDX=u8 PRGD_TIMING=1 timeout 600 python tools/e2e_breakdown.py 5 > gpurun_out/e2e_u8.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_u8.log 2>&1; echo "rc=$?" >> gpurun_out/bench_u8.log
