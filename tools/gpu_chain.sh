mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_chains.py tests/test_gpu_parity.py tests/test_gpu_parity_long.py -q -k "not 4e6 and not full_50steps" > gpurun_out/pytest_chain.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_chain.log
