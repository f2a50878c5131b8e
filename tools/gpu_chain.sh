mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "weighted or maximal or one_step" > gpurun_out/pytest_w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_w.log
