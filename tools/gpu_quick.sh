# parity tests + dense-phase diagnostics (+ optional bench) on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 200 python tools/dense_phases.py 5 "" 12 > gpurun_out/phases5.log 2>&1
timeout 120 python tools/dense_phases.py 3 "" 8 > gpurun_out/phases3.log 2>&1
timeout 120 python tools/dense_phases.py 4 "" 8 > gpurun_out/phases4.log 2>&1
if [ "$1" = "bench" ]; then timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; fi
tail -3 gpurun_out/pytest_gpu.log
