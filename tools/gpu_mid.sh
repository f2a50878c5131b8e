# parity + bench with the middle-split passes enabled
mkdir -p gpurun_out
PRGD_MIDDLE=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_mid.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mid.log
PRGD_MIDDLE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_mid.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_def.log 2>&1
