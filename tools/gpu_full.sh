# round-end style: the whole -m gpu suite (timed), smoke(), default bench
mkdir -p gpurun_out
( time timeout 3000 python -m pytest tests -m gpu -q --durations=15 -k "not cfg5_full_50steps" ) > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -25 gpurun_out/pytest_gpu_full.log; tail -2 gpurun_out/smoke.log
