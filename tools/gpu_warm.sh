mkdir -p gpurun_out
for c in 5 4 3; do S=""; timeout 300 python tools/dense_phases.py $c "" 10 2>&1 | tail -2 | cut -c1-200; done
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c90-190
timeout 600 python bench.py --config 4 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c90-190
timeout 600 python bench.py --config 3 --step-size 0.5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c90-190
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -q -x -k "not cfg5_full_50steps" 2>&1 | tail -3
