# full GPU suite + smoke, then the default bench and the per-config bench lines (final build)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --rank 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_r1.log 2>&1
for c in 1 2 3 4 6; do
  S=1.0; [ $c = 3 ] && S=0.5
  timeout 600 python bench.py --config $c --step-size $S --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1
  timeout 600 python bench.py --config $c --step-size $S --step-rule adaptive --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg${c}_ad.log 2>&1
done
timeout 600 python bench.py --step-rule adaptive --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg5_ad.log 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
