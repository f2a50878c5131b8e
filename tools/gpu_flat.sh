mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -x -q -k "not 4e6 and not full_50steps" > gpurun_out/flat_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/flat_pytest.log
tail -2 gpurun_out/flat_pytest.log
for mode in 0 1; do
  PRGD_ROWPLAN=$mode timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/flat_bench_$mode.log 2>&1
  echo "rowplan=$mode"; tail -1 gpurun_out/flat_bench_$mode.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({g: t['ms'] for g,t in d['roofline']['kernels'].items()})"
done
