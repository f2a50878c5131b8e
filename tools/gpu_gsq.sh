# sliced pass A suffix: forced-slice parity test, config-5 A/B (default slicing vs the row-plan
# gather), slice-size sweep, iterate comparison against the previous build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sliced" > gpurun_out/pytest_gsq.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gsq.log
tail -3 gpurun_out/pytest_gsq.log
for v in 1 "" 1 "" 8 4; do
  PRGD_GSQ_SLICES=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/gsq_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/gsq_$v.log'):
    if l.startswith('{'): j=json.loads(l); k=j['roofline']['kernels']; print('slices=$v', j['value'], j['ms_per_step'], {n: k[n]['ms'] for n in ('passA_suffix','passB_suffix','passB_prefix','marginals')})"
done
timeout 300 python tools/cmp_variant.py paper_2501_13385_b200/libprgd_base.so paper_2501_13385_b200/libprgd.so 5 0 3 2>&1 | grep cfg
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -x -q -m gpu > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
tail -3 gpurun_out/pytest_iter.log
