mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "sliced or one_step" > gpurun_out/pytest_gsq.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gsq.log
tail -2 gpurun_out/pytest_gsq.log
for v in 1 "" 1 ""; do
  PRGD_GSQ_SLICES=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/gsq_$v.log 2>&1
  python -c "
import json
for l in open('gpurun_out/gsq_$v.log'):
    if l.startswith('{'): j=json.loads(l); k=j['roofline']['kernels']; print('slices=$v', j['value'], j['ms_per_step'], {n: k[n]['ms'] for n in ('passA_suffix','passB_suffix','passB_prefix','marginals')})"
done
