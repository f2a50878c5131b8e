# A/B of the pass-B suffix overlap (PRGD_NO_OVERLAP) on configs 5 / 3 / 2, iterate comparison
# against the previous build (libprgd_base.so), e2e breakdown, quick parity subset
mkdir -p gpurun_out
for c in 5 3 2; do
  S=1.0; [ $c = 3 ] && S=0.5
  for v in 1 0 1 0; do
    PRGD_NO_OVERLAP=$v timeout 600 python bench.py --config $c --step-size $S --no-cpu-baseline --no-e2e > gpurun_out/ovl_${c}_$v.log 2>&1
    python -c "
import json,sys
for l in open('gpurun_out/ovl_${c}_$v.log'):
    if l.startswith('{'): j=json.loads(l); print('cfg $c no_overlap=$v', j['value'], j['ms_per_step'])"
  done
done
for c in "5 200000 3" "3 0 3" "2 0 5"; do
  timeout 300 python tools/cmp_variant.py paper_2501_13385_b200/libprgd_base.so paper_2501_13385_b200/libprgd.so $c 2>&1 | grep cfg
done
PRGD_TIMING=1 timeout 300 python tools/e2e_breakdown.py 5 2>&1 | grep -v "^\[prgd\] \(step\|eval\|update\)" | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
tail -3 gpurun_out/pytest_iter.log
