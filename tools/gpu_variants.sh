# dense-sweep phase timings and golden parity for experimental library variants
mkdir -p gpurun_out
for v in base $VARIANTS; do
  if [ "$v" = base ]; then L=paper_2501_13385_b200/libprgd.so; else L=paper_2501_13385_b200/libprgd_$v.so; fi
  for c in 4 5 3; do PRGD_LIB_PATH=$L timeout 300 python tools/dense_phases.py $c "" 8 > gpurun_out/var_${v}_$c.log 2>&1; done
  PRGD_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_parity_long.py -q -k "cfg4 or cfg3 or cfg5_full_1step" > gpurun_out/var_${v}_pytest.log 2>&1
done
for v in base $VARIANTS; do echo "== $v"; tail -n1 gpurun_out/var_${v}_4.log | cut -c1-200; tail -n1 gpurun_out/var_${v}_5.log | cut -c1-200; tail -n1 gpurun_out/var_${v}_3.log | cut -c1-200; tail -n1 gpurun_out/var_${v}_pytest.log; done
