# bench each gpurun_var_*.so variant of the library (experiments)
mkdir -p gpurun_out
for f in gpurun_var_*.so; do
  n=${f%.so}
  PRGD_LIB_PATH=$PWD/$f timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/$n.log 2>&1
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/var_default.log 2>&1
