# bench A/B of libprgd_base.so vs the current build, iterate comparison and dense phases
mkdir -p gpurun_out
NOTEST=1 VALS="paper_2501_13385_b200/libprgd_base.so paper_2501_13385_b200/libprgd.so" VAR=PRGD_LIB_PATH bash tools/gpu_ab.sh
for c in "1 0 5" "2 0 5" "4 0 5" "6 0 5" "5 200000 3" "3 0 3"; do
  timeout 300 python tools/cmp_variant.py paper_2501_13385_b200/libprgd_base.so paper_2501_13385_b200/libprgd.so $c 2>&1 | grep cfg
done
for c in 5 4; do timeout 300 python tools/dense_phases.py $c "" 25 | tail -1; done
