mkdir -p gpurun_out
for c in 5 4 3 2; do timeout 300 python tools/cmp_variant.py paper_2501_13385_b200/libprgd.so paper_2501_13385_b200/libprgd_c1.so $c 0 3 2>&1 | tail -1; done
for v in "" _c1; do timeout 300 env PRGD_LIB_PATH=paper_2501_13385_b200/libprgd$v.so python tools/dense_phases.py 5 "" 8 2>&1 | tail -1 | cut -c1-230; timeout 300 env PRGD_LIB_PATH=paper_2501_13385_b200/libprgd$v.so python tools/dense_phases.py 4 "" 8 2>&1 | tail -1 | cut -c1-230; done
for v in "" _c1; do PRGD_LIB_PATH=paper_2501_13385_b200/libprgd$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200; done
