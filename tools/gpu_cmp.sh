# bitwise comparison and timing of the in-tree library against an experimental variant ($VAR)
mkdir -p gpurun_out
for c in 5 4 3 2; do timeout 300 python tools/cmp_variant.py paper_2501_13385_b200/libprgd.so paper_2501_13385_b200/libprgd_$VAR.so $c 0 3 2>&1 | tail -1; done
for v in "" _$VAR; do timeout 300 env PRGD_LIB_PATH=paper_2501_13385_b200/libprgd$v.so python tools/dense_phases.py 5 "" 8 2>&1 | tail -1 | cut -c1-230; done
for v in "" _$VAR; do PRGD_LIB_PATH=paper_2501_13385_b200/libprgd$v.so timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c90-200; done
