mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --profile-steps 1"
PRGD_MIDDLE=1 $CMD > gpurun_out/plain.log 2>&1 && PRGD_MIDDLE=1 ncu --set full --clock-control none --import-source on -k regex:"k_mid_sddmm_r" -s 0 -c 1 -o gpurun_out/prof_mid $CMD > gpurun_out/ncu_mid.log 2>&1
