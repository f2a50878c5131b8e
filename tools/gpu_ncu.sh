# launch list + full capture of the pass kernels and the dense rounding kernel (config 5)
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --profile-steps 1"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k_seg|k_dense_round|k_back_level|k_table' -s 60 -c 14 \
    -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
