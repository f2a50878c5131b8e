mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum,l1tex__t_sectors.sum,smsp__warps_active.avg.pct_of_peak_sustained_active"
timeout 300 python tools/ncu_step.py 5 "" 1 > gpurun_out/ncu_r1_plain.log 2>&1 && \
timeout 900 ncu --profile-from-start off --clock-control none --metrics $M --csv python tools/ncu_step.py 5 "" 1 > gpurun_out/ncu_r1.csv 2> gpurun_out/ncu_r1.err
timeout 300 python tools/ncu_step.py 5 > gpurun_out/ncu_r16_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:"k_flat|k_seg" -o gpurun_out/flat_full python tools/ncu_step.py 5 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
