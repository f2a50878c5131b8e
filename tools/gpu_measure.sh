# Measurement lease (round 2, final build): FP64 peak with its clock record, the default bench line, the r = 1
# HBM diagnostic, per-config bench lines, one ncu-counted PRGD step at config 5 (per-kernel DRAM
# bytes, DMMA / FP64 pipe utilisation) -> tools/ncu_table.py -> profiles/r02_ncu_kernels.json, and
# the ncu launch list of the bench command.
mkdir -p gpurun_out
Q=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap
nvidia-smi --query-gpu=$Q --format=csv -lms 100 > gpurun_out/fp64_clocks.csv & CP=$!
./tools/fp64_peak.bin > gpurun_out/fp64_peak.log 2>&1
kill $CP
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --rank 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_r1.log 2>&1
for c in 1 2 3 4 6; do
  S=1.0; [ $c = 3 ] && S=0.5
  timeout 600 python bench.py --config $c --step-size $S --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1
  timeout 600 python bench.py --config $c --step-size $S --step-rule adaptive --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg${c}_ad.log 2>&1
done
timeout 600 python bench.py --step-rule adaptive --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg5_ad.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --profile-steps 1"
timeout 600 python tools/ncu_step.py 5 > gpurun_out/ncu_step_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --clock-control none --metrics $M --csv python tools/ncu_step.py 5 > gpurun_out/ncu_step.csv 2> gpurun_out/ncu_step.err
timeout 600 $CMD > gpurun_out/launch_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "ncu rc=$?"
# full ncu captures of the SpMM pipeline kernel and the cluster rounding (one launch each)
timeout 1200 ncu --profile-from-start off --clock-control none --set full --import-source on \
    -k regex:"k_spmm_pipe|k_round_cs|k_flat_sddmm" -c 4 -o gpurun_out/full_head python tools/ncu_step.py 5 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
