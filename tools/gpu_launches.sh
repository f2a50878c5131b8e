# ncu launch list (device time per kernel) of a short config-5 bench run; optional full capture regex in $1
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --profile-steps 1"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
if [ -n "$1" ]; then
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-0} -c ${3:-4} \
    -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
fi
echo "rc=$?"
