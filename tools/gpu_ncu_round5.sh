# ncu source-level capture of one k_round_cs launch at config 5 (diagnostic)
mkdir -p gpurun_out
timeout 300 python tools/ncu_step.py 5 > gpurun_out/r5_plain.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_round_cs -c 1 \
  -o gpurun_out/round5 python tools/ncu_step.py 5 > gpurun_out/r5_ncu.log 2>&1
echo "rc=$?"
