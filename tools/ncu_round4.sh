#!/bin/bash
# ncu source-level capture of one k_round_cs launch at config 4 (diagnostic)
mkdir -p gpurun_out
timeout 300 python tools/dense_phases.py 4 "" 3 > gpurun_out/r4_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_round_cs -s 2 -c 1 \
  -o gpurun_out/round4 -f python tools/dense_phases.py 4 "" 3 > gpurun_out/r4_ncu.log 2>&1
ncu -i gpurun_out/round4.ncu-rep --page source --csv --print-source sass > gpurun_out/round4_src.csv 2>&1
ncu -i gpurun_out/round4.ncu-rep --page source --csv --print-source cuda > gpurun_out/round4_cu.csv 2>&1
ls -la gpurun_out/ | tail -5
