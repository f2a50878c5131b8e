# dense-phase diagnostics only (config 5 and 4)
mkdir -p gpurun_out
timeout 200 python tools/dense_phases.py 5 "" 12 > gpurun_out/phases5.log 2>&1
timeout 120 python tools/dense_phases.py 4 "" 8 > gpurun_out/phases4.log 2>&1
