mkdir -p gpurun_out
for c in 5 3 4; do timeout 300 python tools/dense_phases.py $c "" 8 > gpurun_out/phases_$c.log 2>&1; done
