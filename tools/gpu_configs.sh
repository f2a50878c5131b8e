# bench line per config (no e2e / cpu baseline), theory and adaptive rules
mkdir -p gpurun_out
for c in 1 2 3 4 5 6; do
  for rule in theory adaptive; do
    timeout 600 python bench.py --config $c --step-rule $rule --no-cpu-baseline --no-e2e --steps 20 --warmup 5 2>/dev/null | grep "^{" > gpurun_out/cfg_${c}_${rule}.json
  done
done
