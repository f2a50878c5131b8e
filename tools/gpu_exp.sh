# A/B of an environment switch on the config-5 bench groups: bash tools/gpu_exp.sh VAR
mkdir -p gpurun_out
for v in "" 1; do
  env $1=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/exp_$v.log 2>&1
  tail -2 gpurun_out/exp_$v.log | head -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']
print('$1=$v', d['value'], d['ms_per_step'], {g:t['ms'] for g,t in k.items()})"
done
