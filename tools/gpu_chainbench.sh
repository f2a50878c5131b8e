mkdir -p gpurun_out
N15=$(python -c "print(','.join(['16']*15))")
timeout 900 python bench.py --path chains --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/chain_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/chain_cfg5.log
timeout 900 python bench.py --config 5 --n-override $N15 --rank 8 --m 1000000 --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/chain_refused.log 2>&1; echo "rc=$?" >> gpurun_out/chain_refused.log
timeout 900 python bench.py --config 4 --path chains --no-e2e --no-cpu-baseline > gpurun_out/chain_cfg4.log 2>&1
timeout 900 python bench.py --config 2 --path chains --no-e2e --no-cpu-baseline > gpurun_out/chain_cfg2.log 2>&1
for f in chain_cfg5 chain_refused chain_cfg4 chain_cfg2; do tail -2 gpurun_out/$f.log | head -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']
  print('$f', d['value'], d['ms_per_step'], {g:(t['ms'],t['achieved'],t['frac']) for g,t in k.items()})
except Exception as e: print('$f', 'ERR', e)"; done
