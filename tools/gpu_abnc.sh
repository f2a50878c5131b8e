# cluster vs one-CTA dense kernels (PRGD_NO_CLUSTER=0 / 1) per config
mkdir -p gpurun_out
for c in ${CFGS:-1 2 4 6}; do for v in 0 1; do
  S=1.0; [ $c = 3 ] && S=0.5
  PRGD_NO_CLUSTER=$v timeout 600 python bench.py --config $c --step-size $S --no-cpu-baseline --no-e2e > gpurun_out/abnc.log 2>&1
  python - gpurun_out/abnc.log $c $v <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        j = json.loads(l); k = j["roofline"]["kernels"]
        print("cfg", sys.argv[2], "nocluster", sys.argv[3], j["value"], {n: v["ms"] for n, v in k.items() if n.startswith("dense")})
PY
done; done
