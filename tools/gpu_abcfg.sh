# A/B of libprgd_base.so vs the current build on configs ${CFGS:-3 5}, iterate comparison
mkdir -p gpurun_out
for c in ${CFGS:-3 5}; do
  S=1.0; [ $c = 3 ] && S=0.5
  for lib in paper_2501_13385_b200/libprgd_base.so paper_2501_13385_b200/libprgd.so; do
    PRGD_LIB_PATH=$lib timeout 600 python bench.py --config $c --step-size $S --no-cpu-baseline --no-e2e > gpurun_out/abcfg.log 2>&1
    python - gpurun_out/abcfg.log $c $(basename $lib) <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        j = json.loads(l); k = j["roofline"]["kernels"]
        print("cfg", sys.argv[2], sys.argv[3], j["value"], {n: v["ms"] for n, v in k.items() if v["ms"] > 0.05})
PY
  done
done
for c in "1 0 5" "2 0 5" "4 0 5" "6 0 5" "5 200000 3" "3 0 3"; do
  timeout 300 python tools/cmp_variant.py paper_2501_13385_b200/libprgd_base.so paper_2501_13385_b200/libprgd.so $c 2>&1 | grep cfg
done
