# quick bench (no e2e / cpu baseline) + group times
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${1:-} > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/bench.log"):
    if l.startswith("{"):
        r = json.loads(l)
        print("value", r["value"], "ms", r["ms_per_step"], {k: round(v, 3) for k, v in r["roofline"]["group_ms"].items()})
PY
