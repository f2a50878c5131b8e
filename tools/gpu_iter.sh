# quick iteration on the GPU box: dense-sweep phases, parity subset, default bench
mkdir -p gpurun_out
for c in 5 4; do timeout 300 python tools/dense_phases.py $c "" 8; done > gpurun_out/phases.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_iter.log
tail -4 gpurun_out/phases.log; tail -3 gpurun_out/pytest_iter.log
python - <<'PY'
import json
for l in open("gpurun_out/bench_iter.log"):
    if l.startswith("{"):
        j = json.loads(l); k = j["roofline"]["kernels"]
        print("value", j["value"], "ms", j["ms_per_step"], "e2e", j.get("e2e", {}).get("value"),
              {n: v["ms"] for n, v in k.items()})
PY
