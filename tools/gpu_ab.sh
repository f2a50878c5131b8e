# A/B of an environment switch on the default bench (config 5), then the parity subset.
# usage: VAR=PRGD_SPMM_PIPE bash tools/gpu_ab.sh
mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        j = json.loads(l); k = j["roofline"]["kernels"]
        print(sys.argv[1], "value", j["value"], "ms", j["ms_per_step"], {n: v["ms"] for n, v in k.items()})
PY
}
for v in ${VALS:-0 1}; do
  f=gpurun_out/ab_$(basename "$v").log
  env $VAR=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > $f 2>&1
  summ $f; tail -2 $f | grep -v "^{" | tail -2
done
[ -n "$NOTEST" ] || timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
tail -5 gpurun_out/pytest_iter.log
