# pipelined vs row-plan SpMM (PRGD_SPMM_PIPE=1 / 0) at interior ranks ${RANKS:-16 1}
mkdir -p gpurun_out
for R in ${RANKS:-16 1}; do for v in ${VALS:-0 1}; do
  PRGD_SPMM_PIPE=$v timeout 600 python bench.py --rank $R --no-cpu-baseline --no-e2e > gpurun_out/abr_${R}_$v.log 2>&1
  python - gpurun_out/abr_${R}_$v.log <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        j = json.loads(l); k = j["roofline"]["kernels"]
        print(sys.argv[1], j["value"], k["passB_prefix"]["ms"], k["passB_suffix"]["ms"])
PY
done; done
