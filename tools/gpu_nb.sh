bash tools/gpu_quick.sh
for nb in 1 2 4 8; do PRGD_GATHER_BLOCKS=$nb timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_nb$nb.log 2>&1; done
