"""One PRGD step of a config under the CUDA profiler range, for ncu:

    ncu --profile-from-start off --metrics ... python tools/ncu_step.py [cfg] [m]

Sets up the workload like bench.py (observations through tt_eval_at), runs 3 warm-up steps,
then one step in profiling mode (direct launches, the same kernels as the captured graph)
between cudaProfilerStart / cudaProfilerStop, so the profiled launches are exactly one step in
launch order (tools/ncu_table.py maps them to bench.py's kernel groups)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2501_13385_b200 as pkg  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
m = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
rank = None
if len(sys.argv) > 3:           # optional TT-rank override (the r = 1 HBM diagnostic)
    rank = int(sys.argv[3])
pr = synth.make_problem(cfg, m=m)
if rank is not None:
    pr.r = (1,) + (rank,) * (pr.d - 1) + (1,)
    pr.truth = [c[:pr.r[k], :, :pr.r[k + 1]].copy() for k, c in enumerate(pr.truth)]
    pr.init = [c[:pr.r[k], :, :pr.r[k + 1]].copy() for k, c in enumerate(pr.init)]
t = pkg.TTContext(pr.n, pr.r)
t.set_cores(pr.truth)
y = pr.observations(t.eval_at(pr.idx))
t.close()
ctx = pkg.TTContext(pr.n, pr.r)
ctx.set_observations(pr.idx, y)
ctx.set_cores(pr.init)
for _ in range(3):
    ctx.step(1.0)
ctx.sync()
ctx.set_profiling(True)
ctx.step(1.0)            # direct launches once (events created), then the profiled step
ctx.sync()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ctx.step(1.0)
ctx.sync()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one step:", ctx.get_profile())
ctx.close()
