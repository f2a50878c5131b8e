"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck), one tool per run:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Both paths (tables, chains), config 1 and a reduced config 2, one theory step, one adaptive
step, the weighted retraction, the spectral init and tt_eval_at; direct launches (profiling mode)
so the sanitizer sees every kernel, then the captured-graph step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2501_13385_b200 as pkg  # noqa: E402
import synth  # noqa: E402

for cfg, m in [(1, None), (2, 20_000)]:
    pr = synth.make_problem(cfg, m=m)
    t = pkg.TTContext(pr.n, pr.r)
    t.set_cores(pr.truth)
    y = pr.observations(t.eval_at(pr.idx))
    t.close()
    for path in ("tables", "chains"):
        ctx = pkg.TTContext(pr.n, pr.r, path=path)
        ctx.set_observations(pr.idx, y)
        if path == "tables":
            ctx.spectral_init()
        else:
            ctx.set_cores(pr.init if pr.init is not None else pr.truth)
        ctx.set_profiling(True)
        ctx.step(1.0)
        ctx.set_profiling(False)
        ctx.step(1.0)
        ctx.set_metric("vee", 0.0, "adaptive")
        ctx.step(1.0)
        ctx.set_metric("vee", 0.0, "theory")
        ctx.set_retraction("weighted")
        ctx.step(1.0)
        v = ctx.eval_at(pr.idx[:100])
        print(cfg, path, "residual", ctx.residual_norm(), "eval", float(np.abs(v).sum()), flush=True)
        ctx.close()
print("sanitize workload done")
