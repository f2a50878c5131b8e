"""Diagnostic: wall time of tt_spectral_init at a config, and the relative error of the
spectral init against the truth (and against the perturbed-truth init)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_13385_b200 as pkg  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pr = synth.make_problem(cfg)
t = pkg.TTContext(pr.n, pr.r)
t.set_cores(pr.truth)
y = pr.observations(t.eval_at(pr.idx))
ctx = pkg.TTContext(pr.n, pr.r)
ctx.set_observations(pr.idx, y)
for rep in range(2):
    t0 = time.perf_counter()
    ctx.spectral_init()
    t1 = time.perf_counter()
    print(f"cfg{cfg} m={pr.m} spectral init {1e3 * (t1 - t0):.1f} ms; residual {ctx.residual_norm():.4e}")
for it in range(20):
    ctx.step(1.0)
print("after 20 steps residual", ctx.residual_norm())
ctx.set_cores(pr.init)
print("perturbed-truth init residual", ctx.residual_norm())
