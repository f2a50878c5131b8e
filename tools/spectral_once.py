"""Diagnostic: one tt_spectral_init at a config (for ncu launch lists)."""
import os
import sys

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
ctx.spectral_init()
print("done", ctx.get_core(0).shape)
