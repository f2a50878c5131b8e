"""Diagnostic: rounding parity error vs the oracle for a given libprgd.so (PRGD_LIB env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2501_13385_b200 as pkg  # noqa: E402
import synth  # noqa: E402

for cfg, m, steps in [(2, 20000, 3), (2, 20000, 10), (4, None, 10), (6, None, 3)]:
    pr = synth.make_problem(cfg, m=m)
    y = pr.observations(oracle.eval_at(pr.truth, pr.idx))
    c = pkg.TTContext(pr.n, pr.r)
    c.set_observations(pr.idx, y)
    c.set_cores(pr.init)
    ref = pr.init
    errs = []
    for _ in range(steps):
        c.step(1.0)
        ref = oracle.prgd_step(ref, pr.idx, y, pr.n, pr.r, 1.0)
        errs.append(oracle.tt_diff_norm(c.get_cores(), ref))
    print(cfg, m, steps, " ".join(f"{e:.2e}" for e in errs), flush=True)
    c.close()
