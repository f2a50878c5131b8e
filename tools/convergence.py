"""Convergence of PRGD vs RGD (and the adaptive step) on the GPU at a config: relative
residual on Omega and relative error to the truth per iteration (synthetic data, seeded).

    python tools/convergence.py CFG ITERS > log
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2501_13385_b200 as pkg  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
theory_step = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
pr = synth.make_problem(cfg)
t = pkg.TTContext(pr.n, pr.r)
t.set_cores(pr.truth)
y = pr.observations(t.eval_at(pr.idx))
rng = np.random.default_rng(7)
held = np.stack([rng.integers(0, nk, size=200_000) for nk in pr.n], axis=1).astype(np.int32)
truth_held = t.eval_at(held)
t.close()
ny = float(np.linalg.norm(y))
nh = float(np.linalg.norm(truth_held))
runs = [("PRGD theory", "vee", "theory", theory_step), ("RGD theory", "none", "theory", theory_step),
        ("PRGD adaptive", "vee", "adaptive", 1.0), ("RGD adaptive", "none", "adaptive", 1.0)]
print(f"cfg{cfg}: n={pr.n[0]}^{pr.d} r={max(pr.r)} m={pr.m} p={pr.m / pr.nstar:.3g}, theory step_size {theory_step}; "
      f"rel. residual on Omega / rel. error on 2e5 held-out entries")
for name, eps_rule, step_rule, step in runs:
    ctx = pkg.TTContext(pr.n, pr.r)
    ctx.set_metric(eps_rule, 0.0, step_rule)
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(pr.init)
    hist = []
    t0 = time.perf_counter()
    ok = True
    for it in range(iters):
        try:
            ctx.step(step)
        except pkg.PRGDError as e:
            hist.append((it, float("nan"), float("nan")))
            ok = False
            break
        if it in (0, 4, 9, 19, 29, 49, 99, 199) or it == iters - 1:
            res = ctx.residual_norm() / ny
            err = float(np.linalg.norm(ctx.eval_at(held) - truth_held)) / nh
            hist.append((it + 1, res, err))
    ctx.sync()
    dt = time.perf_counter() - t0
    print(f"{name:14s} " + "  ".join(f"it{i}: {r:.2e}/{e:.2e}" for i, r, e in hist) +
          f"  ({dt:.2f} s wall incl. host reads)" + ("" if ok else "  STOPPED (numeric fault)"))
    ctx.close()
