"""Diagnostic: Jacobi sweeps and per-phase cycles of the dense sweeps (cluster rounding).

    python tools/dense_phases.py [cfg] [m] [steps] [step_size]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2501_13385_b200 as pkg  # noqa: E402
import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
m = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
step_size = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
pr = synth.make_problem(cfg, m=m)
t = pkg.TTContext(pr.n, pr.r)
t.set_cores(pr.truth)
clean = t.eval_at(pr.idx)
t.close()
y = pr.observations(clean)
ctx = pkg.TTContext(pr.n, pr.r)
ctx.set_observations(pr.idx, y)
ctx.set_cores(pr.init)
NAMES = {0: "r2l_qr", 1: "r2l_push", 2: "l2r_qr", 3: "trunc", 4: "l2r_prod", 5: "orth_qr",
         8: "gram", 9: "reduce", 10: "chol", 11: "apply", 12: "racc", 15: "certify", 16: "fullJacobi",
         20: "round_total"}
COUNTS = {17: "cert_fail", 18: "qr_fallbacks", 14: "cross_sweeps", 19: "full_sweeps", 6: "orth_cholqr_ok", 21: "chols", 22: "first_order", 23: "cholqr_calls"}
prev = np.zeros(29)
for i in range(steps):
    show = i >= steps - 3
    ctx.step(step_size)
    e = ctx.debug("eps")
    dl = e - prev
    prev = e.copy()
    cyc = dl[5:]
    if show: print(f"step {i} res {ctx.residual_norm():.4e} jacobi_sweeps {dl[4]:.0f} " +
          " ".join(f"{n}={cyc[j] / 1.965e3:.0f}us" for j, n in NAMES.items()) + " " +
          " ".join(f"{n}={cyc[j]:.0f}" for j, n in COUNTS.items()))
