"""Diagnostic: Jacobi sweeps and per-phase cycles of the dense sweeps at config 5."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth, paper_2501_13385_b200 as pkg

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
pr = synth.make_problem(cfg, m=200000)
t = pkg.TTContext(pr.n, pr.r); t.set_cores(pr.truth); clean = t.eval_at(pr.idx); t.close()
y = pr.observations(clean)
ctx = pkg.TTContext(pr.n, pr.r); ctx.set_observations(pr.idx, y); ctx.set_cores(pr.init)
names = ["r2l_qr", "r2l_prod", "l2r_qr", "jacobi", "l2r_prod+orth_gram", "orth_qr", "n_cholqr_ok", "n_fallback_early"]
prev = np.zeros(13)
for i in range(5):
    ctx.step(1.0)
    e = ctx.debug("eps")
    dl = e - prev; prev = e.copy()
    print(f"step {i} res {ctx.residual_norm():.4e} sweeps {dl[4]:.0f} " +
          " ".join(f"{n}={dl[5 + j] / 1.9e3:.0f}us" for j, n in enumerate(names[:5])) +
          f" fallback_late={dl[10]:.0f} cholqr_ok={dl[11]:.0f} fallback_early={dl[12]:.0f}")
