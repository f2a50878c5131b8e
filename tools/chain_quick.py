import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, oracle, synth
import paper_2501_13385_b200 as pkg
for cfg, m in [(1, None), (2, 50000), (5, 100000)]:
    pr = synth.make_problem(cfg, m=m)
    y = pr.observations(oracle.eval_at(pr.truth, pr.idx))
    init = pr.init if pr.init is not None else oracle.spectral_init(pr.idx, y, pr.n, pr.r)
    ctx = pkg.TTContext(pr.n, pr.r, path="chains")
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(init)
    print(cfg, 'res', ctx.residual_norm(), np.linalg.norm(oracle.residual(init, pr.idx, y)), flush=True)
    ctx.step(1.0)
    ref = oracle.prgd_step(init, pr.idx, y, pr.n, pr.r, 1.0)
    print(cfg, 'one step err', oracle.tt_diff_norm(ctx.get_cores(), ref), flush=True)
    ctx.close()
