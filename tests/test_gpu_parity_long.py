"""Long GPU parity against stored oracle iterates (tests/golden, written by
tools/make_golden.py from synth + oracle only): the configurations BASELINE.json's north star
names at their full sizes, through the C-ABI, in bench.py's launch configuration.

Tolerances (BASELINE.json north star): relative Frobenius error of the iterate (gauge-free,
block-TT QR norm) <= 1e-11 after one step from the identical state and <= 1e-8 after 50
iterations; intermediate saved iterates <= 1e-8; residual norms <= 1e-8 relative plus a
1e-10 ||y|| floor for residuals converged to rounding noise (config 4)."""
import numpy as np
import pytest

import oracle
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2501_13385_b200 as p
    p.load()
    return p


@pytest.mark.parametrize("case,path", [("cfg3_full_50steps", "tables"), ("cfg4_full_50steps", "tables"),
                                       ("cfg5_4e6_50steps", "tables"),
                                       # full config 5: the 10-step reference (its step 1 is the one-step
                                       # check at 1e-11; cfg5_full_1step.npz holds the same first iterate
                                       # and is kept for tools / the CPU fingerprint test only, so that
                                       # the suite draws the 3e7-sample problem twice, not four times)
                                       ("cfg5_full_10steps", "tables"),
                                       # the per-sample chain path on the same references
                                       ("cfg3_full_50steps", "chains"), ("cfg4_full_50steps", "chains"),
                                       ("cfg5_4e6_50steps", "chains"), ("cfg5_full_10steps", "chains")])
def test_golden_iterates(pkg, case, path):
    cfg, m, step, steps, keep = G.CASES[case]
    gold = G.load(case)                     # a missing file fails the test (no skip)
    pr = G.problem(cfg, m)
    assert G.input_sha(pr) == gold["sha"], "stale golden file: synth inputs changed"
    y = G.observations(pr)
    assert pr.m == gold["m"]
    assert abs(float(np.sum(y)) - gold["ysum"]) <= 1e-10 * np.sqrt(gold["ysq"] * pr.m)
    assert abs(float(np.dot(y, y)) - gold["ysq"]) <= 1e-12 * gold["ysq"]
    ctx = pkg.TTContext(pr.n, pr.r, path=path)
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(pr.init)
    res0 = ctx.residual_norm()
    assert abs(res0 - gold["res"][0]) <= 1e-11 * gold["res"][0]
    errs = {}
    for it in range(1, gold["steps"] + 1):
        ctx.step(step)
        if it < len(gold["res"]):
            r = ctx.residual_norm()
            # relative 1e-8, plus a floor for the runs that converge to machine precision
            # (config 4: residual ~5e-13 ||y||, rounding noise of two independent runs).  The
            # iterate bar 1e-8 itself implies |res_gpu - res_orc| <= ||P_Omega(T_gpu - T_orc)||
            # ~ 1e-8 ||y||; 1e-10 ||y|| keeps the check well inside that
            tol = 1e-8 * gold["res"][it] + 1e-10 * np.sqrt(gold["ysq"])
            assert abs(r - gold["res"][it]) <= tol, (it, r, gold["res"][it])
        if it in gold["iterates"]:
            err = oracle.tt_diff_norm(ctx.get_cores(), gold["iterates"][it])
            errs[it] = err
            assert err <= (1e-11 if it == 1 else 1e-8), (it, err)
    ctx.close()
    print(f"{case} ({path}): relative errors {errs}")
