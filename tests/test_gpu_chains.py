"""GPU parity of the per-sample chain path (TT_PATH_CHAINS, chains.cu) against the oracle:
the per-mode buckets (A0) bit-exact, evaluation / residual entrywise, one step <= 1e-11 and
50 steps <= 1e-8 relative Frobenius (BASELINE.json north star) on the BASELINE configs at
oracle-friendly sizes, the adaptive rule, and a shape the table planner refuses (d = 15,
n = 16, r = 8: 16^7 / 16^8-row tables), where TT_PATH_AUTO resolves to the chains."""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2501_13385_b200 as p
    p.load()
    return p


def problem(cfg, m=None, **kw):
    pr = synth.make_problem(cfg, m=m, **kw)
    y = pr.observations(oracle.eval_at(pr.truth, pr.idx))
    init = pr.init if pr.init is not None else oracle.spectral_init(pr.idx, y, pr.n, pr.r)
    return pr, y, init


def context(pkg, pr, y, init, path="chains"):
    ctx = pkg.TTContext(pr.n, pr.r, path=path)
    assert ctx.path == "chains"
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(init)
    return ctx


# d = 15, n = 16, r = 8: max(N_L, N_R) = 16^8 = 2^32 rows > 2^30, so the planner refuses tables
REFUSED = dict(n=(16,) * 15, r=(1,) + (8,) * 14 + (1,))

CASES = [(1, None, {}), (2, 50_000, {}), (3, 100_000, {}), (4, 100_000, {}), (5, 200_000, {}),
         (6, None, {})]


@pytest.mark.parametrize("cfg,m,kw", CASES)
def test_chain_buckets_eval_and_one_step(pkg, cfg, m, kw):
    pr, y, init = problem(cfg, m, **kw)
    ctx = context(pkg, pr, y, init)
    ref_b = oracle.stable_buckets(pr.idx, pr.n)
    for k in range(pr.d):
        assert np.array_equal(ctx.debug("perm_mode", k), ref_b[k][0].astype(np.int32))
        assert np.array_equal(ctx.debug("offs_mode", k), ref_b[k][1].astype(np.int64))
    rng = np.random.default_rng(8)
    held = np.stack([rng.integers(0, nk, 5000) for nk in pr.n], axis=1).astype(np.int32)
    for q in (pr.idx[:20000], held):
        got = ctx.eval_at(q)
        ref = oracle.eval_at(init, q)
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    g_ref = oracle.residual(init, pr.idx, y)
    assert np.max(np.abs(ctx.debug("resid") - g_ref)) <= 1e-13 * max(np.max(np.abs(y)), 1e-300)
    assert abs(ctx.residual_norm() - np.linalg.norm(g_ref)) <= 1e-12 * np.linalg.norm(g_ref)
    ref, info = oracle.prgd_step(init, pr.idx, y, pr.n, pr.r, 1.0, return_info=True)
    for k in range(pr.d):       # h of the current iterate (A3), by bucket pieces
        np.testing.assert_allclose(ctx.debug("h", k), info["h"][k], rtol=1e-12,
                                   atol=1e-14 * max(info["h"][k].max(), 1e-300))
    ctx.step(1.0)
    eps = ctx.debug("eps")
    assert eps[0] == pytest.approx(info["eps"], rel=1e-12)
    assert eps[2] == pytest.approx(info["alpha"], rel=1e-12)
    err = oracle.tt_diff_norm(ctx.get_cores(), ref)
    assert err <= 1e-11, err
    ctx.close()


@pytest.mark.parametrize("cfg,m", [(1, None), (2, 50_000), (6, None)])   # cfg 3-5: test_gpu_parity_long
def test_chain_many_steps(pkg, cfg, m):
    pr, y, init = problem(cfg, m)
    ctx = context(pkg, pr, y, init)
    T = init
    for _ in range(50):
        ctx.step(1.0)
        T = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, 1.0)
    assert oracle.tt_diff_norm(ctx.get_cores(), T) <= 1e-8
    ref = float(np.linalg.norm(oracle.residual(T, pr.idx, y)))
    assert abs(ctx.residual_norm() - ref) <= 1e-8 * max(ref, 1e-300) + 1e-10 * np.linalg.norm(y)
    ctx.close()


@pytest.mark.parametrize("cfg,m,eps_rule", [(1, None, "vee"), (2, 50_000, "none"), (5, 100_000, "vee")])
def test_chain_adaptive_step(pkg, cfg, m, eps_rule):
    pr, y, init = problem(cfg, m)
    ctx = context(pkg, pr, y, init)
    ctx.set_metric(eps_rule, 0.0, "adaptive")
    T = init
    for it in range(3):
        ctx.step(1.0)
        T, info = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, 1.0, eps_rule=eps_rule,
                                   step_rule="adaptive", return_info=True)
        alpha = ctx.debug("eps")[2]
        assert abs(alpha - info["alpha"]) <= 1e-10 * info["alpha"], (it, alpha, info["alpha"])
        assert oracle.tt_diff_norm(ctx.get_cores(), T) <= 1e-10
    ctx.close()


def test_table_path_refused_shape_runs_on_chains(pkg):
    # a shape the table planner refuses: AUTO resolves to chains, TABLES is unsupported
    assert pkg.plan(REFUSED["n"], REFUSED["r"]) == (0, 0, 0)
    with pytest.raises(pkg.PRGDError) as ei:
        pkg.TTContext(REFUSED["n"], REFUSED["r"], path="tables")
    assert ei.value.code == pkg.TT_ERR_UNSUPPORTED
    pr, y, init = problem(5, 1_000_000, **REFUSED)
    ctx = pkg.TTContext(pr.n, pr.r)
    assert ctx.path == "chains"
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(init)
    T = init
    for it in range(1, 11):
        ctx.step(1.0)
        T = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, 1.0)
        if it in (1, 10):
            err = oracle.tt_diff_norm(ctx.get_cores(), T)
            assert err <= (1e-11 if it == 1 else 1e-9), (it, err)
    ctx.close()


def test_chain_edge_cases(pkg):
    pr, y, init = problem(1)
    # out-of-range observed index, empty Omega, stepping without cores
    ctx = pkg.TTContext(pr.n, pr.r, path="chains")
    bad = pr.idx.copy()
    bad[7, 2] = -1
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.set_observations(bad, y)
    assert ei.value.code == pkg.TT_ERR_INDEX
    ctx.set_observations(np.zeros((0, pr.d), np.int32), np.zeros(0))
    ctx.set_cores(init)
    assert ctx.residual_norm() == 0.0
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.step(1.0)
    assert ei.value.code == pkg.TT_ERR_STATE
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.eval_at(bad[:10])
    assert ei.value.code == pkg.TT_ERR_INDEX
    ctx.close()
    # the path is fixed before data is set
    ctx = pkg.TTContext(pr.n, pr.r)
    ctx.set_cores(init)
    with pytest.raises(pkg.PRGDError) as ei:
        ctx._check(ctx.lib.tt_set_path(ctx._h, pkg.PATHS["chains"]), "tt_set_path")
    assert ei.value.code == pkg.TT_ERR_STATE
    ctx.close()
    # one observed entry, d = 2; odd ranks; a slice with no samples
    rng = np.random.default_rng(3)
    n, r = (7, 5), (1, 2, 1)
    cores = [rng.standard_normal((r[k], n[k], r[k + 1])) for k in range(2)]
    idx = np.array([[3, 4]], dtype=np.int32)
    yy = np.array([0.25])
    ctx = pkg.TTContext(n, r, path="chains")
    ctx.set_observations(idx, yy)
    ctx.set_cores(cores)
    ctx.step(1.0)
    assert oracle.tt_diff_norm(ctx.get_cores(), oracle.prgd_step(cores, idx, yy, n, r, 1.0)) <= 1e-11
    ctx.close()


def test_chain_maximal_rank_adaptive(pkg):
    # r = 32 on the chain path: 32-lane chains, contraction tiles 4 x 4, adaptive D at rank 64
    rng = np.random.default_rng(22)
    n, r = (8, 40, 40, 8), (1, 8, 32, 8, 1)
    truth = [rng.standard_normal((r[k], n[k], r[k + 1])) / math.sqrt(r[k + 1]) for k in range(4)]
    lin = rng.choice(math.prod(n), size=30_000, replace=False)
    idx = np.stack(np.unravel_index(lin, n), axis=1).astype(np.int32)
    y = oracle.eval_at(truth, idx)
    init = [c + 0.05 * rng.standard_normal(c.shape) for c in truth]
    ctx = pkg.TTContext(n, r, path="chains")
    ctx.set_observations(idx, y)
    ctx.set_cores(init)
    ctx.set_metric("vee", 0.0, "adaptive")
    T = init
    for _ in range(2):
        ctx.step(1.0)
        T = oracle.prgd_step(T, idx, y, n, r, 1.0, step_rule="adaptive")
        assert oracle.tt_diff_norm(ctx.get_cores(), T) <= 1e-10
    ctx.close()
