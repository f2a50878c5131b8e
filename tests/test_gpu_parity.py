"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same
seeded inputs.  Tolerances: bucketing bit-exact; evaluation /
residual entrywise <= 1e-13 relative to max|v|; one step <= 1e-11 relative
Frobenius (tensor, gauge-free, via the block-TT QR-sweep norm); 50 steps <= 1e-8."""
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
    clean = oracle.eval_at(pr.truth, pr.idx)
    y = pr.observations(clean)
    init = pr.init if pr.init is not None else oracle.spectral_init(pr.idx, y, pr.n, pr.r)
    return pr, y, init


def context(pkg, pr, y, init):
    ctx = pkg.TTContext(pr.n, pr.r)
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(init)
    return ctx


# Sizes the oracle finishes in seconds; each spans many buckets, split buckets
# (cfg3's 256 prefix rows hold ~3k samples each) and ragged tails.
CASES = [
    (1, None, {}),
    (2, None, {}),
    (3, 200_000, {}),
    (4, 200_000, {}),
    (5, 400_000, {}),
    (6, None, {}),     # QST workload shape: d=10, n=4, r=4, 80,000 samples
]


@pytest.mark.parametrize("cfg,m,kw", CASES)
def test_bucketing_bit_exact(pkg, cfg, m, kw):
    pr, y, init = problem(cfg, m, **kw)
    ctx = context(pkg, pr, y, init)
    KL, NL, NR = pkg.plan(pr.n, pr.r)
    assert KL == oracle.split_point(pr.n) and ctx.path == "tables"
    o = oracle.stable_order(pr.idx, pr.n, KL)
    assert np.array_equal(ctx.debug("perm_pre"), o["perm_pre"].astype(np.int32))
    assert np.array_equal(ctx.debug("perm_suf"), o["perm_suf"].astype(np.int32))
    assert np.array_equal(ctx.debug("offs_l"), o["offs_L"].astype(np.int64))
    assert np.array_equal(ctx.debug("offs_r"), o["offs_R"].astype(np.int64))
    ctx.close()


@pytest.mark.parametrize("cfg,m,kw", CASES)
def test_eval_residual_and_weights(pkg, cfg, m, kw):
    pr, y, init = problem(cfg, m, **kw)
    ctx = context(pkg, pr, y, init)
    rng = np.random.default_rng(7)
    held = np.stack([rng.integers(0, nk, 5000) for nk in pr.n], axis=1).astype(np.int32)
    for q in (pr.idx[:20000], held):
        got = ctx.eval_at(q)
        ref = oracle.eval_at(init, q)
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    g_ref = oracle.residual(init, pr.idx, y)
    g = ctx.debug("resid")
    assert np.max(np.abs(g - g_ref)) <= 1e-13 * max(np.max(np.abs(y)), 1e-300)
    res = ctx.residual_norm()
    assert abs(res - np.linalg.norm(g_ref)) <= 1e-12 * np.linalg.norm(g_ref)
    ctx.step(1.0)
    _, info = oracle.prgd_step(init, pr.idx, y, pr.n, pr.r, 1.0, return_info=True)
    eps = ctx.debug("eps")
    assert eps[0] == pytest.approx(info["eps"], rel=1e-12)
    assert eps[3] == pytest.approx(info["p"], rel=1e-15)
    assert eps[2] == pytest.approx(info["alpha"], rel=1e-12)
    for k in range(pr.d):
        np.testing.assert_allclose(ctx.debug("phi", k), info["phi"][k], rtol=1e-13)
    ctx.close()


@pytest.mark.parametrize("cfg,m,kw", CASES)
def test_one_step_parity(pkg, cfg, m, kw):
    pr, y, init = problem(cfg, m, **kw)
    ctx = context(pkg, pr, y, init)
    ctx.step(1.0)
    got = ctx.get_cores()
    ref, info = oracle.prgd_step(init, pr.idx, y, pr.n, pr.r, 1.0, return_info=True)
    # stage parity up to the QR gauge: U_gpu_k = D_{k-1} U_ref_k D_k with D = diag(+-1)
    # (CholeskyQR2 gives R with a positive diagonal, LAPACK's Householder need not);
    # Y_k transforms the same way (its interfaces are built from U).
    dprev = np.ones(1)
    for k in range(pr.d):
        Ur = info["U"][k]
        U = ctx.debug("u", k).reshape(Ur.shape) * dprev[:, None, None]
        dk = np.sign(np.einsum("ajb,ajb->b", U, Ur)) if k < pr.d - 1 else np.ones(Ur.shape[2])
        U = U * dk[None, None, :]
        np.testing.assert_allclose(U, Ur, rtol=0, atol=1e-11 * np.abs(Ur).max())
        Yr = info["Y"][k]
        Yk = ctx.debug("y", k).reshape(Yr.shape) * dprev[:, None, None] * dk[None, None, :]
        np.testing.assert_allclose(Yk, Yr, rtol=0, atol=1e-10 * np.abs(Yr).max())
        dprev = dk
    err = oracle.tt_diff_norm(got, ref)
    assert err <= 1e-11, err
    # output gauge: cores 0..d-2 left-orthogonal (A14)
    for k in range(pr.d - 1):
        Lk = got[k].reshape(-1, got[k].shape[2])
        np.testing.assert_allclose(Lk.T @ Lk, np.eye(Lk.shape[1]), atol=1e-12)
    ctx.close()


@pytest.mark.parametrize("cfg,m,steps", [(1, None, 50), (2, None, 50), (4, 300_000, 50), (6, None, 50)])
def test_many_steps_parity(pkg, cfg, m, steps):
    pr, y, init = problem(cfg, m)
    ctx = context(pkg, pr, y, init)
    T = init
    for _ in range(steps):
        ctx.step(1.0)
        T = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, 1.0)
    got = ctx.get_cores()
    err = oracle.tt_diff_norm(got, T)
    assert err <= 1e-8, err
    res = ctx.residual_norm()
    ref = float(np.linalg.norm(oracle.residual(T, pr.idx, y)))
    # relative 1e-8 plus a floor for residuals converged to rounding noise (config 4); the
    # iterate bar implies |res_gpu - res_orc| <~ 1e-8 ||y||
    assert abs(res - ref) <= 1e-8 * max(ref, 1e-300) + 1e-10 * np.linalg.norm(y)
    ctx.close()


def test_rules_rgd_fixed_raw(pkg):
    pr, y, init = problem(2, 50_000)
    for kw in [dict(eps_rule="none"), dict(eps_rule="fixed", eps_value=0.37),
               dict(eps_rule="vee", step_rule="raw")]:
        ctx = context(pkg, pr, y, init)
        ctx.set_metric(kw.get("eps_rule", "vee"), kw.get("eps_value", 0.0), kw.get("step_rule", "theory"))
        step = 0.5 if kw.get("step_rule") == "raw" else 1.0
        ctx.step(step)
        ref = oracle.prgd_step(init, pr.idx, y, pr.n, pr.r, step, **kw)
        assert oracle.tt_diff_norm(ctx.get_cores(), ref) <= 1e-11, kw
        ctx.close()


# Adaptive (steepest) step, PAPER.md:236-238 (and RGD's, 150-152, with eps_rule "none"): one
# more pass over Omega (the tangent vector at every sample).  Configs 1-3 and a config-5
# subsample: every table level shape, split buckets and the DMMA / fallback table kernels.
@pytest.mark.parametrize("cfg,m,eps_rule", [(1, None, "vee"), (2, 50_000, "vee"), (2, 50_000, "none"),
                                            (6, None, "vee"), (6, None, "none"),
                                            (3, 100_000, "vee"), (5, 200_000, "vee")])
def test_adaptive_step_matches_oracle(pkg, cfg, m, eps_rule):
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
        err = oracle.tt_diff_norm(ctx.get_cores(), T)
        assert err <= 1e-10, (it, err)
    ctx.close()


# Spectral initialisation at scale: the GPU's sparse TT-SVD of
# p^{-1} P_Omega(y) (Gram + Jacobi per mode, tt_spectral_init; config 3's 4096-row unfolding by
# the right Gram) against the oracle's dense Alg. 1 (numpy SVD of the densified tensor) on the
# shapes of configs 1-6.
@pytest.mark.parametrize("cfg,kw", [(1, {}), (2, dict(n=(20, 20, 20, 20), m=40_000)),
                                    (3, dict(m=60_000)),    # full 256x256x128 shape: r_1 n_2 = 4096 rows
                                    (4, dict(n=(2,) * 14, m=3_000)),
                                    (5, dict(n=(6,) * 6, r=(1, 4, 4, 4, 4, 4, 1), m=20_000)),
                                    (6, {})])
def test_spectral_init_matches_dense_tt_svd(pkg, cfg, kw):
    pr = synth.make_problem(cfg, **kw)
    y = pr.observations(oracle.eval_at(pr.truth, pr.idx))
    ctx = pkg.TTContext(pr.n, pr.r)
    ctx.set_observations(pr.idx, y)
    ctx.spectral_init()
    got = ctx.get_cores()
    ref = oracle.spectral_init(pr.idx, y, pr.n, pr.r)
    err = oracle.tt_diff_norm(got, ref)
    assert err <= 1e-9, err
    for k in range(pr.d - 1):                     # orthonormal columns (Alg. 1)
        Lk = got[k].reshape(-1, got[k].shape[2])
        np.testing.assert_allclose(Lk.T @ Lk, np.eye(Lk.shape[1]), atol=1e-12)
    ctx.step(1.0)                                 # the init feeds the step
    ref1 = oracle.prgd_step(got, pr.idx, y, pr.n, pr.r, 1.0)
    assert oracle.tt_diff_norm(ctx.get_cores(), ref1) <= 1e-11
    ctx.close()


def test_exact_fit_is_noop_and_edge_cases(pkg):
    pr, _, init = problem(1)
    # Integer cores: every chain product is exact in fp64 in any order, so G = 0
    # exactly on both sides -> eps = 0 -> the step is a no-op (reading R4).
    rng = np.random.default_rng(5)
    icores = [rng.integers(-2, 3, size=c.shape).astype(np.float64) for c in init]
    yi = oracle.eval_at(icores, pr.idx)
    ctx = context(pkg, pr, yi, icores)
    assert ctx.residual_norm() == 0.0
    ctx.step(1.0)
    for k in range(pr.d):
        np.testing.assert_array_equal(ctx.get_core(k), icores[k])
    ctx.close()
    # y = T_l(Omega) up to rounding: eps is tiny but nonzero; the tensor moves <= 1e-13
    y = oracle.eval_at(init, pr.idx)
    ctx = context(pkg, pr, y, init)
    ctx.step(1.0)
    assert oracle.tt_diff_norm(ctx.get_cores(), init) <= 1e-13
    ctx.close()
    # out-of-range observation index
    ctx = pkg.TTContext(pr.n, pr.r)
    bad = pr.idx.copy()
    bad[5, 1] = pr.n[1]
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.set_observations(bad, y)
    assert ei.value.code == pkg.TT_ERR_INDEX
    # empty Omega: residual 0, step refused
    ctx.set_observations(np.zeros((0, pr.d), np.int32), np.zeros(0))
    ctx.set_cores(init)
    assert ctx.residual_norm() == 0.0
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.step(1.0)
    assert ei.value.code == pkg.TT_ERR_STATE
    assert ctx.eval_at(np.zeros((0, pr.d), np.int32)).shape == (0,)
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.eval_at(bad[:10])
    assert ei.value.code == pkg.TT_ERR_INDEX
    ctx.close()
    # stepping before cores are set
    ctx = pkg.TTContext(pr.n, pr.r)
    ctx.set_observations(pr.idx, y)
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.step(1.0)
    assert ei.value.code == pkg.TT_ERR_STATE
    ctx.close()


def test_single_sample_and_matrix_case(pkg):
    # degenerate sizes: d = 2 (matrix completion), one observed entry
    rng = np.random.default_rng(3)
    n, r = (7, 5), (1, 2, 1)
    cores = [rng.standard_normal((r[k], n[k], r[k + 1])) for k in range(2)]
    idx = np.array([[3, 4]], dtype=np.int32)
    y = np.array([0.25])
    ctx = pkg.TTContext(n, r)
    ctx.set_observations(idx, y)
    ctx.set_cores(cores)
    ctx.step(1.0)
    ref = oracle.prgd_step(cores, idx, y, n, r, 1.0)
    assert oracle.tt_diff_norm(ctx.get_cores(), ref) <= 1e-11
    ctx.close()


def test_maximal_rank_and_rule_limits(pkg):
    # r = 32 = kMaxRank: rank-2r = 64 unfoldings exceed the cluster sweeps' S <= 32 and take
    # the single-CTA Householder path; the adaptive rule evaluates its denominator by
    # per-sample chains of the rank-64 tangent TT (2r > 32); the spectral init's third step
    # (r_2 n_3 = 1280 > 1024 rows) takes the right-Gram path.
    rng = np.random.default_rng(21)
    n, r = (8, 40, 40, 8), (1, 8, 32, 8, 1)
    truth = [rng.standard_normal((r[k], n[k], r[k + 1])) / math.sqrt(r[k + 1]) for k in range(4)]
    N = math.prod(n)
    lin = rng.choice(N, size=30_000, replace=False)
    idx = np.stack(np.unravel_index(lin, n), axis=1).astype(np.int32)
    y = oracle.eval_at(truth, idx)
    init = [c + 0.05 * rng.standard_normal(c.shape) for c in truth]
    ctx = pkg.TTContext(n, r)
    ctx.set_observations(idx, y)
    ctx.set_cores(init)
    T = init
    for _ in range(2):
        ctx.step(1.0)
        T = oracle.prgd_step(T, idx, y, n, r, 1.0)
        assert oracle.tt_diff_norm(ctx.get_cores(), T) <= 1e-11
    ctx.set_metric("vee", 0.0, "adaptive")
    for _ in range(2):
        ctx.step(1.0)
        T, info = oracle.prgd_step(T, idx, y, n, r, 1.0, step_rule="adaptive", return_info=True)
        alpha = ctx.debug("eps")[2]
        assert abs(alpha - info["alpha"]) <= 1e-10 * info["alpha"], (alpha, info["alpha"])
        assert oracle.tt_diff_norm(ctx.get_cores(), T) <= 1e-10
    ctx.spectral_init()
    assert oracle.tt_diff_norm(ctx.get_cores(), oracle.spectral_init(idx, y, n, r)) <= 1e-9
    ctx.close()


def test_full_size_config5_properties(pkg):
    # BASELINE config 5 at full size (3e7 samples, bench.py's launch configuration): A0 bucketing
    # bit-exact against the oracle's stable order; tt_eval_at on 1e4 sampled indices against the
    # oracle; then properties that hold at any size over three steps toward a rank-16 truth whose
    # values are cheap to form exactly (bond-diagonal cores: T(x) = sum_a prod_k c_k[a, x_k],
    # evaluated here in chunks): finite, left-orthogonal output cores, monotonically decreasing
    # residual, and the returned iterate's values on sampled indices equal the oracle's
    # evaluation of the returned cores.
    pr = synth.make_problem(5)
    rng = np.random.default_rng(55)
    KL, NL, NR = pkg.plan(pr.n, pr.r)
    R = pr.r[1]
    c = [rng.uniform(0.5, 1.5, size=(R, nk)) for nk in pr.n]
    y = np.empty(pr.m)
    for s0 in range(0, pr.m, 1 << 20):
        blk = pr.idx[s0:s0 + (1 << 20)]
        acc = np.ones((blk.shape[0], R))
        for k in range(pr.d):
            acc *= c[k][:, blk[:, k]].T
        y[s0:s0 + blk.shape[0]] = acc.sum(axis=1)
    truth = []
    for k in range(pr.d):
        r0, r1 = pr.r[k], pr.r[k + 1]
        core = np.zeros((r0, pr.n[k], r1))
        for a in range(R):
            core[0 if r0 == 1 else a, :, 0 if r1 == 1 else a] = c[k][a]
        truth.append(core)
    ctx = pkg.TTContext(pr.n, pr.r)
    ctx.set_observations(pr.idx, y)
    o = oracle.stable_order(pr.idx, pr.n, KL)
    assert np.array_equal(ctx.debug("perm_pre"), o["perm_pre"].astype(np.int32))
    assert np.array_equal(ctx.debug("perm_suf"), o["perm_suf"].astype(np.int32))
    assert np.array_equal(ctx.debug("offs_l"), o["offs_L"].astype(np.int64))
    assert np.array_equal(ctx.debug("offs_r"), o["offs_R"].astype(np.int64))
    del o
    q = np.stack([rng.integers(0, nk, size=10_000) for nk in pr.n], axis=1).astype(np.int32)
    ctx.set_cores(truth)
    assert ctx.residual_norm() <= 1e-12 * np.linalg.norm(y)     # the values above are T*(Omega)
    init = [t + 0.05 * rng.standard_normal(t.shape) * np.abs(t).max() for t in truth]
    ctx.set_cores(init)
    np.testing.assert_allclose(ctx.eval_at(q), oracle.eval_at(init, q), rtol=0,
                               atol=1e-12 * np.abs(oracle.eval_at(init, q)).max())
    res = [ctx.residual_norm()]
    for _ in range(3):
        ctx.step(1.0)
        res.append(ctx.residual_norm())
        cores = ctx.get_cores()
        assert all(np.all(np.isfinite(cc)) for cc in cores)
        for k in range(pr.d - 1):
            Lk = cores[k].reshape(-1, cores[k].shape[2])
            np.testing.assert_allclose(Lk.T @ Lk, np.eye(Lk.shape[1]), atol=1e-12)
        ref = oracle.eval_at(cores, q)
        np.testing.assert_allclose(ctx.eval_at(q), ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    assert all(b < a for a, b in zip(res, res[1:])), res
    assert res[-1] < 0.1 * res[0], res
    ctx.close()


# Weighted retraction W^{-1/2} SVD_r^tt W^{1/2} (Remark; tt_set_retraction) on
# both paths: one step <= 1e-11, ten steps <= 1e-9 against the oracle's "weighted" retraction.
@pytest.mark.parametrize("cfg,m,path,steps", [(1, None, "tables", 1), (2, 50_000, "tables", 10),
                                              (5, 200_000, "tables", 1), (6, None, "tables", 1),
                                              (2, 50_000, "chains", 1)])
def test_weighted_retraction(pkg, cfg, m, path, steps):
    pr, y, init = problem(cfg, m)
    ctx = pkg.TTContext(pr.n, pr.r, path=path)
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(init)
    ctx.set_retraction("weighted")
    T = init
    for it in range(steps):
        ctx.step(1.0)
        T = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, 1.0, retraction="weighted")
    err = oracle.tt_diff_norm(ctx.get_cores(), T)
    assert err <= (1e-11 if steps == 1 else 1e-9), err
    plain = oracle.prgd_step(init, pr.idx, y, pr.n, pr.r, 1.0)
    if steps == 1:
        assert oracle.tt_diff_norm(plain, T) > 1e-9      # the variant is a different iterate
    ctx.close()


# Numeric faults (reading R6, include/prgd.h): tt_prgd_step is asynchronous, so a fault raised on
# the device is reported by the next synchronising call as TT_ERR_NUMERIC, once (the flag is
# cleared when read), and the faulting update leaves the iterate unchanged (noop).
@pytest.mark.parametrize("path", ["tables", "chains"])
def test_numeric_faults_reported_by_next_sync(pkg, path):
    pr, y, init = problem(2, 20_000)
    # NaN in an observed value: the residual is not finite
    ybad = y.copy()
    ybad[17] = np.nan
    ctx = pkg.TTContext(pr.n, pr.r, path=path)
    ctx.set_observations(pr.idx, ybad)
    ctx.set_cores(init)
    ctx.step(1.0)                                    # enqueued: no status yet
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.sync()
    assert ei.value.code == pkg.TT_ERR_NUMERIC
    ctx.sync()                                       # reported once
    for k in range(pr.d):
        np.testing.assert_array_equal(ctx.get_core(k), init[k])
    ctx.close()
    # rank-deficient right Gram: a zero last core makes P_{d-1} = 0 (Cholesky breakdown)
    zero = [c.copy() for c in init]
    zero[-1][:] = 0.0
    ctx = pkg.TTContext(pr.n, pr.r, path=path)
    ctx.set_observations(pr.idx, y)
    ctx.set_cores(zero)
    ctx.step(1.0)
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.residual_norm()
    assert ei.value.code == pkg.TT_ERR_NUMERIC and "Cholesky" in str(ei.value)
    got = ctx.get_cores()
    assert all(np.array_equal(a, b) for a, b in zip(got, zero))
    ctx.close()


# Race detection by determinism (compute-sanitizer is closed on this GPU pool, profiles/
# r02_sanitizer.md): every reduction of the library has a fixed order, so two independent runs of
# the same steps must give bit-identical cores and residuals; a shared-memory or cluster race
# would show up as run-to-run differences.
@pytest.mark.parametrize("cfg,m,path,rule", [(2, 50_000, "tables", "theory"), (2, 50_000, "chains", "theory"),
                                             (5, 200_000, "tables", "adaptive"), (4, 100_000, "tables", "theory"),
                                             (3, 100_000, "tables", "theory")])
def test_bitwise_deterministic(pkg, cfg, m, path, rule):
    pr, y, init = problem(cfg, m)
    outs = []
    for rep in range(2):
        ctx = pkg.TTContext(pr.n, pr.r, path=path)
        ctx.set_observations(pr.idx, y)
        ctx.set_cores(init)
        ctx.set_metric("vee", 0.0, rule)
        res = []
        for _ in range(3):
            ctx.step(0.5 if cfg == 3 else 1.0)
            res.append(ctx.residual_norm())
        outs.append((ctx.get_cores(), res, ctx.debug("resid")))
        ctx.close()
    (c0, r0, g0), (c1, r1, g1) = outs
    assert r0 == r1
    assert all(np.array_equal(a, b) for a, b in zip(c0, c1))
    assert np.array_equal(g0, g1)


# A14 alone (tt_debug_round) on constructed rank-2r block TTs whose bond-1 spectrum is known: the
# kept group ends in a weak direction (0.3) just above the discarded group (0.25 / 0.299), so the
# cluster truncation's norm-ordered split is not the answer from the start (the
# cross-angle exit of the one-sided Jacobi must not certify a wrong split).  d = 3,
# n = (20, 10, 16), r = (1, 8, 8, 1): B_0 = U diag(sigma) (U orthonormal 20 x 16), B_1 B_2 an
# orthonormal right part, so W^<1> = U diag(sigma) Q^T exactly.  Against the oracle's
# numpy-SVD TT-rounding (Alg. 1), tensors compared.
@pytest.mark.parametrize("gap", [0.05, 1e-3])
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_rounding_weak_kept_direction(pkg, gap, seed):
    rng = np.random.default_rng(100 + seed)
    n, r = (20, 10, 16), (1, 8, 8, 1)
    kept = np.array([5.0, 4.5, 4.0, 3.5, 3.0, 2.5, 2.0, 0.3])
    disc = np.array([0.3 - gap, 0.2, 0.1, 0.05, 1e-3, 1e-4, 1e-6, 1e-8])
    sig = np.concatenate([kept, disc])[rng.permutation(16)]
    U, _ = np.linalg.qr(rng.standard_normal((20, 16)))
    Q, _ = np.linalg.qr(rng.standard_normal((10 * 16, 16)))
    B0 = (U * sig[None, :])[None, :, :]                       # [1][20][16]
    B1 = Q.T.reshape(16, 10, 16)                              # [16][10][16]
    B2 = np.eye(16)[:, :, None]                               # [16][16][1]
    ref = oracle.tt_round([B0, B1, B2], r)
    ctx = pkg.TTContext(n, r)
    e0 = ctx.debug("eps")
    ctx.debug_round([B0, B1, B2])
    got = ctx.get_cores()
    e1 = ctx.debug("eps")
    err = oracle.tt_diff_norm(got, ref)
    assert err <= 1e-11, (err, e1[4] - e0[4])
    np.testing.assert_allclose(got[0].reshape(20, 8).T @ got[0].reshape(20, 8), np.eye(8), atol=1e-12)
    # bond 1 kept exactly the kept singular directions: the first core spans U's kept columns
    Uk = U[:, np.isin(sig, kept)]
    P0 = got[0].reshape(20, 8)
    np.testing.assert_allclose(np.linalg.svd(Uk.T @ P0, compute_uv=False), np.ones(8), atol=1e-12)
    print(f"seed {seed} gap {gap}: err {err:.2e}, Jacobi sweeps {int(e1[4] - e0[4])}, "
          f"cross {int(e1[5 + 14] - e0[5 + 14])}, full {int(e1[5 + 19] - e0[5 + 19])}, "
          f"cert failures {int(e1[5 + 17] - e0[5 + 17])}")
    ctx.close()


@pytest.mark.parametrize("cfg,m,nslices", [(5, 400_000, 3), (3, 200_000, 5), (2, None, 7), (4, 200_000, 2)])
def test_sliced_suffix_pass(pkg, cfg, m, nslices, monkeypatch):
    """Pass A suffix by slices of g (the default once g exceeds one ~48 MB slice, i.e. at config
    5's full size) forced at oracle-sized inputs: H_R-based weights, pass B through the staged
    g, one step and three steps against the oracle, and the same iterates as the row-plan
    gather up to the summation order of H_R."""
    pr, y, init = problem(cfg, m)
    monkeypatch.setenv("PRGD_GSQ_SLICES", str(nslices))
    ctx = context(pkg, pr, y, init)
    monkeypatch.setenv("PRGD_GSQ_SLICES", "1")
    ref_ctx = context(pkg, pr, y, init)
    ctx.residual_norm()
    ref, info = oracle.prgd_step(init, pr.idx, y, pr.n, pr.r, 1.0, return_info=True)
    ctx.step(1.0)
    ref_ctx.step(1.0)
    eps = ctx.debug("eps")
    assert eps[0] == pytest.approx(info["eps"], rel=1e-12)
    assert eps[2] == pytest.approx(info["alpha"], rel=1e-12)
    for k in range(pr.d):
        np.testing.assert_allclose(ctx.debug("phi", k), info["phi"][k], rtol=1e-13)
    assert oracle.tt_diff_norm(ctx.get_cores(), ref) <= 1e-11
    assert oracle.tt_diff_norm(ctx.get_cores(), ref_ctx.get_cores()) <= 1e-13
    step = 0.5 if cfg == 3 else 1.0
    T = ref
    for _ in range(2):
        ctx.step(step)
        T = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, step)
    assert oracle.tt_diff_norm(ctx.get_cores(), T) <= 1e-10
    ctx.close()
    ref_ctx.close()


# tt_set_observations_u8 (include/prgd.h): byte multi-indices are widened on the device and then
# bucketed exactly like the int32 call, so everything downstream must be bit-identical -- the
# bucketing, the residual vector, and the iterates of two steps -- on both paths; sizes with a
# ragged tail of the 16-indices-per-thread widening kernel (m d not a multiple of 16).
@pytest.mark.parametrize("cfg,m,path", [(2, 50_001, "tables"), (2, 50_001, "chains"), (3, 100_003, "tables"),
                                        (5, 200_001, "tables"), (1, None, "tables")])
def test_byte_indices_identical_to_int32(pkg, cfg, m, path):
    pr, y, init = problem(cfg, m)
    assert pr.idx.max() < 256
    outs = []
    for dt in (np.int32, np.uint8):
        ctx = pkg.TTContext(pr.n, pr.r, path=path)
        ctx.set_observations(pr.idx.astype(dt), y)
        ctx.set_cores(init)
        res = [ctx.residual_norm()]
        g = ctx.debug("resid")
        for _ in range(2):
            ctx.step(0.5 if cfg == 3 else 1.0)
            res.append(ctx.residual_norm())
        outs.append((ctx.get_cores(), res, g))
        ctx.close()
    (c0, r0, g0), (c1, r1, g1) = outs
    assert r0 == r1
    assert np.array_equal(g0, g1)
    assert all(np.array_equal(a, b) for a, b in zip(c0, c1))


def test_byte_indices_errors(pkg):
    # an index outside [0, n_k) is reported like the int32 call; mode sizes above 256 are refused
    pr, y, init = problem(2, 1000)
    ctx = pkg.TTContext(pr.n, pr.r)
    bad = pr.idx.astype(np.uint8)
    bad[17, 2] = pr.n[2]
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.set_observations(bad, y)
    assert ei.value.code == pkg.TT_ERR_INDEX
    ctx.set_observations(pr.idx.astype(np.uint8), y)        # the context stays usable
    ctx.set_cores(init)
    assert np.isfinite(ctx.residual_norm())
    ctx.close()
    ctx = pkg.TTContext([300, 20, 20], [1, 2, 2, 1])
    with pytest.raises(pkg.PRGDError) as ei:
        ctx.set_observations(np.zeros((4, 3), np.uint8), np.zeros(4))
    assert ei.value.code == pkg.TT_ERR_ARG
    ctx.close()
