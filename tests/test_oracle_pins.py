"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the passage of PAPER.md / SPEC.md it pins, and the mistake it
would catch.  Brute-force references live in tests/_brute.py and share no code
with oracle/."""
import itertools
import math

import numpy as np
import pytest

import oracle
import synth
from tests import _brute as bf


def rand_tt(rng, n, r, scale=1.0):
    return [scale * rng.standard_normal((r[k], n[k], r[k + 1])) for k in range(len(n))]


def all_indices(n):
    return np.array(list(itertools.product(*[range(k) for k in n])), dtype=np.int32)


# ----------------------------------------------------------------- A1 evaluation
@pytest.mark.parametrize("n,r", [((4, 5, 3), (1, 2, 3, 1)), ((3, 2, 4, 2), (1, 3, 2, 2, 1)),
                                 ((6, 7), (1, 3, 1))])
def test_eval_matches_entrywise_products(n, r):
    # catches a transposed slice, wrong mode order or dropped core.
    rng = np.random.default_rng(0)
    cores = rand_tt(rng, n, r)
    idx = all_indices(n)
    v = oracle.eval_at(cores, idx)
    ref = np.array([bf.entry(cores, x) for x in idx])
    np.testing.assert_allclose(v, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    np.testing.assert_allclose(oracle.to_dense(cores), bf.dense(cores), rtol=1e-13, atol=1e-13)


def test_eval_spec_examples():
    # all-ones rank-1 TT -> 1; zero slice annihilates; rank-1 = outer product.
    ones = [np.ones((1, 2, 1)) for _ in range(3)]
    assert np.all(oracle.eval_at(ones, all_indices((2, 2, 2))) == 1.0)
    rng = np.random.default_rng(1)
    cores = rand_tt(rng, (3, 4, 5), (1, 2, 2, 1))
    cores[1][:, 2, :] = 0.0
    idx = all_indices((3, 4, 5))
    v = oracle.eval_at(cores, idx)
    assert np.all(v[idx[:, 1] == 2] == 0.0) and np.any(v[idx[:, 1] != 2] != 0.0)
    u = [rng.standard_normal(k) for k in (3, 4, 5)]
    r1 = [u[0][None, :, None], u[1][None, :, None], u[2][None, :, None]]
    np.testing.assert_allclose(oracle.to_dense(r1), np.einsum("i,j,k->ijk", *u), rtol=1e-14)


# ----------------------------------------------------------------- A3 weights
def test_mode_sums_are_row_norms_of_unfoldings():
    # diag(M_i(G) M_i(G)^T) — catches summing g instead of g^2 or wrong mode.
    rng = np.random.default_rng(2)
    n = (4, 3, 5)
    idx = all_indices(n)[rng.choice(60, 25, replace=False)]
    g = rng.standard_normal(25)
    G = bf.sampled_dense(n, idx, g)
    h = oracle.mode_sums(g, idx, n)
    for k in range(3):
        Mk = np.moveaxis(G, k, 0).reshape(n[k], -1)
        np.testing.assert_allclose(h[k], (Mk * Mk).sum(axis=1), rtol=1e-14)


def test_vee_norm_and_weights_spec_examples():
    # two entries in one mode-1 slice with values 3 and 4 -> 5.
    idx = np.array([[0, 0, 0], [0, 1, 1]], dtype=np.int32)
    assert oracle.vee_norm(np.array([3.0, 4.0]), idx, (2, 2, 2)) == 5.0
    # one observed entry v at x -> diag[i][x_i] = eps + v^2, others eps; eps = v^2
    v = 1.5
    idx = np.array([[1, 0, 2]], dtype=np.int32)
    h = oracle.mode_sums(np.array([v]), idx, (2, 3, 4))
    eps, w, phi = oracle.build_weights(h, 3)
    assert eps == v * v
    for k, xk in enumerate(idx[0]):
        expect = np.full(w[k].shape, eps)
        expect[xk] = eps + v * v
        np.testing.assert_array_equal(w[k], expect)
        np.testing.assert_allclose(phi[k], expect ** (1 / 12), rtol=1e-15)
    # zero residual -> eps = 0 flags the no-op branch (reading R4)
    eps0, _, _ = oracle.build_weights(oracle.mode_sums(np.zeros(1), idx, (2, 3, 4)), 3)
    assert eps0 == 0.0


def test_theory_step_and_os_examples():
    # SPEC.md:393 (Thm 4.1): alpha = 1.001 eps^{1/2}/p
    assert oracle.theory_step(1.0, 0.5) == pytest.approx(2.002, abs=1e-15)
    assert oracle.theory_step(4.0, 1.0) == pytest.approx(2.002, abs=1e-15)
    # SPEC.md:460 / PAPER.md:521: (100^3, r=5, OS=7) -> dim 3450, |Omega| 24150
    assert oracle.os_dim((100,) * 3, (1, 5, 5, 1)) == 3450
    assert oracle.os_to_m((100,) * 3, (1, 5, 5, 1), 7) == 24150
    # 10 qubits, Pauli tensor 4^10, r=4, OS=200 -> "around 7.6%"
    m = oracle.os_to_m((4,) * 10, (1,) + (4,) * 9 + (1,), 200)
    assert m == 80000 and abs(m / 4 ** 10 - 0.076) < 0.001


# ----------------------------------------------------------------- Prop 3.1 / Lemma 4.2
def test_component_weighting_prop31():
    # W T = [T_k ×_2 G_k^{1/(2m)}] — catches scaling the wrong mode/power.
    rng = np.random.default_rng(3)
    n, r = (3, 4, 2), (1, 2, 2, 1)
    cores = rand_tt(rng, n, r)
    w = [rng.uniform(0.5, 3.0, k) for k in n]
    d = 3
    phi2 = [wk ** (1 / (2 * d)) for wk in w]          # G^{1/(2m)} diagonal
    lhs = bf.dense(cores) * bf.weight_diag(n, w, d)
    rhs = oracle.to_dense(oracle.weight_cores(cores, phi2, 1.0))
    np.testing.assert_allclose(rhs, lhs, rtol=1e-13)


def test_norm_equivalence_lemma42():
    # eps^{1/2} ||Z||^2 <= ||Z||_W^2 <= (eps + ||G||_vee^2)^{1/2} ||Z||^2
    rng = np.random.default_rng(4)
    n = (4, 3, 5)
    idx = all_indices(n)[rng.choice(60, 30, replace=False)]
    g = rng.standard_normal(30)
    h = oracle.mode_sums(g, idx, n)
    eps, w, _ = oracle.build_weights(h, 3)
    D = bf.weight_diag(n, w, 3)
    vee2 = oracle.vee_norm(g, idx, n) ** 2
    for _ in range(20):
        Z = rng.standard_normal(n)
        zw = float((D * Z * Z).sum())
        zf = float((Z * Z).sum())
        assert math.sqrt(eps) * zf <= zw * (1 + 1e-14)
        assert zw <= math.sqrt(eps + vee2) * zf * (1 + 1e-14)


# ----------------------------------------------------------------- A5 / A6
def test_left_orthogonalize_and_right_grams():
    # L(U_k)^T L(U_k) = I, tensor unchanged; PAPER.md:104-110 / 358:
    # P_k equals the Gram of the right part T^{>=k+1} computed entry by entry.
    rng = np.random.default_rng(5)
    n, r = (3, 4, 3, 2), (1, 2, 3, 2, 1)
    cores = rand_tt(rng, n, r)
    U = oracle.left_orthogonalize(cores)
    for k in range(3):
        L = U[k].reshape(-1, U[k].shape[2])
        np.testing.assert_allclose(L.T @ L, np.eye(L.shape[1]), atol=1e-13)
    np.testing.assert_allclose(oracle.to_dense(U), bf.dense(cores), rtol=1e-12, atol=1e-12)
    P = oracle.right_grams(U)
    for k in range(3):                       # P[k] = P_{k+1}: right part from core k+1 on
        tail = U[k + 1:]
        cols = []
        for x in itertools.product(*[range(c.shape[1]) for c in tail]):
            v = np.eye(tail[0].shape[0])
            for c, xi in zip(tail, x):
                v = v @ c[:, xi, :]
            cols.append(v[:, 0])
        R = np.array(cols).T
        np.testing.assert_allclose(P[k], R @ R.T, rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------- A7-A11 projection
def _weights_for(rng, n, idx, g, d):
    h = oracle.mode_sums(g, idx, n)
    return oracle.build_weights(h, d)


@pytest.mark.parametrize("n,r", [((3, 4, 3), (1, 2, 2, 1)), ((2, 2, 2), (1, 1, 1, 1)),
                                 ((2, 3, 2, 3), (1, 2, 2, 2, 1))])
@pytest.mark.parametrize("rule", ["vee", "none"])
def test_gradient_equals_bruteforce_jacobian_projection(n, r, rule):
    # Lemma P~ = W^{-1/2} P_That W^{1/2} and the closed form
    # (356-360): the PRGD direction P~_T W^{-1} G must equal J (J^T D J)^+ J^T G
    # (W-orthogonal projection onto range J).  Catches a missing Gram inverse,
    # a missing gauge projection, wrong phi power or a wrong last-core rule.
    rng = np.random.default_rng(6)
    d = len(n)
    cores = rand_tt(rng, n, r)
    N = math.prod(n)
    idx = all_indices(n)[rng.choice(N, max(2, int(0.6 * N)), replace=False)]
    g = rng.standard_normal(idx.shape[0])
    eps, w, phi = oracle.build_weights(oracle.mode_sums(g, idx, n), d, rule)
    ghat = oracle.precondition_residual(g, idx, phi)
    tv = oracle.tangent_direction(cores, phi, idx, ghat)
    got = oracle.to_dense(oracle.tangent_sum(tv["Ttil"], tv["A"]))
    Dw = bf.weight_diag(n, w, d)
    G = bf.sampled_dense(n, idx, g)
    ref = bf.weighted_tangent_projection(cores, Dw, G / Dw)    # P~ (W^{-1} G)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-10 * np.abs(ref).max())


@pytest.mark.parametrize("n,r", [((3, 4, 3), (1, 2, 2, 1)), ((2, 3, 2, 3), (1, 2, 2, 2, 1))])
@pytest.mark.parametrize("rule", ["vee", "none"])
def test_adaptive_step_equals_bruteforce_steepest_step(n, r, rule):
    # eq. `PRGD stepsize` and, for W = I, RGD's step:
    # alpha = ||D||_W^2 / ||P_Omega D||^2 with D the dense brute-force W-projection of W^{-1}G.
    # Also the line-search identity ||D||_W^2 = <G, D> (D is the W-orthogonal projection of
    # W^{-1}G), so alpha minimises f(T - alpha D).  Catches a numerator without the weights,
    # a dropped component, non-orthogonal components or a wrong denominator.
    rng = np.random.default_rng(11)
    d = len(n)
    cores = rand_tt(rng, n, r)
    N = math.prod(n)
    idx = all_indices(n)[rng.choice(N, max(2, int(0.6 * N)), replace=False)]
    g = rng.standard_normal(idx.shape[0])
    eps, w, phi = oracle.build_weights(oracle.mode_sums(g, idx, n), d, rule)
    ghat = oracle.precondition_residual(g, idx, phi)
    tv = oracle.tangent_direction(cores, phi, idx, ghat)
    alpha, num, den = oracle.adaptive_step(1.0, tv["U"], tv["Ahat"], tv["Ttil"], tv["A"], idx)
    Dw = bf.weight_diag(n, w, d)
    G = bf.sampled_dense(n, idx, g)
    Dref = bf.weighted_tangent_projection(cores, Dw, G / Dw)
    num_ref = float(np.sum(Dw * Dref * Dref))
    dv = Dref[tuple(idx.T)]
    den_ref = float(dv @ dv)
    assert abs(num - num_ref) <= 1e-9 * num_ref
    assert abs(den - den_ref) <= 1e-9 * den_ref
    assert abs(num_ref - float(g @ dv)) <= 1e-9 * num_ref          # <G, D> = ||D||_W^2
    assert abs(alpha - num_ref / den_ref) <= 1e-9 * alpha
    assert abs(oracle.adaptive_step(0.5, tv["U"], tv["Ahat"], tv["Ttil"], tv["A"], idx)[0]
               - 0.5 * alpha) <= 1e-12 * alpha


def test_adaptive_prgd_step_minimises_objective_along_direction():
    # The adaptive step is the exact minimiser of f(T_l - alpha D) over alpha
    # (`argmin_alpha`), f = 1/2 sum_Omega (T - y)^2 evaluated densely.
    rng = np.random.default_rng(12)
    n, r = (4, 3, 4), (1, 2, 2, 1)
    truth = rand_tt(rng, n, r)
    T0 = oracle.tt_add(truth, rand_tt(rng, n, r, 0.3))
    T0 = oracle.tt_round(T0, r)
    N = math.prod(n)
    idx = all_indices(n)[rng.choice(N, int(0.7 * N), replace=False)]
    y = oracle.eval_at(truth, idx)
    _, info = oracle.prgd_step(T0, idx, y, n, r, 1.0, step_rule="adaptive", return_info=True)
    D = oracle.to_dense(oracle.tangent_sum(info["Ttil"], info["A"]))
    T = bf.dense(T0)
    Y = bf.sampled_dense(n, idx, y)
    mask = bf.sampled_dense(n, idx, np.ones(idx.shape[0])) > 0

    def f(a):
        return 0.5 * float(np.sum(((T - a * D) - Y)[mask] ** 2))

    a = info["alpha"]
    assert a > 0
    for t in (0.9, 0.99, 1.01, 1.1):
        assert f(a) < f(t * a)


def test_projection_idempotent_selfadjoint_and_components_orthogonal():
    # SPEC.md:306/322-323 idempotence & self-adjointness in <.,.>_W; Lemma component
    # orthogonal; Def. 3.2 weighted orthogonality.
    rng = np.random.default_rng(7)
    n, r = (3, 4, 3, 2), (1, 2, 3, 2, 1)
    d = 4
    cores = rand_tt(rng, n, r)
    idx_all = all_indices(n)
    g = rng.standard_normal(idx_all.shape[0])
    eps, w, phi = oracle.build_weights(oracle.mode_sums(g, idx_all, n), d)
    Dw = bf.weight_diag(n, w, d)
    sq = np.sqrt(Dw).ravel()                               # W^{1/2} entry factors

    def Pt(Z):                                             # P~_T Z for dense Z
        zhat = Z.ravel() * sq
        tv = oracle.tangent_direction(cores, phi, idx_all, zhat)
        return oracle.to_dense(oracle.tangent_sum(tv["Ttil"], tv["A"])), tv

    Z1, Z2 = rng.standard_normal(n), rng.standard_normal(n)
    X, tv = Pt(Z1)
    XX, _ = Pt(X)
    np.testing.assert_allclose(XX, X, rtol=1e-10, atol=1e-11 * np.abs(X).max())
    Y, _ = Pt(Z2)
    lhs, rhs = float((Dw * X * Z2).sum()), float((Dw * Z1 * Y).sum())
    assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1.0)
    assert float((Dw * X * X).sum()) <= float((Dw * Z1 * Z1).sum()) * (1 + 1e-12)
    comps = []
    for k in range(d):
        Ak = [tv["Ttil"][i] if i != k else tv["A"][k] for i in range(d)]
        comps.append(oracle.to_dense(Ak))
    for i in range(d):
        for j in range(i + 1, d):
            ip = float((Dw * comps[i] * comps[j]).sum())
            assert abs(ip) <= 1e-10 * math.sqrt(float((Dw * comps[i] ** 2).sum()) *
                                                float((Dw * comps[j] ** 2).sum())) + 1e-14
    for k in range(d - 1):
        T = tv["Ttil"][k]
        Gm = np.einsum("ajb,j,ajc->bc", T, phi[k] ** 2, T)
        np.testing.assert_allclose(Gm, np.eye(T.shape[2]), atol=1e-12)
        # gauge condition [A_k, Ttil_k]_W = 0
        gauge = np.einsum("ajb,j,ajc->bc", tv["A"][k], phi[k] ** 2, T)
        assert np.abs(gauge).max() <= 1e-11 * max(1.0, np.abs(tv["A"][k]).max())


def test_matrix_case_textbook_projector():
    # m = 2: the fixed-rank matrix tangent projector UU^T Z + Z VV^T - UU^T Z VV^T at
    # That = W^{1/2} T, conjugated by W^{-1/2}, G^{1/(4m)} = w^{1/8}.
    rng = np.random.default_rng(8)
    n, r = (7, 6), (1, 3, 1)
    cores = rand_tt(rng, n, r)
    idx = all_indices(n)[rng.choice(42, 30, replace=False)]
    g = rng.standard_normal(30)
    eps, w, phi = oracle.build_weights(oracle.mode_sums(g, idx, n), 2)
    tv = oracle.tangent_direction(cores, phi, idx, oracle.precondition_residual(g, idx, phi))
    got = oracle.to_dense(oracle.tangent_sum(tv["Ttil"], tv["A"]))
    s1, s2 = w[0] ** 0.125, w[1] ** 0.125                      # W^{1/2} row / column factors
    That = s1[:, None] * bf.dense(cores) * s2[None, :]
    Uu, _, Vt = np.linalg.svd(That)
    Uu, V = Uu[:, :3], Vt[:3].T
    Ghat = bf.sampled_dense(n, idx, g) / s1[:, None] / s2[None, :]
    Pu, Pv = Uu @ Uu.T, V @ V.T
    ref = (Pu @ Ghat + Ghat @ Pv - Pu @ Ghat @ Pv) / s1[:, None] / s2[None, :]
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())


# ----------------------------------------------------------------- A13-A14 retraction
def test_tt_svd_exact_and_quasi_optimal():
    # Alg. 1: exact on TT-rank-r input; left-orthogonal output;
    # quasi-optimality tail bound.
    rng = np.random.default_rng(9)
    n, r = (4, 5, 3, 4), (1, 2, 3, 2, 1)
    X = bf.dense(rand_tt(rng, n, r))
    C = oracle.tt_svd(X, r)
    np.testing.assert_allclose(oracle.to_dense(C), X, rtol=1e-10, atol=1e-12 * np.abs(X).max())
    for k in range(3):
        L = C[k].reshape(-1, C[k].shape[2])
        np.testing.assert_allclose(L.T @ L, np.eye(L.shape[1]), atol=1e-12)
    Z = rng.standard_normal((5, 5, 5))
    rr = (1, 2, 2, 1)
    err2 = float(((oracle.to_dense(oracle.tt_svd(Z, rr)) - Z) ** 2).sum())
    tail = 0.0
    for i in (1, 2):
        s = np.linalg.svd(Z.reshape(5 ** i, -1), compute_uv=False)
        tail += float((s[rr[i]:] ** 2).sum())
    assert err2 <= tail * (1 + 1e-10)


@pytest.mark.parametrize("n,r", [((3, 4, 3), (1, 2, 2, 1)), ((2, 2, 2, 2, 2), (1, 2, 2, 2, 2, 1)),
                                 ((5, 4), (1, 2, 1))])
def test_rounding_equals_dense_tt_svd(n, r):
    # structured TT-rounding of the rank-2r update == Alg. 1 on the
    # densified W_l; idempotent on manifold points.
    rng = np.random.default_rng(10)
    cores = rand_tt(rng, n, r)
    A = rand_tt(rng, n, r, 0.3)
    Ttil = oracle.left_orthogonalize(cores)
    B = oracle.assemble(Ttil, A, 0.7)
    dense_W = oracle.to_dense(B)
    # A13 check: B represents T - alpha sum_k [Ttil..A_k..Ttil]
    ref_W = bf.dense(Ttil) - 0.7 * sum(
        bf.dense([Ttil[i] if i != k else A[k] for i in range(len(n))]) for k in range(len(n)))
    np.testing.assert_allclose(dense_W, ref_W, rtol=1e-12, atol=1e-12 * np.abs(ref_W).max())
    got = oracle.to_dense(oracle.tt_round(B, r))
    ref = oracle.to_dense(oracle.tt_svd(dense_W, r))
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-11 * np.abs(ref).max())
    same = oracle.to_dense(oracle.tt_round(cores, r))
    np.testing.assert_allclose(same, bf.dense(cores), rtol=1e-10, atol=1e-11 * np.abs(same).max())


def test_diff_norm_matches_dense():
    rng = np.random.default_rng(11)
    n, r = (3, 4, 5), (1, 2, 3, 1)
    a, b = rand_tt(rng, n, r), rand_tt(rng, n, r)
    da, db = bf.dense(a), bf.dense(b)
    assert oracle.tt_diff_norm(a, b) == pytest.approx(np.linalg.norm(da - db) / np.linalg.norm(db), rel=1e-12)
    assert oracle.tt_norm(a) == pytest.approx(np.linalg.norm(da), rel=1e-13)


# ----------------------------------------------------------------- whole step
def test_zero_gradient_at_truth_is_noop():
    # Noiseless data, T_l = T*: G = 0 -> eps = 0 -> T_{l+1} = T_l (reading R4).
    rng = np.random.default_rng(12)
    n, r = (5, 4, 6), (1, 2, 2, 1)
    T = rand_tt(rng, n, r)
    idx = all_indices(n)[rng.choice(120, 60, replace=False)]
    y = oracle.eval_at(T, idx)                      # bitwise T_l(Omega): G = 0 exactly
    new, info = oracle.prgd_step(T, idx, y, n, r, 1.0, return_info=True)
    assert info["noop"]
    assert all(np.array_equal(a, b) for a, b in zip(new, T))
    # values from an independent evaluation differ by rounding only: eps tiny, step ~1e-14
    y2 = np.array([bf.entry(T, x) for x in idx])
    new2 = oracle.prgd_step(T, idx, y2, n, r, 1.0)
    assert oracle.tt_diff_norm(new2, T) <= 1e-13


def test_full_observation_rgd_converges_quadratically():
    # p = 1, W = I, raw alpha = 1: T_{l+1} = SVD_r(T_l - P_T(T_l - T*)), error O(e^2)
    # (PAPER.md:715-720).  Catches any first-order error in projection or retraction.
    rng = np.random.default_rng(13)
    n, r = (4, 5, 4), (1, 2, 2, 1)
    Tstar = rand_tt(rng, n, r)
    idx = all_indices(n)
    y = np.array([bf.entry(Tstar, x) for x in idx])
    errs = []
    for delta in (1e-2, 1e-3):
        T0 = [c + delta * rng.standard_normal(c.shape) for c in Tstar]
        e0 = oracle.tt_diff_norm(T0, Tstar)
        T1 = oracle.prgd_step(T0, idx, y, n, r, 1.0, eps_rule="none", step_rule="raw")
        errs.append((e0, oracle.tt_diff_norm(T1, Tstar)))
    for e0, e1 in errs:
        assert e1 < 50 * e0 * e0
    assert errs[1][1] < errs[0][1] * 0.05


def test_geometric_decay_on_exact_low_rank_data():
    # Noiseless, generous sampling (cfg1 recipe): error decays geometrically under the
    # theory step (Thm 4.1); ratio < 1 for >= 90% of iterations.
    import synth
    pr = synth.make_problem(1)
    y = oracle.eval_at(pr.truth, pr.idx)
    T = oracle.spectral_init(pr.idx, y, pr.n, pr.r)
    errs = [oracle.tt_diff_norm(T, pr.truth)]
    for _ in range(40):
        T = oracle.prgd_step(T, pr.idx, y, pr.n, pr.r, 1.0)
        errs.append(oracle.tt_diff_norm(T, pr.truth))
    ratios = np.array(errs[6:]) / np.array(errs[5:-1])
    assert np.mean(ratios < 1.0) >= 0.9
    assert errs[-1] < 1e-3 * errs[0]


# ----------------------------------------------------------------- A0 bucketing
def test_stable_order_matches_python_sort():
    # Stable sort is unique: compare with Python's sorted() on explicit tuples.
    rng = np.random.default_rng(14)
    n = (3, 5, 2, 4)
    idx = rng.integers(0, 1, size=(200, 4)).astype(np.int32)
    for k in range(4):
        idx[:, k] = rng.integers(0, n[k], 200)
    KL = oracle.split_point(n)
    o = oracle.stable_order(idx, n, KL)
    pre = sorted(range(200), key=lambda s: (tuple(idx[s, :KL]), tuple(idx[s, KL:][::-1]), s))
    suf = sorted(range(200), key=lambda s: (tuple(idx[s, KL:][::-1]), tuple(idx[s, :KL]), s))
    assert list(o["perm_pre"]) == pre and list(o["perm_suf"]) == suf
    assert o["offs_L"][-1] == 200 and o["offs_R"][-1] == 200
    P = o["P"][o["perm_pre"]]
    assert np.all(np.diff(P) >= 0)
    for j in range(len(o["offs_L"]) - 1):
        assert np.all(P[o["offs_L"][j]:o["offs_L"][j + 1]] == j)


def test_split_point():
    assert oracle.split_point((16,) * 10) == 5
    assert oracle.split_point((2,) * 24) == 12
    assert oracle.split_point((50,) * 4) == 2
    assert oracle.split_point((256, 256, 128)) == 1
    assert oracle.split_point((20, 20, 20)) == 1


def test_stable_buckets_match_python_sort():
    # Per-mode buckets (the chain path): perm_k = the stable order of the
    # sample ids by x_k, i.e. Python's sorted() on the key (x_{s,k}, s); offs_k = exclusive
    # cumulative bucket counts, empty buckets included.
    rng = np.random.default_rng(17)
    n = (3, 7, 1, 4)
    m = 250
    idx = np.stack([rng.integers(0, nk, m) for nk in n], axis=1).astype(np.int32)
    idx[:, 1] = np.where(idx[:, 1] == 5, 6, idx[:, 1])          # bucket 5 of mode 1 stays empty
    out = oracle.stable_buckets(idx, n)
    for k in range(len(n)):
        perm, offs = out[k]
        assert list(perm) == sorted(range(m), key=lambda s: (int(idx[s, k]), s))
        assert len(offs) == n[k] + 1 and offs[0] == 0 and offs[-1] == m
        for j in range(n[k]):
            assert offs[j + 1] - offs[j] == int(np.sum(idx[:, k] == j))
            assert np.all(idx[perm[offs[j]:offs[j + 1]], k] == j)
    assert out[1][1][6] == out[1][1][5]


# ----------------------------------------------------------------- weighted retraction
def test_weighted_retraction_matches_dense_definition():
    # Remark at PAPER.md:365-367: T_{l+1} = W^{-1/2} SVD_r^tt(W^{1/2} W_l).  Dense check: W_l
    # densified from the step's rank-2r blocks, W^{+-1/2} as the Kronecker diagonal
    # prod_k phi_{k,x_k}^{+-1} applied entrywise, SVD_r^tt as the literal dense
    # Alg. 1 (tt_svd); with eps_rule "none" (phi = 1) the two retractions coincide.
    pr = synth.make_problem(1, seed=99, n=(5, 6, 4), r=(1, 2, 2, 1), m=60)
    y = oracle.eval_at(pr.truth, pr.idx)
    T0 = [c + 0.3 * np.random.default_rng(1).standard_normal(c.shape) for c in pr.truth]
    new, info = oracle.prgd_step(T0, pr.idx, y, pr.n, pr.r, 1.0, return_info=True,
                                 retraction="weighted")
    Wd = oracle.to_dense(info["B"])
    D = np.einsum("i,j,k->ijk", *info["phi"])
    ref = oracle.to_dense(oracle.tt_svd(Wd * D, pr.r)) / D
    assert np.linalg.norm(oracle.to_dense(new) - ref) <= 1e-12 * np.linalg.norm(ref)
    plain = oracle.to_dense(oracle.prgd_step(T0, pr.idx, y, pr.n, pr.r, 1.0))
    assert np.linalg.norm(plain - ref) > 1e-6 * np.linalg.norm(ref)     # a different iterate
    a = oracle.prgd_step(T0, pr.idx, y, pr.n, pr.r, 1.0, eps_rule="none", retraction="weighted")
    b = oracle.prgd_step(T0, pr.idx, y, pr.n, pr.r, 1.0, eps_rule="none")
    assert oracle.tt_diff_norm(a, b) <= 1e-13


def test_spectral_init_rescales_by_inverse_p():
    # BASELINE.json config 1 / SPEC.md:371-376: T_0 = SVD_r^tt(p^{-1} P_Omega(y)).  At full TT rank
    # (r_k = min(prod_{i<=k} n_i, prod_{i>k} n_i)) Alg. 1 is exact, so the initial tensor must equal
    # the zero-filled observations divided by p = |Omega| / prod(n) entrywise: a x p or missing
    # rescaling fails by a factor p^2 or p.
    rng = np.random.default_rng(31)
    n = (3, 4, 2)
    r = (1, 3, 2, 1)
    N = 24
    lin = rng.choice(N, size=9, replace=False)
    idx = np.stack(np.unravel_index(lin, n), axis=1).astype(np.int32)
    y = rng.standard_normal(9)
    T0 = oracle.to_dense(oracle.spectral_init(idx, y, n, r))
    ref = np.zeros(n)
    ref[tuple(idx.T)] = y * (N / 9.0)
    np.testing.assert_allclose(T0, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


def test_step_length_theory_rule_worked_examples():
    # Thm 4.1: alpha_l = 1.001 eps_l^{1/2} / p; SPEC.md:393 worked values 2.002 at
    # (eps, p) = (1, 0.5) and (4, 1) -- through the rule prgd_step actually calls (A12).
    assert oracle.step_length(1.001, 1.0, 0.5) == pytest.approx(2.002, rel=1e-15)
    assert oracle.step_length(1.001, 4.0, 1.0) == pytest.approx(2.002, rel=1e-15)
    assert oracle.step_length(0.5, 9.0, 0.25) == pytest.approx(6.0, rel=1e-15)
    assert oracle.step_length(0.3, None, 0.2) == pytest.approx(1.5, rel=1e-15)   # W = I: step / p
    assert oracle.step_length(0.7, 123.0, 0.01, "raw") == 0.7
    # and prgd_step reports exactly that alpha for its own eps and p
    pr = synth.make_problem(1)
    y = oracle.eval_at(pr.truth, pr.idx)
    T0 = [c + 0.1 for c in pr.truth]
    _, info = oracle.prgd_step(T0, pr.idx, y, pr.n, pr.r, 1.001, return_info=True)
    assert info["alpha"] == pytest.approx(1.001 * math.sqrt(info["eps"]) / 0.3, rel=1e-15)
