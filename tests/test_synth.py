"""Seeded input generator: determinism, shapes, sampling without replacement (CPU)."""
import math

import numpy as np
import pytest

import synth


@pytest.mark.parametrize("cfg,m", [(1, None), (2, None), (3, 5000), (4, 5000), (5, 20000), (6, None)])
def test_shapes_and_determinism(cfg, m):
    a = synth.make_problem(cfg, m=m)
    b = synth.make_problem(cfg, m=m)
    assert a.idx.dtype == np.int32 and a.idx.shape[1] == len(a.n)
    assert np.array_equal(a.idx, b.idx)
    for k in range(a.d):
        assert a.truth[k].shape == (a.r[k], a.n[k], a.r[k + 1])
        assert np.array_equal(a.truth[k], b.truth[k])
        assert a.idx[:, k].min() >= 0 and a.idx[:, k].max() < a.n[k]
    lin = np.zeros(a.m, dtype=np.int64)
    for k in range(a.d):
        lin = lin * a.n[k] + a.idx[:, k]
    assert np.unique(lin).size == a.m              # Omega is a set (reading R12)


def test_config_sizes():
    assert synth.make_problem(1).m == 2400
    assert synth.make_problem(2).m == 312500
    assert synth.mps_ranks(24, 8) == (1, 2, 4) + (8,) * 19 + (4, 2, 1)
    p5 = synth.make_problem(5, m=100000)
    assert p5.meta["duplicates"] == 100000 - p5.m


def test_qst_pauli_tensor_matches_dense_measurements():
    # Config 6: T*(a) = sum_{i,j} rho(i,j) W_a(i,j), rho = u u^dagger from the
    # bond-2 MPS, W_a the Kronecker product of the Pauli matrices; real
    # TT of rank s^2 = 4; unit trace (a = all identities).  Dense check at d = 5 (1024 entries).
    import itertools
    import oracle
    p = synth.make_problem(6, n=(4,) * 5, m=100)
    assert p.r == (1, 4, 4, 4, 4, 1)
    U = p.meta["mps"]
    u = U[0][0]                                      # [2, s1]
    for c in U[1:]:
        u = np.einsum("pa,aib->pib", u, c).reshape(-1, c.shape[2])
    u = u[:, 0]                                      # 2^5 amplitudes, qubit 1 most significant
    rho = np.outer(u, np.conj(u))
    assert math.isclose(np.trace(rho).real, 1.0, rel_tol=1e-12)
    idx = np.array(list(itertools.product(range(4), repeat=5)), dtype=np.int32)
    got = oracle.eval_at(p.truth, idx)
    ref = np.empty(idx.shape[0])
    for t, a in enumerate(idx):
        W = np.ones((1, 1), dtype=np.complex128)
        for ak in a:
            W = np.kron(W, synth.PAULI[ak])
        v = np.sum(rho * W)
        assert abs(v.imag) <= 1e-13
        ref[t] = v.real
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13)
    assert math.isclose(got[0], 1.0, rel_tol=1e-12)  # tr(rho)
    assert synth.make_problem(6).m == 80000          # OS = 200 at n = 10


def test_mps_unit_norm():
    p = synth.make_problem(4, m=10)
    assert math.isclose(synth._sq_norm_tt(p.truth), 1.0, rel_tol=1e-12)


def test_noise_models():
    p = synth.make_problem(2, m=1000)
    clean = np.ones(p.m) * 2.0
    y = p.observations(clean)
    np.testing.assert_allclose(y - clean, 1e-3 * 2.0 * p.noise_unit)
    p3 = synth.make_problem(3, m=1000)
    np.testing.assert_allclose(p3.observations(clean) - clean, 0.01 * p3.noise_unit)
