"""Seeded input generator: determinism, shapes, sampling without replacement (CPU)."""
import math

import numpy as np
import pytest

import synth


@pytest.mark.parametrize("cfg,m", [(1, None), (2, None), (3, 5000), (4, 5000), (5, 20000)])
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
