"""The stored oracle iterates (tests/golden) exist for every long-parity case and still match
the seeded inputs synth produces (CPU; the full-size config 5 fingerprint is checked by the
GPU test itself, since drawing 3e7 indices is slow here)."""
import numpy as np
import pytest

from tests import _golden as G


@pytest.mark.parametrize("case", sorted(G.CASES))
def test_golden_file_present_and_consistent(case):
    gold = G.load(case)
    cfg, m, step, steps, keep = G.CASES[case]
    assert gold["steps"] == steps and gold["step_size"] == step
    assert sorted(gold["iterates"]) == sorted(keep)
    res = gold["res"]
    assert np.all(np.isfinite(res))
    assert steps == 1 or res[-1] < res[0]                      # the oracle run descended
    if m is not None or cfg != 5:
        pr = G.problem(cfg, m)
        assert G.input_sha(pr) == gold["sha"]
        assert pr.m == gold["m"]
