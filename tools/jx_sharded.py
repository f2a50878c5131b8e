"""Diagnostic: print the sharded two-context parity errors (tests/test_gpu_sharded.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import test_gpu_sharded as t  # noqa: E402

orig = oracle.tt_diff_norm


def wrap(a, b, relative=True):
    v = orig(a, b, relative)
    print(f"  diff {v:.3e}", flush=True)
    return v


oracle.tt_diff_norm = wrap
for args in [(2, 20000, 3, "theory"), (5, 60000, 2, "theory"), (2, 20000, 2, "adaptive")]:
    print(args, flush=True)
    try:
        t.test_sharded_two_contexts_match_oracle(*args)
    except AssertionError as e:
        print("  FAIL", str(e)[:80])
