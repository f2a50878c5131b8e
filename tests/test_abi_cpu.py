"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/prgd.h declares, and the host-side validation / planning behaves as
documented (no compute calls)."""
import ctypes
import re

import pytest

import paper_2501_13385_b200 as pkg


def header_symbols():
    text = open(pkg.HEADER).read()
    return sorted(set(re.findall(r"PRGD_API\s+(?:const\s+)?\w+\*?\s+(tt_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = pkg.load()
    syms = header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    raw = ctypes.CDLL(pkg.LIB_PATH)
    for s in syms:
        assert getattr(raw, s) is not None


def test_plan_split_and_validation():
    assert pkg.plan((16,) * 10, (1,) + (16,) * 9 + (1,)) == (5, 16 ** 5, 16 ** 5)
    assert pkg.plan((256, 256, 128), (1, 16, 16, 1)) == (1, 256, 256 * 128)
    assert pkg.plan((2,) * 24, (1, 2, 4) + (8,) * 19 + (4, 2, 1)) == (12, 4096, 4096)
    assert pkg.plan((20, 20, 20), (1, 2, 2, 1)) == (1, 20, 400)
    assert pkg.plan((7, 5), (1, 2, 1)) == (1, 7, 5)
    bad = [((4, 4), (1, 5, 1), pkg.TT_ERR_RANK),          # r_1 > min(n_1, n_2)
           ((4, 4, 4), (2, 2, 2, 1), pkg.TT_ERR_RANK),     # r_0 != 1
           ((2, 3, 2), (1, 2, 5, 1), pkg.TT_ERR_RANK),     # r_2 > r_1 n_2 = 6? no: > n_3 r_3 = 2
           ((4,), (1, 1), pkg.TT_ERR_ARG),                 # d < 2
           ((100,) * 4, (1, 33, 33, 33, 1), pkg.TT_ERR_UNSUPPORTED)]
    for n, r, code in bad:
        with pytest.raises(pkg.PRGDError) as ei:
            pkg.plan(n, r)
        assert ei.value.code == code, (n, r)
    # shapes whose prefix / suffix tables cannot fit resolve to the per-sample chain path
    # (tt_plan reports K_L = 0): 2^40 rows per side, or d = 16 binary-free n = 16 (16^8 rows)
    assert pkg.plan((1 << 20,) * 4, (1, 2, 2, 2, 1)) == (0, 0, 0)
    assert pkg.plan((16,) * 16, (1,) + (8,) * 15 + (1,)) == (0, 0, 0)


def test_create_validates_before_touching_the_device():
    lib = pkg.load()
    h = ctypes.c_void_p()
    rc = lib.tt_create(2, pkg._i64((4, 4)), pkg._i64((1, 5, 1)), ctypes.byref(h))
    assert rc == pkg.TT_ERR_RANK and not h.value
    assert lib.tt_destroy(None) == pkg.TT_OK
    assert lib.tt_last_error(None) == b"no context"
    assert lib.tt_profile_name(0) == b"tables_C" and lib.tt_profile_name(99) == b""


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(pkg.PRGDError) as ei:
        pkg.TTContext((20, 20, 20), (1, 2, 2, 1))
    assert ei.value.code == pkg.TT_ERR_CUDA
