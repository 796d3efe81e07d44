"""CPU: the C-ABI library loads, exports every symbol include/l1b.h declares,
and refuses to compute without a GPU (no silent CPU fallback)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "l1b.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"^[A-Za-z_][\w \*]*?\b(l1b_\w+)\s*\(", text, flags=re.M))
    return sorted(names)


def test_header_declares_abi():
    names = declared_functions()
    assert "l1b_solve" in names and "l1b_generate" in names and len(names) >= 25


def test_library_exports_every_declared_symbol():
    from paper_1503_03520_b200 import _native

    lib = _native.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    bound = {s[0] for s in _native.SIGNATURES}
    assert set(declared_functions()) == bound


def test_library_is_sm100a_only():
    from paper_1503_03520_b200 import _native

    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_host_rng_primitives_match_oracle(oracle):
    """The product's host RNG streams (std::mt19937_64) equal the oracle's."""
    import numpy as np

    from paper_1503_03520_b200 import _native as N

    lib = N.load()
    assert lib.l1b_mix_seed(3, 0) == oracle.mix_seed(3, 0)
    mp = np.empty(1000, dtype=np.uint32)
    N.check(lib.l1b_realize_permutation(1000, 77, mp.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    ref_map = np.empty(1000, dtype=np.uint32)
    inv = np.empty(1000, dtype=np.uint32)
    oracle.lib.lo_permutation_realize(1000, 77, ref_map.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                      inv.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    np.testing.assert_array_equal(mp, ref_map)
    sig = np.empty(500)
    N.check(lib.l1b_realize_spectrum_uniform(500, 0.0, 10.0, 0.1, 9, sig.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    ref = np.empty(500)
    oracle.lib.lo_spectrum_uniform(500, 0.0, 10.0, 0.1, 9, ref.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    np.testing.assert_array_equal(sig, ref)


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1503_03520_b200 import l1bench

    with pytest.raises(Exception):
        l1bench.build_instance(64, stages=1)


def test_invalid_arguments_map_to_value_error():
    from paper_1503_03520_b200 import l1bench

    with pytest.raises(ValueError):
        l1bench.SolverConfig(id="bogus").to_c()
    with pytest.raises(ValueError):
        l1bench.build_instance(1)  # ExperimentConfig: dimensions must be at least 2


def test_solver_cfg_default_takes_the_arithmetic_from_the_environment():
    """l1b_solver_cfg_default (SolverConfig's defaults, solvers.hpp:19-38): the
    reference's bits unless L1B_ARITH=fma -- the switch of callers without a
    field for the mode (the reference-side drop-in)."""
    from paper_1503_03520_b200 import _native as N

    lib = N.load()
    old = os.environ.pop("L1B_ARITH", None)
    try:
        c = N.SolverCfg()
        lib.l1b_solver_cfg_default(ctypes.byref(c))
        assert c.arith == 0 and c.max_iters == 100000 and c.block == 256
        os.environ["L1B_ARITH"] = "fma"
        lib.l1b_solver_cfg_default(ctypes.byref(c))
        assert c.arith == 1
        os.environ["L1B_ARITH"] = "exact"
        lib.l1b_solver_cfg_default(ctypes.byref(c))
        assert c.arith == 0
    finally:
        os.environ.pop("L1B_ARITH", None)
        if old is not None:
            os.environ["L1B_ARITH"] = old


def _plan_mirror(kmax, iters):
    ks, kmin = [], min(6, kmax)
    launches, r = iters // kmax + (1 if iters % kmax >= kmin else 0), iters
    while launches > 0 and r >= kmin:
        k = min((r + launches - 1) // launches, kmax)
        down = (k + 2) % 4
        k = max(k - down if k > down else kmin, kmin)
        if k > r:
            break
        ks.append(k)
        r -= k
        launches -= 1
    return ks


def test_tile_launch_plan():
    """l1b_tile_plan: the tile launches a step of `iters` iterations takes --
    every launch K = 2 mod 4 (the rotation of the four x buffers) and at most
    kmax, fewer than 6 iterations (kmax for K = 2) left to the two-iteration /
    single launches, the iterations spread evenly over the launches."""
    from paper_1503_03520_b200 import _native as N

    lib = N.load()

    def plan(kmax, iters):
        cap = iters // 2 + 2
        ks, cnt = (ctypes.c_int * cap)(), ctypes.c_int()
        assert lib.l1b_tile_plan(kmax, iters, ks, cap, ctypes.byref(cnt)) == 0
        return [ks[i] for i in range(cnt.value)]

    assert plan(14, 20) == [10, 10] and plan(14, 29) == [14, 14] and plan(14, 5) == []
    assert sorted(plan(14, 500)) == [10] + [14] * 35 and plan(0, 100) == []
    for kmax in (2, 6, 10, 14):
        for iters in list(range(0, 130)) + [499, 500, 501, 1000, 12345]:
            p = plan(kmax, iters)
            assert p == _plan_mirror(kmax, iters), (kmax, iters)
            assert all(k % 4 == 2 and min(6, kmax) <= k <= kmax for k in p)
            assert 0 <= iters - sum(p) < min(6, kmax) + (4 if kmax > 6 else 0) or not p
            if p:
                assert max(p) - min(p) <= 4 or kmax == 14  # spread evenly
    out = ctypes.c_int()
    assert lib.l1b_tile_plan(12, 100, None, 0, ctypes.byref(out)) != 0  # K must be 2 mod 4
