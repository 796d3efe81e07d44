"""GPU: the reference-side drop-in (integration/l1bench_b200.cpp), compiled
against the reference's own headers: an instance built by the reference's
build_instance is solved by l1bench::run_solver and by
l1bench::b200::run_solver on the same host objects."""
import ctypes
import os

import numpy as np
import pytest

from conftest import ROOT
from gpu_util import need_cuda

pytestmark = pytest.mark.gpu

SO = os.path.join(ROOT, "integration", "_build", "libl1bench_b200_dropin.so")


@pytest.mark.parametrize("solver,iters,tol", [("fista", 200, 1e-10), ("ista", 100, 1e-10),
                                              ("fista_bt", 150, 1e-10), ("ista_bt", 100, 1e-10),
                                              ("cd", 10, 1e-10), ("newton_cg", 2, 1e-9)])
def test_dropin_matches_reference(solver, iters, tol):
    need_cuda()
    if not os.path.exists(SO):
        pytest.skip("integration/_build not built (needs the reference headers)")
    lib = ctypes.CDLL(SO)
    out = np.zeros(6)
    rc = lib.b200_dropin_compare(solver.encode(), ctypes.c_uint64(2048), ctypes.c_uint32(2),
                                 ctypes.c_int(1), ctypes.c_uint64(7), ctypes.c_uint64(iters),
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert rc == 0
    rel_dx, rel_df, n_ref, n_b200, st_ref, st_b200 = out
    assert n_ref == n_b200 and st_ref == st_b200
    assert rel_dx < tol and rel_df < tol


def test_dropin_contracted_arithmetic_from_the_environment():
    """L1B_ARITH=fma: the binding (whose SolverConfig has no arithmetic field)
    runs the tile kernel with fused multiply-adds on a reference-built instance
    with n > 2^20 -- within 1e-12 of l1bench::run_solver, same iteration count
    and status; without the variable the iterates are the reference's bits."""
    need_cuda()
    if not os.path.exists(SO):
        pytest.skip("integration/_build not built (needs the reference headers)")
    lib = ctypes.CDLL(SO)

    def compare():
        out = np.zeros(6)
        rc = lib.b200_dropin_compare(b"fista", ctypes.c_uint64((1 << 20) + 4096), ctypes.c_uint32(4),
                                     ctypes.c_int(1), ctypes.c_uint64(7), ctypes.c_uint64(30),
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        assert rc == 0
        return out

    old = os.environ.pop("L1B_ARITH", None)
    try:
        rel_dx, rel_df, n_ref, n_b200, st_ref, st_b200 = compare()
        assert rel_dx == 0.0 and rel_df < 1e-12 and n_ref == n_b200 and st_ref == st_b200
        os.environ["L1B_ARITH"] = "fma"
        rel_dx, rel_df, n_ref, n_b200, st_ref, st_b200 = compare()
        assert 0.0 < rel_dx < 1e-12 and rel_df < 1e-12 and n_ref == n_b200 and st_ref == st_b200
    finally:
        os.environ.pop("L1B_ARITH", None)
        if old is not None:
            os.environ["L1B_ARITH"] = old
