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
