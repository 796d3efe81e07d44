"""Parity of the recomputing single-kernel FISTA path (k_iter_rc.cu: r_k and
r_{k-1} rebuilt from x_k, x_{k-1}, objective recorded one kernel late) on
instances with many warp segments, ragged ends (n not a multiple of the
segment or of 4) and 1..4 stages: iterates bit-identical to the oracle's
restatement of fista_run (solvers.cpp:290-380) and to the stored-residual
kernel (k_fused.cu), objectives within 1e-12."""
import math
import os

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu

TH = 2 * math.pi / 10


def _solve(inst, iters, rc, **cfg):
    from paper_1503_03520_b200 import l1bench

    old = os.environ.get("L1B_ITER_RC")
    os.environ["L1B_ITER_RC"] = "1" if rc else "0"
    try:
        x = np.empty(inst.n)
        tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=iters, op="matrix_free", **cfg), x)
    finally:
        if old is None:
            del os.environ["L1B_ITER_RC"]
        else:
            os.environ["L1B_ITER_RC"] = old
    return tr, x


@pytest.mark.parametrize("n,stages", [(100003, 4), (50001, 3), (20005, 2), (7777, 1), (4096, 4), (449, 4)])
def test_rc_matches_oracle_and_stored_kernel(oracle, n, stages):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=n, stages=stages, q=1, s_divisor=100, seed=5, theta=TH)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    assert np.array_equal(inst.b, oi.b)
    iters = 60
    tr, x = _solve(inst, iters, rc=True)
    otr, ox = oracle.fista(oi, max_iters=iters)
    assert tr.iterations == iters and tr.status == l1bench.StopReason.iter_budget
    np.testing.assert_array_equal(x, ox)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-12
    np.testing.assert_array_equal(tr.iters(), otr["iter"])
    tr0, x0 = _solve(inst, iters, rc=False)
    np.testing.assert_array_equal(x, x0)
    assert rel_err(tr.objectives(), tr0.objectives()) < 1e-13
    np.testing.assert_array_equal([s.nnz for s in tr.samples], [s.nnz for s in tr0.samples])


def test_rc_stops_like_the_reference(oracle):
    """Target / fixed-point stops decided one kernel late must land on the same
    iteration with the same x (the extra x_{k+1} is discarded)."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=3001, stages=4, q=1, s_divisor=50, seed=9, theta=TH)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    otr, ox = oracle.fista(oi, max_iters=400)
    f = otr["objective"]
    assert f[37] < f[:37].min()
    target = float(f[37] + 0.25 * (f[:37].min() - f[37]))  # first reached at iteration 37
    tr, x = _solve(inst, 400, rc=True, target_objective=target)
    otr2, ox2 = oracle.fista(oi, max_iters=400, target=target)
    assert tr.status == l1bench.StopReason.target_reached
    assert tr.iterations == int(otr2["iter"][-1]) == 37
    np.testing.assert_array_equal(x, ox2)
    for k in (0, 1, 2):  # budgets at and right after the start
        tr, x = _solve(inst, k, rc=True)
        otr3, ox3 = oracle.fista(oi, max_iters=k)
        assert tr.iterations == k
        np.testing.assert_array_equal(x, ox3)
        assert rel_err(tr.objectives(), otr3["objective"]) < 1e-12


def test_rc_session_stepping_matches_solve():
    """Session API: K steps then end (the flush records the last iterate)."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=30011, stages=4, q=1, s_divisor=100, seed=4, theta=TH)
    tr, x = _solve(inst, 25, rc=True)
    s = l1bench.Session(inst, l1bench.SolverConfig(max_iters=100, op="matrix_free"))
    s.step(10)
    s.step(15)
    x2 = np.empty(inst.n)
    tr2 = s.end(x2)
    np.testing.assert_array_equal(x, x2)
    assert tr2.iterations == 25
    assert rel_err(tr.objectives(), tr2.objectives()) == 0.0
