"""GPU edge cases against the oracle / reference semantics: minimum
dimensions, odd sizes, zero budgets, immediate targets, time budget, bad
arguments."""
import math

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu
TH = 2 * math.pi / 10


@pytest.mark.parametrize("n,stages,m_ratio", [(2, 1, 2.0), (3, 2, 1.0), (5, 3, 1.4), (7, 4, 2.0), (33, 1, 1.0)])
def test_tiny_instances_all_solvers(oracle, n, stages, m_ratio):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=n, stages=stages, m_ratio=m_ratio, q=1, s_divisor=2, seed=13, theta=TH)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    np.testing.assert_array_equal(inst.b, oi.b)
    for got, want in zip(inst.op.csr(), oracle.csr(oi.op)):
        np.testing.assert_array_equal(got, want)
    for got, want in zip(inst.op.csc(), oracle.csc(oi.op)):
        np.testing.assert_array_equal(got, want)
    otr, ox = oracle.fista(oi, max_iters=60)
    for op in ("sparse", "matrix_free"):
        x = np.empty(n)
        tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=60, op=op), x)
        f, fo = tr.objectives(), otr["objective"]
        if op == "matrix_free":  # the reference's own products: same trajectory, same stop
            np.testing.assert_array_equal(x, ox)
            assert len(f) == len(fo) and tr.status == l1bench.StopReason(otr["status"])
        k = min(len(f), len(fo))  # CSR/CSC rounding can move an exact fixed point by an iteration
        assert rel_err(f[:k], fo[:k]) < 1e-10
        assert rel_err(x, ox) < 1e-10
    x = np.empty(n)
    tr = l1bench.coordinate_descent_run(inst, l1bench.SolverConfig(max_iters=5, varpi=2, seed=4), x)
    otr, ox = oracle.cd(oi, max_iters=5, varpi=2, seed=4)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-10 and rel_err(x, ox) < 1e-10
    x = np.empty(n)
    tr = l1bench.pcdm_run(inst, l1bench.SolverConfig(max_iters=5, block=2, seed=4), x)
    otr, ox = oracle.pcdm(oi, max_iters=5, block=2, seed=4)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-10 and rel_err(x, ox) < 1e-10
    x = np.empty(n)
    tr = l1bench.newton_cg_run(inst, l1bench.SolverConfig(max_iters=3), x)
    otr, ox = oracle.newton_cg(oi, max_iters=3)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-8


@pytest.mark.parametrize("solver", ["fista", "ista", "cd", "pcdm", "newton_cg"])
def test_zero_budget_and_immediate_target(solver):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=64, stages=2, q=1, s_divisor=8, seed=2, theta=TH)
    x = np.full(inst.n, 7.0)
    tr = l1bench.run_solver(inst, l1bench.SolverConfig(id=solver, max_iters=0, block=8), x)
    assert tr.status == l1bench.StopReason.iter_budget and tr.iterations == 0
    assert len(tr.samples) == 1 and np.all(x == 0.0)
    f0 = 0.5 * float(np.dot(inst.b, inst.b))
    assert tr.samples[0].objective == pytest.approx(f0, rel=1e-14)
    tr = l1bench.run_solver(inst, l1bench.SolverConfig(id=solver, target_objective=2 * f0, block=8))
    assert tr.status == l1bench.StopReason.target_reached and tr.iterations == 0 and tr.reached_target


@pytest.mark.parametrize("solver", ["fista", "cd", "pcdm"])
def test_time_budget(solver):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=256, stages=1, q=1, s_divisor=8, seed=2, theta=TH)
    tr = l1bench.run_solver(inst, l1bench.SolverConfig(id=solver, max_seconds=1e-9, block=8))
    assert tr.status == l1bench.StopReason.time_budget and tr.iterations == 0


def test_bad_arguments():
    need_cuda()
    from paper_1503_03520_b200 import _native as N
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=64, stages=1, q=1, s_divisor=8, seed=2, theta=TH)
    for bad in (dict(eta=0.0), dict(eta=1.0), dict(mu=0.0), dict(varpi=0), dict(max_seconds=0.0),
                dict(omega=65), dict(l_fixed=-1.0)):
        with pytest.raises(ValueError):
            l1bench.fista_run(inst, l1bench.SolverConfig(**bad))
    with pytest.raises(ValueError):
        l1bench.build_instance(n=64, tau=0.0)
    with pytest.raises(ValueError):
        l1bench.build_instance(n=64, m_ratio=0.5)
    with pytest.raises(N.L1bUnsupported):  # sessions keep L constant
        l1bench.Session(inst, l1bench.SolverConfig(l_policy=l1bench.LPolicy.backtracking))
    with pytest.raises(ValueError):  # bad spectrum in from_host (Spectrum::validate)
        l1bench.ProblemInstance.from_host(4, 2, [(0, 0.3)], [1.0, 2.0], np.zeros(4), -1.0)
    with pytest.raises(RuntimeError):
        l1bench.ProblemInstance.from_host(4, 2, [(0, 0.3)], [1.0, 0.0], np.zeros(4), 1.0)
