"""GPU: FISTA / ISTA with LPolicy::backtracking (k_bt.cu) against the oracle's
restatement (pinned bit-exact to the reference in test_oracle.py): same
backtrack counts, matvec counts and sampled iterations; objectives and
iterates within 1e-10 (the products are the reference's own sweeps; the sums
are grid reductions, which the bound test's 1e-12 slack absorbs)."""
import math

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu
TH = 2 * math.pi / 10


@pytest.mark.parametrize("kw,solver", [
    (dict(n=512, stages=2, q=1, s_divisor=20, seed=4), "fista"),
    (dict(n=1000, stages=1, q=2, s_divisor=50, seed=7), "ista"),
    (dict(n=300, stages=3, left_stages=1, permute=True, q=1, s_divisor=10, seed=9), "fista"),
    (dict(n=4097, stages=4, q=1, s_divisor=100, seed=3), "fista"),
])
def test_backtracking_matches_oracle(oracle, kw, solver):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(kw, theta=TH)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    iters = 150
    x = np.empty(inst.n)
    cfg = l1bench.SolverConfig(id=solver, max_iters=iters, l_policy=l1bench.LPolicy.backtracking, seed=11)
    tr = l1bench.run_solver(inst, cfg, x)
    otr, ox = oracle.fista(oi, max_iters=iters, backtracking=True, accelerated=solver == "fista", seed=11)
    np.testing.assert_array_equal(tr.iters(), otr["iter"])
    np.testing.assert_array_equal([s.extra for s in tr.samples], otr["extra"])
    np.testing.assert_array_equal([s.matvecs for s in tr.samples], otr["matvecs"])
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-10
    assert rel_err(x, ox) < 1e-10
    assert sum(s.extra for s in tr.samples) > 0


def test_backtracking_target_and_fixed_L():
    """A target stops it like the spectrum policy; l_fixed overrides the policy
    (LipschitzState: the fixed value wins) and then equals the spectrum path with
    that L."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=2048, stages=2, q=1, s_divisor=40, seed=5, theta=TH)
    full = l1bench.run_solver(inst, l1bench.SolverConfig(max_iters=300, l_policy=l1bench.LPolicy.backtracking))
    target = float(full.objectives()[120])
    tr = l1bench.run_solver(inst, l1bench.SolverConfig(max_iters=300, target_objective=target,
                                                       l_policy=l1bench.LPolicy.backtracking))
    assert tr.status == l1bench.StopReason.target_reached and tr.iterations <= 120
    L = inst.info.gram_lmax * 1.5
    a = l1bench.run_solver(inst, l1bench.SolverConfig(max_iters=50, l_fixed=L, l_policy=l1bench.LPolicy.backtracking))
    b = l1bench.run_solver(inst, l1bench.SolverConfig(max_iters=50, l_fixed=L))
    assert rel_err(a.objectives(), b.objectives()) < 1e-12


@pytest.mark.parametrize("kw", [dict(n=700, stages=2, q=1, seed=4),
                                dict(n=300, stages=3, left_stages=1, permute=True, q=2, seed=9)])
def test_estimate_gram_lmax_matches_oracle(oracle, kw):
    """estimate_gram_lmax (linops.cpp:757-778) on the device vs the oracle
    (same normal() draws, same sweeps; the dot products are grid sums)."""
    import ctypes as C

    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(kw, theta=TH, s_divisor=20)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    st = oi.op.c_struct()
    for iters, seed in ((30, 11), (5, 2)):
        want = oracle.lib.lo_estimate_gram_lmax(C.byref(st), iters, seed)
        got = inst.op.estimate_gram_lmax(iters, seed)
        assert abs(got - want) <= 1e-12 * abs(want)
        assert got <= inst.info.gram_lmax * (1 + 1e-12)
