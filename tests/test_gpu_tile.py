"""The tile kernel (k_iter_rc.cu fista_tb_kernel: K FISTA iterations per
launch, 16-warp tiles with their x halos exchanged in shared memory, the
eroded tile ends recomputed by the neighbouring tiles) against the
two-iteration kernel (L1B_TB=0) and the oracle's restatement of fista_run
(solvers.cpp:290-380): iterates bit-identical in the exact arithmetic and within 1e-12 in the
contracted one (scaled rotations), objectives within 1e-12, the same stop; a stop inside a launch is replayed
from the launch's inputs."""
import math
import os

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu

TH = 2 * math.pi / 10


def _solve(inst, tile, k=None, **cfg):
    """tile: None = the default choice for the size, True = forced (L1B_TB=2,
    any n), False = off (L1B_TB=0)."""
    from paper_1503_03520_b200 import l1bench

    env = {"L1B_TB": {None: "1", True: "2", False: "0"}[tile]}
    if k is not None:
        env["L1B_TB_K"] = str(k)
    old = {key: os.environ.get(key) for key in env}
    os.environ.update(env)
    try:
        x = np.empty(inst.n)
        tr = l1bench.fista_run(inst, l1bench.SolverConfig(op="matrix_free", **cfg), x)
    finally:
        for key, v in old.items():
            if v is None:
                del os.environ[key]
            else:
                os.environ[key] = v
    return tr, x


@pytest.mark.parametrize("n,stages,k", [(100003, 4, 10), (50001, 3, 14), (20005, 2, 6), (7777, 1, 10),
                                        (3001, 4, 14), (449, 4, 10), (300007, 4, 2)])
def test_tile_matches_oracle_and_two_iteration_kernel(oracle, n, stages, k):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=n, stages=stages, q=1, s_divisor=100, seed=5, theta=TH)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    iters = 63  # K-launches, then two-iteration launches and a single one
    tr, x = _solve(inst, True, k, max_iters=iters)
    assert tr.ran("fista_tile"), tr.path
    otr, ox = oracle.fista(oi, max_iters=iters)
    assert tr.iterations == iters and tr.status == l1bench.StopReason.iter_budget
    np.testing.assert_array_equal(x, ox)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-12
    np.testing.assert_array_equal(tr.iters(), otr["iter"])
    np.testing.assert_array_equal([s.nnz for s in tr.samples], otr["nnz"])
    tr2, x2 = _solve(inst, False, max_iters=iters)
    assert not tr2.ran("fista_tile")
    np.testing.assert_array_equal(x, x2)
    assert rel_err(tr.objectives(), tr2.objectives()) < 1e-13


@pytest.mark.parametrize("n,stages", [(1 << 20 | 4099, 4), (1 << 21, 3)])
def test_tile_default_at_large_n_fma(oracle, n, stages):
    """Above 2^20 the tile kernel is the default.  In the contracted arithmetic
    both it and the two-iteration kernel rotate in the scaled form (two
    independent fmas per pair, prod cos carried by sigma) with the same
    operations per entry: bit-identical to each other, within 1e-12 of the
    oracle's fista_run restatement, same supports."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=n, stages=stages, q=1, s_divisor=1000, seed=3, theta=TH)
    inst = l1bench.build_instance(**kw)
    tr, x = _solve(inst, None, max_iters=40, arith="fma")
    assert tr.ran("fista_tile") and tr.ran("fma"), tr.path
    tr2, x2 = _solve(inst, False, max_iters=40, arith="fma")
    assert not tr2.ran("fista_tile") and tr2.ran("fma")
    np.testing.assert_array_equal(x, x2)
    assert rel_err(tr.objectives(), tr2.objectives()) < 1e-13
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=40)
    assert np.max(np.abs(x - ox)) < 1e-12 * np.max(np.abs(ox))
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-12
    np.testing.assert_array_equal([s.nnz for s in tr.samples], otr["nnz"])
    assert tr.iterations == tr2.iterations == 40



@pytest.mark.parametrize("n,stages,k", [(100003, 4, 10), (50001, 3, 14), (20005, 2, 6), (7777, 1, 10),
                                        (3001, 4, 14), (449, 4, 10), (4098, 4, 6), (300007, 4, 2)])
def test_tile_fma_scaled_rotations_match_oracle(oracle, n, stages, k):
    """Contracted arithmetic on forced tiles at sizes whose ends fall inside a
    tile (the entries a stage leaves unpaired take 1 / cos(theta) in the
    scaled form): within 1e-12 of the oracle, same supports, nnz trace and
    stop."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=n, stages=stages, q=1, s_divisor=100, seed=5, theta=TH)
    inst = l1bench.build_instance(**kw)
    iters = 63
    tr, x = _solve(inst, True, k, max_iters=iters, arith="fma")
    assert tr.ran("fista_tile") and tr.ran("fma"), tr.path
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=iters)
    assert tr.iterations == iters
    assert np.max(np.abs(x - ox)) < 1e-12 * np.max(np.abs(ox))
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-12
    np.testing.assert_array_equal([s.nnz for s in tr.samples], otr["nnz"])


def test_steep_rotations_keep_the_exact_arithmetic(oracle):
    """|cos(theta)| < 1/4: the scaled form of the contracted arithmetic is not
    used -- arith = "fma" is declined (flag not set) and the exact kernels run:
    the oracle's iterates bit for bit."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=(1 << 20) + 4099, stages=4, q=1, s_divisor=1000, seed=5, theta=0.47 * math.pi)
    inst = l1bench.build_instance(**kw)
    tr, x = _solve(inst, None, max_iters=41, arith="fma")
    assert tr.ran("fista_tile") and not tr.ran("fma"), tr.path
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=41)
    np.testing.assert_array_equal(x, ox)
    tr2, x2 = _solve(inst, False, max_iters=41, arith="fma")
    assert not tr2.ran("fista_tile") and not tr2.ran("fma")
    np.testing.assert_array_equal(x2, ox)



@pytest.mark.parametrize("stop_at", [11, 12, 13, 17, 18, 19, 20])
def test_stop_inside_a_tile_launch_is_replayed(stop_at):
    """A target met at iteration stop_at: launches of K = 10 cover 1-10,
    11-20, ...; only the last two iterates of a launch are stored, so stops at
    11..18 are replayed from x_10, x_9.  Same stop, iterations, status and x
    as the two-iteration kernel."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=200003, stages=4, q=1, s_divisor=100, seed=2, theta=TH)
    full, _ = _solve(inst, False, max_iters=40)
    f = full.objectives()
    it = list(full.iters())
    target = float(f[it.index(stop_at)] * (1 + 1e-9))
    assert all(v > target for v in f[:it.index(stop_at)])  # first met at stop_at
    tr, x = _solve(inst, True, 10, max_iters=40, target_objective=target)
    tr2, x2 = _solve(inst, False, max_iters=40, target_objective=target)
    assert tr.ran("fista_tile")
    assert tr.status == tr2.status == l1bench.StopReason.target_reached
    assert tr.iterations == tr2.iterations == stop_at
    np.testing.assert_array_equal(x, x2)
    assert rel_err(tr.objectives(), tr2.objectives()) < 1e-13


def test_tile_session_steps_and_profile():
    """Session.step in odd chunks (K-launches + remainders) and profile
    (timed K-launches) give the one-call solve's iterates."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=(1 << 20) + 12345, stages=4, q=1, s_divisor=1000, seed=3, theta=TH)
    old = os.environ.get("L1B_TB")
    os.environ["L1B_TB"] = "1"
    try:
        cfg = l1bench.SolverConfig(max_iters=57, op="matrix_free")
        s = l1bench.Session(inst, cfg)
        assert s.kernel_mode() == 6
        k, span, valid = s.tile_geometry()
        assert k == 14 and span % 240 == 0 and valid == span - 2 * 104
        # launches spread evenly, each K = 2 mod 4; fewer than 6 left over: two-iteration / single launches
        assert s.tile_plan(20) == [10, 10] and sorted(s.tile_plan(500)) == [10] + [14] * 35
        assert s.tile_plan(29) == [14, 14] and sorted(s.tile_plan(34)) == [10, 10, 14] and s.tile_plan(27) == [14, 10]
        assert s.tile_plan(5) == [] and s.tile_plan(6) == [6] and s.tile_plan(14) == [14]
        s.step(3)
        s.profile(30)
        s.step(24)
        x = np.empty(inst.n)
        tr = s.end(x)
    finally:
        if old is None:
            del os.environ["L1B_TB"]
        else:
            os.environ["L1B_TB"] = old
    tr2, x2 = _solve(inst, False, max_iters=57)
    np.testing.assert_array_equal(x, x2)
    assert tr.iterations == 57
    assert rel_err(tr.objectives(), tr2.objectives()) < 1e-13


@pytest.mark.parametrize("iters", [24, 27, 34, 41])
def test_remainder_runs_as_a_shorter_tile_launch(oracle, iters):
    """K = 14: 24 = 10 + 14, 27 = 14 + 10 + 2 + 1, 34 = 10 + 10 + 14, 41 = 14 + 14 + 10 + 2 + 1 --
    a remainder of 6 or more takes its own tile launch (K = 2 mod 4, the
    iterations spread evenly), the rest two-iteration and single launches: the
    oracle's iterates bit for bit, and a target met inside a shorter launch is
    replayed from that launch's own inputs."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=150001, stages=4, q=1, s_divisor=100, seed=7, theta=TH)
    inst = l1bench.build_instance(**kw)
    tr, x = _solve(inst, True, 14, max_iters=iters)
    assert tr.ran("fista_tile") and tr.iterations == iters
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=iters)
    np.testing.assert_array_equal(x, ox)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-12
    # a stop three iterations before the end: inside the last tile launch or after it
    f, it = tr.objectives(), list(tr.iters())
    stop_at = iters - 3
    target = float(f[it.index(stop_at)] * (1 + 1e-9))
    if all(v > target for v in f[:it.index(stop_at)]):
        tr1, x1 = _solve(inst, True, 14, max_iters=iters, target_objective=target)
        tr2, x2 = _solve(inst, False, max_iters=iters, target_objective=target)
        assert tr1.iterations == tr2.iterations == stop_at
        assert tr1.status == tr2.status == l1bench.StopReason.target_reached
        np.testing.assert_array_equal(x1, x2)


def test_ista_on_tiles(oracle):
    """ISTA (no momentum: beta = 0 in every iteration of a launch) through the
    tile kernel: the oracle's ista iterates bit for bit."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=60013, stages=3, q=1, s_divisor=100, seed=9, theta=TH)
    inst = l1bench.build_instance(**kw)
    env = {"L1B_TB": "2", "L1B_TB_K": "10"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        x = np.empty(inst.n)
        tr = l1bench.ista_run(inst, l1bench.SolverConfig(op="matrix_free", max_iters=37), x)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    assert tr.ran("fista_tile"), tr.path
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=37, accelerated=False)
    np.testing.assert_array_equal(x, ox)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-12


def test_tile_random_shapes_and_angles(oracle):
    """Seeded sweep over sizes (ends of [0, n) anywhere inside a tile, n odd and
    even, smaller than one tile and several tiles long), stage counts, launch
    lengths and rotation angles (including ones the scaled form declines): the
    exact arithmetic gives the oracle's bits, the contracted one stays within
    1e-12 with the same support, and says whether it was applied."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    rng = np.random.default_rng(20261021)
    for case in range(14):
        n = int(rng.integers(300, 9000))
        stages = int(rng.integers(1, 5))
        k = int(rng.choice([2, 6, 10, 14]))
        theta = float(rng.choice([0.3, TH, 1.0, 1.2, 1.4, -0.8, 2.2]))
        iters = int(rng.integers(k + 1, 3 * k + 6))
        kw = dict(n=n, stages=stages, q=1, s_divisor=50, seed=100 + case, theta=theta)
        inst = l1bench.build_instance(**kw)
        otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=iters)
        tr, x = _solve(inst, True, k, max_iters=iters)
        assert tr.ran("fista_tile"), (kw, k, iters)
        np.testing.assert_array_equal(x, ox, err_msg=f"{kw} k={k} iters={iters}")
        assert rel_err(tr.objectives(), otr["objective"]) < 1e-12
        trf, xf = _solve(inst, True, k, max_iters=iters, arith="fma")
        assert trf.ran("fista_tile")
        assert trf.ran("fma") == (abs(math.cos(theta)) >= 0.25), (kw, trf.path)
        assert np.max(np.abs(xf - ox)) <= 1e-12 * max(np.max(np.abs(ox)), 1e-300), (kw, k, iters)
        np.testing.assert_array_equal(np.nonzero(xf)[0], np.nonzero(ox)[0])
        assert rel_err(trf.objectives(), otr["objective"]) < 1e-12
