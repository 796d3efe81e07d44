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


def _solve(inst, iters, rc, env=None, **cfg):
    """rc: recomputing kernels (else the stored-residual one); env: extra
    switches, e.g. L1B_PERSIST=0 (no cooperative loop: two-iteration launches
    on any n) or L1B_RC2=0 (one iteration per launch)."""
    from paper_1503_03520_b200 import l1bench

    env = dict(env or {}, L1B_ITER_RC="1" if rc else "0")
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        x = np.empty(inst.n)
        tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=iters, op="matrix_free", **cfg), x)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
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


# (the switches are read once per process by the library, so each mode below
# runs in a subprocess of its own)
_MODES = {"loop": {}, "pairs": {"L1B_PERSIST": "0"}, "single": {"L1B_PERSIST": "0", "L1B_RC2": "0"}}


def _mode_run(mode, kw, iters, target=None, arith="exact"):
    import json
    import subprocess
    import sys

    code = (
        "import json, sys, numpy as np; sys.path.insert(0, '.');"
        "from paper_1503_03520_b200 import l1bench;"
        f"inst = l1bench.build_instance(**{kw!r});"
        "x = np.empty(inst.n);"
        f"cfg = l1bench.SolverConfig(max_iters={iters}, op='matrix_free', arith={arith!r}"
        + (f", target_objective={target!r}" if target is not None else "") + ");"
        "tr = l1bench.fista_run(inst, cfg, x);"
        "np.save(sys.argv[1], x);"
        "print(json.dumps({'f': list(tr.objectives()), 'it': [int(s.iter) for s in tr.samples],"
        " 'nnz': [int(s.nnz) for s in tr.samples], 'status': int(tr.status), 'k': int(tr.iterations),"
        " 'launches': l1bench.launch_count()}))")
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "x.npy")
        env = dict(os.environ, **_MODES[mode])
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        p = subprocess.run([sys.executable, "-c", code, out], cwd=root, env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        return json.loads(p.stdout.strip().splitlines()[-1]), np.load(out)


@pytest.mark.parametrize("n,stages", [(100003, 4), (30001, 3), (20005, 2), (7777, 1)])
def test_two_iteration_kernel_matches_single_and_oracle(oracle, n, stages):
    """fista_rc2_kernel (two iterations per launch) vs one iteration per launch
    and vs the oracle: identical x, objectives within 1e-12."""
    need_cuda()
    kw = dict(n=n, stages=stages, q=1, s_divisor=100, seed=5, theta=TH)
    iters = 41  # odd: the last launch is a single iteration
    tp, xp = _mode_run("pairs", kw, iters)
    ts, xs = _mode_run("single", kw, iters)
    np.testing.assert_array_equal(xp, xs)
    assert tp["it"] == ts["it"] and tp["k"] == ts["k"] == iters
    assert rel_err(tp["f"], ts["f"]) < 1e-13
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=iters)
    np.testing.assert_array_equal(xp, ox)
    assert rel_err(tp["f"], otr["objective"]) < 1e-12


# The contracted arithmetic (SolverConfig.arith = "fma", L1B_ARITH_FMA): every
# a*b + c of the matrix-free FISTA kernels is one fused multiply-add.  Not the
# reference's bits any more; the bar is the north star's parity contract at
# 1e-12 (x, objectives) with identical sample iterations and supports.
@pytest.mark.parametrize("mode", ["pairs", "single"])
@pytest.mark.parametrize("n,stages", [(100003, 4), (30001, 3), (20005, 2), (7777, 1)])
def test_fma_kernels_match_oracle(oracle, n, stages, mode):
    need_cuda()
    kw = dict(n=n, stages=stages, q=1, s_divisor=100, seed=5, theta=TH)
    iters = 201  # odd: the two-iteration path ends with a single-iteration launch
    tf, xf = _mode_run(mode, kw, iters, arith="fma")
    te, xe = _mode_run(mode, kw, iters, arith="exact")
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=iters)
    np.testing.assert_array_equal(xe, ox)  # the exact build: the reference's bits
    assert not np.array_equal(xf, ox), "fma build produced the exact bits: contraction not active"
    assert rel_err(xf, ox) < 1e-12
    assert rel_err(tf["f"], otr["objective"]) < 1e-12
    assert tf["it"] == [int(i) for i in otr["iter"]] and tf["k"] == iters
    np.testing.assert_array_equal(np.nonzero(xf)[0], np.nonzero(ox)[0])
    assert tf["nnz"] == [int(v) for v in otr["nnz"]]


def test_fma_kernels_stop_like_the_reference(oracle):
    """A target between two iterates' objectives stops the fma build on the
    reference's iteration."""
    need_cuda()
    kw = dict(n=30001, stages=4, q=1, s_divisor=50, seed=9, theta=TH)
    oi = oracle.build_instance(**kw)
    otr, _ = oracle.fista(oi, max_iters=400)
    f = otr["objective"]
    for k in (37, 38):
        target = float(f[k] + 0.5 * (f[:k].min() - f[k]))
        tp, xp = _mode_run("pairs", kw, 400, target, arith="fma")
        otr2, ox2 = oracle.fista(oi, max_iters=400, target=target)
        assert tp["k"] == int(otr2["iter"][-1]) == k
        assert rel_err(xp, ox2) < 1e-12


def test_two_iteration_kernel_stops_like_the_reference(oracle):
    need_cuda()
    kw = dict(n=3001, stages=4, q=1, s_divisor=50, seed=9, theta=TH)
    oi = oracle.build_instance(**kw)
    otr, _ = oracle.fista(oi, max_iters=400)
    f = otr["objective"]
    for k in (37, 38):  # the stop lands on the first / second iteration of a launch
        assert f[k] < f[:k].min()
        target = float(f[k] + 0.25 * (f[:k].min() - f[k]))
        tp, xp = _mode_run("pairs", kw, 400, target)
        otr2, ox2 = oracle.fista(oi, max_iters=400, target=target)
        assert tp["k"] == int(otr2["iter"][-1]) == k
        np.testing.assert_array_equal(xp, ox2)


@pytest.mark.parametrize("stages", [4, 2])
def test_two_iteration_kernel_large_n(oracle, stages):
    """Above the cooperative-loop size (n > 2^20): the default path."""
    need_cuda()
    kw = dict(n=(1 << 20) + 12345, stages=stages, q=1, s_divisor=1000, seed=3, theta=TH)
    tp, xp = _mode_run("loop", kw, 12)
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=12)
    np.testing.assert_array_equal(xp, ox)
    assert rel_err(tp["f"], otr["objective"]) < 1e-12


def _pair_instance(oracle, n, off, q, seed):
    """Single-stage instance with the given stage offset, built by the oracle
    (b = A x* + tau A (A^T A)^-1 g) and uploaded as-is."""
    import ctypes as C

    from pyoracle import Instance, _ptr

    js = oracle.mix_seed(seed, 0)
    op = oracle.spec(n, stages=1, q=q, job_seed=js)
    op.right_offset = np.array([off], dtype=np.int32)
    s = max(1, n // 50)
    rng = oracle.rng(oracle.mix_seed(js, 4))
    sup = np.empty(s, dtype=np.uint32)
    vals = np.empty(s)
    oracle.lib.lo_uniform_sparse_solution(n, s, 10.0, C.byref(rng), _ptr(sup, C.c_uint32), _ptr(vals, C.c_double))
    gen = oracle.rng(oracle.mix_seed(js, 5))
    b = np.empty(op.m)
    st = op.c_struct()
    noise = oracle.lib.lo_generate_instance(C.byref(st), 1.0, _ptr(sup, C.c_uint32), _ptr(vals, C.c_double), s,
                                            0.9, C.byref(gen), _ptr(b, C.c_double))
    return Instance(op, 1.0, b, sup, vals, float(noise), js)


@pytest.mark.parametrize("n,off", [(4096, 0), (4095, 1), (2047, 0), (1000, 1), (513, 0), (6, 1), (3, 0),
                                   (12001, 1), (16384, 0)])
def test_pair_small_kernel_bit_identical(oracle, n, off):
    """The pair-local kernel for single-stage instances (an 8-CTA cluster, the
    default for n <= 16384) against the oracle and the window kernel
    (L1B_PAIR_SMALL=0): identical iterates, samples, stop."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    oi = _pair_instance(oracle, n, off, q=1, seed=n + off)
    inst = l1bench.ProblemInstance.from_host(oi.m, n, [(off, TH)], oi.op.sigma, oi.b, 1.0, oi.support, oi.values)
    iters = 300
    tr, x = _solve(inst, iters, rc=True)
    otr, ox = oracle.fista(oi, max_iters=iters)
    np.testing.assert_array_equal(x, ox)
    np.testing.assert_array_equal(tr.iters(), otr["iter"])
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-12
    for mode in ("0",):
        tw, xw = _solve(inst, iters, rc=True, env={"L1B_PAIR_SMALL": mode})
        np.testing.assert_array_equal(x, xw)
        np.testing.assert_array_equal(tr.iters(), tw.iters())
        assert tr.status == tw.status
        np.testing.assert_array_equal([s.nnz for s in tr.samples], [s.nnz for s in tw.samples])


def test_pair_small_kernel_target_stop(oracle):
    """C1-style run to a target objective: same stopping iteration as the oracle."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    oi = _pair_instance(oracle, 4096, 0, q=1, seed=77)
    inst = l1bench.ProblemInstance.from_host(oi.m, 4096, [(0, TH)], oi.op.sigma, oi.b, 1.0, oi.support,
                                             oi.values)
    f0 = 0.5 * float((oi.b ** 2).sum())
    target = oi.f_star() + 1e-8 * (f0 - oi.f_star())
    tr, x = _solve(inst, 100000, rc=True, target_objective=target)
    otr, ox = oracle.fista(oi, max_iters=100000, target=target)
    assert tr.status == l1bench.StopReason.target_reached
    np.testing.assert_array_equal(tr.iters(), otr["iter"])
    np.testing.assert_array_equal(x, ox)
