"""GPU parity at BASELINE.json's OWN configuration sizes (SURVEY.md 8(d)
tall reading), against the unmodified reference built
from its sources (oracle/_ref) or the oracle pinned to it:

  C2  n=2^15, q=1, seed 1: block PCDM (B=256, 100 epochs) vs the oracle's
      lo_pcdm, and the reference's own serial CD (solvers.cpp:414-482) bit for
      bit -- both on the pair-local path (asserted through l1b_summary.path)
  C3  n=2^19, q=2 (kappa ~ 1e6), seed 2: the first Newton step (PCG count,
      objective), a Hessian-vector probe (solvers.cpp:188-200) and the final
      objective of the 30-step run within the smoothing band tau*n*mu of the
      reference's own 30-step run (trajectories part at this kappa,
      SURVEY.md 0.7 / 8(c))
  C4  n=2^27, 4 stages, q=1, seed 3: sigma, b and x* of the device generator
      bit-identical to the reference's generator; the first 4 FISTA iterations
      bit-identical (exact arithmetic) / within 1e-12 (fma) of fista_run
  C5  n=2^32, q=0, seed 4: rank 7 of the 8-way row split -- its sigma window,
      the fill stream window it draws and L = sigma_max^2 against the oracle's
      sequential mt19937_64 streams over all 2^32 draws

These run minutes of single-threaded reference CPU work (C4: ~20 GB of host
memory); the GPU box has the cores and memory for them."""
import ctypes
import math
import os
import threading

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu

TH = 2 * math.pi / 10
C2 = dict(n=1 << 15, stages=1, q=1, s_divisor=100, seed=1, theta=TH)
C3 = dict(n=1 << 19, stages=1, q=2, s_divisor=1000, seed=2, theta=TH)
C4 = dict(n=1 << 27, stages=4, q=1, s_divisor=1000, seed=3, theta=TH)
C5 = dict(n=1 << 32, stages=4, q=0, s_divisor=10000, seed=4, theta=TH)
MU = 1e-5


# ---------------------------------------------------------------- C2 ------
def test_c2_block_pcdm_matches_oracle(oracle):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(**C2)
    x = np.empty(inst.n)
    tr = l1bench.pcdm_run(inst, l1bench.SolverConfig(max_iters=100, block=256, seed=1), x)
    assert tr.ran("pcdm_pair"), f"pair-local path not taken (path={tr.path:#x})"
    assert tr.iterations == 100 and tr.status == l1bench.StopReason.iter_budget
    otr, ox = oracle.pcdm(oracle.build_instance(**C2), max_iters=100, block=256, seed=1)
    np.testing.assert_array_equal([s.extra for s in tr.samples], otr["extra"])  # applied updates
    assert rel_err(x, ox) < 1e-10
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-10
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])
    np.testing.assert_array_equal([s.nnz for s in tr.samples], otr["nnz"])


def test_c2_serial_cd_matches_reference(reference):
    """The reference's algorithm on the C2 instance: serial randomized CD,
    100 sweeps, seed 1 -- iterates bit for bit."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(**C2)
    x = np.empty(inst.n)
    tr = l1bench.coordinate_descent_run(inst, l1bench.SolverConfig(max_iters=100, seed=1), x)
    assert tr.ran("pcdm_pair"), f"pair-local path not taken (path={tr.path:#x})"
    ri = reference.build_instance(**C2)
    rtr, rx = ri.solve("cd", max_iters=100, seed=1)
    np.testing.assert_array_equal(x, rx)
    np.testing.assert_array_equal(tr.iters(), rtr["iter"])
    np.testing.assert_array_equal([s.extra for s in tr.samples], rtr["extra"])
    np.testing.assert_array_equal([s.nnz for s in tr.samples], rtr["nnz"])
    assert rel_err(tr.objectives(), rtr["objective"]) < 1e-12
    np.testing.assert_allclose([s.matvecs for s in tr.samples], rtr["matvecs"], rtol=1e-14)


# ---------------------------------------------------------------- C3 ------
@pytest.fixture(scope="module")
def c3(reference):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    return l1bench.build_instance(**C3), reference.build_instance(**C3)


def test_c3_generator_matches_reference(c3):
    inst, ri = c3
    np.testing.assert_array_equal(inst.b, ri.b())
    np.testing.assert_array_equal(inst.sigma(), ri.sigma())


def test_c3_first_newton_step_matches_reference(c3):
    from paper_1503_03520_b200 import l1bench

    inst, ri = c3
    x = np.empty(inst.n)
    tr = l1bench.newton_cg_run(inst, l1bench.SolverConfig(max_iters=1, mu=MU), x)
    assert tr.ran("pcg_pair"), f"pair-local PCG not taken (path={tr.path:#x})"
    rtr, rx = ri.solve("newton_cg", max_iters=1, mu=MU)
    assert tr.total_pcg_iterations == rtr["total_pcg_iterations"] > 0
    np.testing.assert_array_equal([s.extra for s in tr.samples], rtr["extra"])
    assert rel_err(tr.objectives(), rtr["objective"]) < 1e-10
    assert rel_err(x, rx) < 1e-10


def test_c3_hessvec_probe_matches_reference(c3):
    """One Hessian-vector product at the reference's first Newton iterate
    (dense, all |x_i| ~ mu .. 10) on a seeded direction."""
    torch = need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst, ri = c3
    _, x1 = ri.solve("newton_cg", max_iters=1, mu=MU)
    v = np.random.default_rng(7).uniform(-1.0, 1.0, inst.n)
    want = ri.smoothed_hessvec(x1, MU, v)
    got = l1bench.smoothed_hessvec(inst, torch.from_numpy(x1).cuda(), MU, torch.from_numpy(v).cuda())
    assert rel_err(got.cpu().numpy(), want) < 1e-13


def test_c3_thirty_steps_within_smoothing_band(c3):
    """The C3 run itself: 30 Newton steps on both sides.  At kappa ~ 1e6 the
    PCG trajectories part under summation-order rounding (the reference
    itself does), so the final objectives are compared within
    the pdNCG smoothing band tau*n*mu, and the supports by |x_i| > 10 mu."""
    from paper_1503_03520_b200 import l1bench

    inst, ri = c3
    x = np.empty(inst.n)
    tr = l1bench.newton_cg_run(inst, l1bench.SolverConfig(max_iters=30, mu=MU), x)
    rtr, rx = ri.solve("newton_cg", max_iters=30, mu=MU)
    assert tr.iterations == 30 == rtr["newton_steps"] or tr.status == l1bench.StopReason(rtr["status"])
    band = inst.tau * inst.n * MU
    assert abs(tr.final_objective - rtr["final_objective"]) <= band, (tr.final_objective, rtr["final_objective"])
    f_star = inst.objective_at_planted()
    assert tr.final_objective >= f_star - band
    sup, rsup = np.abs(x) > 10 * MU, np.abs(rx) > 10 * MU
    # the planted support is found by both, and the large-entry supports agree
    # but for entries within the smoothing scale of the threshold
    xs = inst.x_star.support
    assert sup[xs].all() and rsup[xs].all()
    differ = np.nonzero(sup != rsup)[0]
    assert np.all(np.minimum(np.abs(x[differ]), np.abs(rx[differ])) < 100 * MU), differ[:10]


# ---------------------------------------------------------------- C4 ------
@pytest.fixture(scope="module")
def c4(reference):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    ri = reference.build_instance(**C4)
    inst = l1bench.build_instance(lazy_sparse=True, **C4)
    return inst, ri


def test_c4_generator_bit_exact(c4):
    inst, ri = c4
    assert (inst.n, inst.m) == (1 << 27, 1 << 28)
    np.testing.assert_array_equal(inst.sigma(), ri.sigma())
    np.testing.assert_array_equal(inst.b, ri.b())
    sup, val = ri.x_star()
    np.testing.assert_array_equal(inst.x_star.support, sup)
    np.testing.assert_array_equal(inst.x_star.values, val)
    assert inst.info.gram_lmax == ri.gram_lmax
    # ||e|| is a reduction: the device sums in a tree, the reference left to right
    assert abs(inst.noise_norm - ri.noise_norm) <= 1e-12 * ri.noise_norm


def test_c4_first_iterations_match_fista_run(c4):
    """C4 itself (n = 2^27) against the reference's own fista_run, 8
    iterations (~50 s of reference CPU time): the tile kernel (one launch of 6
    iterations on chip-resident tiles, then a two-iteration launch) and the
    two-iteration kernel alone (L1B_TB=0), each in the exact arithmetic (the
    reference's bits) and in the contracted one (<= 1e-12, same support); then,
    without the reference, the default 14-iteration tile launch against the
    two-iteration kernel over 16 iterations, bit for bit in both arithmetics."""
    from paper_1503_03520_b200 import l1bench

    inst, ri = c4

    def run(tile, arith, iters, k=None):
        env = {"L1B_TB": "1" if tile else "0"}
        if k:
            env["L1B_TB_K"] = str(k)
        old = {key: os.environ.get(key) for key in env}
        os.environ.update(env)
        try:
            x = np.empty(inst.n)
            tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=iters, arith=arith), x)
        finally:
            for key, v in old.items():
                if v is None:
                    del os.environ[key]
                else:
                    os.environ[key] = v
        assert tr.ran("fista_tile") == tile and tr.ran("fista_two_iter"), f"path={tr.path:#x}"
        assert tr.ran("fma") == (arith == "fma"), f"path={tr.path:#x}"
        return tr, x

    iters = 8
    rtr, rx = ri.solve("fista", max_iters=iters)
    xfs = []
    for tile in (True, False):
        for arith in ("exact", "fma"):
            tr, x = run(tile, arith, iters, k=6)
            np.testing.assert_array_equal(tr.iters(), rtr["iter"])
            assert rel_err(tr.objectives(), rtr["objective"]) < 1e-12
            np.testing.assert_array_equal([s.nnz for s in tr.samples], rtr["nnz"])
            if arith == "exact":
                np.testing.assert_array_equal(x, rx)
            else:
                assert rel_err(x, rx) < 1e-12
                np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(rx)[0])
                xfs.append(x)
    # (the same operations per entry in both kernels: the contracted arithmetic too is
    # independent of the launch shape -- and of the row split, which runs the second kernel)
    np.testing.assert_array_equal(xfs[0], xfs[1])
    del xfs, rx
    for arith in ("exact", "fma"):
        tr1, x1 = run(True, arith, 16)
        tr2, x2 = run(False, arith, 16)
        np.testing.assert_array_equal(x1, x2)
        assert rel_err(tr1.objectives(), tr2.objectives()) < 1e-13
        np.testing.assert_array_equal([s.nnz for s in tr1.samples], [s.nnz for s in tr2.samples])


# ---------------------------------------------------------------- C5 ------
def _oracle_window(oracle, seed, count, lo, hi, spectrum, shift, wlo, whi):
    L = oracle.lib
    L.lo_uniform_stream_window.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double)]
    out = np.empty(whi - wlo)
    vmin, vmax = ctypes.c_double(), ctypes.c_double()
    L.lo_uniform_stream_window(seed, count, lo, hi, spectrum, shift, wlo, whi, out.ctypes.data,
                               ctypes.byref(vmin), ctypes.byref(vmax))
    return out, vmin.value, vmax.value


def test_c5_rank_shard_streams_match_oracle(oracle):
    """Rank 7 of the 8-way split of C5 (rows [7 * 2^29, 2^32)): the sigma
    window the shard holds and its L = sigma_max^2 over all 2^32 draws, and the
    fill-stream window its generator draws (same device call, same window),
    against the oracle's sequential streams (ctypes releases the GIL: the two
    2^32-draw streams run on two host threads)."""
    torch = need_cuda()
    from paper_1503_03520_b200 import _native as N
    from paper_1503_03520_b200 import l1bench

    n = C5["n"]
    sh = l1bench.build_instance(lazy_sparse=True, shard=(7, 8), **C5)
    info = sh.info
    assert (int(info.row_begin), int(info.row_end)) == (7 << 29, n)
    sa, sig = sh.sigma_window()
    sb = sa + len(sig)
    assert sa <= int(info.row_begin) and sb == n
    job = oracle.mix_seed(C5["seed"], 0)
    res = {}

    def run(key, *a):
        res[key] = _oracle_window(oracle, *a)

    th = [threading.Thread(target=run, args=("sigma", oracle.mix_seed(job, 3), n, 0.0, 1.0, 1, 0.1, sa, sb)),
          threading.Thread(target=run, args=("fill", oracle.mix_seed(job, 5), n, -0.9, 0.9, 0, 0.0, sa, sb))]
    for t in th:
        t.start()
    # the fill window through the call the shard generator makes (abi.cu l1b_generate)
    fill = torch.empty(sb - sa, dtype=torch.float64, device="cuda")
    exact = ctypes.c_int()
    N.check(N.load().l1b_device_uniform_draws(0, oracle.mix_seed(job, 5), n, -0.9, 0.9, 0, 0.0, sa, sb, 12,
                                              ctypes.c_void_p(fill.data_ptr()), None, None, ctypes.byref(exact)))
    got_fill = fill.cpu().numpy()
    for t in th:
        t.join()
    want_sig, smin, smax = res["sigma"]
    want_fill, _, _ = res["fill"]
    np.testing.assert_array_equal(sig, want_sig)
    np.testing.assert_array_equal(got_fill, want_fill)
    assert info.gram_lmax == smax * smax
    assert info.cert_kappa == (smax / smin) * (smax / smin)
