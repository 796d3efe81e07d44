"""The pair-local CD / PCDM epochs (k_pcdm.cu cd_pair_kernel, coordinate
stream drawn on the device by mt_stream_indices + cd_walk_kernel) against the
direct epoch kernel (L1B_PCDM_PAIR=0: host draws, cd_epoch_plan_kernel) and
the oracle's block-PCDM restatement: identical iterates and applied counts;
objectives agree to the summation order (the pair kernel folds per-pair
partials)."""
import math
import os

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu

TH = 2 * math.pi / 10


def _run(inst, solver, pair, **cfg):
    from paper_1503_03520_b200 import l1bench

    old = os.environ.get("L1B_PCDM_PAIR")
    os.environ["L1B_PCDM_PAIR"] = "1" if pair else "0"
    try:
        x = np.empty(inst.n)
        tr = l1bench.run_solver(inst, l1bench.SolverConfig(id=solver, **cfg), x)
    finally:
        if old is None:
            del os.environ["L1B_PCDM_PAIR"]
        else:
            os.environ["L1B_PCDM_PAIR"] = old
    return tr, x


@pytest.mark.parametrize("n,block,solver,epochs", [(4096, 256, "pcdm", 12), (3001, 512, "pcdm", 9),
                                                   (20000, 64, "pcdm", 7), (1000, 1, "cd", 6),
                                                   (4097, 1, "cd", 3), (65536, 1024, "pcdm", 4),
                                                   (8192, 256, "pcdm", 150),    # three chunks, drawn ahead
                                                   (65536, 256, "pcdm", 520)])  # > 2^25 draws: a rewind
def test_pair_epochs_match_direct_epochs(n, block, solver, epochs):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=n, stages=1, q=1, s_divisor=50, seed=7, theta=TH)
    kw = dict(max_iters=epochs, block=block, seed=3)
    if solver == "cd":
        kw = dict(max_iters=epochs, seed=3, varpi=4)
    tr_p, x_p = _run(inst, solver, True, **kw)
    tr_d, x_d = _run(inst, solver, False, **kw)
    assert tr_p.ran("pcdm_pair") and not tr_d.ran("pcdm_pair"), (tr_p.path, tr_d.path)
    np.testing.assert_array_equal(x_p, x_d)
    np.testing.assert_array_equal([s.extra for s in tr_p.samples], [s.extra for s in tr_d.samples])
    np.testing.assert_array_equal([s.nnz for s in tr_p.samples], [s.nnz for s in tr_d.samples])
    np.testing.assert_allclose([s.matvecs for s in tr_p.samples], [s.matvecs for s in tr_d.samples],
                               rtol=1e-15)
    assert rel_err(tr_p.objectives(), tr_d.objectives()) < 1e-12
    assert tr_p.iterations == tr_d.iterations == epochs
    assert tr_p.status == tr_d.status


def test_pair_pcdm_matches_oracle_c2_shape(oracle):
    """The C2 recipe (one stage, q = 1, s = n/100, seed 1, blocks of 256) at
    n = 2^13, 30 epochs."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=8192, stages=1, q=1, s_divisor=100, seed=1, theta=TH)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    tr, x = _run(inst, "pcdm", True, max_iters=30, block=256, seed=1)
    assert tr.ran("pcdm_pair"), tr.path
    otr, ox = oracle.pcdm(oi, max_iters=30, block=256, seed=1)
    assert rel_err(x, ox) < 1e-10
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-10
    np.testing.assert_array_equal([s.extra for s in tr.samples], otr["extra"])
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])


def test_pair_pcdm_target_stop_matches_direct():
    """A target met mid-chunk: both paths stop at the same epoch with the same x."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=4096, stages=1, q=1, s_divisor=100, seed=2, theta=TH)
    full, _ = _run(inst, "pcdm", False, max_iters=40, block=128, seed=9)
    f = full.objectives()
    target = float(f[17] * (1 + 1e-9))  # first met at or before epoch 17
    tr_p, x_p = _run(inst, "pcdm", True, max_iters=40, block=128, seed=9, target_objective=target)
    tr_d, x_d = _run(inst, "pcdm", False, max_iters=40, block=128, seed=9, target_objective=target)
    assert tr_p.ran("pcdm_pair") and not tr_d.ran("pcdm_pair")
    assert tr_p.status == tr_d.status == l1bench.StopReason.target_reached
    assert tr_p.iterations == tr_d.iterations <= 17
    np.testing.assert_array_equal(x_p, x_d)


def test_pair_path_not_taken_for_two_stages():
    """Two stages couple neighbouring pairs: the pair path must decline (the
    switch changes nothing) and the results stay those of the direct path."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=4096, stages=2, q=1, s_divisor=50, seed=7, theta=TH)
    tr_p, x_p = _run(inst, "pcdm", True, max_iters=5, block=256, seed=3)
    tr_d, x_d = _run(inst, "pcdm", False, max_iters=5, block=256, seed=3)
    assert not tr_p.ran("pcdm_pair") and tr_p.path == tr_d.path
    np.testing.assert_array_equal(x_p, x_d)
    np.testing.assert_array_equal(tr_p.objectives(), tr_d.objectives())


@pytest.mark.parametrize("n,block,solver,epochs,shift", [(1000, 1, "cd", 6, 3), (4097, 1, "cd", 4, 1),
                                                         (4096, 256, "pcdm", 10, 3), (3001, 512, "pcdm", 6, 2),
                                                         (65536, 1024, "pcdm", 3, 4), (8192, 256, "pcdm", 150, 5)])
def test_redrawn_draws_match_direct_and_oracle(oracle, n, block, solver, epochs, shift):
    """Draws the reference rejects (x >= UINT64_MAX - UINT64_MAX % n) come once
    per ~2^64/n draws, so the walk's redraw handling (B = 1: blocks extended by
    rejected draws, cd_b1_starts_kernel; B > 1: kPrevRej candidates) never meets
    a real stream.  L1B_TEST_INDEX_REJECT=s (and the oracle's
    lo_set_index_reject) lower the limit so ~2^-s of the draws are redrawn:
    the pair path, the direct path and the oracle must still agree."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=n, stages=1, q=1, s_divisor=50, seed=7, theta=TH)
    inst = l1bench.build_instance(**kw)
    cfg = dict(max_iters=epochs, seed=3, varpi=4) if solver == "cd" else dict(max_iters=epochs, block=block, seed=3)
    tr_0, x_0 = _run(inst, solver, True, **cfg)
    os.environ["L1B_TEST_INDEX_REJECT"] = str(shift)
    oracle.set_index_reject(shift)
    try:
        tr_p, x_p = _run(inst, solver, True, **cfg)
        tr_d, x_d = _run(inst, solver, False, **cfg)
        oi = oracle.build_instance(**kw)
        if solver == "cd":
            otr, ox = oracle.cd(oi, **cfg)
        else:
            otr, ox = oracle.pcdm(oi, **cfg)
    finally:
        del os.environ["L1B_TEST_INDEX_REJECT"]
        oracle.set_index_reject(0)
    assert tr_p.ran("pcdm_pair") and not tr_d.ran("pcdm_pair"), (tr_p.path, tr_d.path)
    assert not np.array_equal(x_0, x_p)  # the hook moved the stream
    np.testing.assert_array_equal(x_p, x_d)
    np.testing.assert_array_equal([s.extra for s in tr_p.samples], [s.extra for s in tr_d.samples])
    np.testing.assert_array_equal([s.extra for s in tr_p.samples], otr["extra"])
    assert rel_err(x_p, ox) < 1e-10
    assert rel_err(tr_p.objectives(), otr["objective"]) < 1e-10
