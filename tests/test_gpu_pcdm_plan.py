"""The planned PCDM epoch (k_pcdm.cu cd_epoch_plan_kernel: per-slot records +
shared-memory hash of the block's steps) against the direct epoch kernel
(cd_epoch_kernel, L1B_PCDM_PLAN=0) and the oracle's block-PCDM restatement:
identical iterates, applied counts and objectives."""
import math
import os

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu

TH = 2 * math.pi / 10


def _run(inst, solver, planned, **cfg):
    from paper_1503_03520_b200 import l1bench

    env = {"L1B_PCDM_PLAN": "1" if planned else "0", "L1B_PCDM_PAIR": "0"}  # pair-local path off
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        x = np.empty(inst.n)
        tr = l1bench.run_solver(inst, l1bench.SolverConfig(id=solver, **cfg), x)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    assert tr.ran("pcdm_plan" if planned else "pcdm_direct"), f"path={tr.path:#x}"
    return tr, x


@pytest.mark.parametrize("n,stages,block,solver", [(4096, 1, 256, "pcdm"), (6000, 2, 128, "pcdm"),
                                                   (3001, 1, 512, "pcdm"), (2048, 2, 1, "cd"),
                                                   (1000, 1, 1, "cd")])
def test_planned_epochs_match_direct_epochs(n, stages, block, solver):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=n, stages=stages, q=1, s_divisor=50, seed=7, theta=TH)
    kw = dict(max_iters=12, block=block, seed=3)
    if solver == "cd":
        kw = dict(max_iters=6, seed=3)
    tr_p, x_p = _run(inst, solver, True, **kw)
    tr_d, x_d = _run(inst, solver, False, **kw)
    np.testing.assert_array_equal(x_p, x_d)
    np.testing.assert_array_equal(tr_p.objectives(), tr_d.objectives())
    np.testing.assert_array_equal([s.extra for s in tr_p.samples], [s.extra for s in tr_d.samples])
    assert tr_p.iterations == tr_d.iterations


def test_planned_pcdm_matches_oracle(oracle):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(n=4096, stages=1, q=1, s_divisor=100, seed=1, theta=TH)
    inst = l1bench.build_instance(**kw)
    oi = oracle.build_instance(**kw)
    tr, x = _run(inst, "pcdm", True, max_iters=10, block=256, seed=1)
    otr, ox = oracle.pcdm(oi, max_iters=10, block=256, seed=1)
    assert rel_err(x, ox) < 1e-10
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-10
    np.testing.assert_array_equal([s.extra for s in tr.samples], otr["extra"])
