"""GPU: the pair-local PCG loop of Newton-CG (k_ncg.cu pcg_pair_kernel, one
right stage, identity permutations -- C1-C3's operators) against the oracle's
newton_cg (solvers.cpp:487-568 restated) and against the CSR/CSC PCG loop
(L1B_PCG_PAIR=0), for both stage offsets and odd / even n."""
import ctypes as C
import math
import os

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu
THETA = 2 * math.pi / 10


def _instance(oracle, n, off, q, seed):
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


def _run(inst, steps, pair):
    from paper_1503_03520_b200 import l1bench

    old = os.environ.get("L1B_PCG_PAIR")
    os.environ["L1B_PCG_PAIR"] = "1" if pair else "0"
    try:
        x = np.empty(inst.n)
        tr = l1bench.newton_cg_run(inst, l1bench.SolverConfig(max_iters=steps), x)
    finally:
        if old is None:
            del os.environ["L1B_PCG_PAIR"]
        else:
            os.environ["L1B_PCG_PAIR"] = old
    return tr, x


@pytest.mark.parametrize("n,off,q", [(1024, 0, 0), (3001, 1, 1), (3000, 1, 0), (2049, 0, 1), (7, 1, 0)])
def test_pair_pcg_matches_oracle_and_csr_loop(oracle, n, off, q):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    oi = _instance(oracle, n, off, q, seed=5 + n)
    inst = l1bench.ProblemInstance.from_host(oi.m, n, [(off, THETA)], oi.op.sigma, oi.b, 1.0, oi.support,
                                             oi.values)
    steps = 6
    tp, xp = _run(inst, steps, pair=True)
    tc, xc = _run(inst, steps, pair=False)
    otr, ox = oracle.newton_cg(oi, max_iters=steps)
    ext = np.array([s.extra for s in tp.samples])
    np.testing.assert_array_equal(ext, otr["extra"])  # PCG iterations per Newton step
    np.testing.assert_array_equal(ext, [s.extra for s in tc.samples])
    assert rel_err(tp.objectives(), otr["objective"]) < 1e-10
    assert rel_err(tp.objectives(), tc.objectives()) < 1e-10
    assert rel_err(xp, ox) < 1e-9
    assert tp.total_pcg_iterations == tc.total_pcg_iterations
