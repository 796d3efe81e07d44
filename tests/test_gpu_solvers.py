"""GPU parity of coordinate descent (serial CD = the reference sampler; block
PCDM = the C2 mapping restated in oracle/l1oracle.c:lo_pcdm) and of Newton-CG
(pdNCG) against the reference traces."""
import numpy as np
import pytest

from conftest import golden_kwargs, load_golden
from gpu_util import device_build, need_cuda, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cd", "odd", "perm"])
def test_serial_cd_matches_reference(name):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    g = load_golden(name)
    inst = device_build(name)
    x = np.empty(inst.n)
    tr = l1bench.coordinate_descent_run(inst, l1bench.SolverConfig(max_iters=20, varpi=4, seed=5), x)
    assert tr.status == l1bench.StopReason.iter_budget
    assert rel_err(tr.objectives(), g["cd_obj"]) < 1e-10
    np.testing.assert_array_equal([s.extra for s in tr.samples], g["cd_extra"])
    np.testing.assert_allclose([s.matvecs for s in tr.samples], g["cd_matvecs"], rtol=1e-14)
    assert rel_err(x, g["cd_x"]) < 1e-10


@pytest.mark.parametrize("name,block", [("cd", 64), ("k4", 256), ("perm", 16)])
def test_block_pcdm_matches_oracle(oracle, name, block):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = device_build(name)
    oi = oracle.build_instance(**golden_kwargs(name))
    x = np.empty(inst.n)
    tr = l1bench.pcdm_run(inst, l1bench.SolverConfig(max_iters=25, block=block, seed=1), x)
    otr, ox = oracle.pcdm(oi, max_iters=25, block=block, seed=1)
    assert rel_err(tr.objectives(), otr["objective"]) < 1e-10
    np.testing.assert_array_equal([s.extra for s in tr.samples], otr["extra"])
    assert rel_err(x, ox) < 1e-10
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])
    # objective decreases towards f* (the planted optimum)
    assert tr.objectives()[-1] < tr.objectives()[0]
    assert tr.objectives()[-1] >= inst.objective_at_planted() * (1 - 1e-12)


@pytest.mark.parametrize("name,exact_steps", [("ncg", 8), ("cd", 8), ("odd", 4)])
def test_newton_cg_matches_reference(name, exact_steps):
    """Step-level parity while the PCG trajectories coincide; pdNCG is not
    reproducible across summation orders once kappa is large (SURVEY.md 0.7:
    the reference itself moves 891 -> 886 PCG iterations under 1e-16 operator
    rounding), so later steps are held to the smoothing band tau*n*mu."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    g = load_golden(name)
    inst = device_build(name)
    x = np.empty(inst.n)
    mu = 1e-5
    tr = l1bench.newton_cg_run(inst, l1bench.SolverConfig(max_iters=8, mu=mu), x)
    assert tr.status == l1bench.StopReason(int(g["ncg_status"]))
    np.testing.assert_array_equal(tr.iters(), g["ncg_iter"])
    ext, gext = np.array([s.extra for s in tr.samples]), g["ncg_extra"]
    same = len(ext) if np.array_equal(ext, gext) else int(np.argmax(ext != gext))
    assert same >= min(exact_steps, len(gext)), (ext, gext)
    obj = tr.objectives()
    assert rel_err(obj[:same], g["ncg_obj"][:same]) < 1e-10
    # after the trajectories part, both keep descending to the same optimum:
    # objective within 1e-3 relative of the reference's at every later step
    assert np.all(np.abs(obj - g["ncg_obj"]) <= 1e-3 * np.abs(g["ncg_obj"]))
    if same == len(gext):
        assert tr.total_pcg_iterations == int(g["ncg_pcg"])
        assert rel_err(x, g["ncg_x"]) < 1e-9


def test_pcg_single_solve_matches_reference(reference):
    """Per-operation parity: one PCG solve of the smoothed
    Newton system at a non-trivial x, same preconditioner -- via the first
    Newton step of newton_cg_run against pcg_solve on the reference."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    g = load_golden("ncg")
    kw = golden_kwargs("ncg")
    ri = reference.build_instance(**kw)
    inst = device_build("ncg")
    tr1 = l1bench.newton_cg_run(inst, l1bench.SolverConfig(max_iters=1))
    rtr, _ = ri.solve("newton_cg", max_iters=1)
    assert tr1.total_pcg_iterations == rtr["total_pcg_iterations"]
    assert rel_err(tr1.objectives(), rtr["objective"]) < 1e-12
