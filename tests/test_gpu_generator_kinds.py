"""The generator's SolutionRule kinds (bench.cpp:281-301) against the
reference's own build_instance (oracle/_ref): spectral_sparse_solution
(solution.cpp:77-113) and the two-value support, with the uniform and
alternating spectra, permuted or not -- x*, sigma and b bit-exact."""
import math

import numpy as np
import pytest

from gpu_util import need_cuda

pytestmark = pytest.mark.gpu

TH = 2 * math.pi / 10


@pytest.mark.parametrize("kw", [
    dict(n=4096, stages=1, solution="spectral"),
    dict(n=4099, stages=4, solution="spectral", s1_fraction=0.25),
    dict(n=3000, stages=2, left_stages=1, permute=True, solution="spectral", s1_fraction=1.0),
    dict(n=2048, stages=3, solution="two_value"),
    dict(n=2049, stages=2, permute=True, solution="two_value", value_a=3.5, value_b=-0.25),
    dict(n=1024, stages=1, solution="uniform"),
])
def test_solution_kinds_match_reference(reference, kw):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(kw, q=1, s_divisor=64, seed=11, theta=TH)
    inst = l1bench.build_instance(**kw)
    ri = reference.build_instance(**kw)
    xs = inst.x_star
    sup, val = ri.x_star()
    np.testing.assert_array_equal(np.asarray(xs.support, dtype=np.int64), np.asarray(sup, dtype=np.int64))
    np.testing.assert_array_equal(np.asarray(xs.values), np.asarray(val))
    np.testing.assert_array_equal(inst.sigma(), ri.sigma())
    np.testing.assert_array_equal(inst.b, ri.b())
    assert inst.objective_at_planted() == pytest.approx(ri.f_star, rel=1e-13)


def test_spectral_solution_rejected_on_banded_shards():
    need_cuda()
    from paper_1503_03520_b200 import _native as N
    from paper_1503_03520_b200.distributed import CudaShard
    from paper_1503_03520_b200 import l1bench

    with pytest.raises(Exception):
        CudaShard(dict(n=4096, stages=2, solution="spectral"), 0, 2, 0, l1bench.SolverConfig(max_iters=5))
