"""Instance files and traces (serialize.cpp:182-294): instances written by the
reference's save_instance load onto the device bit for bit (and solve like the
reference), instances written by l1bench.save_instance load into the
reference's load_instance bit for bit, and write_trace_csv keeps the
reference's columns and number formats."""
import csv
import math

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu

TH = 2 * math.pi / 10


@pytest.mark.parametrize("kw", [dict(n=2048, stages=4), dict(n=1500, stages=2, left_stages=1, permute=True),
                                dict(n=1024, stages=1, solution="spectral")])
def test_reference_file_loads_on_device(tmp_path, reference, kw):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(kw, q=1, s_divisor=64, seed=4, theta=TH)
    ri = reference.build_instance(**kw)
    path = tmp_path / "ref.l1i"
    reference.save_instance(ri, path)
    inst = l1bench.load_instance(str(path))
    np.testing.assert_array_equal(inst.b, ri.b())
    np.testing.assert_array_equal(inst.sigma(), ri.sigma())
    sup, val = ri.x_star()
    np.testing.assert_array_equal(inst.x_star.support, sup)
    np.testing.assert_array_equal(inst.x_star.values, val)
    assert inst.noise_norm == ri.noise_norm and inst.cert_kappa == ri.cert_kappa
    assert inst.objective_at_planted() == pytest.approx(ri.f_star, rel=1e-14)
    x = np.empty(inst.n)
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=30), x)
    rtr, rx = ri.solve("fista", max_iters=30)
    assert rel_err(x, rx) < 1e-10
    assert rel_err(tr.objectives(), rtr["objective"]) < 1e-10


@pytest.mark.parametrize("kw", [dict(n=2048, stages=4), dict(n=1500, stages=2, left_stages=1, permute=True)])
def test_device_file_loads_in_reference(tmp_path, reference, kw):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(kw, q=1, s_divisor=64, seed=9, theta=TH)
    inst = l1bench.build_instance(**kw)
    path = tmp_path / "dev.l1i"
    l1bench.save_instance(inst, str(path))
    ri = reference.load_instance(path)
    np.testing.assert_array_equal(ri.b(), inst.b)
    np.testing.assert_array_equal(ri.sigma(), inst.sigma())
    sup, val = ri.x_star()
    np.testing.assert_array_equal(sup, inst.x_star.support)
    np.testing.assert_array_equal(val, inst.x_star.values)
    assert ri.noise_norm == inst.noise_norm
    # and back: the round trip keeps the device instance
    back = l1bench.load_instance(str(path))
    np.testing.assert_array_equal(back.b, inst.b)
    assert back.stages(True) == inst.stages(True) and back.stages(False) == inst.stages(False)
    for w in (1, 2):
        a, c = back.perm(w), inst.perm(w)
        assert (a is None and c is None) or np.array_equal(a, c)


def test_trace_csv_format(tmp_path):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(n=1024, stages=2, q=1, s_divisor=64, seed=2, theta=TH)
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=12))
    path = tmp_path / "t.csv"
    l1bench.write_trace_csv(tr, str(path))
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["solver", "iter", "elapsed_s", "objective", "nnz_x", "matvecs", "extra"]
    assert len(rows) == 1 + len(tr.samples)
    for r, s in zip(rows[1:], tr.samples):
        assert r[0] == "fista" and int(r[1]) == s.iter and float(r[3]) == s.objective
        assert r[2] == "%.6f" % s.elapsed_s and r[5] == "%.3f" % s.matvecs
