"""The reference's own experiment driver on the device: run_experiment
(src/bench.cpp:364-457, unchanged, from the reference library built by
oracle/Makefile) with its run_solver calls (:414, :450) bound to
l1bench::b200::run_solver by integration/libl1bench_b200_interpose.so
(integration/run_experiment_b200), against the same driver on the reference's
CPU solvers (integration/run_experiment_ref).  Presets from the reference's
catalog (src/bench.cpp:472-587).  The device build must launch kernels (the
interposition took effect) and every summary.csv row must agree: same solver,
status and target-reached flag, targets and final objectives within 1e-10."""
import csv
import os
import re
import subprocess

import pytest

from conftest import ROOT
from gpu_util import need_cuda

pytestmark = pytest.mark.gpu

BUILD = os.path.join(ROOT, "integration", "_build")


def _run(exe, preset, out, n=None):
    cmd = [os.path.join(BUILD, exe), preset, str(out)] + ([str(n)] if n else [])
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr + p.stdout
    launches = int(re.search(r"device_launches=(\d+)", p.stdout).group(1))
    with open(os.path.join(out, "summary.csv")) as f:
        rows = list(csv.DictReader(f))
    return rows, launches


def _rel(a, b):
    a, b = float(a), float(b)
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("preset,n", [("smoke", None), ("nontrivial-sweep", 1024)])
def test_run_experiment_on_device_matches_reference(tmp_path, preset, n):
    need_cuda()
    for exe in ("run_experiment_ref", "run_experiment_b200"):
        if not os.path.exists(os.path.join(BUILD, exe)):
            pytest.skip("integration/_build not built (needs the reference headers)")
    ref, l_ref = _run("run_experiment_ref", preset, tmp_path / "cpu", n)
    dev, l_dev = _run("run_experiment_b200", preset, tmp_path / "gpu", n)
    assert l_ref == 0 and l_dev > 0, "run_solver was not interposed"
    assert len(dev) == len(ref) > 0
    for r, d in zip(ref, dev):
        key = (r["instance"], r["solver"])
        assert (d["instance"], d["solver"]) == key
        assert d["status"] == r["status"], key
        assert d["reached"] == r["reached"], key
        assert _rel(d["target"], r["target"]) < 1e-10, key
        assert _rel(d["final_objective"], r["final_objective"]) < 1e-10, key
        if r["solver"] in ("fista", "ista"):
            assert float(d["matvecs_total"]) == float(r["matvecs_total"]), key
    for sub in ("instances", "traces", "plots"):
        assert sorted(os.listdir(tmp_path / "gpu" / sub)) == sorted(os.listdir(tmp_path / "cpu" / sub))
