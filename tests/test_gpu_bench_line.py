"""The bench lines the driver parses, on a small instance: the one-GPU line
and the N > 1 line (row-sharded native NCCL driver) at one rank -- every key
of the contract present, the e2e and roofline blocks filled, the timings
positive.  Guards bench.py / distributed.bench_main against regressions that
would only surface in the round-end scaling run."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def _check(d):
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    # (the tile kernel, n > 2^20 on one GPU, is bound by the FP64 pipe and says so;
    # its HBM side rides along in r["hbm"])
    assert r["achieved"] > 0 and r["peak"] > 0
    assert (r["bound"], r["unit"]) in (("hbm", "GB/s"), ("fp64", "TFLOP/s"))
    if r["bound"] == "fp64":
        assert r["hbm"]["unit"] == "GB/s" and r["hbm"]["achieved"] > 0 and r["hbm"]["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


def test_single_gpu_line():
    from gpu_util import need_cuda

    need_cuda()
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--n", str(1 << 21), "--steps", "20",
                        "--warmup", "4", "--no-cpu", "--no-configs"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    d = _line(p.stdout)
    _check(d)
    assert d["n_gpus"] == 1 and d["steps"] == 20
    assert d["other_arith"]["value"] > 0 and d["sparse_path"]["value"] > 0
    assert "k500" in d["e2e_more"] and "serving_resident_operator" in d["e2e_more"]


def test_sharded_line_one_rank():
    from gpu_util import need_cuda

    need_cuda()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--force-dist", "--columns", str(1 << 22), "--steps", "20", "--warmup", "4", "--no-cpu"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    d = _line(p.stdout)
    _check(d)
    assert d["config"]["driver"].startswith("native")
    assert d["roofline"]["per_rank"] and d["roofline"]["aggregate_frac"] > 0
    assert d["iterations_timed"] == 20
