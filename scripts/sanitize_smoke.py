"""Small end-to-end exercise of every kernel family, for compute-sanitizer."""
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1503_03520_b200 import l1bench  # noqa: E402

TH = 2 * math.pi / 10
for kw in [dict(n=1000, stages=4, q=1, s_divisor=50, seed=3), dict(n=101, stages=3, q=2, seed=11, s_divisor=10),
           dict(n=777, stages=1, q=1, s_divisor=20, seed=5, solution="spectral"),
           dict(n=515, stages=2, q=1, s_divisor=20, seed=6, solution="two_value"),
           dict(n=96, m_ratio=1.5, stages=3, left_stages=2, permute=True, q=1, seed=7, s_divisor=16)]:
    inst = l1bench.build_instance(theta=TH, **kw)
    banded = not kw.get("permute")
    x = torch.randn(inst.n, dtype=torch.float64, device="cuda")
    y = torch.randn(inst.m, dtype=torch.float64, device="cuda")
    for path in (["sparse", "sweep", "fused"] if banded else ["sparse", "sweep"]):
        inst.op.apply(x, path=path)
        inst.op.apply_transpose(y, path=path)
    inst.op.gram_diagonal()
    l1bench.verify_optimality(inst, 1e-8)
    for op in (["sparse", "matrix_free"] if banded else ["sparse"]):
        l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=30, op=op))
        l1bench.ista_run(inst, l1bench.SolverConfig(max_iters=10, op=op))
    l1bench.coordinate_descent_run(inst, l1bench.SolverConfig(max_iters=3, varpi=4))
    l1bench.pcdm_run(inst, l1bench.SolverConfig(max_iters=3, block=16))
    l1bench.newton_cg_run(inst, l1bench.SolverConfig(max_iters=2, pcg_max_iters=50))
    torch.cuda.synchronize()
# emulated shards (matrix-free single kernel + CSR/CSC)
import test_gpu_shards as T  # noqa: E402
from pyoracle import Oracle  # noqa: E402  (the shard tests' checker)

ORC = Oracle()
T.KW = dict(n=4096, stages=4, q=1, s_divisor=100, seed=3, theta=TH)
for op in ("matrix_free", "sparse"):
    T.test_shards_reproduce_single_device_fista(2, op, ORC)
T.KW_PERM = dict(n=1024, stages=2, left_stages=1, permute=True, q=1, s_divisor=50, seed=6, theta=TH)
T.test_general_shards_reproduce_single_device_fista(2, ORC)
# the C2 path at a small size: jump-started coordinate stream, sorted look-back,
# device walk over several segments, event masks, the cp.async epoch kernel,
# fold; serial CD (B = 1); with a target (cooperative epochs)
c2 = l1bench.build_instance(n=8192, stages=1, q=1, s_divisor=100, seed=1, theta=TH)
l1bench.pcdm_run(c2, l1bench.SolverConfig(max_iters=30, block=256, seed=1))
l1bench.coordinate_descent_run(c2, l1bench.SolverConfig(max_iters=5, seed=1))
l1bench.pcdm_run(c2, l1bench.SolverConfig(max_iters=10, block=256, seed=1, target_objective=1.0))
torch.cuda.synchronize()
print("sanitize smoke done")
