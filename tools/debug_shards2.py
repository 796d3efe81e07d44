"""Debug: iteration-1 x of single-device fused, sharded fused and the oracle."""
import ctypes as C
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_1503_03520_b200 import _native as N  # noqa: E402
from paper_1503_03520_b200 import l1bench  # noqa: E402
from paper_1503_03520_b200.distributed import device_view  # noqa: E402
from pyoracle import Oracle  # noqa: E402
from test_gpu_shards import KW, _allreduce, _exchange, _shards  # noqa: E402

O = Oracle()
oi = O.build_instance(**KW)
g = O.apply_transpose(oi.op, -oi.b)
L = O.gram_lmax(oi.op)
inv_l = 1.0 / L
thr = oi.tau * inv_l
v = 0.0 - inv_l * g
trial = np.where(v > thr, v - thr, np.where(v < -thr, v + thr, 0.0))

for op in ["matrix_free", "sparse"]:
    inst = l1bench.build_instance(**KW)
    sess = l1bench.Session(inst, l1bench.SolverConfig(max_iters=3, op=op))
    b = N.ShardBuffers()
    N.check(N.load().l1b_session_buffers(sess._s, C.byref(b)))
    x1 = device_view(b.x_win, inst.n, torch.device("cuda", 0))
    sess.step(1)
    torch.cuda.synchronize()
    x1 = x1.cpu().numpy()
    print(op, "single vs oracle: mismatches", int((x1 != trial).sum()), "max", float(np.abs(x1 - trial).max()))
    shards = _shards(2, 3, op)
    _allreduce(shards)
    for s in shards:
        s.finalize()
    _exchange(shards, "r_y_win")
    for s in shards:
        s.k1()
    torch.cuda.synchronize()
    xs = np.concatenate([s.x_win[s.halo:s.halo + s.own].cpu().numpy() for s in shards])
    print(op, "shards vs oracle: mismatches", int((xs != trial).sum()), "max", float(np.abs(xs - trial).max()))
    ry = np.concatenate([s.r_y_win[s.halo:s.halo + s.own].cpu().numpy() for s in shards])
    print(op, "shard r_y == -b:", bool(np.array_equal(ry, 0.0 - oi.b[: inst.n])))
    sg = shards[0]
    print("rank0 window halo", sg.r_y_win[:6].cpu().numpy(), "own0", (0.0 - oi.b[:2]))
