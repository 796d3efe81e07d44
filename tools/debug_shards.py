"""Debug: first bitwise mismatch between sharded (emulated on one GPU) and
single-device matrix-free FISTA state."""
import ctypes as C
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from paper_1503_03520_b200 import _native as N  # noqa: E402
from paper_1503_03520_b200 import l1bench  # noqa: E402
from paper_1503_03520_b200.distributed import device_view  # noqa: E402
from test_gpu_shards import KW, _allreduce, _exchange, _shards  # noqa: E402

world, iters = 2, 6
inst = l1bench.build_instance(**KW)
cfg = l1bench.SolverConfig(max_iters=iters, op="matrix_free")
sess = l1bench.Session(inst, cfg)
b = N.ShardBuffers()
N.check(N.load().l1b_session_buffers(sess._s, C.byref(b)))
n = inst.n
x1 = device_view(b.x_win, n, torch.device("cuda", 0))
ry1 = device_view(b.r_y_win, 2 * n, torch.device("cuda", 0))
shards = _shards(world, iters, "matrix_free")
_allreduce(shards)
for s in shards:
    s.finalize()
_exchange(shards, "r_y_win")
for it in range(iters):
    sess.step(1)
    for s in shards:
        s.k1()
    _exchange(shards, "x_win")
    torch.cuda.synchronize()
    xs = torch.cat([s.x_win[s.halo:s.halo + s.own] for s in shards])
    d = (xs != x1).nonzero().flatten()
    print("iter", it + 1, "x mismatches", d.numel(), d[:10].tolist())
    for s in shards:
        s.k2()
    _allreduce(shards)
    for s in shards:
        s.finalize()
    _exchange(shards, "r_y_win")
    torch.cuda.synchronize()
    rys = torch.cat([s.r_y_win[s.halo:s.halo + s.own] for s in shards])
    d = (rys != ry1[:n]).nonzero().flatten()
    print("iter", it + 1, "r_y mismatches", d.numel(), d[:10].tolist(),
          float((rys - ry1[:n]).abs().max()))
    sc = [s.scal.cpu().numpy() for s in shards]
    print("  scal", sc[0])
