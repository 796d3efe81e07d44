"""Where the end-to-end (host buffers -> C ABI -> host) time goes at C4."""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1503_03520_b200 import l1bench  # noqa: E402

C4 = dict(n=1 << 27, m_ratio=2.0, stages=4, q=1, shift=0.1, s_divisor=1000, gamma=10.0, tau=1.0,
          theta=2 * math.pi / 10, seed=3)
inst = l1bench.build_instance(lazy_sparse=True, **C4)
sig, b, xs = inst.sigma(), inst.b, inst.x_star
m, n = inst.m, inst.n
del inst
stages = [((4 - 1 - i) % 2, C4["theta"]) for i in range(4)]
x = np.empty(n)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = l1bench.ProblemInstance.from_host(m, n, stages, sig, b, 1.0, xs.support, xs.values)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tr = l1bench.fista_run(p, l1bench.SolverConfig(max_iters=20), x)
    t2 = time.perf_counter()
    del p
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rep {rep}: create {t1 - t0:.3f}s  solve(20 it + x D2H) {t2 - t1:.3f}s (device {tr.elapsed_s:.4f}s)  free {t3 - t2:.3f}s")
