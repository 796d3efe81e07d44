"""Where the C4 solve's device time goes: trace timestamps of l1b_solve."""
import math
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1503_03520_b200 import l1bench  # noqa: E402

inst = l1bench.build_instance(n=1 << 27, stages=4, q=1, s_divisor=1000, seed=3, theta=2 * math.pi / 10,
                              lazy_sparse=True)
for rep in range(2):
    torch.cuda.synchronize()
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=500))
    el = [s.elapsed_s for s in tr.samples]
    its = [s.iter for s in tr.samples]
    pick = [0, 1, 2, 3, 4, 6, 10, 20, 50, 100, 200, 300, 400, 499, 500]
    print("rep", rep, "total", tr.elapsed_s, [(its[i], round(el[i] * 1e3, 3)) for i in pick if i < len(el)])

# the same 500 iterations through a Session (bench.py's path), CUDA events
for rep in range(2):
    cfg = l1bench.SolverConfig(max_iters=600)
    sess = l1bench.Session(inst, cfg)
    stream = torch.cuda.ExternalStream(inst.stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sess.step(500)
    e1.record(stream)
    torch.cuda.synchronize()
    print("session step(500) ms", e0.elapsed_time(e1))
    sess.end()
# solve again with a wall clock around it
import time  # noqa: E402
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=500))
    torch.cuda.synchronize()
    print("fista_run wall ms", (time.perf_counter() - t) * 1e3, "device elapsed ms", tr.elapsed_s * 1e3)
