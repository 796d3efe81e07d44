import sys, time, math
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1503_03520_b200 import l1bench
from bench import C4
torch.cuda.set_device(0)
inst = l1bench.build_instance(device=0, lazy_sparse=True, **C4)
sig, b, xs = inst.sigma(), inst.b, inst.x_star
m, n = inst.m, inst.n
stages = [((4 - 1 - i) % 2, C4["theta"]) for i in range(4)]
def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = a
    return t.numpy()
psig, pb = pinned(sig), pinned(b)
px = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
for label, s_, b_, x_ in [("pageable", sig, b, np.empty(n)), ("pinned", psig, pb, px), ("pinned2", psig, pb, px)]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    p = l1bench.ProblemInstance.from_host(m, n, stages, s_, b_, inst.tau, xs.support, xs.values, device=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    tr = l1bench.fista_run(p, l1bench.SolverConfig(max_iters=20), x_)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(label, "create %.1f ms" % ((t1 - t0) * 1e3), "solve+d2h %.1f ms" % ((t2 - t1) * 1e3), "iters", tr.iterations, "dev %.1f ms" % (tr.elapsed_s * 1e3))
    del p
