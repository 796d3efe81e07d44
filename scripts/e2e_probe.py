"""e2e pass breakdown (create / solve / free) and device memory per pass."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1503_03520_b200 import l1bench
from bench import C4
torch.cuda.set_device(0)
inst = l1bench.build_instance(device=0, lazy_sparse=True, **C4)
ARITH = sys.argv[2] if len(sys.argv) > 2 else "fma"
sig, b, xs = inst.sigma(), inst.b, inst.x_star
m, n = inst.m, inst.n
stages = [((4 - 1 - i) % 2, C4["theta"]) for i in range(4)]
def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[:] = a
    return t.numpy()
psig, pb = pinned(sig), pinned(b)
px = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 500
for rep in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    p = l1bench.ProblemInstance.from_host(m, n, stages, psig, pb, inst.tau, xs.support, xs.values, device=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    tr = l1bench.fista_run(p, l1bench.SolverConfig(max_iters=K, arith=ARITH), px)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    del p
    torch.cuda.synchronize(); t3 = time.perf_counter()
    free, tot = torch.cuda.mem_get_info()
    print(f"pass {rep}: create {(t1-t0)*1e3:.1f} ms solve+d2h {(t2-t1)*1e3:.1f} ms (device {tr.elapsed_s*1e3:.1f}) "
          f"free {(t3-t2)*1e3:.1f} ms; total {(t3-t0)*1e3:.1f} ms; device free {free/1e9:.1f} GB", flush=True)
