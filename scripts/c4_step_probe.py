"""Session.step vs Session.profile on the C4 instance (same kernels): outer
CUDA-event time per iteration, and the sum of per-launch event times."""
import math
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1503_03520_b200 import l1bench  # noqa: E402

inst = l1bench.build_instance(n=1 << 27, stages=4, q=1, s_divisor=1000, seed=3, theta=2 * math.pi / 10,
                              lazy_sparse=True)
stream = torch.cuda.ExternalStream(inst.stream)


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


for rep in range(2):
    for mode in ("step", "profile", "step20"):
        sess = l1bench.Session(inst, l1bench.SolverConfig(max_iters=2000))
        sess.step(4)
        if mode == "step":
            ms, _ = timed(lambda: sess.step(500))
            extra = ""
        elif mode == "profile":
            ms, k = timed(lambda: sess.profile(500))
            extra = f" sum-of-launches {k[0]:.1f} ms"
        else:
            def f():
                for _ in range(25):
                    sess.step(20)
            ms, _ = timed(f)
            extra = ""
        print(f"rep {rep} {mode:8s} {ms:8.2f} ms  {ms / 500:.4f} ms/iter{extra}", flush=True)
        sess.end()
