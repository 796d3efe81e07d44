"""Per-iteration device time of the small-instance FISTA paths (C1 shape)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1503_03520_b200 import l1bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
st = int(sys.argv[2]) if len(sys.argv) > 2 else 1
inst = l1bench.build_instance(n=n, stages=st, q=1, s_divisor=100, seed=0, theta=2 * math.pi / 10)
stream = torch.cuda.ExternalStream(inst.stream)
for it in (8, 64, 512):
    s = l1bench.Session(inst, l1bench.SolverConfig(max_iters=100000, op="matrix_free"))
    s.step(4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.step(it)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"n={n} stages={st} chunk={it}: {e0.elapsed_time(e1) * 1000 / it:.2f} us/iteration")
    s.end()
