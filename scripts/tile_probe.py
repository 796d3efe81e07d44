"""A/B of the tile kernel (K iterations per launch) against the two-iteration
kernel on C4: device time of K timed iterations after a warm-up, per arith."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_03520_b200 import l1bench  # noqa: E402

C4 = dict(n=1 << 27, stages=4, q=1, s_divisor=1000, seed=3)


def run(inst, env, iters, arith):
    os.environ.update(env)
    cfg = l1bench.SolverConfig(max_iters=iters + 40, op="matrix_free", arith=arith)
    s = l1bench.Session(inst, cfg)
    stream = torch.cuda.ExternalStream(inst.stream)
    s.step(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s.step(iters)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kms = s.profile(20)
    s.end()
    return {"env": env, "arith": arith, "iters": iters, "ips": 1000 * iters / ms, "prof_ms_per_iter": kms[0] / 20}


inst = l1bench.build_instance(**C4)
out = []
for arith in ("fma", "exact"):
    for env in ({"L1B_TB": "0"}, {"L1B_TB": "1", "L1B_TB_K": "10"}, {"L1B_TB": "1", "L1B_TB_K": "14"}):
        for iters in (20 if False else 100, 500):
            r = run(inst, env, iters, arith)
            print(json.dumps(r), flush=True)
            out.append(r)
