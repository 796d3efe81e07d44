"""Timing of the device mt19937_64 streams (k_rng.cu) and of the generator
with / without them (L1B_DEVICE_RNG)."""
import ctypes
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1503_03520_b200 import _native as N, l1bench  # noqa: E402

lib = N.load()
res = {}


def draws(count, wlo, whi, reduce=True):
    out = torch.empty(max(whi - wlo, 1), dtype=torch.float64, device="cuda")
    vmin, vmax, ex = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    torch.cuda.synchronize()
    t = time.perf_counter()
    N.check(lib.l1b_device_uniform_draws(0, 12345, count, 0.0, 10.0, 1, 0.1, wlo, whi, 12,
                                         ctypes.c_void_p(out.data_ptr()),
                                         ctypes.byref(vmin) if reduce else None,
                                         ctypes.byref(vmax) if reduce else None, ctypes.byref(ex)))
    return time.perf_counter() - t


draws(1 << 20, 0, 1 << 20)  # warm-up (charpoly, polys, module load)
res["draws_2^27_store_s"] = draws(1 << 27, 0, 1 << 27)
res["draws_2^27_store_s_again"] = draws(1 << 27, 0, 1 << 27)
res["draws_2^32_reduce_only_s"] = draws(1 << 32, 0, 0)
res["draws_2^32_window_2^29_s"] = draws(1 << 32, 7 << 29, 8 << 29, reduce=False)
kw = dict(n=1 << 27, stages=4, q=1, s_divisor=1000, seed=3, theta=2 * math.pi / 10, lazy_sparse=True)
for v in ("0", "1"):
    os.environ["L1B_DEVICE_RNG"] = v
    torch.cuda.synchronize()
    t = time.perf_counter()
    inst = l1bench.build_instance(**kw)
    torch.cuda.synchronize()
    res[f"generate_c4_device_rng={v}_s"] = time.perf_counter() - t
    if v == "0":
        b0 = inst.b[: 1 << 20].copy()
    else:
        import numpy as np
        res["c4_b_prefix_equal"] = bool(np.array_equal(b0, inst.b[: 1 << 20]))
    del inst
print(json.dumps(res))
