import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden")
THETA = 2 * math.pi / 10
CASES = ["c1", "k4", "perm", "odd", "ncg", "cd"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from pyoracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libl1ref.so not built (reference sources absent)")
    return Reference()


def golden_kwargs(name):
    """build_instance arguments of each golden case (tests/golden/make_golden.py)."""
    sys.path.insert(0, GOLDEN)
    import make_golden

    kw = dict(make_golden.CASES[name])
    if kw.pop("sigma", None) == "log1":
        from pyoracle import log_spaced_sigma

        kw["sigma"] = log_spaced_sigma(kw["n"], 1.0)
    kw["theta"] = THETA
    return kw


def spec_from_golden(g):
    """OpSpec (oracle) from a golden record."""
    from pyoracle import OpSpec

    op = OpSpec(int(g["m"]), int(g["n"]), g["right_offset"], g["right_theta"], g["left_offset"],
                g["left_theta"], g["sigma"])
    if "p1" in g:
        op.p1 = g["p1"].astype(np.uint32)
        op.p2 = g["p2"].astype(np.uint32)
        op.p1_inv = np.argsort(op.p1).astype(np.uint32)
        op.p2_inv = np.argsort(op.p2).astype(np.uint32)
    return op
