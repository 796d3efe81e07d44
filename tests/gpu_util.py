"""Helpers shared by the GPU parity tests."""
import numpy as np
import pytest


def need_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    return torch


def rel_err(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(float(np.max(np.abs(want))) if want.size else 0.0, 1e-300)
    return float(np.max(np.abs(got - want))) / scale if want.size else 0.0


def device_build(name):
    from conftest import golden_kwargs
    from paper_1503_03520_b200 import l1bench

    kw = golden_kwargs(name)
    return l1bench.build_instance(**kw)
