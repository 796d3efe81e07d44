"""B200-native hot path of the arXiv 1503.03520 l1-least-squares benchmark.

``paper_1503_03520_b200.l1bench`` mirrors the reference's generator/solver API;
the work runs in ``lib/libl1b.so`` (hand-written sm_100a CUDA behind the C ABI
in ``include/l1b.h``).  There is no CPU fallback.
"""
from . import _native  # noqa: F401

__all__ = ["l1bench"]
