"""C4 session: warm-up, then tile launches (for ncu -k fista_tb_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_03520_b200 import l1bench  # noqa: E402

arith = sys.argv[1] if len(sys.argv) > 1 else "fma"
inst = l1bench.build_instance(n=1 << 27, stages=4, q=1, s_divisor=1000, seed=3)
s = l1bench.Session(inst, l1bench.SolverConfig(max_iters=100, op="matrix_free", arith=arith))
s.step(60)
s.end()
