"""The native shard driver (l1b_session_attach_nccl / nccl_start / nccl_steps /
nccl_finish): the per-launch loop k1 -> halos -> NCCL all-reduce -> finalize
issued by the library with its own communicator, the steady state replayed
from a CUDA graph.  One GPU per box here, and NCCL refuses two ranks on one
device, so the communicator has one rank (the all-reduce and the graph capture
are real, the halo send / recv has no neighbour; that host logic is the one
tests/test_distributed_gloo.py runs at world 2-4).  The iterates must equal
the reference's fista_run (the oracle, tests/test_oracle.py pins it) bit for
bit in the exact arithmetic, whether the launches come from the graph, from
direct launches or from the timed (event-bracketed) path, and a restarted
session (a new b streamed from the host) must reproduce them."""
import math
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
KW = dict(n=(1 << 16) + 48, stages=4, q=1, s_divisor=100, seed=3, theta=2 * math.pi / 10)
LAUNCHES = 15  # 30 FISTA iterations


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out, arith):
    sys.path.insert(0, os.path.join(HERE, ".."))
    import torch
    import torch.distributed as dist

    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    stream = torch.cuda.Stream(0)
    torch.cuda.set_stream(stream)
    cfg = l1bench.SolverConfig(max_iters=2 * LAUNCHES, op="matrix_free", arith=arith)
    be = CudaShard(KW, 0, 1, 0, cfg)
    assert be.native_ok, "expected the lagged two-iteration shard protocol"
    be.attach_nccl()
    res = {}
    for run in ("mixed", "graph"):
        if run == "graph":  # serving: the same b again from pinned host memory, x_0 = 0
            b = be.inst.b[:be.own].copy()
            lo, bw = be.inst.b_window()
            be.inst.set_rhs(b, bw)
            be.restart()
        k0 = l1bench.launch_count()
        be.native_start()
        if run == "mixed":
            be.native_steps(1, graph=False)  # launch 0 direct (j % 4 == 0)
            be.native_steps(6, graph=True)  # three replays of the graph starting at j % 4 == 2
            ms = be.native_steps(3, graph=False, timed=True)
            assert ms > 0.0
            be.native_steps(5, graph=True)  # two replays (j % 4 == 0) + one direct launch
        else:
            be.native_steps(LAUNCHES, graph=True)
        be.native_finish()
        x = np.empty(be.own)
        tr = be.read(x)
        res[run] = (x, tr.objectives(), [s.iter for s in tr.samples], l1bench.launch_count() - k0)
    np.savez(os.path.join(out, f"{arith}.npz"), x_mixed=res["mixed"][0], f_mixed=res["mixed"][1],
             it_mixed=res["mixed"][2], x_graph=res["graph"][0], f_graph=res["graph"][1],
             it_graph=res["graph"][2], launches=[res["mixed"][3], res["graph"][3]])
    be.sess.end()
    dist.destroy_process_group()


@pytest.mark.parametrize("arith", ["exact", "fma"])
def test_native_driver_matches_reference(tmp_path, oracle, arith):
    from gpu_util import need_cuda, rel_err

    need_cuda()
    mp.spawn(_worker, args=(_port(), str(tmp_path), arith), nprocs=1, join=True)
    z = np.load(tmp_path / f"{arith}.npz")
    otr, ox = oracle.fista(oracle.build_instance(**KW), max_iters=2 * LAUNCHES)
    of = np.asarray(otr["objective"])
    for run in ("mixed", "graph"):
        x, f = z[f"x_{run}"], z[f"f_{run}"]
        if arith == "exact":
            np.testing.assert_array_equal(x, ox)
        else:
            assert rel_err(x, ox) < 1e-12
            np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])
        assert list(z[f"it_{run}"]) == list(otr["iter"])
        assert np.max(np.abs(f - of) / np.abs(of)) < 1e-12
    # graph replays and direct launches: the same bits
    np.testing.assert_array_equal(z["x_mixed"], z["x_graph"])
    np.testing.assert_array_equal(z["f_mixed"], z["f_graph"])
    # the library's kernels of graph replays are counted (2 per launch + start + flush + finish)
    assert z["launches"][0] == z["launches"][1] and z["launches"][0] >= 2 * LAUNCHES
