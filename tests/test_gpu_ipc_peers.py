"""Peer halos between PROCESSES (the one-process-per-GPU layout): two ranks on
the same device exchange cudaIpc handles of their x buffers
(CudaShard.attach_peers_ipc), the kernels store the halo entries into the
other process's buffers, and the scalar all-reduce (gloo here, NCCL on a box)
orders the steps.  Nothing waits on another rank inside a kernel.  Must equal
the single-device run bit for bit."""
import math
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
KW = dict(n=4096, stages=4, q=1, s_divisor=100, seed=3, theta=2 * math.pi / 10)
ITERS = 30


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, os.path.join(HERE, ".."))
    import torch
    import torch.distributed as dist

    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard, fista_distributed

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    be = CudaShard(KW, rank, world, 0, l1bench.SolverConfig(max_iters=ITERS))
    be.attach_peers_ipc()
    assert be.peer_halos
    tr, x = fista_distributed(be, ITERS + 2)
    np.savez(os.path.join(out, f"r{rank}.npz"), x=x, f=tr.objectives())
    dist.barrier()
    dist.destroy_process_group()


def test_ipc_peer_halos_two_processes(tmp_path, oracle):
    import torch

    from gpu_util import need_cuda

    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(**KW)
    x_ref = np.empty(inst.n)
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=ITERS, op="matrix_free"), x_ref)
    mp.spawn(_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    x = np.concatenate([p["x"] for p in parts])
    np.testing.assert_array_equal(x, x_ref)
    f = parts[0]["f"]
    assert np.max(np.abs(f - tr.objectives()) / np.abs(tr.objectives())) < 1e-12
    # and the reference's fista_run restated (the oracle), bit for bit
    otr, ox = oracle.fista(oracle.build_instance(**KW), max_iters=ITERS)
    np.testing.assert_array_equal(x, ox)
    of = np.asarray(otr["objective"])
    assert np.max(np.abs(f - of) / np.abs(of)) < 1e-12
