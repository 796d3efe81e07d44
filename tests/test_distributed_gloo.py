"""CPU, world_size 2 and 3 over gloo: the row-sharded FISTA driver
(paper_1503_03520_b200/distributed.py) with the numpy stand-in backend equals
the single-process oracle FISTA (the reference's fista_run restated)."""
import math
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ITERS = 40
KW = dict(n=96, stages=4, q=1, s_divisor=16, seed=3, theta=2 * math.pi / 10)
# a permuted operator with left stages: not banded -> reduce-scatter / all-gather path
KW_PERM = dict(n=80, stages=2, left_stages=1, permute=True, q=1, s_divisor=16, seed=5,
               theta=2 * math.pi / 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, single):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.join(HERE, "..", "oracle"))
    sys.path.insert(0, os.path.join(HERE, ".."))
    import torch.distributed as dist

    from dist_cpu_backend import CpuShard, CpuShardGeneral, CpuShardRc, CpuShardRc2, CpuShardSingle
    from paper_1503_03520_b200.distributed import fista_distributed
    from pyoracle import Oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    oracle = Oracle()
    inst = oracle.build_instance(**(KW_PERM if single == "general" else KW))
    cls = {"two": CpuShard, "single": CpuShardSingle, "rc": CpuShardRc, "rc2": CpuShardRc2,
           "general": CpuShardGeneral}[single]
    be = cls(oracle, inst, rank, world, ITERS)
    samples, x_own = fista_distributed(be, ITERS + 5)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), f=np.array([s[1] for s in samples]),
             it=np.array([s[0] for s in samples]), x=x_own)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,single", [(2, "two"), (3, "two"), (2, "single"), (3, "single"),
                                          (2, "rc"), (3, "rc"), (2, "rc2"), (3, "rc2"), (4, "rc2"),
                                          (2, "general"), (3, "general")])
def test_sharded_fista_matches_single_process(tmp_path, oracle, world, single):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), single), nprocs=world, join=True)
    inst = oracle.build_instance(**(KW_PERM if single == "general" else KW))
    tr, x_ref = oracle.fista(inst, max_iters=ITERS)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for p in parts[1:]:  # every rank saw the same all-reduced objective trace
        np.testing.assert_array_equal(p["f"], parts[0]["f"])
    f = parts[0]["f"]
    np.testing.assert_array_equal(parts[0]["it"], np.arange(ITERS + 1))
    np.testing.assert_allclose(f, tr["objective"], rtol=1e-12)
    x = np.concatenate([p["x"] for p in parts])
    assert np.max(np.abs(x - x_ref)) <= 1e-12 * np.max(np.abs(x_ref))
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(x_ref)[0])


def test_partition_balanced():
    from paper_1503_03520_b200.distributed import partition

    parts = partition(1 << 27, 8)
    assert parts[0][0] == 0 and parts[-1][1] == 1 << 27
    assert all(b - a == 1 << 24 for a, b in parts)
    assert all(parts[i][1] == parts[i + 1][0] for i in range(7))
