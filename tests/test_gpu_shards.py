"""GPU: row-block shards (distributed.CudaShard) on ONE device.  The ranks are
emulated sequentially in one process -- halo exchanges and the scalar
all-reduce become tensor copies between the shards' buffers, no kernel ever
waits on another -- and must reproduce the single-device FISTA run."""
import math

import numpy as np
import pytest

from gpu_util import need_cuda, rel_err

pytestmark = pytest.mark.gpu

KW = dict(n=4096, stages=4, q=1, s_divisor=100, seed=3, theta=2 * math.pi / 10)


def _shards(world, iters, op="auto", stored=False):
    import os

    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard

    cfg = l1bench.SolverConfig(max_iters=iters, op=op)
    os.environ["L1B_ITER_RC"] = "0" if stored else "1"  # read at session begin
    try:
        return [CudaShard(KW, r, world, 0, cfg) for r in range(world)]
    finally:
        del os.environ["L1B_ITER_RC"]


def _exchange(shards, name):
    for g, s in enumerate(shards):
        win, h, own = getattr(s, name), s.halo, s.own
        if g > 0:
            left = shards[g - 1]
            win[0:h].copy_(getattr(left, name)[left.own:left.own + h])
        if g < len(shards) - 1:
            right = shards[g + 1]
            win[own + h:own + 2 * h].copy_(getattr(right, name)[h:2 * h])


def _exchange_many(shards, getter):
    lists = [getter(s) for s in shards]
    for g, s in enumerate(shards):
        for w, (win, h) in enumerate(lists[g]):
            own = s.own
            if g > 0:
                lwin, _ = lists[g - 1][w]
                win[0:h].copy_(lwin[shards[g - 1].own:shards[g - 1].own + h])
            if g < len(shards) - 1:
                rwin, _ = lists[g + 1][w]
                win[own + h:own + 2 * h].copy_(rwin[h:2 * h])


def oracle_check(oracle, kw, iters, x, f, exact):
    """The shards against the reference's fista_run restated (the oracle,
    pinned bit-exact to the reference in tests/test_oracle.py)."""
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=iters)
    if exact:
        np.testing.assert_array_equal(x, ox)
    else:
        assert rel_err(x, ox) < 1e-10
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])
    of = np.asarray(otr["objective"])
    assert len(f) == len(of)
    assert np.max(np.abs(f - of) / np.abs(of)) < 1e-12


def _allreduce(shards):
    bufs = [getattr(s, "scal_now", s.scal) for s in shards]  # scal8 after a two-iteration step
    tot = sum(b.clone() for b in bufs)
    for b in bufs:
        b.copy_(tot)


@pytest.mark.parametrize("world,op", [(2, "sparse"), (3, "sparse"), (2, "matrix_free"), (3, "matrix_free"),
                                     (4, "matrix_free"), (2, "stored"), (3, "stored")])
def test_shards_reproduce_single_device_fista(world, op, oracle):
    torch = need_cuda()
    from paper_1503_03520_b200 import l1bench

    iters = 60
    stored = op == "stored"  # stored-residual single kernel (L1B_ITER_RC=0)
    op = "matrix_free" if stored else op
    inst = l1bench.build_instance(**KW)
    x_ref = np.empty(inst.n)
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=iters, op=op), x_ref)
    b_ref = inst.b
    shards = _shards(world, iters, op, stored)
    assert shards[0].lagged == (op == "matrix_free" and not stored)
    for s in shards:  # the shard's own rows of b are the global b, bit for bit
        a, e = s.inst.info.row_begin, s.inst.info.row_end
        np.testing.assert_array_equal(s.inst.b[: e - a], b_ref[a:e])
    _allreduce(shards)
    for s in shards:
        s.finalize()
    single = shards[0].single
    assert single == (op == "matrix_free")
    if single:
        _exchange_many(shards, lambda s: s.initial_halos())
    else:
        _exchange(shards, "r_y_win")
    for _ in range(iters):
        if single:  # one kernel per iteration, then the halos of x_{k+1} / r_{k+1}
            for s in shards:
                s.k1()
            _exchange_many(shards, lambda s: s.next_halos())
            _allreduce(shards)
            for s in shards:
                s.finalize()
            continue
        for s in shards:
            s.k1()
        _exchange(shards, "x_win")
        for s in shards:
            s.k2()
        _allreduce(shards)
        for s in shards:
            s.finalize()
        _exchange(shards, "r_y_win")
    if shards[0].lagged:  # the last iterate's objective: flush, all-reduce, finalize
        for s in shards:
            s.flush()
        _allreduce(shards)
        for s in shards:
            s.finalize()
    torch.cuda.synchronize()
    outs = [s.finish() for s in shards]
    for t, _ in outs[1:]:
        np.testing.assert_array_equal(t.objectives(), outs[0][0].objectives())
    assert rel_err(outs[0][0].objectives(), tr.objectives()) < 1e-12
    x = np.concatenate([o[1] for o in outs])
    if op == "matrix_free":  # same products entry by entry: sharding changes nothing
        np.testing.assert_array_equal(x, x_ref)
    assert rel_err(x, x_ref) < 1e-12
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(x_ref)[0])
    oracle_check(oracle, KW, iters, x, outs[0][0].objectives(), exact=op == "matrix_free")


def test_shard_rows_match_global_rows():
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    inst = l1bench.build_instance(**KW)
    gp, gi, gv = inst.op.csr()
    for s in _shards(3, 5, "sparse"):
        info = s.inst.info
        a, e, h = int(info.row_begin), int(info.row_end), int(info.halo)
        ptr = np.zeros(info.m + 1, dtype=np.uint64)
        import ctypes as C

        from paper_1503_03520_b200 import _native as N

        idx = np.empty(info.nnz, dtype=np.uint32)
        val = np.empty(info.nnz)
        N.check(N.load().l1b_export_csr(s.inst._h, ptr.ctypes.data_as(C.POINTER(C.c_uint64)),
                                        idx.ctypes.data_as(C.POINTER(C.c_uint32)),
                                        val.ctypes.data_as(C.POINTER(C.c_double))))
        lo, hi = int(gp[a]), int(gp[e])
        np.testing.assert_array_equal(idx.astype(np.int64) + (a - h), gi[lo:hi].astype(np.int64))
        np.testing.assert_array_equal(val, gv[lo:hi])


KW_PERM = dict(n=4096, stages=2, left_stages=1, permute=True, q=1, s_divisor=100, seed=6,
               theta=2 * math.pi / 10)


@pytest.mark.parametrize("world", [2, 3])
def test_general_shards_reproduce_single_device_fista(world, oracle):
    """Permuted operator with a left stage (not banded): row blocks of A,
    columns of x split; the reduce-scatter of g and the all-gather of x are
    emulated by sums / copies between the shards' buffers."""
    torch = need_cuda()
    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard

    iters = 50
    inst = l1bench.build_instance(**KW_PERM)
    x_ref = np.empty(inst.n)
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=iters, op="sparse"), x_ref)
    cfg = l1bench.SolverConfig(max_iters=iters)
    shards = [CudaShard(KW_PERM, r, world, 0, cfg) for r in range(world)]
    assert all(s.general for s in shards)
    b_ref = inst.b
    for s in shards:  # the shard's rows of b are the global b, bit for bit
        a, e = s.inst.info.row_begin, s.inst.info.row_end
        np.testing.assert_array_equal(s.inst.b[: e - a], b_ref[a:e])
    cs = shards[0].n_pad // world
    _allreduce(shards)
    for s in shards:
        s.finalize()
    for _ in range(iters):
        for s in shards:
            s.k1()
        tot = sum(s.g_full.clone() for s in shards)  # reduce-scatter (every slice)
        for s in shards:
            s.g_full.copy_(tot)
        for s in shards:
            s.prox()
        for src in shards:  # all-gather of the own slices
            sl = src.x_full[src.rank * cs:(src.rank + 1) * cs]
            for dst in shards:
                if dst is not src:
                    dst.x_full[src.rank * cs:(src.rank + 1) * cs].copy_(sl)
        for s in shards:
            s.k2()
        _allreduce(shards)
        for s in shards:
            s.finalize()
    torch.cuda.synchronize()
    outs = [s.finish() for s in shards]
    for t, _ in outs[1:]:
        np.testing.assert_array_equal(t.objectives(), outs[0][0].objectives())
    assert rel_err(outs[0][0].objectives(), tr.objectives()) < 1e-12
    x = np.concatenate([o[1] for o in outs])
    assert x.shape == x_ref.shape
    assert rel_err(x, x_ref) < 1e-12
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(x_ref)[0])
    oracle_check(oracle, KW_PERM, iters, x, outs[0][0].objectives(), exact=False)


@pytest.mark.parametrize("world", [2, 3])
def test_peer_halos_reproduce_single_device_fista(world, oracle):
    """The kernels store the halo entries straight into the neighbours' x
    buffers (l1b_session_attach_peers; same device here, NVLink peers on a
    box): no halo exchange at all, the scalar all-reduce orders the steps."""
    torch = need_cuda()
    from paper_1503_03520_b200 import l1bench

    iters = 40
    inst = l1bench.build_instance(**KW)
    x_ref = np.empty(inst.n)
    tr = l1bench.fista_run(inst, l1bench.SolverConfig(max_iters=iters, op="matrix_free"), x_ref)
    shards = _shards(world, iters, "matrix_free")
    for g, s in enumerate(shards):
        s.attach_peers_direct(shards[g - 1] if g > 0 else None, shards[g + 1] if g + 1 < world else None)
        assert s.peer_halos
    _allreduce(shards)
    for s in shards:
        s.finalize()
    for _ in range(iters):
        for s in shards:  # every rank's kernel of this step before any rank's next one
            s.k1()
        _allreduce(shards)
        for s in shards:
            s.finalize()
    for s in shards:
        s.flush()
    _allreduce(shards)
    for s in shards:
        s.finalize()
    torch.cuda.synchronize()
    outs = [s.finish() for s in shards]
    x = np.concatenate([o[1] for o in outs])
    np.testing.assert_array_equal(x, x_ref)
    assert rel_err(outs[0][0].objectives(), tr.objectives()) < 1e-12
    oracle_check(oracle, KW, iters, x, outs[0][0].objectives(), exact=True)


def test_shards_in_contracted_arithmetic_give_the_tile_kernels_bits(oracle):
    """n > 2^20, arith = fma: the single device runs the tile kernel (14
    iterations per launch), the two emulated ranks the two-iteration kernel on
    their row blocks -- both in the scaled form with the same operations per
    entry, so the row split changes no bit; within 1e-12 of the oracle."""
    torch = need_cuda()
    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard

    kw = dict(n=(1 << 20) + 4096, stages=4, q=1, s_divisor=1000, seed=3, theta=2 * math.pi / 10)
    iters = 30
    cfg = l1bench.SolverConfig(max_iters=iters, op="matrix_free", arith="fma")
    inst = l1bench.build_instance(**kw)
    x_ref = np.empty(inst.n)
    tr = l1bench.fista_run(inst, cfg, x_ref)
    assert tr.ran("fista_tile") and tr.ran("fma"), tr.path
    shards = [CudaShard(kw, r, 2, 0, cfg) for r in range(2)]
    assert shards[0].single and shards[0].lagged and shards[0].pairs
    _allreduce(shards)
    for s in shards:
        s.finalize()
    _exchange_many(shards, lambda s: s.initial_halos())
    for _ in range(iters // 2):  # two iterations per k1
        for s in shards:
            s.k1()
        _exchange_many(shards, lambda s: s.next_halos())
        _allreduce(shards)
        for s in shards:
            s.finalize()
    for s in shards:
        s.flush()
    _allreduce(shards)
    for s in shards:
        s.finalize()
    torch.cuda.synchronize()
    outs = [s.finish() for s in shards]
    assert outs[0][0].iterations == iters
    x = np.concatenate([o[1] for o in outs])
    np.testing.assert_array_equal(x, x_ref)
    assert rel_err(outs[0][0].objectives(), tr.objectives()) < 1e-12
    otr, ox = oracle.fista(oracle.build_instance(**kw), max_iters=iters)
    assert rel_err(x, ox) < 1e-12
    np.testing.assert_array_equal(np.nonzero(x)[0], np.nonzero(ox)[0])
