"""GPU: std::mt19937_64 streams drawn on the device (k_rng.cu) -- chunks
started by jump-ahead, a 16-ary jump tree -- bit-identical to the oracle's
sequential streams (Spectrum::uniform, linops.cpp:323-331; the l1_subgradient
fill, instance.cpp:33-35), and the generator built on them identical to the
sequential host replay (L1B_DEVICE_RNG=0) and to the oracle."""
import ctypes
import math
import os

import numpy as np
import pytest

from gpu_util import need_cuda

pytestmark = pytest.mark.gpu


def _draws(seed, count, lo, hi, spectrum, shift, wlo, whi, min_log2_chunk):
    torch = need_cuda()
    from paper_1503_03520_b200 import _native as N

    out = torch.empty(max(whi - wlo, 1), dtype=torch.float64, device="cuda")
    vmin, vmax, exact = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    N.check(N.load().l1b_device_uniform_draws(0, seed, count, lo, hi, spectrum, shift, wlo, whi,
                                              min_log2_chunk, ctypes.c_void_p(out.data_ptr()),
                                              ctypes.byref(vmin), ctypes.byref(vmax), ctypes.byref(exact)))
    torch.cuda.synchronize()
    return out[: whi - wlo].cpu().numpy(), vmin.value, vmax.value, exact.value


def _oracle_spectrum(oracle, n, hi, shift, seed):
    out = np.empty(n)
    oracle.lib.lo_spectrum_uniform(n, 0.0, hi, shift, seed, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


@pytest.mark.parametrize("count,wlo,whi,chunk", [
    (3_000_001, 1_000_003, 2_500_017, 10),   # 2930 chunks: three jump levels
    (200_000, 0, 200_000, 12),               # 49 chunks: two levels
    (1000, 0, 1000, 12),                     # one chunk, no jump
    (70_000, 69_990, 70_000, 8),             # window at the very end
])
def test_spectrum_stream_bit_exact(oracle, count, wlo, whi, chunk):
    seed = oracle.mix_seed(oracle.mix_seed(3, 0), 3)
    got, vmin, vmax, exact = _draws(seed, count, 0.0, 10.0, 1, 0.1, wlo, whi, chunk)
    want = _oracle_spectrum(oracle, count, 10.0, 0.1, seed)
    assert exact == 1
    np.testing.assert_array_equal(got, want[wlo:whi])
    assert vmin == want.min() and vmax == want.max()


def test_fill_stream_bit_exact(oracle):
    n = 300_007
    seed = oracle.mix_seed(oracle.mix_seed(9, 0), 5)
    got, _, _, _ = _draws(seed, n, -0.9, 0.9, 0, 0.0, 0, n, 6)  # 4096 chunks of 2^7
    want = np.empty(n)
    r = oracle.rng(seed)
    oracle.lib.lo_l1_subgradient(ctypes.c_uint64(n), None, None, ctypes.c_uint64(0), ctypes.c_double(0.9),
                                 ctypes.byref(r), want.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    np.testing.assert_array_equal(got, want)


def test_c4_sized_spectrum_stream_matches_host_replay():
    """n = 2^26 draws (default chunking: 4096 chunks of 2^14) against the
    library's own sequential host stream."""
    from paper_1503_03520_b200 import _native as N

    n = 1 << 26
    seed = N.load().l1b_mix_seed(N.load().l1b_mix_seed(3, 0), 3)
    got, vmin, vmax, exact = _draws(seed, n, 0.0, 10.0, 1, 0.1, 0, n, 12)
    want = np.empty(n)
    N.check(N.load().l1b_realize_spectrum_uniform(n, 0.0, 10.0, 0.1, seed,
                                                  want.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    assert exact == 1
    np.testing.assert_array_equal(got, want)
    assert vmin == want.min() and vmax == want.max()


def _with_env(val, fn):
    old = os.environ.get("L1B_DEVICE_RNG")
    os.environ["L1B_DEVICE_RNG"] = val
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["L1B_DEVICE_RNG"]
        else:
            os.environ["L1B_DEVICE_RNG"] = old


@pytest.mark.parametrize("kw", [
    dict(n=4096, stages=4, q=1, s_divisor=100, seed=3),
    dict(n=5000, stages=2, left_stages=1, permute=True, q=2, s_divisor=50, seed=6),
    dict(n=4096, stages=1, q=1, s_divisor=100, seed=2, solution="spectral", s1_fraction=0.5),
    dict(n=3001, stages=3, alternating=(2.0, 0.5), s_divisor=30, seed=8),
    dict(n=2048, stages=2, q=1, s_divisor=64, seed=9, solution="two_value"),
])
def test_generator_device_rng_equals_host_and_oracle(oracle, kw):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(kw, theta=2 * math.pi / 10)
    dev = _with_env("1", lambda: l1bench.build_instance(**kw))
    host = _with_env("0", lambda: l1bench.build_instance(**kw))
    np.testing.assert_array_equal(dev.sigma(), host.sigma())
    np.testing.assert_array_equal(dev.b, host.b)
    np.testing.assert_array_equal(dev.x_star.support, host.x_star.support)
    np.testing.assert_array_equal(dev.x_star.values, host.x_star.values)
    assert dev.noise_norm == host.noise_norm
    if kw.get("solution", "uniform") == "uniform" and "alternating" not in kw:
        okw = {k: v for k, v in kw.items() if k not in ("solution", "s1_fraction")}
        oi = oracle.build_instance(**okw)
        np.testing.assert_array_equal(dev.b, oi.b)


def test_shard_device_rng_ragged_and_single_rank():
    """A shard layout whose windows reach both stream ends (world 1) and an
    uneven 5-way split of an n that is no multiple of the chunking."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard

    kw = dict(n=70001, stages=4, q=2, s_divisor=70, seed=12, theta=2 * math.pi / 10)
    whole = _with_env("0", lambda: l1bench.build_instance(**kw))
    cfg = l1bench.SolverConfig(max_iters=2)
    for world in (1, 5):
        shards = _with_env("1", lambda: [CudaShard(kw, r, world, 0, cfg) for r in range(world)])
        for s in shards:
            a, e = s.inst.info.row_begin, s.inst.info.row_end
            np.testing.assert_array_equal(s.inst.b[: e - a], whole.b[a:e])
            assert s.inst.info.gram_lmax == whole.info.gram_lmax


def test_shards_device_rng_reproduce_global_instance():
    """Row-block shards draw only their windows of the fill stream and reduce
    sigma over the whole stream without storing it: same b rows as the whole
    instance, same L."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench
    from paper_1503_03520_b200.distributed import CudaShard

    kw = dict(n=40000, stages=4, q=1, s_divisor=100, seed=3, theta=2 * math.pi / 10)
    whole = _with_env("0", lambda: l1bench.build_instance(**kw))
    cfg = l1bench.SolverConfig(max_iters=4)
    shards = _with_env("1", lambda: [CudaShard(kw, r, 3, 0, cfg) for r in range(3)])
    for s in shards:
        a, e = s.inst.info.row_begin, s.inst.info.row_end
        np.testing.assert_array_equal(s.inst.b[: e - a], whole.b[a:e])
        assert s.inst.info.gram_lmax == whole.info.gram_lmax
        assert s.inst.info.cert_kappa == whole.info.cert_kappa


@pytest.mark.parametrize("n,pieces", [(32768, [100_000]), (1_000_003, [1, 311, 313, 40_000, 3]),
                                      (4096, [312] * 7), ((1 << 31), [5000]),
                                      # several jump-started chunks of 312 x 256 draws per piece
                                      (32768, [3_300_000]), (1_000_003, [200_000, 500_001, 79_872, 90_000])])
def test_coordinate_index_stream_bit_exact(oracle, n, pieces):
    """The pair-local CD / PCDM coordinate stream (mt_stream_indices, continued
    over several launches) against std::mt19937_64 reduced like uniform_index:
    raw % n, the redraw marker where raw >= UINT64_MAX - UINT64_MAX % n."""
    torch = need_cuda()
    from paper_1503_03520_b200 import _native as N

    seed = oracle.mix_seed(1, 7)
    cap = sum(-(-max(p, 1) // 312) * 312 for p in pieces)
    out = torch.empty(cap, dtype=torch.int32, device="cuda")
    arr = (ctypes.c_uint64 * len(pieces))(*pieces)
    drawn = ctypes.c_uint64()
    N.check(N.load().l1b_device_index_stream(0, seed, n, arr, len(pieces), ctypes.c_void_p(out.data_ptr()),
                                             ctypes.byref(drawn)))
    torch.cuda.synchronize()
    assert drawn.value == sum(-(-p // 312) * 312 for p in pieces)
    got = out[: drawn.value].cpu().numpy().view(np.uint32)
    r = oracle.rng(seed)
    raw = np.array([oracle.lib.lo_rng_next(ctypes.byref(r)) for _ in range(drawn.value)], dtype=np.uint64)
    lim = np.uint64((1 << 64) - 1 - ((1 << 64) - 1) % n)
    want = np.where(raw >= lim, np.uint64(0xFFFFFFFF), raw % np.uint64(n)).astype(np.uint32)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("kw", [dict(n=3001, stages=3, alternating=(2.0, 0.5), s_divisor=30, seed=8),
                                dict(n=4096, stages=1, alternating=(0.1, 100.0), s_divisor=64, seed=5),
                                dict(n=70001, stages=4, alternating=(3.0, 0.25), s_divisor=100, seed=2)])
def test_alternating_spectrum_matches_reference(reference, kw):
    """SpectrumRule::Kind::alternating (Spectrum::alternating, linops.cpp:332-335)
    built on the device against the reference's own build_instance (the
    unmodified reference library): sigma, b and x* bit for bit."""
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    kw = dict(kw, theta=2 * math.pi / 10)
    dev = l1bench.build_instance(**kw)
    ref = reference.build_instance(**kw)
    np.testing.assert_array_equal(dev.sigma(), ref.sigma())
    np.testing.assert_array_equal(dev.b, ref.b())
    np.testing.assert_array_equal(dev.x_star.support, ref.x_star()[0])
    np.testing.assert_array_equal(dev.x_star.values, ref.x_star()[1])


@pytest.mark.parametrize("n,s,seed", [(1000, 1000, 1), (1000, 1, 2), (4096, 40, 3), (1 << 15, 327, 4),
                                      (5000, 4000, 9), ((1 << 20) + 7, 10_000, 5), (1 << 27, 134_217, None),
                                      (1 << 32, 429_496, None)])
def test_device_floyd_sampling_matches_reference(oracle, n, s, seed):
    """uniform_sparse_solution (solution.cpp:47-75) on the device against the
    oracle's sequential Floyd sampling on the same stream: support and values
    bit for bit (C4's and C5's own seeds and sizes included; s = n chooses all)."""
    need_cuda()
    from paper_1503_03520_b200 import _native as N

    if seed is None:  # the generator's seed for x* of C4 / C5: mix_seed(job seed, 4)
        seed = oracle.mix_seed(oracle.mix_seed(3 if n == 1 << 27 else 4, 0), 4)
    sup = np.empty(s, dtype=np.uint32)
    val = np.empty(s)
    on_dev = ctypes.c_int()
    N.check(N.load().l1b_device_uniform_sparse_solution(
        0, n, s, 10.0, seed, sup.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
        val.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(on_dev)))
    assert on_dev.value == 1
    rng = oracle.rng(seed)
    osup = np.empty(s, dtype=np.uint32)
    oval = np.empty(s)
    oracle.lib.lo_uniform_sparse_solution(n, s, 10.0, ctypes.byref(rng), osup.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                          oval.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    np.testing.assert_array_equal(sup, osup)
    np.testing.assert_array_equal(val, oval)


@pytest.mark.parametrize("n,seed", [(2, 1), (3, 2), (17, 3), (1000, 4), (1 << 16, 5), (1_000_003, 6),
                                    (1 << 24, 7)])
def test_device_permutation_matches_reference(oracle, n, seed):
    """Permutation::realize (linops.cpp:224-239, Fisher-Yates with
    uniform_index) on the device against the oracle's sequential shuffle on the
    same stream, bit for bit."""
    need_cuda()
    from paper_1503_03520_b200 import _native as N

    got = np.empty(n, dtype=np.uint32)
    on_dev = ctypes.c_int()
    N.check(N.load().l1b_device_realize_permutation(0, n, seed, got.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                                     ctypes.byref(on_dev)))
    assert on_dev.value == 1
    want = np.empty(n, dtype=np.uint32)
    inv = np.empty(n, dtype=np.uint32)
    oracle.lib.lo_permutation_realize(n, seed, want.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                      inv.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    np.testing.assert_array_equal(got, want)
