"""CPU: the mt19937_64 jump-ahead behind the device generator (k_rng.cu).

The host restatement of the jump (characteristic polynomial by
Berlekamp-Massey, t^(2^e) mod P by squaring, the window correlation) must land
exactly where stepping the oracle's sequential std::mt19937_64 (rng.hpp:14-56
restated in oracle/l1oracle.c) lands."""
import ctypes

import numpy as np
import pytest


@pytest.mark.parametrize("seed,e", [(5489, 0), (7, 1), (12345, 5), (99, 10), (3, 14),
                                    (2**63 + 5, 15), (0, 18)])
def test_jump_lands_on_sequential_stream(oracle, seed, e):
    from paper_1503_03520_b200 import _native as N

    lib = N.load()
    count = 700  # > 2 x 312: the jumped window regenerates the following words too
    got = np.empty(count, dtype=np.uint64)
    N.check(lib.l1b_mt_draws_after_jump(seed, e, count, got.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    r = oracle.rng(seed)
    nxt = oracle.lib.lo_rng_next
    for _ in range(1 << e):
        nxt(ctypes.byref(r))
    want = np.array([nxt(ctypes.byref(r)) for _ in range(count)], dtype=np.uint64)
    np.testing.assert_array_equal(got, want)


def test_mix_seeded_generator_streams(oracle):
    """The job seeds the generator uses (mix_seed(job, 3) sigma, 5 fill)."""
    from paper_1503_03520_b200 import _native as N

    lib = N.load()
    for salt in (3, 5):
        seed = oracle.mix_seed(oracle.mix_seed(3, 0), salt)
        got = np.empty(400, dtype=np.uint64)
        N.check(lib.l1b_mt_draws_after_jump(seed, 12, 400, got.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
        r = oracle.rng(seed)
        for _ in range(1 << 12):
            oracle.lib.lo_rng_next(ctypes.byref(r))
        want = np.array([oracle.lib.lo_rng_next(ctypes.byref(r)) for _ in range(400)], dtype=np.uint64)
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("seed,chunk", [(1, 1), (7, 2), (2**64 - 3, 5)])
def test_chunk_jump_lands_on_sequential_stream(oracle, seed, chunk):
    """The coordinate-stream chunks (mt_stream_indices): chunk c starts at
    t^(c J) mod P, J = 312 x 256, by one carry-less multiplication mod P per
    chunk -- the same stream position as stepping c J draws."""
    from paper_1503_03520_b200 import _native as N

    lib = N.load()
    J = 312 * 256
    count = 700
    got = np.empty(count, dtype=np.uint64)
    N.check(lib.l1b_mt_draws_after_chunk_jump(seed, chunk, count,
                                              got.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    r = oracle.rng(seed)
    nxt = oracle.lib.lo_rng_next
    for _ in range(chunk * J):
        nxt(ctypes.byref(r))
    want = np.array([nxt(ctypes.byref(r)) for _ in range(count)], dtype=np.uint64)
    np.testing.assert_array_equal(got, want)
