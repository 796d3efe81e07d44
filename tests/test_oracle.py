"""CPU: pins the oracle restatement (oracle/l1oracle.c) against the golden
vectors the reference wrote (tests/golden), the reference itself when it is
built (oracle/_ref), SPEC.md's known answers and an independent dense
assembly of A from its definitions (proj/tests/oracles.hpp:15-79)."""
import math

import numpy as np
import pytest

from conftest import CASES, golden_kwargs, load_golden, spec_from_golden


def test_mt19937_64_known_answer(oracle):
    # C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64
    r = oracle.rng(5489)
    for _ in range(9999):
        oracle.lib.lo_rng_next(r)
    assert int(oracle.lib.lo_rng_next(r)) == 9981545732273789042


@pytest.mark.parametrize("name", CASES)
def test_generator_bit_exact(oracle, name):
    g = load_golden(name)
    inst = oracle.build_instance(**golden_kwargs(name))
    assert inst.m == g["m"] and inst.n == g["n"]
    np.testing.assert_array_equal(inst.op.sigma, g["sigma"])
    np.testing.assert_array_equal(inst.support, g["support"])
    np.testing.assert_array_equal(inst.values, g["values"])
    np.testing.assert_array_equal(inst.b, g["b"])
    assert inst.noise_norm == g["noise_norm"]
    assert inst.f_star() == pytest.approx(float(g["f_star"]), rel=1e-15)
    if "p1" in g:
        np.testing.assert_array_equal(inst.op.p1, g["p1"])
        np.testing.assert_array_equal(inst.op.p2, g["p2"])


@pytest.mark.parametrize("name", CASES)
def test_rows_columns_bit_exact(oracle, name):
    g = load_golden(name)
    op = spec_from_golden(g)
    for got, key in ((oracle.csr(op), "csr"), (oracle.csc(op), "csc")):
        np.testing.assert_array_equal(got[0], g[f"{key}_ptr"])
        np.testing.assert_array_equal(got[1], g[f"{key}_idx"])
        np.testing.assert_array_equal(got[2], g[f"{key}_val"])
    np.testing.assert_array_equal(oracle.gram_diagonal(op), g["gram_diag"])


@pytest.mark.parametrize("name", CASES)
def test_operator_probes_bit_exact(oracle, name):
    g = load_golden(name)
    op = spec_from_golden(g)
    np.testing.assert_array_equal(oracle.apply(op, g["probe_x"]), g["probe_ax"])
    np.testing.assert_array_equal(oracle.apply_transpose(op, g["probe_y"]), g["probe_aty"])
    np.testing.assert_array_equal(oracle.gram_inverse(op, g["probe_x"]), g["probe_ginv"])


@pytest.mark.parametrize("name", CASES)
def test_solvers_bit_exact(oracle, name):
    g = load_golden(name)
    inst = oracle.build_instance(**golden_kwargs(name))
    tr, x = oracle.fista(inst, max_iters=3000, target=float(g["fista_target"]))
    np.testing.assert_array_equal(tr["iter"], g["fista_iter"])
    np.testing.assert_array_equal(tr["objective"], g["fista_obj"])
    np.testing.assert_array_equal(tr["nnz"], g["fista_nnz"])
    np.testing.assert_array_equal(tr["matvecs"], g["fista_matvecs"])
    assert tr["status"] == int(g["fista_status"])
    np.testing.assert_array_equal(x, g["fista_x"])
    tr, x = oracle.fista(inst, max_iters=50, accelerated=False)
    np.testing.assert_array_equal(tr["objective"], g["ista_obj"])
    np.testing.assert_array_equal(x, g["ista_x"])
    if "ncg_obj" in g:
        tr, x = oracle.newton_cg(inst, max_iters=8)
        np.testing.assert_array_equal(tr["objective"], g["ncg_obj"])
        np.testing.assert_array_equal(tr["extra"], g["ncg_extra"])
        np.testing.assert_array_equal(x, g["ncg_x"])
    if "cd_obj" in g:
        tr, x = oracle.cd(inst, max_iters=20, varpi=4, seed=5)
        np.testing.assert_array_equal(tr["objective"], g["cd_obj"])
        np.testing.assert_array_equal(tr["extra"], g["cd_extra"])
        np.testing.assert_array_equal(tr["matvecs"], g["cd_matvecs"])
        np.testing.assert_array_equal(x, g["cd_x"])


def test_certificate(oracle):
    for name in CASES:
        g = load_golden(name)
        inst = oracle.build_instance(**golden_kwargs(name))
        c = oracle.verify(inst, 1e-8)
        assert c["passed"]
        assert c["max_support_violation"] == g["cert"][0]
        assert c["max_offsupport_violation"] == g["cert"][1]


# ---- an independent dense oracle (proj/tests/oracles.hpp:15-79 restated) ----

def dense_stage(n, offset, theta):
    g = np.eye(n)
    c, s = math.cos(theta), math.sin(theta)
    for k in range(offset, n - 1, 2):
        g[k, k], g[k, k + 1], g[k + 1, k], g[k + 1, k + 1] = c, -s, s, c
    return g


def dense_perm(mp):
    m = len(mp)
    P = np.zeros((m, m))
    P[np.arange(m), mp] = 1.0
    return P


def dense_operator(op):
    right = np.eye(op.n)
    for o, t in zip(op.right_offset, op.right_theta):
        right = right @ dense_stage(op.n, int(o), float(t))
    left = np.eye(op.m)
    for o, t in zip(op.left_offset, op.left_theta):
        left = left @ dense_stage(op.m, int(o), float(t))
    sig = np.zeros((op.m, op.n))
    sig[np.arange(op.n), np.arange(op.n)] = op.sigma
    P1 = dense_perm(op.p1) if op.p1 is not None else np.eye(op.m)
    P2 = dense_perm(op.p2) if op.p2 is not None else np.eye(op.m)
    return P1 @ left @ P2 @ sig @ right.T


@pytest.mark.parametrize("name", ["perm", "odd"])
def test_dense_definition(oracle, name):
    g = load_golden(name)
    op = spec_from_golden(g)
    A = dense_operator(op)
    x, y = g["probe_x"], g["probe_y"]
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    assert rel(oracle.apply(op, x), A @ x) < 1e-12
    assert rel(oracle.apply_transpose(op, y), A.T @ y) < 1e-12
    ptr, idx, val = oracle.csr(op)
    D = np.zeros_like(A)
    for i in range(op.m):
        D[i, idx[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
    assert np.max(np.abs(D - A)) < 1e-12
    assert np.all(np.abs(A[D == 0]) < 1e-14)
    np.testing.assert_allclose(oracle.gram_diagonal(op), np.diag(A.T @ A), rtol=1e-12)


# ---- SPEC.md known answers ---------------------------------------------------

def _spec(oracle_mod, m, n, sigma, right=(), theta=0.0):
    from pyoracle import OpSpec

    return OpSpec(m, n, np.array([o for o in right], dtype=np.int32), np.full(len(right), theta),
                  np.zeros(0, dtype=np.int32), np.zeros(0), np.array(sigma, dtype=np.float64))


def test_spec_known_answers(oracle):
    import pyoracle

    op = _spec(pyoracle, 4, 2, [1.0, 2.0], right=[0], theta=0.0)
    np.testing.assert_array_equal(oracle.apply(op, [1.0, 1.0]), [1, 2, 0, 0])
    np.testing.assert_array_equal(oracle.apply_transpose(op, [1, 1, 1, 1.0]), [1, 2])
    op = _spec(pyoracle, 2, 2, [1.0, 2.0], right=[0], theta=math.pi / 4)
    np.testing.assert_allclose(oracle.gram_diagonal(op), [2.5, 2.5], rtol=1e-15)
    assert oracle.lib.lo_soft_threshold(1.5, 1.0) == 0.5
    assert oracle.lib.lo_soft_threshold(-0.3, 0.5) == 0.0
    assert oracle.lib.lo_soft_threshold(-2.0, 0.5) == -1.5
    assert oracle.lib.lo_cd_damping(2, 1, 5) == 1.0
    assert oracle.lib.lo_cd_damping(2, 3, 5) == 1.5
    op = _spec(pyoracle, 2, 2, [1.0, 4.0 ** 0.5])
    np.testing.assert_array_equal(oracle.gram_inverse(op, [1.0, 4.0]), [1.0, 1.0])   # SPEC.md "no stages"


@pytest.mark.parametrize("stages,expected", [(1, 16), (2, 38), (3, 56), (4, 62)])
def test_spec_gram_sparsity(oracle, stages, expected):
    # nnz(A^T A) for 1-4 alternating stages, n=8, m=16, theta=2pi/10
    inst = oracle.build_instance(8, stages=stages, q=1, seed=3, s_divisor=8, theta=2 * math.pi / 10)
    A = dense_operator(inst.op)
    assert int(np.sum(np.abs(A.T @ A) > 1e-12)) == expected


def test_oracle_matches_live_reference(oracle, reference):
    kw = dict(n=300, m_ratio=1.7, stages=3, left_stages=1, permute=True, q=2, seed=42, s_divisor=20,
              theta=0.37)
    oi = oracle.build_instance(**kw)
    ri = reference.build_instance(**kw)
    np.testing.assert_array_equal(oi.b, ri.b())
    for a, b in zip(oracle.csr(oi.op), ri.csr()):
        np.testing.assert_array_equal(a, b)
    tr, x = oracle.fista(oi, max_iters=200)
    rtr, rx = ri.solve("fista", max_iters=200)
    np.testing.assert_array_equal(tr["objective"], rtr["objective"])
    np.testing.assert_array_equal(x, rx)


@pytest.mark.parametrize("kw,solver", [
    (dict(n=512, stages=2, q=1, s_divisor=20, seed=4), "fista"),
    (dict(n=1000, stages=1, q=2, s_divisor=50, seed=7), "ista"),
    (dict(n=300, stages=3, left_stages=1, permute=True, q=1, s_divisor=10, seed=9), "fista"),
])
def test_oracle_backtracking_matches_reference(oracle, reference, kw, solver):
    """LPolicy::backtracking (solvers.cpp:99-120, 325-343): power-iteration seed
    (estimate_gram_lmax, linops.cpp:757-778, normal() draws), halving per
    iteration, doubling until the quadratic bound holds -- bit for bit."""
    import math

    kw = dict(kw, theta=2 * math.pi / 10)
    oi, ri = oracle.build_instance(**kw), reference.build_instance(**kw)
    otr, ox = oracle.fista(oi, max_iters=200, backtracking=True, accelerated=solver == "fista", seed=11)
    rtr, rx = ri.solve(solver, max_iters=200, backtracking=True, seed=11)
    np.testing.assert_array_equal(ox, rx)
    for key in ("objective", "extra", "matvecs", "iter"):
        np.testing.assert_array_equal(otr[key], rtr[key])
    assert otr["extra"].sum() > 0  # backtracks happened
