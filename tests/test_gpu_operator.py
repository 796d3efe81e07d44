"""GPU parity of the generator and the operator kernels against the oracle /
reference golden vectors.  Bar: indices and everything the reference computes
with the same operation order bit-exact; SpMV products (different summation
order) within 1e-13 relative."""
import numpy as np
import pytest

from conftest import CASES, load_golden
from gpu_util import device_build, need_cuda, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", CASES)
def test_generator_bit_exact(name):
    need_cuda()
    g = load_golden(name)
    inst = device_build(name)
    assert (inst.m, inst.n) == (int(g["m"]), int(g["n"]))
    np.testing.assert_array_equal(inst.sigma(), g["sigma"])
    xs = inst.x_star
    np.testing.assert_array_equal(xs.support, g["support"])
    np.testing.assert_array_equal(xs.values, g["values"])
    np.testing.assert_array_equal(inst.b, g["b"])  # sweeps in reference order: bit-exact
    assert inst.noise_norm == pytest.approx(float(g["noise_norm"]), rel=1e-14)
    assert inst.objective_at_planted() == pytest.approx(float(g["f_star"]), rel=1e-14)
    assert inst.cert_kappa == float(g["cert_kappa"])
    assert inst.op.gram_lmax() == float(g["gram_lmax"])


@pytest.mark.parametrize("name", CASES)
def test_csr_csc_bit_exact(name):
    need_cuda()
    g = load_golden(name)
    inst = device_build(name)
    for got, key in ((inst.op.csr(), "csr"), (inst.op.csc(), "csc")):
        np.testing.assert_array_equal(got[0], g[f"{key}_ptr"])
        np.testing.assert_array_equal(got[1], g[f"{key}_idx"])
        np.testing.assert_array_equal(got[2], g[f"{key}_val"])


@pytest.mark.parametrize("name", CASES)
def test_products(name):
    torch = need_cuda()
    g = load_golden(name)
    inst = device_build(name)
    x = torch.tensor(g["probe_x"], device="cuda")
    y = torch.tensor(g["probe_y"], device="cuda")
    # matrix-free sweeps: the reference's own operation order -> bit-exact
    np.testing.assert_array_equal(inst.op.apply(x, path="sweep").cpu().numpy(), g["probe_ax"])
    np.testing.assert_array_equal(inst.op.apply_transpose(y, path="sweep").cpu().numpy(), g["probe_aty"])
    np.testing.assert_array_equal(inst.op.apply_gram_inverse(x).cpu().numpy(), g["probe_ginv"])
    np.testing.assert_array_equal(inst.op.gram_diagonal().cpu().numpy(), g["gram_diag"])
    if "p1" not in g and len(g["left_offset"]) == 0:  # banded: the fused matrix-free kernels
        np.testing.assert_array_equal(inst.op.apply(x, path="fused").cpu().numpy(), g["probe_ax"])
        np.testing.assert_array_equal(inst.op.apply_transpose(y, path="fused").cpu().numpy(), g["probe_aty"])
    # CSR / CSC SpMV kernels
    assert rel_err(inst.op.apply(x).cpu().numpy(), g["probe_ax"]) < 1e-13
    assert rel_err(inst.op.apply_transpose(y).cpu().numpy(), g["probe_aty"]) < 1e-13


@pytest.mark.parametrize("name", CASES)
def test_certificate(name):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    g = load_golden(name)
    inst = device_build(name)
    rep = l1bench.verify_optimality(inst, 1e-8)
    assert rep.passed
    assert rep.max_support_violation == float(g["cert"][0])
    assert rep.max_offsupport_violation == float(g["cert"][1])


def test_certificate_detects_perturbation():
    torch = need_cuda()
    from paper_1503_03520_b200 import l1bench

    g = load_golden("k4")
    b = g["b"].copy()
    b[int(g["support"][0])] += 1.0  # SPEC.md: b perturbed by +1 -> fail
    inst = l1bench.ProblemInstance.from_host(
        int(g["m"]), int(g["n"]), list(zip(g["right_offset"], g["right_theta"])), g["sigma"], b,
        float(g["tau"]), g["support"], g["values"])
    assert not l1bench.verify_optimality(inst, 1e-8).passed


@pytest.mark.parametrize("name", ["perm", "k4"])
def test_from_host_matches_generated(name):
    need_cuda()
    from paper_1503_03520_b200 import l1bench

    g = load_golden(name)
    inst = l1bench.ProblemInstance.from_host(
        int(g["m"]), int(g["n"]), list(zip(g["right_offset"], g["right_theta"])), g["sigma"], g["b"],
        float(g["tau"]), g["support"], g["values"],
        left_stages=list(zip(g["left_offset"], g["left_theta"])),
        p1=g.get("p1"), p2=g.get("p2"))
    for got, key in ((inst.op.csr(), "csr"), (inst.op.csc(), "csc")):
        np.testing.assert_array_equal(got[1], g[f"{key}_idx"])
        np.testing.assert_array_equal(got[2], g[f"{key}_val"])


def test_large_properties():
    """n = 2^22, 4 stages: structure (nnz = 8n-16, |col-row| <= 4), adjoint
    identity and SpMV == sweep products at full size."""
    torch = need_cuda()
    from paper_1503_03520_b200 import l1bench

    n = 1 << 22
    inst = l1bench.build_instance(n, stages=4, q=1, s_divisor=1000, seed=3)
    assert inst.info.nnz == 8 * n - 16
    assert inst.info.m_active == n
    gen = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    y = torch.randn(2 * n, dtype=torch.float64, device="cuda", generator=gen)
    ax = inst.op.apply(x)
    aty = inst.op.apply_transpose(y)
    lhs, rhs = float(torch.dot(ax, y)), float(torch.dot(x, aty))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0) * 10
    assert float(torch.max(torch.abs(ax - inst.op.apply(x, path="sweep")))) <= 1e-13 * float(torch.max(torch.abs(ax)))
    assert float(torch.max(torch.abs(aty - inst.op.apply_transpose(y, path="sweep")))) <= 1e-13 * float(torch.max(torch.abs(aty)))
    # fused matrix-free == stage-by-stage sweeps, bit for bit, at full size
    assert torch.equal(inst.op.apply(x, path="fused"), inst.op.apply(x, path="sweep"))
    assert torch.equal(inst.op.apply_transpose(y, path="fused"), inst.op.apply_transpose(y, path="sweep"))
    ptr, idx, _ = inst.op.csr()
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr[: n + 1].astype(np.int64)))
    assert np.max(np.abs(idx.astype(np.int64) - rows)) <= 4
