"""Writes the golden vectors of tests/golden/*.npz from the UNMODIFIED reference
compiled by oracle/Makefile (oracle/_ref/libl1ref.so).  Run in the build
container, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Every case is built through the reference's own public API (ExperimentConfig +
enumerate_jobs + build_instance, OperatorSpec::row/column, run_solver, ...) via
oracle/ref_shim.cpp; nothing here re-implements the algorithm.
"""
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import Reference, log_spaced_sigma  # noqa: E402

THETA = 2 * math.pi / 10

# (name, build_instance kwargs) -- small enough for committed fixtures
CASES = {
    # C1 mapping: n=2^12, m=2n, k=1, log-spaced sigma (kappa=100), s=n/100, seed 0
    "c1": dict(n=4096, stages=1, s_divisor=100, seed=0, sigma="log1"),
    # 4-stage banded instance (C4/C5 structure) at desk scale, q=1
    "k4": dict(n=2048, stages=4, s_divisor=100, q=1, seed=3),
    # general operator: seeded P1/P2, left stages, odd m (random_spec-like)
    "perm": dict(n=96, m_ratio=1.5, stages=3, left_stages=2, permute=True, q=1, seed=7, s_divisor=16),
    # odd n, alternating-offset stages, q=2
    "odd": dict(n=101, m_ratio=2.0, stages=2, q=2, seed=11, s_divisor=10),
    # pdNCG-style instance (q=0 keeps the PCG trajectory well conditioned)
    "ncg": dict(n=1024, stages=1, q=0, seed=2, s_divisor=100),
    # C2-like for CD
    "cd": dict(n=512, stages=1, q=1, seed=1, s_divisor=100),
}


def build(ref, kw):
    kw = dict(kw)
    sig = kw.pop("sigma", None)
    if sig == "log1":
        kw["sigma"] = log_spaced_sigma(kw["n"], 1.0)
    return ref.build_instance(theta=THETA, **kw)


def main():
    ref = Reference()
    for name, kw in CASES.items():
        ri = build(ref, kw)
        out = dict(m=ri.m, n=ri.n, tau=ri.tau, sigma=ri.sigma(), b=ri.b(), noise_norm=ri.noise_norm,
                   cert_kappa=ri.cert_kappa, f_star=ri.f_star, gram_lmax=ri.gram_lmax)
        sup, val = ri.x_star()
        out.update(support=sup, values=val)
        p1, p2 = ri.perm(1), ri.perm(2)
        if p1 is not None:
            out.update(p1=p1, p2=p2)
        rs, ls = ri.stages(True), ri.stages(False)
        out.update(right_offset=np.array([s[0] for s in rs], dtype=np.int32),
                   right_theta=np.array([s[1] for s in rs]),
                   left_offset=np.array([s[0] for s in ls], dtype=np.int32),
                   left_theta=np.array([s[1] for s in ls]))
        csr, csc = ri.csr(), ri.csc()
        out.update(csr_ptr=csr[0], csr_idx=csr[1], csr_val=csr[2],
                   csc_ptr=csc[0], csc_idx=csc[1], csc_val=csc[2])
        out["gram_diag"] = ri.gram_diagonal()
        rng = np.random.default_rng(1234)
        xv = rng.standard_normal(ri.n)
        yv = rng.standard_normal(ri.m)
        out.update(probe_x=xv, probe_ax=ri.apply(xv), probe_y=yv, probe_aty=ri.apply_transpose(yv),
                   probe_ginv=ri.gram_inverse(xv))
        cert = ri.verify(1e-8)
        out.update(cert=np.array([cert["max_support_violation"], cert["max_offsupport_violation"]]))
        f0 = 0.5 * float(np.dot(out["b"], out["b"]))
        target = ri.f_star + 1e-8 * max(f0 - ri.f_star, 0.0)
        out["fista_target"] = target
        tr, x = ri.solve("fista", max_iters=3000, target=target)
        out.update(fista_iter=tr["iter"], fista_obj=tr["objective"], fista_nnz=tr["nnz"],
                   fista_matvecs=tr["matvecs"], fista_status=tr["status"], fista_x=x)
        tr, x = ri.solve("ista", max_iters=50)
        out.update(ista_obj=tr["objective"], ista_x=x)
        if name in ("ncg", "odd", "cd"):
            tr, x = ri.solve("newton_cg", max_iters=8)
            out.update(ncg_iter=tr["iter"], ncg_obj=tr["objective"], ncg_extra=tr["extra"],
                       ncg_x=x, ncg_pcg=tr["total_pcg_iterations"], ncg_status=tr["status"])
        if name in ("cd", "odd", "perm"):
            tr, x = ri.solve("cd", max_iters=20, varpi=4, seed=5)
            out.update(cd_obj=tr["objective"], cd_extra=tr["extra"], cd_matvecs=tr["matvecs"], cd_x=x)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: m={ri.m} n={ri.n} nnz={len(csr[1])} fista_iters={out['fista_iter'][-1]} "
              f"-> {os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    main()
