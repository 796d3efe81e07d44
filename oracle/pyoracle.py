"""ctypes front-end for the CPU checkers.

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline / --impl reference), never by the product package.

* :class:`Oracle` wraps ``oracle/liboracle.so`` -- the plain-C restatement of the
  reference path (``oracle/l1oracle.c``).
* :class:`Reference` wraps ``oracle/_ref/libl1ref.so`` -- the unmodified
  reference sources built by ``oracle/Makefile`` -- through ``ref_shim.cpp``.

``build_instance`` restates ``bench.cpp:216-316`` (enumerate_jobs seed
derivation + build_instance) on top of the oracle's RNG and operator.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libl1ref.so")

u64, i32, u32, f64 = C.c_uint64, C.c_int32, C.c_uint32, C.c_double
P = C.POINTER


def _ptr(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(P(ctype))


class LoRng(C.Structure):
    _fields_ = [("mt", u64 * 312), ("idx", C.c_int)]


class LoOp(C.Structure):
    _fields_ = [
        ("m", u64), ("n", u64), ("n_right", u32), ("n_left", u32),
        ("right_offset", P(i32)), ("right_theta", P(f64)),
        ("left_offset", P(i32)), ("left_theta", P(f64)),
        ("p1", P(u32)), ("p2", P(u32)), ("p1_inv", P(u32)), ("p2_inv", P(u32)),
        ("sigma", P(f64)),
    ]


class LoSample(C.Structure):
    _fields_ = [("iter", u64), ("objective", f64), ("nnz", u64), ("matvecs", f64), ("extra", u64)]


class LoSummary(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("reached_target", C.c_int), ("final_objective", f64),
        ("total_matvecs", f64), ("total_pcg_iterations", u64), ("newton_steps", u64),
        ("matvecs_to_target", f64), ("n_samples", u64), ("n_samples_total", u64),
    ]


class LoCfg(C.Structure):
    _fields_ = [
        ("max_iters", u64), ("has_target", C.c_int), ("target", f64),
        ("mu", f64), ("eta", f64), ("grad_tol_rel", f64),
        ("pcg_max_iters", u64), ("ls_max_backtracks", u64), ("l_fixed", f64),
        ("varpi", u64), ("omega", u64), ("seed", u64), ("block", u64), ("accelerated", C.c_int),
        ("backtracking", C.c_int),
    ]


class LoCert(C.Structure):
    _fields_ = [("max_support_violation", f64), ("max_offsupport_violation", f64),
                ("threshold", f64), ("pass_", C.c_int)]


class LoPcg(C.Structure):
    _fields_ = [("iterations", u64), ("converged", C.c_int), ("negative_curvature", C.c_int),
                ("rel_residual", f64)]


def llround(x: float) -> int:
    """std::llround for the non-negative values build_instance uses."""
    return int(math.floor(x + 0.5))


@dataclass
class OpSpec:
    """Realised operator description A = P1 G~ P2 Sigma G^T (linops.hpp:159-206)."""

    m: int
    n: int
    right_offset: np.ndarray
    right_theta: np.ndarray
    left_offset: np.ndarray
    left_theta: np.ndarray
    sigma: np.ndarray
    p1: np.ndarray | None = None
    p2: np.ndarray | None = None
    p1_inv: np.ndarray | None = None
    p2_inv: np.ndarray | None = None
    _keep: list = field(default_factory=list, repr=False)

    def c_struct(self) -> LoOp:
        for name in ("right_offset", "left_offset"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.int32))
        for name in ("right_theta", "left_theta", "sigma"):
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.float64))
        return LoOp(
            self.m, self.n, len(self.right_offset), len(self.left_offset),
            _ptr(self.right_offset, i32), _ptr(self.right_theta, f64),
            _ptr(self.left_offset, i32), _ptr(self.left_theta, f64),
            _ptr(self.p1, u32), _ptr(self.p2, u32), _ptr(self.p1_inv, u32), _ptr(self.p2_inv, u32),
            _ptr(self.sigma, f64),
        )


@dataclass
class Instance:
    """Tall instance as built by build_instance (bench.cpp:253-316)."""

    op: OpSpec
    tau: float
    b: np.ndarray
    support: np.ndarray
    values: np.ndarray
    noise_norm: float
    job_seed: int

    @property
    def m(self):
        return self.op.m

    @property
    def n(self):
        return self.op.n

    def x_star_dense(self):
        x = np.zeros(self.n)
        x[self.support] = self.values
        return x

    def f_star(self):
        """objective_at_planted (instance.cpp:49-51)."""
        return self.tau * float(np.sum(np.abs(self.values))) + 0.5 * self.noise_norm * self.noise_norm


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.lo_rng_seed.argtypes = [P(LoRng), u64]
        L.lo_rng_next.argtypes = [P(LoRng)]
        L.lo_rng_next.restype = u64
        L.lo_mix_seed.argtypes = [u64, u64]
        L.lo_mix_seed.restype = u64
        L.lo_uniform_unit.argtypes = [P(LoRng)]
        L.lo_uniform_unit.restype = f64
        L.lo_uniform_in.argtypes = [P(LoRng), f64, f64]
        L.lo_uniform_in.restype = f64
        L.lo_uniform_index.argtypes = [P(LoRng), u64]
        L.lo_uniform_index.restype = u64
        L.lo_apply_stage.argtypes = [P(f64), u64, C.c_int, f64, C.c_int]
        for fn in ("lo_apply", "lo_apply_transpose", "lo_apply_gram_inverse"):
            getattr(L, fn).argtypes = [P(LoOp), P(f64), P(f64)]
        L.lo_gram_diagonal.argtypes = [P(LoOp), P(f64)]
        L.lo_gram_lmax.argtypes = [P(LoOp)]
        L.lo_estimate_gram_lmax.argtypes = [P(LoOp), u64, u64]
        L.lo_estimate_gram_lmax.restype = f64
        L.lo_gram_lmax.restype = f64
        L.lo_permutation_realize.argtypes = [u64, u64, P(u32), P(u32)]
        L.lo_spectrum_uniform.argtypes = [u64, f64, f64, f64, u64, P(f64)]
        L.lo_ws_create.argtypes = [u64]
        L.lo_ws_create.restype = C.c_void_p
        L.lo_ws_free.argtypes = [C.c_void_p]
        for fn in ("lo_row", "lo_column"):
            getattr(L, fn).argtypes = [P(LoOp), u64, C.c_void_p, P(u32), P(f64)]
            getattr(L, fn).restype = u64
        for fn in ("lo_build_csr", "lo_build_csc"):
            getattr(L, fn).argtypes = [P(LoOp), P(u64), P(u32), P(f64), u64]
            getattr(L, fn).restype = u64
        L.lo_uniform_sparse_solution.argtypes = [u64, u64, f64, P(LoRng), P(u32), P(f64)]
        L.lo_uniform_sparse_solution.restype = u64
        L.lo_generate_instance.argtypes = [P(LoOp), f64, P(u32), P(f64), u64, f64, P(LoRng), P(f64)]
        L.lo_generate_instance.restype = f64
        L.lo_verify_optimality.argtypes = [P(LoOp), f64, P(f64), P(u32), P(f64), u64, f64]
        L.lo_verify_optimality.restype = LoCert
        L.lo_fista.argtypes = [P(LoOp), f64, P(f64), P(LoCfg), P(LoSample), u64, P(f64)]
        L.lo_fista.restype = LoSummary
        L.lo_newton_cg.argtypes = [P(LoOp), f64, P(f64), P(LoCfg), P(LoSample), u64, P(f64)]
        L.lo_newton_cg.restype = LoSummary
        L.lo_cd.argtypes = [P(LoOp), f64, P(f64), P(LoCfg), P(u64), P(u32), P(f64), P(u64),
                            P(LoSample), u64, P(f64)]
        L.lo_cd.restype = LoSummary
        L.lo_pcdm.argtypes = [P(LoOp), f64, P(f64), P(LoCfg), P(u64), P(u32), P(f64), P(u64),
                              P(u32), P(LoSample), u64, P(f64)]
        L.lo_pcdm.restype = LoSummary
        L.lo_pcg_at.argtypes = [P(LoOp), f64, f64, P(f64), P(f64), P(f64), f64, u64, P(f64)]
        L.lo_pcg_at.restype = LoPcg
        L.lo_soft_threshold.argtypes = [f64, f64]
        L.lo_soft_threshold.restype = f64
        L.lo_cd_damping.argtypes = [u64, u64, u64]
        L.lo_cd_damping.restype = f64
        L.lo_set_index_reject.argtypes = [C.c_int]
        L.lo_objective.argtypes = [P(LoOp), f64, P(f64), P(f64)]
        L.lo_objective.restype = f64

    # -- rng ---------------------------------------------------------------
    def rng(self, seed: int) -> LoRng:
        r = LoRng()
        self.lib.lo_rng_seed(C.byref(r), seed)
        return r

    def mix_seed(self, seed: int, salt: int) -> int:
        return int(self.lib.lo_mix_seed(seed, salt))

    # -- operator ------------------------------------------------------------
    def apply(self, op: OpSpec, x):
        s = op.c_struct()
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(op.m)
        self.lib.lo_apply(C.byref(s), _ptr(x, f64), _ptr(y, f64))
        return y

    def apply_transpose(self, op: OpSpec, y):
        s = op.c_struct()
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.empty(op.n)
        self.lib.lo_apply_transpose(C.byref(s), _ptr(y, f64), _ptr(x, f64))
        return x

    def gram_inverse(self, op: OpSpec, v):
        s = op.c_struct()
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty(op.n)
        self.lib.lo_apply_gram_inverse(C.byref(s), _ptr(v, f64), _ptr(out, f64))
        return out

    def gram_diagonal(self, op: OpSpec):
        s = op.c_struct()
        d = np.empty(op.n)
        self.lib.lo_gram_diagonal(C.byref(s), _ptr(d, f64))
        return d

    def gram_lmax(self, op: OpSpec) -> float:
        s = op.c_struct()
        return float(self.lib.lo_gram_lmax(C.byref(s)))

    def _lines(self, op: OpSpec, rows: bool):
        s = op.c_struct()
        dim = op.m if rows else op.n
        nst = len(op.right_offset) + len(op.left_offset)
        per = max(2, 2 * (1 + nst)) * (2 ** min(nst, 6))
        cap = max(16, per * max(op.m, op.n))
        while True:
            ptr = np.zeros(dim + 1, dtype=np.uint64)
            idx = np.empty(cap, dtype=np.uint32)
            val = np.empty(cap, dtype=np.float64)
            fn = self.lib.lo_build_csr if rows else self.lib.lo_build_csc
            nnz = int(fn(C.byref(s), _ptr(ptr, u64), _ptr(idx, u32), _ptr(val, f64), cap))
            if nnz != 2**64 - 1:
                return ptr, idx[:nnz].copy(), val[:nnz].copy()
            cap *= 4

    def csr(self, op: OpSpec):
        """Rows of A from OperatorSpec::row (linops.cpp:597-619)."""
        return self._lines(op, True)

    def csc(self, op: OpSpec):
        """Columns of A from OperatorSpec::column (linops.cpp:566-595)."""
        return self._lines(op, False)

    def row(self, op: OpSpec, i: int):
        s = op.c_struct()
        ws = self.lib.lo_ws_create(max(op.m, op.n))
        idx = np.empty(max(op.m, op.n), dtype=np.uint32)
        val = np.empty(max(op.m, op.n))
        k = self.lib.lo_row(C.byref(s), i, ws, _ptr(idx, u32), _ptr(val, f64))
        self.lib.lo_ws_free(ws)
        return idx[:k].copy(), val[:k].copy()

    def column(self, op: OpSpec, j: int):
        s = op.c_struct()
        ws = self.lib.lo_ws_create(max(op.m, op.n))
        idx = np.empty(max(op.m, op.n), dtype=np.uint32)
        val = np.empty(max(op.m, op.n))
        k = self.lib.lo_column(C.byref(s), j, ws, _ptr(idx, u32), _ptr(val, f64))
        self.lib.lo_ws_free(ws)
        return idx[:k].copy(), val[:k].copy()

    # -- generator -----------------------------------------------------------
    def spec(self, n, m_ratio=2.0, stages=1, left_stages=0, permute=False, q=1, shift=0.1,
             theta=2 * math.pi / 10, job_seed=0, sigma=None) -> OpSpec:
        """Operator part of build_instance (bench.cpp:255-279) + finalize (linops.cpp:394-416)."""
        m = llround(m_ratio * float(n))
        ro = np.array([(stages - 1 - i) % 2 for i in range(stages)], dtype=np.int32)
        lo_ = np.array([(left_stages - 1 - i) % 2 for i in range(left_stages)], dtype=np.int32)
        op = OpSpec(m, n, ro, np.full(stages, theta), lo_, np.full(left_stages, theta),
                    np.empty(0))
        if permute:
            for which, salt in (("p1", 1), ("p2", 2)):
                mp = np.empty(m, dtype=np.uint32)
                inv = np.empty(m, dtype=np.uint32)
                self.lib.lo_permutation_realize(m, self.mix_seed(job_seed, salt), _ptr(mp, u32),
                                                _ptr(inv, u32))
                setattr(op, which, mp)
                setattr(op, which + "_inv", inv)
        if sigma is None:
            sig = np.empty(n)
            self.lib.lo_spectrum_uniform(n, 0.0, math.pow(10.0, q), shift,
                                         self.mix_seed(job_seed, 3), _ptr(sig, f64))
        else:
            sig = np.ascontiguousarray(sigma, dtype=np.float64)
        op.sigma = sig
        return op

    def build_instance(self, n, m_ratio=2.0, stages=1, left_stages=0, permute=False, q=1,
                       shift=0.1, s_divisor=128, gamma=10.0, tau=1.0, theta=2 * math.pi / 10,
                       seed=1, sigma=None, fill_bound=0.9) -> Instance:
        """bench.cpp:216-316 for a single-job config (job.seed = mix_seed(seed, 0))."""
        job_seed = self.mix_seed(seed, 0)
        op = self.spec(n, m_ratio, stages, left_stages, permute, q, shift, theta, job_seed, sigma)
        s = max(1, n // s_divisor)
        rng = self.rng(self.mix_seed(job_seed, 4))
        sup = np.empty(s, dtype=np.uint32)
        vals = np.empty(s)
        self.lib.lo_uniform_sparse_solution(n, s, gamma, C.byref(rng), _ptr(sup, u32), _ptr(vals, f64))
        gen = self.rng(self.mix_seed(job_seed, 5))
        b = np.empty(op.m)
        st = op.c_struct()
        noise = self.lib.lo_generate_instance(C.byref(st), tau, _ptr(sup, u32), _ptr(vals, f64), s,
                                              fill_bound, C.byref(gen), _ptr(b, f64))
        return Instance(op, tau, b, sup, vals, float(noise), job_seed)

    def verify(self, inst: Instance, tol: float):
        st = inst.op.c_struct()
        c = self.lib.lo_verify_optimality(C.byref(st), inst.tau, _ptr(inst.b, f64),
                                          _ptr(inst.support, u32), _ptr(inst.values, f64),
                                          len(inst.support), tol)
        return dict(max_support_violation=c.max_support_violation,
                    max_offsupport_violation=c.max_offsupport_violation,
                    threshold=c.threshold, passed=bool(c.pass_))

    # -- solvers -------------------------------------------------------------
    @staticmethod
    def cfg(max_iters=100000, target=None, mu=1e-5, eta=0.1, grad_tol_rel=1e-8,
            pcg_max_iters=1000, ls_max_backtracks=50, l_fixed=0.0, varpi=1, omega=0, seed=0,
            block=256, accelerated=True, backtracking=False) -> LoCfg:
        return LoCfg(max_iters, 0 if target is None else 1, 0.0 if target is None else target,
                     mu, eta, grad_tol_rel, pcg_max_iters, ls_max_backtracks, l_fixed, varpi, omega,
                     seed, block, 1 if accelerated else 0, 1 if backtracking else 0)

    def _run(self, fn, inst: Instance, cfg: LoCfg, extra_args=(), cap=200000):
        st = inst.op.c_struct()
        samples = (LoSample * cap)()
        x = np.empty(inst.n)
        summ = fn(C.byref(st), inst.tau, _ptr(inst.b, f64), C.byref(cfg), *extra_args, samples, cap,
                  _ptr(x, f64))
        k = int(summ.n_samples)
        tr = dict(
            iter=np.array([samples[i].iter for i in range(k)], dtype=np.int64),
            objective=np.array([samples[i].objective for i in range(k)]),
            nnz=np.array([samples[i].nnz for i in range(k)], dtype=np.int64),
            matvecs=np.array([samples[i].matvecs for i in range(k)]),
            extra=np.array([samples[i].extra for i in range(k)], dtype=np.int64),
            status=int(summ.status), reached_target=bool(summ.reached_target),
            final_objective=float(summ.final_objective), total_matvecs=float(summ.total_matvecs),
            total_pcg_iterations=int(summ.total_pcg_iterations),
            newton_steps=int(summ.newton_steps), matvecs_to_target=float(summ.matvecs_to_target),
        )
        return tr, x

    def fista(self, inst, **kw):
        return self._run(self.lib.lo_fista, inst, self.cfg(**kw))

    def newton_cg(self, inst, **kw):
        return self._run(self.lib.lo_newton_cg, inst, self.cfg(**kw))

    def set_index_reject(self, s):
        """Test hook: CD / PCDM coordinate draws redrawn with probability
        ~2^-s (0 = the reference's limit); mirrors L1B_TEST_INDEX_REJECT."""
        self.lib.lo_set_index_reject(int(s))

    def cd(self, inst, csc=None, csr=None, **kw):
        csc = csc or self.csc(inst.op)
        csr = csr or self.csr(inst.op)
        args = (_ptr(csc[0], u64), _ptr(csc[1], u32), _ptr(csc[2], f64), _ptr(csr[0], u64))
        return self._run(self.lib.lo_cd, inst, self.cfg(**kw), args)

    def pcdm(self, inst, csc=None, csr=None, **kw):
        csc = csc or self.csc(inst.op)
        csr = csr or self.csr(inst.op)
        args = (_ptr(csc[0], u64), _ptr(csc[1], u32), _ptr(csc[2], f64), _ptr(csr[0], u64),
                _ptr(csr[1], u32))
        return self._run(self.lib.lo_pcdm, inst, self.cfg(**kw), args)

    def pcg_at(self, inst, mu, x, rhs, precond, eta, max_iters):
        st = inst.op.c_struct()
        x, rhs, precond = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, rhs, precond))
        step = np.empty(inst.n)
        r = self.lib.lo_pcg_at(C.byref(st), inst.tau, mu, _ptr(x, f64), _ptr(rhs, f64),
                               _ptr(precond, f64), eta, max_iters, _ptr(step, f64))
        return step, dict(iterations=int(r.iterations), converged=bool(r.converged),
                          negative_curvature=bool(r.negative_curvature))

    def objective(self, inst, x):
        st = inst.op.c_struct()
        x = np.ascontiguousarray(x, dtype=np.float64)
        return float(self.lib.lo_objective(C.byref(st), inst.tau, _ptr(inst.b, f64), _ptr(x, f64)))


# ---------------------------------------------------------------------------
# The reference itself (oracle/_ref/libl1ref.so)


class RefSample(C.Structure):
    _fields_ = [("iter", u64), ("elapsed_s", f64), ("objective", f64), ("nnz", u64),
                ("matvecs", f64), ("extra", u64)]


class RefSummary(C.Structure):
    _fields_ = [("status", C.c_int), ("reached_target", C.c_int), ("final_objective", f64),
                ("elapsed_s", f64), ("total_matvecs", f64), ("total_pcg_iterations", u64),
                ("newton_steps", u64), ("time_to_target", f64), ("matvecs_to_target", f64),
                ("n_samples_total", u64)]


class RefCfg(C.Structure):
    _fields_ = [("id", C.c_char_p), ("max_iters", u64), ("max_seconds", f64),
                ("has_target", C.c_int), ("target", f64), ("mu", f64), ("eta", f64),
                ("grad_tol_rel", f64), ("pcg_max_iters", u64), ("ls_max_backtracks", u64),
                ("l_fixed", f64), ("varpi", u64), ("omega", u64), ("seed", u64),
                ("backtracking", C.c_int)]


class Reference:
    """The unmodified reference (oracle/_ref/libl1ref.so), via ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_instance.argtypes = [u64, f64, u64, u64, C.c_int, C.c_int, f64, u64, f64, f64,
                                         f64, u64, P(f64)]
        L.ref_build_instance.restype = C.c_void_p
        L.ref_build_instance2.argtypes = L.ref_build_instance.argtypes + [C.c_int, f64, f64, f64]
        L.ref_build_instance2.restype = C.c_void_p
        L.ref_next_spectrum_alternating.argtypes = [C.c_int, f64, f64]
        L.ref_save_instance.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_save_instance.restype = C.c_int
        L.ref_load_instance.argtypes = [C.c_char_p]
        L.ref_load_instance.restype = C.c_void_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_dims.argtypes = [C.c_void_p, P(u64), P(u64)]
        for fn in ("ref_tau", "ref_noise_norm", "ref_cert_kappa", "ref_f_star", "ref_gram_lmax"):
            getattr(L, fn).argtypes = [C.c_void_p]
            getattr(L, fn).restype = f64
        L.ref_get_b.argtypes = [C.c_void_p, P(f64)]
        L.ref_get_sigma.argtypes = [C.c_void_p, P(f64)]
        L.ref_xstar_nnz.argtypes = [C.c_void_p]
        L.ref_xstar_nnz.restype = u64
        L.ref_get_xstar.argtypes = [C.c_void_p, P(u32), P(f64)]
        L.ref_get_perm.argtypes = [C.c_void_p, C.c_int, P(u32)]
        L.ref_n_stages.argtypes = [C.c_void_p, C.c_int]
        L.ref_n_stages.restype = u32
        L.ref_stage.argtypes = [C.c_void_p, C.c_int, u32, P(i32), P(f64)]
        for fn in ("ref_row", "ref_column"):
            getattr(L, fn).argtypes = [C.c_void_p, u64, P(u32), P(f64)]
            getattr(L, fn).restype = u64
        for fn in ("ref_apply", "ref_apply_transpose", "ref_gram_inverse"):
            getattr(L, fn).argtypes = [C.c_void_p, P(f64), P(f64)]
        L.ref_gram_diagonal.argtypes = [C.c_void_p, P(f64)]
        L.ref_objective.argtypes = [C.c_void_p, P(f64)]
        L.ref_objective.restype = f64
        L.ref_verify.argtypes = [C.c_void_p, f64, P(f64)]
        L.ref_smoothed_hessvec.argtypes = [C.c_void_p, P(f64), f64, P(f64), P(f64)]
        L.ref_smoothed_gradient.argtypes = [C.c_void_p, P(f64), f64, P(f64)]
        L.ref_smoothed_objective.argtypes = [C.c_void_p, P(f64), f64]
        L.ref_smoothed_objective.restype = f64
        L.ref_pcg.argtypes = [C.c_void_p, P(f64), f64, P(f64), P(f64), f64, u64, P(f64), P(u64),
                              P(C.c_int)]
        L.ref_solve.argtypes = [C.c_void_p, P(RefCfg), P(RefSample), u64, P(u64), P(RefSummary),
                                P(f64)]

    SOLUTION_KINDS = {"uniform": 0, "spectral": 1, "two_value": 2}

    def build_instance(self, n, m_ratio=2.0, stages=1, left_stages=0, permute=False, q=1,
                       shift=0.1, s_divisor=128, gamma=10.0, tau=1.0, theta=2 * math.pi / 10,
                       seed=1, sigma=None, solution="uniform", s1_fraction=0.5, value_a=-1e4,
                       value_b=1e-1, alternating=None):
        sig = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float64)
        if alternating is not None:  # SpectrumRule::Kind::alternating (odd_value, even_value)
            self.lib.ref_next_spectrum_alternating(1, float(alternating[0]), float(alternating[1]))
        h = self.lib.ref_build_instance2(n, m_ratio, stages, left_stages, int(permute), q, shift,
                                         s_divisor, gamma, tau, theta, seed, _ptr(sig, f64),
                                         self.SOLUTION_KINDS[solution], s1_fraction, value_a, value_b)
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return RefInstance(self, h)

    def save_instance(self, inst, path):
        """the reference's save_instance (serialize.cpp:182-219)"""
        if self.lib.ref_save_instance(inst.h, str(path).encode()) != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def load_instance(self, path):
        """the reference's load_instance (serialize.cpp:221-281)"""
        h = self.lib.ref_load_instance(str(path).encode())
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return RefInstance(self, h)


class RefInstance:
    def __init__(self, ref: Reference, h):
        self.ref, self.lib, self.h = ref, ref.lib, h
        m, n = u64(), u64()
        self.lib.ref_dims(h, C.byref(m), C.byref(n))
        self.m, self.n = int(m.value), int(n.value)

    def __del__(self):
        try:
            self.lib.ref_free(self.h)
        except Exception:
            pass

    tau = property(lambda s: float(s.lib.ref_tau(s.h)))
    noise_norm = property(lambda s: float(s.lib.ref_noise_norm(s.h)))
    cert_kappa = property(lambda s: float(s.lib.ref_cert_kappa(s.h)))
    f_star = property(lambda s: float(s.lib.ref_f_star(s.h)))
    gram_lmax = property(lambda s: float(s.lib.ref_gram_lmax(s.h)))

    def b(self):
        out = np.empty(self.m)
        self.lib.ref_get_b(self.h, _ptr(out, f64))
        return out

    def sigma(self):
        out = np.empty(self.n)
        self.lib.ref_get_sigma(self.h, _ptr(out, f64))
        return out

    def x_star(self):
        k = int(self.lib.ref_xstar_nnz(self.h))
        sup = np.empty(k, dtype=np.uint32)
        val = np.empty(k)
        self.lib.ref_get_xstar(self.h, _ptr(sup, u32), _ptr(val, f64))
        return sup, val

    def perm(self, which):
        mp = np.empty(self.m, dtype=np.uint32)
        return mp if self.lib.ref_get_perm(self.h, which, _ptr(mp, u32)) else None

    def stages(self, right=True):
        out = []
        for k in range(int(self.lib.ref_n_stages(self.h, int(right)))):
            o, t = i32(), f64()
            self.lib.ref_stage(self.h, int(right), k, C.byref(o), C.byref(t))
            out.append((int(o.value), float(t.value)))
        return out

    def _line(self, fn, i):
        cap = max(self.m, self.n)
        idx = np.empty(cap, dtype=np.uint32)
        val = np.empty(cap)
        k = int(fn(self.h, i, _ptr(idx, u32), _ptr(val, f64)))
        return idx[:k].copy(), val[:k].copy()

    def row(self, i):
        return self._line(self.lib.ref_row, i)

    def column(self, j):
        return self._line(self.lib.ref_column, j)

    def csr(self):
        ptr = [0]
        idx, val = [], []
        for i in range(self.m):
            a, v = self.row(i)
            idx.append(a)
            val.append(v)
            ptr.append(ptr[-1] + len(a))
        return (np.array(ptr, dtype=np.uint64), np.concatenate(idx).astype(np.uint32),
                np.concatenate(val))

    def csc(self):
        ptr = [0]
        idx, val = [], []
        for j in range(self.n):
            a, v = self.column(j)
            idx.append(a)
            val.append(v)
            ptr.append(ptr[-1] + len(a))
        return (np.array(ptr, dtype=np.uint64), np.concatenate(idx).astype(np.uint32),
                np.concatenate(val))

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.m)
        self.lib.ref_apply(self.h, _ptr(x, f64), _ptr(y, f64))
        return y

    def apply_transpose(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        x = np.empty(self.n)
        self.lib.ref_apply_transpose(self.h, _ptr(y, f64), _ptr(x, f64))
        return x

    def gram_inverse(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty(self.n)
        self.lib.ref_gram_inverse(self.h, _ptr(v, f64), _ptr(out, f64))
        return out

    def gram_diagonal(self):
        d = np.empty(self.n)
        self.lib.ref_gram_diagonal(self.h, _ptr(d, f64))
        return d

    def objective(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return float(self.lib.ref_objective(self.h, _ptr(x, f64)))

    def verify(self, tol):
        out = np.empty(3)
        ok = self.lib.ref_verify(self.h, tol, _ptr(out, f64))
        return dict(max_support_violation=out[0], max_offsupport_violation=out[1],
                    threshold=out[2], passed=bool(ok))

    def smoothed_hessvec(self, x, mu, v):
        x, v = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, v))
        out = np.empty(self.n)
        self.lib.ref_smoothed_hessvec(self.h, _ptr(x, f64), mu, _ptr(v, f64), _ptr(out, f64))
        return out

    def smoothed_gradient(self, x, mu):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.n)
        self.lib.ref_smoothed_gradient(self.h, _ptr(x, f64), mu, _ptr(out, f64))
        return out

    def smoothed_objective(self, x, mu):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return float(self.lib.ref_smoothed_objective(self.h, _ptr(x, f64), mu))

    def pcg(self, x, mu, rhs, precond, eta, max_iters):
        x, rhs, precond = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, rhs, precond))
        step = np.empty(self.n)
        it, cv = u64(), C.c_int()
        rc = self.lib.ref_pcg(self.h, _ptr(x, f64), mu, _ptr(rhs, f64), _ptr(precond, f64), eta,
                              max_iters, _ptr(step, f64), C.byref(it), C.byref(cv))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return step, dict(iterations=int(it.value), converged=bool(cv.value))

    def solve(self, solver="fista", max_iters=100000, max_seconds=1e9, target=None, mu=1e-5,
              eta=0.1, grad_tol_rel=1e-8, pcg_max_iters=1000, ls_max_backtracks=50, l_fixed=0.0,
              varpi=1, omega=0, seed=0, cap=200000, backtracking=False):
        cfg = RefCfg(solver.encode(), max_iters, max_seconds, 0 if target is None else 1,
                     0.0 if target is None else target, mu, eta, grad_tol_rel, pcg_max_iters,
                     ls_max_backtracks, l_fixed, varpi, omega, seed, 1 if backtracking else 0)
        samples = (RefSample * cap)()
        ns = u64()
        summ = RefSummary()
        x = np.empty(self.n)
        rc = self.lib.ref_solve(self.h, C.byref(cfg), samples, cap, C.byref(ns), C.byref(summ),
                                _ptr(x, f64))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        k = int(ns.value)
        tr = dict(
            iter=np.array([samples[i].iter for i in range(k)], dtype=np.int64),
            elapsed_s=np.array([samples[i].elapsed_s for i in range(k)]),
            objective=np.array([samples[i].objective for i in range(k)]),
            nnz=np.array([samples[i].nnz for i in range(k)], dtype=np.int64),
            matvecs=np.array([samples[i].matvecs for i in range(k)]),
            extra=np.array([samples[i].extra for i in range(k)], dtype=np.int64),
            status=int(summ.status), reached_target=bool(summ.reached_target),
            final_objective=float(summ.final_objective), elapsed_s_total=float(summ.elapsed_s),
            total_matvecs=float(summ.total_matvecs),
            total_pcg_iterations=int(summ.total_pcg_iterations),
            newton_steps=int(summ.newton_steps), matvecs_to_target=float(summ.matvecs_to_target),
        )
        return tr, x


def log_spaced_sigma(n: int, decades: float = 1.0) -> np.ndarray:
    """C1 spectrum: sigma_i = 10^(decades * i/(n-1)) -> kappa(A^T A) = 10^(2*decades)."""
    # math.pow is glibc pow(), the same routine std::pow calls in the reference build
    return np.array([math.pow(10.0, decades * float(i) / float(n - 1)) for i in range(n)])
