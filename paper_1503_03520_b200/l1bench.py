"""Python mirror of the reference's ``l1bench`` generator/solver API over the
CUDA C ABI (include/l1b.h).

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/l1bench/*.hpp):

==============================  ============================================
reference (C++)                  here
==============================  ============================================
``ExperimentConfig`` + ``build_instance`` (bench.hpp:37-102)   :func:`build_instance`
``ProblemInstance`` (instance.hpp:36-52)                         :class:`ProblemInstance`
``OperatorSpec`` apply / apply_transpose / gram_diagonal (linops.hpp:139-206)  ``ProblemInstance.op``
``verify_optimality`` (instance.hpp:74)                          :func:`verify_optimality`
``SolverConfig`` / ``SolverTrace`` / ``StopReason`` (solvers.hpp:15-66)
``run_solver`` / ``fista_run`` / ``ista_run`` / ``coordinate_descent_run`` / ``newton_cg_run``
``objective`` (solvers.hpp:70)
==============================  ============================================

``std::invalid_argument`` surfaces as :class:`ValueError`, ``std::runtime_error``
as :class:`RuntimeError`.  Device vectors are torch CUDA float64 tensors (torch
is only the device-memory plumbing); everything else is numpy on the host.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


def _lib():
    return N.load()


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _dptr(t) -> int:
    """Device pointer of a contiguous CUDA float64 torch tensor."""
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise ValueError("device vectors must be CUDA float64 torch tensors")
    if not t.is_contiguous():
        raise ValueError("device vectors must be contiguous")
    return t.data_ptr()


def mix_seed(seed: int, salt: int) -> int:
    """splitmix64 finaliser of rng.hpp:19-24."""
    return int(_lib().l1b_mix_seed(seed, salt))


def realize_permutation(n: int, seed: int) -> np.ndarray:
    """Permutation::random(n, seed).map() (linops.cpp:224-239)."""
    out = np.empty(n, dtype=np.uint32)
    N.check(_lib().l1b_realize_permutation(n, seed, _ptr(out, _u32p)))
    return out


def realize_spectrum_uniform(n: int, lo: float, hi: float, shift: float, seed: int) -> np.ndarray:
    """Spectrum::uniform(n, lo, hi, shift, seed).values() (linops.cpp:320-336)."""
    out = np.empty(n)
    N.check(_lib().l1b_realize_spectrum_uniform(n, lo, hi, shift, seed, _ptr(out, _f64p)))
    return out


class StopReason(enum.IntEnum):  # solvers.hpp:24
    target_reached = 0
    iter_budget = 1
    time_budget = 2

    def __str__(self):  # to_string (solvers.cpp:124-131)
        return {0: "target-reached", 1: "iter-budget", 2: "time-budget"}[int(self)]


class LPolicy(enum.IntEnum):
    spectrum = 0
    backtracking = 1


@dataclass
class SolverConfig:  # solvers.hpp:17-41
    id: str = "fista"
    max_iters: int = 100000
    max_seconds: float = 600.0
    target_objective: Optional[float] = None
    mu: float = 1e-5
    eta: float = 0.1
    pcg_max_iters: int = 1000
    ls_max_backtracks: int = 50
    grad_tol_rel: float = 1e-8
    l_policy: LPolicy = LPolicy.spectrum
    l_fixed: Optional[float] = None
    varpi: int = 1
    omega: Optional[int] = None
    seed: int = 0
    block: int = 256  # pcdm: coordinates per block
    op: str = "auto"  # FISTA/ISTA products: "auto" (matrix-free when banded) | "sparse" | "matrix_free"
    # "exact": the reference's separately rounded a*b+c (bit-identical iterates);
    # "fma": fused multiply-adds in the large matrix-free FISTA kernels (<= 1e-12)
    arith: str = "exact"

    _IDS = {"ista": N.ISTA, "fista": N.FISTA, "cd": N.CD, "newton_cg": N.NEWTON_CG, "pcdm": N.PCDM}

    def to_c(self) -> N.SolverCfg:
        if self.id not in self._IDS:
            raise ValueError(f"SolverConfig: unknown solver id '{self.id}'")
        c = N.SolverCfg()
        _lib().l1b_solver_cfg_default(C.byref(c))
        c.solver = self._IDS[self.id]
        c.max_iters = int(self.max_iters)
        c.max_seconds = float(self.max_seconds)
        c.has_target = 0 if self.target_objective is None else 1
        c.target = 0.0 if self.target_objective is None else float(self.target_objective)
        c.mu, c.eta = float(self.mu), float(self.eta)
        c.pcg_max_iters, c.ls_max_backtracks = int(self.pcg_max_iters), int(self.ls_max_backtracks)
        c.grad_tol_rel = float(self.grad_tol_rel)
        if self.l_fixed is not None and not (self.l_fixed > 0.0):
            raise ValueError("SolverConfig: fixed L must be positive")
        c.l_fixed = 0.0 if self.l_fixed is None else float(self.l_fixed)
        c.varpi = int(self.varpi)
        c.omega = 0 if self.omega is None else int(self.omega)
        c.seed = int(self.seed)
        c.block = int(self.block)
        c.l_policy = int(LPolicy(self.l_policy))
        ops = {"auto": N.OP_AUTO, "sparse": N.OP_SPARSE, "matrix_free": N.OP_MATRIX_FREE}
        if self.op not in ops:
            raise ValueError(f"SolverConfig: unknown operator path '{self.op}'")
        c.op = ops[self.op]
        ariths = {"exact": 0, "fma": 1}
        if self.arith not in ariths:
            raise ValueError(f"SolverConfig: unknown arithmetic mode '{self.arith}'")
        c.arith = ariths[self.arith]
        return c


@dataclass
class TraceSample:  # solvers.hpp:45-52
    iter: int
    elapsed_s: float
    objective: float
    nnz: int
    matvecs: float
    extra: int


@dataclass
class SolverTrace:  # solvers.hpp:54-66
    solver: str
    samples: list = field(default_factory=list)
    status: StopReason = StopReason.iter_budget
    reached_target: bool = False
    final_objective: float = math.nan
    elapsed_s: float = 0.0
    total_matvecs: float = 0.0
    total_pcg_iterations: int = 0
    newton_steps: int = 0
    time_to_target: float = math.inf
    matvecs_to_target: float = math.inf
    iterations: int = 0
    path: int = 0  # l1b_summary.path: which kernels ran (L1B_RAN_* flags)

    def ran(self, name: str) -> bool:
        """Did the solve run the kernel family `name` (N.RAN keys, e.g. "pcdm_pair")?"""
        return bool(self.path & N.RAN[name])

    def objectives(self) -> np.ndarray:
        return np.array([s.objective for s in self.samples])

    def iters(self) -> np.ndarray:
        return np.array([s.iter for s in self.samples], dtype=np.int64)


@dataclass
class SparseSolution:  # solution.hpp:13-33
    n: int
    support: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return len(self.support)

    def dense(self) -> np.ndarray:
        x = np.zeros(self.n)
        x[self.support] = self.values
        return x

    def norm1(self) -> float:
        return float(np.sum(np.abs(self.values)))


@dataclass
class CertificateReport:  # instance.hpp:58-63
    max_support_violation: float
    max_offsupport_violation: float
    threshold: float
    passed: bool


def _ext_stream(inst):
    import torch

    if inst._ext is None:
        inst._ext = torch.cuda.ExternalStream(inst.stream)
    return inst._ext


class _Ordered:
    """Orders library work on the problem's stream after the caller's current
    torch stream (inputs ready) and the caller's stream after it (outputs
    ready) -- the C ABI only promises ordering on its own stream."""

    def __init__(self, inst):
        self.inst = inst

    def __enter__(self):
        import torch

        _ext_stream(self.inst).wait_stream(torch.cuda.current_stream())

    def __exit__(self, *a):
        import torch

        torch.cuda.current_stream().wait_stream(_ext_stream(self.inst))


class DeviceOperator:
    """LinearOperator view of a problem's A on the GPU (linops.hpp:139-155).

    ``path="sparse"`` runs the CSR/CSC SpMV kernels, ``path="sweep"`` the
    matrix-free stage sweeps (bit-exact with OperatorSpec::apply)."""

    def __init__(self, inst: "ProblemInstance"):
        self._inst = inst

    def rows(self) -> int:
        return self._inst.m

    def cols(self) -> int:
        return self._inst.n

    def _path(self, path):
        return {"sparse": N.PATH_SPARSE, "sweep": N.PATH_SWEEP, "fused": N.PATH_FUSED}[path]

    def apply(self, x, out=None, path: str = "sparse"):
        import torch

        if x.shape != (self.cols(),):
            raise ValueError(f"OperatorSpec::apply: expected length {self.cols()}, got {tuple(x.shape)}")
        out = torch.empty(self.rows(), dtype=torch.float64, device=x.device) if out is None else out
        with _Ordered(self._inst):
            N.check(_lib().l1b_apply(self._inst._h, self._path(path), _dptr(x), _dptr(out)))
        return out

    def apply_transpose(self, y, out=None, path: str = "sparse"):
        import torch

        if y.shape != (self.rows(),):
            raise ValueError(f"OperatorSpec::apply_transpose: expected length {self.rows()}, got {tuple(y.shape)}")
        out = torch.empty(self.cols(), dtype=torch.float64, device=y.device) if out is None else out
        with _Ordered(self._inst):
            N.check(_lib().l1b_apply_transpose(self._inst._h, self._path(path), _dptr(y), _dptr(out)))
        return out

    def apply_gram_inverse(self, v, out=None):
        import torch

        out = torch.empty(self.cols(), dtype=torch.float64, device=v.device) if out is None else out
        with _Ordered(self._inst):
            N.check(_lib().l1b_gram_inverse(self._inst._h, _dptr(v), _dptr(out)))
        return out

    def gram_diagonal(self, device="cuda"):
        import torch

        out = torch.empty(self.cols(), dtype=torch.float64, device=device)
        with _Ordered(self._inst):
            N.check(_lib().l1b_gram_diagonal(self._inst._h, _dptr(out)))
        return out

    def gram_lmax(self) -> float:
        return self._inst.info.gram_lmax

    def estimate_gram_lmax(self, iters: int = 30, seed: int = 0) -> float:
        """estimate_gram_lmax(op, iters, seed) (linops.hpp:283): power iteration."""
        out = C.c_double()
        N.check(_lib().l1b_estimate_gram_lmax(self._inst._h, int(iters), int(seed), C.byref(out)))
        return float(out.value)

    def csr(self):
        """Rows of A exactly as OperatorSpec::row (linops.cpp:597-619)."""
        info = self._inst.materialize()
        ptr = np.zeros(self.rows() + 1, dtype=np.uint64)
        idx = np.empty(max(info.nnz, 1), dtype=np.uint32)
        val = np.empty(max(info.nnz, 1))
        N.check(_lib().l1b_export_csr(self._inst._h, _ptr(ptr, _u64p), _ptr(idx, _u32p), _ptr(val, _f64p)))
        return ptr, idx[: info.nnz], val[: info.nnz]

    def csc(self):
        """Columns of A exactly as OperatorSpec::column (linops.cpp:566-595)."""
        info = self._inst.materialize()
        ptr = np.zeros(self.cols() + 1, dtype=np.uint64)
        idx = np.empty(max(info.nnz, 1), dtype=np.uint32)
        val = np.empty(max(info.nnz, 1))
        N.check(_lib().l1b_export_csc(self._inst._h, _ptr(ptr, _u64p), _ptr(idx, _u32p), _ptr(val, _f64p)))
        return ptr, idx[: info.nnz], val[: info.nnz]


class ProblemInstance:
    """Device-resident instance (instance.hpp:36-52): operator + b + tau + x*."""

    def __init__(self, handle):
        self._h = handle
        self._ext = None
        self.info = N.ProblemInfo()
        N.check(_lib().l1b_problem_info_get(self._h, C.byref(self.info)))

    @property
    def op(self) -> DeviceOperator:
        # a fresh view per access: a stored one would make instance <-> operator
        # a reference cycle, and `del inst` would not free the device buffers
        return DeviceOperator(self)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                _lib().l1b_problem_free(h)
            except Exception:
                pass

    def materialize(self) -> N.ProblemInfo:
        """Build the CSR/CSC copy of A (if lazy) and refresh ``info``."""
        N.check(_lib().l1b_problem_materialize(self._h))
        N.check(_lib().l1b_problem_info_get(self._h, C.byref(self.info)))
        return self.info

    # -- reference accessors --------------------------------------------------
    @property
    def m(self) -> int:
        return int(self.info.m)

    @property
    def n(self) -> int:
        return int(self.info.n)

    def rows(self) -> int:
        return self.m

    def cols(self) -> int:
        return self.n

    @property
    def tau(self) -> float:
        return float(self.info.tau)

    @property
    def noise_norm(self) -> float:
        return float(self.info.noise_norm)

    @property
    def cert_kappa(self) -> float:
        return float(self.info.cert_kappa)

    def objective_at_planted(self) -> float:  # instance.cpp:49-51
        return float(self.info.f_star)

    @property
    def b(self) -> np.ndarray:
        out = np.empty(self.m)
        N.check(_lib().l1b_problem_get_b(self._h, _ptr(out, _f64p)))
        return out

    def sigma(self) -> np.ndarray:
        out = np.empty(self.n)
        N.check(_lib().l1b_problem_get_sigma(self._h, _ptr(out, _f64p)))
        return out

    def b_window(self):
        """(lo, b[lo:hi]): a banded shard's b on the rows around its block (empty otherwise)."""
        a, e = C.c_uint64(), C.c_uint64()
        N.check(_lib().l1b_problem_get_b_window(self._h, C.byref(a), C.byref(e), None))
        out = np.empty(e.value - a.value)
        N.check(_lib().l1b_problem_get_b_window(self._h, C.byref(a), C.byref(e), _ptr(out, _f64p)))
        return int(a.value), out

    def set_rhs(self, b, b_win=None) -> None:
        """A new right-hand side for the resident operator (l1b_problem_set_rhs):
        host float64 arrays (pinned for full PCIe speed) in the layout of
        ``b`` / ``b_window()``."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        bw = None if b_win is None else np.ascontiguousarray(b_win, dtype=np.float64)
        N.check(_lib().l1b_problem_set_rhs(self._h, _ptr(b, _f64p), _ptr(bw, _f64p)))

    def sigma_window(self):
        """(begin, sigma[begin:end]): the sigma entries this problem holds (shards: a window)."""
        a, e = C.c_uint64(), C.c_uint64()
        N.check(_lib().l1b_problem_get_sigma_window(self._h, C.byref(a), C.byref(e), None))
        out = np.empty(e.value - a.value)
        N.check(_lib().l1b_problem_get_sigma_window(self._h, C.byref(a), C.byref(e), _ptr(out, _f64p)))
        return int(a.value), out

    @property
    def x_star(self) -> SparseSolution:
        s = int(self.info.s)
        sup = np.empty(max(s, 1), dtype=np.uint32)
        val = np.empty(max(s, 1))
        N.check(_lib().l1b_problem_get_xstar(self._h, _ptr(sup, _u32p), _ptr(val, _f64p)))
        return SparseSolution(self.n, sup[:s], val[:s])

    def stages(self, right: bool = True):
        """[(offset, theta)] of the right (G) or left (G~) factor."""
        cnt = C.c_uint32()
        N.check(_lib().l1b_problem_get_stages(self._h, int(right), C.byref(cnt), None, None))
        k = int(cnt.value)
        off = np.empty(max(k, 1), dtype=np.int32)
        th = np.empty(max(k, 1))
        N.check(_lib().l1b_problem_get_stages(self._h, int(right), C.byref(cnt),
                                               off.ctypes.data_as(C.POINTER(C.c_int32)), _ptr(th, _f64p)))
        return [(int(off[i]), float(th[i])) for i in range(k)]

    def perm(self, which: int) -> Optional[np.ndarray]:
        """P1 (which=1) / P2 (which=2) as an m-entry map, None for the identity."""
        ident = C.c_int()
        out = np.empty(self.m, dtype=np.uint32)
        N.check(_lib().l1b_problem_get_perm(self._h, which, C.byref(ident), _ptr(out, _u32p)))
        return None if ident.value else out

    @property
    def stream(self) -> int:
        return int(_lib().l1b_problem_stream(self._h) or 0)

    def set_stream(self, stream_ptr: int):
        N.check(_lib().l1b_problem_set_stream(self._h, stream_ptr))
        self._ext = None

    # -- constructors ---------------------------------------------------------
    @classmethod
    def from_host(cls, m, n, right_stages, sigma, b, tau, x_support=(), x_values=(),
                  left_stages=(), p1=None, p2=None, device: int = 0) -> "ProblemInstance":
        """Upload an instance described on the host (e.g. one the reference
        generated): stages as (offset, theta) pairs in OperatorSpec order."""
        ro = np.array([s[0] for s in right_stages], dtype=np.int32)
        rt = np.array([s[1] for s in right_stages], dtype=np.float64)
        lo = np.array([s[0] for s in left_stages], dtype=np.int32)
        lt = np.array([s[1] for s in left_stages], dtype=np.float64)
        sig = np.ascontiguousarray(sigma, dtype=np.float64)
        bb = np.ascontiguousarray(b, dtype=np.float64)
        if sig.shape != (n,) or bb.shape != (m,):
            raise ValueError("ProblemInstance.from_host: sigma / b size mismatch")
        p1a = None if p1 is None else np.ascontiguousarray(p1, dtype=np.uint32)
        p2a = None if p2 is None else np.ascontiguousarray(p2, dtype=np.uint32)
        d = N.OperatorDesc(m, n, len(ro), _ptr(ro, C.POINTER(C.c_int32)), _ptr(rt, _f64p), len(lo),
                           _ptr(lo, C.POINTER(C.c_int32)), _ptr(lt, _f64p), _ptr(p1a, _u32p),
                           _ptr(p2a, _u32p), _ptr(sig, _f64p))
        sup = np.ascontiguousarray(x_support, dtype=np.uint32)
        val = np.ascontiguousarray(x_values, dtype=np.float64)
        h = C.c_void_p()
        N.check(_lib().l1b_problem_create(device, C.byref(d), float(tau), _ptr(bb, _f64p),
                                          _ptr(sup, _u32p), _ptr(val, _f64p), len(sup), C.byref(h)))
        return cls(h)


def build_instance(n: int, m_ratio: float = 2.0, stages: int = 1, left_stages: int = 0,
                   permute: bool = False, q: Optional[int] = 1, shift: float = 0.1,
                   alternating: Optional[tuple] = None, sigma: Optional[np.ndarray] = None,
                   gamma: float = 10.0, s_divisor: int = 128, tau: float = 1.0,
                   theta: float = 0.6283185307179586, seed: int = 1, job_index: int = 0,
                   fill_bound: float = 0.9, device: int = 0, lazy_sparse: bool = False,
                   solution: str = "uniform", s1_fraction: float = 0.5, value_a: float = -1e4,
                   value_b: float = 1e-1, shard: Optional[tuple] = None) -> ProblemInstance:
    """``build_instance(cfg, enumerate_jobs(cfg)[job_index])`` for a single-job
    ExperimentConfig (bench.cpp:216-316), generated on the GPU.  ``sigma`` gives
    an explicit spectrum (Spectrum::from_values), ``alternating=(odd, even)`` the
    alternating one, otherwise uniform in (0, 10^q] + shift.  ``solution`` is the
    SolutionRule kind (bench.hpp:25-32): "uniform" (default), "spectral"
    (spectral_sparse_solution, s1_fraction) or "two_value" (value_a, value_b).
    ``shard=(rank, world)`` builds only that rank's row block of the default
    even split (banded operators)."""
    sig = None
    g = N.GenDesc()
    g.n, g.m_ratio, g.stages, g.left_stages, g.permute = n, m_ratio, stages, left_stages, int(permute)
    if sigma is not None:
        sig = np.ascontiguousarray(sigma, dtype=np.float64)
        if sig.shape != (n,):
            raise ValueError("Spectrum: realized value count mismatch")
        g.spectrum_kind, g.sigma_explicit = N.SPECTRUM_EXPLICIT, _ptr(sig, _f64p)
    elif alternating is not None:
        g.spectrum_kind, g.odd_value, g.even_value = N.SPECTRUM_ALTERNATING, *alternating
    else:
        g.spectrum_kind, g.q = N.SPECTRUM_UNIFORM_Q, int(q)
    g.shift, g.gamma, g.s_divisor, g.tau, g.theta = shift, gamma, s_divisor, tau, theta
    g.seed, g.job_index, g.fill_bound = seed, job_index, fill_bound
    g.lazy_sparse = int(lazy_sparse)
    kinds = {"uniform": N.SOLUTION_UNIFORM, "spectral": N.SOLUTION_SPECTRAL, "two_value": N.SOLUTION_TWO_VALUE}
    if solution not in kinds:
        raise ValueError(f"SolutionRule: unknown kind '{solution}'")
    g.solution_kind, g.s1_fraction, g.value_a, g.value_b = kinds[solution], s1_fraction, value_a, value_b
    h = C.c_void_p()
    sh = None if shard is None else N.ShardDesc(int(shard[0]), int(shard[1]), 0, 0)
    N.check(_lib().l1b_generate(device, C.byref(g), None if sh is None else C.byref(sh), C.byref(h)))
    return ProblemInstance(h)


# -- instance files and traces (serialize.cpp:182-294) --------------------------
_L1I_MAGIC = b"L1BINST\x01"


def save_instance(inst: ProblemInstance, path: str) -> None:
    """save_instance (serialize.cpp:182-219): magic, u64 header length, the JSON
    header (operator description, tau, ||e||, cert_kappa, |x*|), b as raw
    little-endian doubles, then x* as (u64 index, double) pairs.  The spectrum
    is written as its realised values (the reference's own reader takes them
    back bit for bit)."""
    import json
    import struct

    def perm_json(which):
        mp = inst.perm(which)
        return {"kind": "identity"} if mp is None else {"kind": "explicit", "map": mp.tolist()}

    op = {"version": 1, "m": inst.m, "n": inst.n,
          "spectrum": {"kind": "explicit", "values": inst.sigma().tolist()},
          "right_stages": [{"kind": "paired", "offset": o, "theta": t} for o, t in inst.stages(True)],
          "left_stages": [{"kind": "paired", "offset": o, "theta": t} for o, t in inst.stages(False)],
          "p1": perm_json(1), "p2": perm_json(2)}
    xs = inst.x_star
    header = {"version": 1, "kind": "tall", "m": inst.m, "n": inst.n, "tau": inst.tau,
              "noise_norm": inst.noise_norm, "cert_kappa": inst.cert_kappa, "x_nnz": len(xs.support),
              "op": op}
    head = json.dumps(header, separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(_L1I_MAGIC)
        f.write(struct.pack("<Q", len(head)))
        f.write(head)
        f.write(np.ascontiguousarray(inst.b, dtype="<f8").tobytes())
        rec = np.empty(len(xs.support), dtype=[("i", "<u8"), ("v", "<f8")])
        rec["i"], rec["v"] = xs.support, xs.values
        f.write(rec.tobytes())


def load_instance(path: str, device: int = 0) -> ProblemInstance:
    """load_instance (serialize.cpp:221-281) onto the device: tall instances
    with paired stages; spectrum explicit / uniform (realised values, or the
    seeded draws) / alternating; permutations identity / seeded / explicit."""
    import json
    import struct

    with open(path, "rb") as f:
        if f.read(8) != _L1I_MAGIC:
            raise RuntimeError(f"load_instance: '{path}' is not an instance file")
        (hl,) = struct.unpack("<Q", f.read(8))
        header = json.loads(f.read(hl).decode())
        if header.get("kind") != "tall":
            raise N.L1bUnsupported("load_instance: wide (IGen2) instances are out of scope")
        m, n = int(header["m"]), int(header["n"])
        b = np.frombuffer(f.read(8 * m), dtype="<f8").astype(np.float64)
        s = int(header["x_nnz"])
        rec = np.frombuffer(f.read(16 * s), dtype=[("i", "<u8"), ("v", "<f8")])
        if len(b) != m or len(rec) != s:
            raise RuntimeError(f"load_instance: truncated file '{path}'")
    op = header["op"]
    sp = op["spectrum"]
    if sp["kind"] == "explicit" or (sp["kind"] == "uniform" and "values" in sp):
        sigma = np.asarray(sp["values"], dtype=np.float64)
    elif sp["kind"] == "uniform":
        sigma = realize_spectrum_uniform(n, sp["lo"], sp["hi"], sp["shift"], sp["seed"])
    elif sp["kind"] == "alternating":
        sigma = np.where(np.arange(n) % 2 == 0, float(sp["odd"]), float(sp["even"]))
    else:
        raise ValueError(f"spectrum_from_json: unknown spectrum kind '{sp['kind']}'")

    def stages(lst):
        out = []
        for st in lst:
            if st["kind"] != "paired":
                raise N.L1bUnsupported("load_instance: explicit rotation lists are out of scope")
            out.append((int(st["offset"]), float(st["theta"])))
        return out

    def perm(pj):
        if pj["kind"] == "identity":
            return None
        if pj["kind"] == "seeded":
            return realize_permutation(m, int(pj["seed"]))
        if pj["kind"] == "explicit":
            return np.asarray(pj["map"], dtype=np.uint32)
        raise ValueError(f"perm_from_json: unknown permutation kind '{pj['kind']}'")

    inst = ProblemInstance.from_host(m, n, stages(op["right_stages"]), sigma, b, float(header["tau"]),
                                     rec["i"].astype(np.uint32), rec["v"].copy(),
                                     left_stages=stages(op["left_stages"]), p1=perm(op["p1"]),
                                     p2=perm(op["p2"]), device=device)
    N.check(_lib().l1b_problem_set_meta(inst._h, float(header["noise_norm"]), float(header["cert_kappa"])))
    N.check(_lib().l1b_problem_info_get(inst._h, C.byref(inst.info)))
    return inst


def write_trace_csv(trace: SolverTrace, path: str) -> None:
    """write_trace_csv (serialize.cpp:283-294), same columns and formats."""
    with open(path, "w") as f:
        f.write("solver,iter,elapsed_s,objective,nnz_x,matvecs,extra\n")
        for s in trace.samples:
            f.write("%s,%d,%.6f,%.17g,%d,%.3f,%d\n" % (trace.solver, s.iter, s.elapsed_s, s.objective,
                                                       s.nnz, s.matvecs, s.extra))


def verify_optimality(inst: ProblemInstance, tol: float) -> CertificateReport:
    c = N.Cert()
    N.check(_lib().l1b_verify_optimality(inst._h, float(tol), C.byref(c)))
    return CertificateReport(c.max_support_violation, c.max_offsupport_violation, c.threshold, bool(c.pass_))


def objective(inst: ProblemInstance, x) -> float:
    """tau*||x||_1 + 1/2*||A x - b||^2 for a device vector x (solvers.cpp:145-151)."""
    f = C.c_double()
    with _Ordered(inst):
        N.check(_lib().l1b_objective(inst._h, _dptr(x), C.byref(f)))
    return float(f.value)


def smoothed_hessvec(inst: ProblemInstance, x, mu: float, v):
    """smoothed_hessvec (solvers.cpp:188-200) as newton_cg_run's PCG forms it
    (:536-540): A^T A v + tau d2psi_mu(x) v, on device vectors; returns a new
    CUDA float64 tensor."""
    import torch

    out = torch.empty(inst.n, dtype=torch.float64, device=x.device)
    with _Ordered(inst):
        N.check(_lib().l1b_smoothed_hessvec(inst._h, float(mu), _dptr(x), _dptr(v), _dptr(out)))
    return out


def soft_threshold(v: float, t: float) -> float:  # solvers.cpp:153-157 (host scalar helper)
    if v > t:
        return v - t
    if v < -t:
        return v + t
    return 0.0


def cd_damping(omega: int, varpi: int, n: int) -> float:  # solvers.cpp:266-270
    if n <= 1 or varpi <= 1:
        return 1.0
    return 1.0 + float(omega - 1) * float(varpi - 1) / float(n - 1)


def _trace_from(name: str, samples, k: int, s: N.Summary) -> SolverTrace:
    tr = SolverTrace(name)
    tr.samples = [TraceSample(int(samples[i].iter), samples[i].elapsed_s, samples[i].objective,
                              int(samples[i].nnz), samples[i].matvecs, int(samples[i].extra))
                  for i in range(k)]
    tr.status = StopReason(s.status)
    tr.reached_target = bool(s.reached_target)
    tr.final_objective = s.final_objective
    tr.elapsed_s = s.elapsed_s
    tr.total_matvecs = s.total_matvecs
    tr.total_pcg_iterations = int(s.total_pcg_iterations)
    tr.newton_steps = int(s.newton_steps)
    tr.time_to_target = s.time_to_target
    tr.matvecs_to_target = s.matvecs_to_target
    tr.iterations = int(s.iterations)
    tr.path = int(s.path)
    return tr


def run_solver(inst: ProblemInstance, cfg: SolverConfig, x_out: Optional[np.ndarray] = None,
               cap: int = 1 << 20) -> SolverTrace:
    """run_solver (solvers.cpp:574-581).  When ``x_out`` (float64[n]) is given
    the final iterate is copied into it, like the reference's x_out pointer."""
    c = cfg.to_c()
    # trace capacity: every iteration up to 1000, then every 10th (solvers.cpp:368-371)
    # for ista/fista; one sample per sweep / Newton step otherwise
    if cfg.id in ("fista", "ista"):
        need = min(cfg.max_iters, 1000) + max(0, cfg.max_iters - 1000) // 10 + 3
    else:
        need = cfg.max_iters + 2
    cap = max(1, min(cap, need))
    samples = (N.Sample * cap)()
    summ = N.Summary()
    if x_out is not None:
        if x_out.dtype != np.float64 or x_out.shape != (inst.n,) or not x_out.flags.c_contiguous:
            raise ValueError("x_out must be a contiguous float64 array of length n")
    N.check(_lib().l1b_solve(inst._h, C.byref(c), samples, cap, C.byref(summ), _ptr(x_out, _f64p), None))
    name = {"cd": "cd", "newton_cg": "newton_cg", "fista": "fista", "ista": "ista", "pcdm": "pcdm"}[cfg.id]
    return _trace_from(name, samples, min(int(summ.n_samples), cap), summ)


def _with_id(cfg: SolverConfig, ident: str) -> SolverConfig:
    from dataclasses import replace

    return replace(cfg, id=ident)


def fista_run(inst, cfg: SolverConfig, x_out=None) -> SolverTrace:
    return run_solver(inst, _with_id(cfg, "fista"), x_out)


def ista_run(inst, cfg: SolverConfig, x_out=None) -> SolverTrace:
    return run_solver(inst, _with_id(cfg, "ista"), x_out)


def coordinate_descent_run(inst, cfg: SolverConfig, x_out=None) -> SolverTrace:
    return run_solver(inst, _with_id(cfg, "cd"), x_out)


def newton_cg_run(inst, cfg: SolverConfig, x_out=None) -> SolverTrace:
    return run_solver(inst, _with_id(cfg, "newton_cg"), x_out)


def pcdm_run(inst, cfg: SolverConfig, x_out=None) -> SolverTrace:
    return run_solver(inst, _with_id(cfg, "pcdm"), x_out)


def known_solver(ident: str) -> bool:  # solvers.cpp:570-572 (+ pcdm)
    return ident in SolverConfig._IDS


def fp64_peak(device: int = 0) -> float:
    """Dense FP64 fma throughput of the GPU in TFLOP/s (l1b_fp64_peak)."""
    v = C.c_double()
    N.check(_lib().l1b_fp64_peak(int(device), C.byref(v)))
    return float(v.value)


class Session:
    """Stepping handle over the device-resident FISTA/ISTA loop (bench.py)."""

    def __init__(self, inst: ProblemInstance, cfg: SolverConfig):
        self.inst = inst
        c = cfg.to_c()
        self._s = C.c_void_p()
        N.check(_lib().l1b_session_begin(inst._h, C.byref(c), C.byref(self._s)))
        self._name = cfg.id

    def step(self, iters: int):
        N.check(_lib().l1b_session_step(self._s, int(iters)))

    def profile(self, iters: int):
        ms = (C.c_double * 2)()
        N.check(_lib().l1b_session_profile(self._s, int(iters), ms, 2))
        return [ms[0], ms[1]]

    def kernel_mode(self) -> int:
        """N.KMODE_* of the FISTA kernels this session runs."""
        m = C.c_int()
        N.check(_lib().l1b_session_kernel_mode(self._s, C.byref(m)))
        return int(m.value)

    def tile_geometry(self):
        """(iterations per launch, entries per tile, entries kept per tile) of a
        tile-kernel session (N.KMODE_RECOMPUTE_TILE); zeros otherwise."""
        k, span, valid = C.c_int(), C.c_int64(), C.c_int64()
        N.check(_lib().l1b_session_tile_geometry(self._s, C.byref(k), C.byref(span), C.byref(valid)))
        return int(k.value), int(span.value), int(valid.value)

    def tile_plan(self, iters: int):
        """Lengths of the tile launches step(iters) / profile(iters) take."""
        cap = max(1, int(iters) // 6 + 1)
        ks, cnt = (C.c_int * cap)(), C.c_int()
        N.check(_lib().l1b_session_tile_plan(self._s, int(iters), ks, cap, C.byref(cnt)))
        return [int(ks[i]) for i in range(min(cap, cnt.value))]

    def sync(self):
        stopped, k = C.c_int(), C.c_uint64()
        N.check(_lib().l1b_session_sync(self._s, C.byref(stopped), C.byref(k)))
        return bool(stopped.value), int(k.value)

    def restart(self):
        """x_0 = 0 and iteration 0 again, on the same buffers (serving a new b)."""
        N.check(_lib().l1b_session_restart(self._s))

    def read(self, x_out: Optional[np.ndarray] = None, cap: int = 1 << 16) -> SolverTrace:
        """Shard sessions: the trace and own x so far, without ending."""
        samples = (N.Sample * cap)()
        summ = N.Summary()
        N.check(_lib().l1b_session_read(self._s, samples, cap, C.byref(summ), _ptr(x_out, _f64p)))
        return _trace_from(self._name, samples, min(int(summ.n_samples), cap), summ)

    def end(self, x_out: Optional[np.ndarray] = None, cap: int = 1 << 16) -> SolverTrace:
        samples = (N.Sample * cap)()
        summ = N.Summary()
        s, self._s = self._s, None
        N.check(_lib().l1b_session_end(s, samples, cap, C.byref(summ), _ptr(x_out, _f64p)))
        return _trace_from(self._name, samples, min(int(summ.n_samples), cap), summ)


def launch_count() -> int:
    return int(_lib().l1b_launch_count())
