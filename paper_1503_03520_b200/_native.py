"""ctypes binding of libl1b.so (include/l1b.h).

The CUDA library is the only implementation: if ``lib/libl1b.so`` is missing or
no CUDA device is visible, every compute entry point raises -- there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libl1b.so")

u64, u32, i32, f64 = C.c_uint64, C.c_uint32, C.c_int32, C.c_double
P = C.POINTER
vp = C.c_void_p

# status codes (l1b.h)
OK, EINVAL, ERUNTIME, ELOGIC, ECUDA, ENOMEM, EUNSUPPORTED, ENCCL = range(8)

ISTA, FISTA, CD, NEWTON_CG, PCDM = range(5)
TARGET_REACHED, ITER_BUDGET, TIME_BUDGET = range(3)
PATH_SPARSE, PATH_SWEEP, PATH_FUSED = 0, 1, 2
OP_AUTO, OP_SPARSE, OP_MATRIX_FREE = 0, 1, 2
SPECTRUM_UNIFORM_Q, SPECTRUM_ALTERNATING, SPECTRUM_EXPLICIT = range(3)
SOLUTION_UNIFORM, SOLUTION_SPECTRAL, SOLUTION_TWO_VALUE = range(3)


class OperatorDesc(C.Structure):
    _fields_ = [("m", u64), ("n", u64), ("n_right", u32), ("right_offset", P(i32)),
                ("right_theta", P(f64)), ("n_left", u32), ("left_offset", P(i32)),
                ("left_theta", P(f64)), ("p1", P(u32)), ("p2", P(u32)), ("sigma", P(f64))]


class GenDesc(C.Structure):
    _fields_ = [("n", u64), ("m_ratio", f64), ("stages", u32), ("left_stages", u32),
                ("permute", C.c_int), ("spectrum_kind", C.c_int), ("q", C.c_int), ("shift", f64),
                ("odd_value", f64), ("even_value", f64), ("sigma_explicit", P(f64)),
                ("gamma", f64), ("s_divisor", u64), ("tau", f64), ("theta", f64), ("seed", u64),
                ("job_index", u64), ("fill_bound", f64), ("lazy_sparse", C.c_int),
                ("solution_kind", C.c_int), ("s1_fraction", f64), ("value_a", f64), ("value_b", f64)]


class ShardDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("row_begin", u64), ("row_end", u64)]


class ProblemInfo(C.Structure):
    _fields_ = [("m", u64), ("n", u64), ("m_active", u64), ("nnz", u64), ("s", u64),
                ("tau", f64), ("noise_norm", f64), ("cert_kappa", f64), ("gram_lmax", f64),
                ("f_star", f64), ("device_bytes", u64), ("row_begin", u64), ("row_end", u64),
                ("col_begin", u64), ("col_end", u64), ("csr_lanes", C.c_int),
                ("csc_lanes", C.c_int), ("world", C.c_int), ("rank", C.c_int), ("halo", u64)]


# l1b_session_kernel_mode (include/l1b.h)
KMODE_SPARSE, KMODE_MATRIX_FREE_PAIR, KMODE_STORED_RESIDUAL = 0, 1, 2
KMODE_RECOMPUTE, KMODE_RECOMPUTE_TWO, KMODE_GENERAL_SHARD = 3, 4, 5
KMODE_RECOMPUTE_TILE = 6


class ShardBuffers(C.Structure):
    _fields_ = [("x_win", vp), ("r_y_win", vp), ("scal", vp), ("own", u64), ("halo", u64),
                ("single", C.c_int), ("x_bufs", vp * 4), ("r_bufs", vp * 3), ("x_halo", u64),
                ("r_halo", u64), ("lagged", C.c_int), ("x_nbufs", C.c_int), ("pairs", C.c_int),
                ("scal8", vp), ("general", C.c_int),
                ("g_full", vp),
                ("x_full", vp), ("n_pad", u64), ("col_begin", u64), ("col_count", u64)]


class Cert(C.Structure):
    _fields_ = [("max_support_violation", f64), ("max_offsupport_violation", f64),
                ("threshold", f64), ("pass_", C.c_int)]


class SolverCfg(C.Structure):
    _fields_ = [("solver", C.c_int), ("max_iters", u64), ("max_seconds", f64),
                ("has_target", C.c_int), ("target", f64), ("mu", f64), ("eta", f64),
                ("pcg_max_iters", u64), ("ls_max_backtracks", u64), ("grad_tol_rel", f64),
                ("l_fixed", f64), ("varpi", u64), ("omega", u64), ("seed", u64), ("block", u64),
                ("op", C.c_int), ("l_policy", C.c_int), ("arith", C.c_int)]


class Sample(C.Structure):
    _fields_ = [("iter", u64), ("elapsed_s", f64), ("objective", f64), ("nnz", u64),
                ("matvecs", f64), ("extra", u64)]


class Summary(C.Structure):
    _fields_ = [("status", C.c_int), ("reached_target", C.c_int), ("final_objective", f64),
                ("elapsed_s", f64), ("total_matvecs", f64), ("total_pcg_iterations", u64),
                ("newton_steps", u64), ("time_to_target", f64), ("matvecs_to_target", f64),
                ("n_samples", u64), ("iterations", u64), ("path", u32)]


# l1b_summary.path flags (include/l1b.h L1B_RAN_*)
RAN = {name: 1 << i for i, name in enumerate(
    ["fista_sparse", "fista_mf_pair", "fista_stored", "fista_recompute", "fista_two_iter", "fista_loop",
     "fma", "pcdm_pair", "pcdm_plan", "pcdm_direct", "pcg_pair", "pcg_loop", "pcg_kernels", "host_led",
     "fista_tile"])}


# every symbol include/l1b.h declares: (name, restype, argtypes)
SIGNATURES = [
    ("l1b_abi_version", C.c_int, []),
    ("l1b_last_error", C.c_char_p, []),
    ("l1b_launch_count", u64, []),
    ("l1b_mix_seed", u64, [u64, u64]),
    ("l1b_realize_permutation", C.c_int, [u64, u64, P(u32)]),
    ("l1b_device_realize_permutation", C.c_int, [C.c_int, u64, u64, P(u32), P(C.c_int)]),
    ("l1b_realize_spectrum_uniform", C.c_int, [u64, f64, f64, f64, u64, P(f64)]),
    ("l1b_device_uniform_draws", C.c_int, [C.c_int, u64, u64, f64, f64, C.c_int, f64, u64, u64, u32,
                                           vp, P(f64), P(f64), P(C.c_int)]),
    ("l1b_device_index_stream", C.c_int, [C.c_int, u64, u64, P(u64), u32, vp, P(u64)]),
    ("l1b_mt_draws_after_jump", C.c_int, [u64, u32, u64, P(u64)]),
    ("l1b_mt_draws_after_chunk_jump", C.c_int, [u64, u64, u64, P(u64)]),
    ("l1b_uniform_sparse_solution", C.c_int, [u64, u64, f64, u64, P(u32), P(f64)]),
    ("l1b_device_uniform_sparse_solution", C.c_int, [C.c_int, u64, u64, f64, u64, P(u32), P(f64), P(C.c_int)]),
    ("l1b_generate", C.c_int, [C.c_int, P(GenDesc), P(ShardDesc), P(vp)]),
    ("l1b_problem_create", C.c_int, [C.c_int, P(OperatorDesc), f64, P(f64), P(u32), P(f64), u64,
                                     P(vp)]),
    ("l1b_problem_free", C.c_int, [vp]),
    ("l1b_problem_materialize", C.c_int, [vp]),
    ("l1b_problem_info_get", C.c_int, [vp, P(ProblemInfo)]),
    ("l1b_problem_get_b", C.c_int, [vp, P(f64)]),
    ("l1b_problem_get_sigma", C.c_int, [vp, P(f64)]),
    ("l1b_problem_get_sigma_window", C.c_int, [vp, P(u64), P(u64), P(f64)]),
    ("l1b_problem_get_b_window", C.c_int, [vp, P(u64), P(u64), P(f64)]),
    ("l1b_problem_set_rhs", C.c_int, [vp, P(f64), P(f64)]),
    ("l1b_smoothed_hessvec", C.c_int, [vp, f64, vp, vp, vp]),
    ("l1b_problem_set_meta", C.c_int, [vp, f64, f64]),
    ("l1b_problem_get_stages", C.c_int, [vp, C.c_int, P(u32), P(C.c_int32), P(f64)]),
    ("l1b_problem_get_perm", C.c_int, [vp, C.c_int, P(C.c_int), P(u32)]),
    ("l1b_problem_get_xstar", C.c_int, [vp, P(u32), P(f64)]),
    ("l1b_problem_stream", vp, [vp]),
    ("l1b_problem_set_stream", C.c_int, [vp, vp]),
    ("l1b_apply", C.c_int, [vp, C.c_int, vp, vp]),
    ("l1b_apply_transpose", C.c_int, [vp, C.c_int, vp, vp]),
    ("l1b_gram_inverse", C.c_int, [vp, vp, vp]),
    ("l1b_gram_diagonal", C.c_int, [vp, vp]),
    ("l1b_estimate_gram_lmax", C.c_int, [vp, u64, u64, P(f64)]),
    ("l1b_export_csr", C.c_int, [vp, P(u64), P(u32), P(f64)]),
    ("l1b_export_csc", C.c_int, [vp, P(u64), P(u32), P(f64)]),
    ("l1b_objective", C.c_int, [vp, vp, P(f64)]),
    ("l1b_verify_optimality", C.c_int, [vp, f64, P(Cert)]),
    ("l1b_solver_cfg_default", None, [P(SolverCfg)]),
    ("l1b_solve", C.c_int, [vp, P(SolverCfg), P(Sample), u64, P(Summary), P(f64), vp]),
    ("l1b_session_begin", C.c_int, [vp, P(SolverCfg), P(vp)]),
    ("l1b_session_step", C.c_int, [vp, u64]),
    ("l1b_session_profile", C.c_int, [vp, u64, P(f64), C.c_int]),
    ("l1b_session_sync", C.c_int, [vp, P(C.c_int), P(u64)]),
    ("l1b_session_end", C.c_int, [vp, P(Sample), u64, P(Summary), P(f64)]),
    ("l1b_session_buffers", C.c_int, [vp, P(ShardBuffers)]),
    ("l1b_session_k1", C.c_int, [vp]),
    ("l1b_session_k2", C.c_int, [vp]),
    ("l1b_session_finalize", C.c_int, [vp]),
    ("l1b_session_flush", C.c_int, [vp]),
    ("l1b_session_prox", C.c_int, [vp]),
    ("l1b_session_attach_peers", C.c_int, [vp, P(vp), u64, P(vp), u64]),
    ("l1b_session_export_x_ipc", C.c_int, [vp, vp]),
    ("l1b_session_attach_peers_ipc", C.c_int, [vp, vp, u64, vp, u64]),
    ("l1b_session_kernel_mode", C.c_int, [vp, P(C.c_int)]),
    ("l1b_session_tile_geometry", C.c_int, [vp, P(C.c_int), P(C.c_int64), P(C.c_int64)]),
    ("l1b_session_tile_plan", C.c_int, [vp, C.c_uint64, P(C.c_int), C.c_int, P(C.c_int)]),
    ("l1b_tile_plan", C.c_int, [C.c_int, C.c_uint64, P(C.c_int), C.c_int, P(C.c_int)]),
    ("l1b_fp64_peak", C.c_int, [C.c_int, P(f64)]),
    ("l1b_session_restart", C.c_int, [vp]),
    ("l1b_session_read", C.c_int, [vp, P(Sample), u64, P(Summary), P(f64)]),
    ("l1b_nccl_get_unique_id", C.c_int, [vp]),
    ("l1b_nccl_version", C.c_int, [P(C.c_int)]),
    ("l1b_session_attach_nccl", C.c_int, [vp, vp, C.c_int, C.c_int]),
    ("l1b_session_nccl_start", C.c_int, [vp]),
    ("l1b_session_nccl_steps", C.c_int, [vp, u64, C.c_int, P(f64)]),
    ("l1b_session_nccl_finish", C.c_int, [vp]),
]


class L1bError(RuntimeError):
    """Device / library failure without a reference analogue (ECUDA, ENOMEM, ...)."""


class L1bLogicError(RuntimeError):
    """std::logic_error analogue."""


class L1bUnsupported(RuntimeError):
    pass


_lib = None


def load(path: str = LIB_PATH):
    """Load libl1b.so; raise loudly when it is absent (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (or `make -C paper_1503_03520_b200/csrc`)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.l1b_abi_version() != 1:
        raise ImportError("libl1b ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int):
    if rc == OK:
        return
    msg = (_lib.l1b_last_error() or b"").decode()
    if rc == EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == ERUNTIME:
        raise RuntimeError(msg)  # std::runtime_error
    if rc == ELOGIC:
        raise L1bLogicError(msg)
    if rc == EUNSUPPORTED:
        raise L1bUnsupported(msg)
    raise L1bError(f"[l1b status {rc}] {msg}")
