/*
 * l1b.h -- C ABI of the B200-native l1-least-squares hot path
 *          (min_x tau*||x||_1 + 1/2*||A x - b||^2, arXiv 1503.03520).
 *
 * Plain C: plain pointers, sizes and status codes; no torch or C++ types.
 * Implemented by libl1b.so (paper_1503_03520_b200/lib/), CUDA sm_100a only --
 * there is no CPU path behind any of these entry points.
 *
 * Each group below names the reference interface it replaces (paths relative
 * to /root/reference/proj).  The reference's C++ API throws; this ABI returns
 * a status code and keeps the exception text in l1b_last_error() (thread
 * local), so a host shim can rethrow the same exception type with the same
 * message:
 *   L1B_EINVAL  -> std::invalid_argument   (linops.cpp:13-18, solvers.cpp:133-143)
 *   L1B_ERUNTIME-> std::runtime_error      (solvers.cpp:36-40, 233, 244; linops.cpp:481)
 *   L1B_ELOGIC  -> std::logic_error        (linops.cpp:418-420)
 *   L1B_ECUDA / L1B_ENOMEM / L1B_ENCCL     -> device failures (no reference analogue)
 *
 * Ownership: every device buffer inside an l1b_problem belongs to the library;
 * host buffers passed in are read during the call only; host output buffers
 * belong to the caller.  Device-pointer arguments (d_*) must live on the
 * problem's device; work is ordered on the problem's stream
 * (l1b_problem_stream), calls that return host data synchronise it.
 */
#ifndef L1B_H
#define L1B_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define L1B_ABI_VERSION 1

enum l1b_status {
  L1B_OK = 0,
  L1B_EINVAL = 1,
  L1B_ERUNTIME = 2,
  L1B_ELOGIC = 3,
  L1B_ECUDA = 4,
  L1B_ENOMEM = 5,
  L1B_EUNSUPPORTED = 6,
  L1B_ENCCL = 7
};

int l1b_abi_version(void);
const char* l1b_last_error(void);

/* ------------------------------------------------------------------------ */
/* Host-side generator primitives (bit-exact std::mt19937_64 streams).
 * Replace: rng.hpp:19-45 (mix_seed, uniform_*), Permutation::realize
 * (linops.cpp:224-239), Spectrum::realize (linops.cpp:320-336),
 * uniform_sparse_solution (solution.cpp:47-75).                             */
uint64_t l1b_mix_seed(uint64_t seed, uint64_t salt);
int l1b_realize_permutation(uint64_t n, uint64_t seed, uint32_t* map_out);
/* The same on the device (k_solution.cu: the Fisher-Yates result from its
 * draws alone -- targets sorted, value chains by pointer jumping); the host
 * replay after a redrawn index (*on_device = 0).  n <= 2^32.               */
int l1b_device_realize_permutation(int device, uint64_t n, uint64_t seed, uint32_t* map_out, int* on_device);
int l1b_realize_spectrum_uniform(uint64_t n, double lo, double hi, double shift, uint64_t seed,
                                 double* sigma_out);
/* Device realisation of the per-entry streams (Spectrum::uniform,
 * linops.cpp:323-331, with spectrum = 1; the l1_subgradient fill,
 * instance.cpp:33-35, with spectrum = 0): draws [0, count) of
 * Rng(seed) as lo + (hi - lo) * uniform_unit (+ shift), cut into chunks
 * started by mt19937_64 jump-ahead (k_rng.cu).  Draws [win_lo, win_hi) go to
 * the device buffer d_out; vmin / vmax (host, optional) receive the min / max
 * over all draws; *exact = 0 when a spectrum draw would have been rejected
 * (the stream shifts: replay it with l1b_realize_spectrum_uniform).
 * Chunks hold >= 2^min_log2_chunk draws (at most 4096 chunks). */
int l1b_device_uniform_draws(int device, uint64_t seed, uint64_t count, double lo, double hi,
                             int spectrum, double shift, uint64_t win_lo, uint64_t win_hi,
                             uint32_t min_log2_chunk, double* d_out, double* vmin, double* vmax,
                             int* exact);
/* Device coordinate stream of the pair-local CD / PCDM path (k_rng.cu
 * mt_stream_indices): raw draws of Rng(seed) reduced like uniform_index(rng,
 * n) (rng.hpp:37-45), 0xffffffff where the reference would redraw, into the
 * device buffer d_out.  Drawn in npieces consecutive launches that continue the
 * saved generator state; each piece is rounded up to a multiple of 312 draws
 * (d_out needs room for them); *drawn receives the total.  n < 2^32. */
int l1b_device_index_stream(int device, uint64_t seed, uint64_t n, const uint64_t* piece_counts,
                            uint32_t npieces, uint32_t* d_out, uint64_t* drawn);
/* Host check of the jump polynomials: raw outputs 2^log2_jump ...
 * 2^log2_jump + count - 1 of std::mt19937_64(seed), reached by jumping. */
int l1b_mt_draws_after_jump(uint64_t seed, uint32_t log2_jump, uint64_t count, uint64_t* out);
/* The same through t^(chunk * 79872) mod P: the start of chunk `chunk` of a
 * coordinate stream (l1b_device_index_stream draws chunks of 312 x 256). */
int l1b_mt_draws_after_chunk_jump(uint64_t seed, uint64_t chunk, uint64_t count, uint64_t* out);
/* Returns s through *s_out; support (ascending) and values need capacity s. */
int l1b_uniform_sparse_solution(uint64_t n, uint64_t s, double gamma, uint64_t rng_seed,
                                uint32_t* support_out, double* values_out);
/* The same on the device (k_solution.cu: Floyd's sampling from the draws
 * alone -- first occurrences by a stable sort, chains by relaxation); the
 * host replay when a draw the reference redraws occurs (*on_device = 0).   */
int l1b_device_uniform_sparse_solution(int device, uint64_t n, uint64_t s, double gamma, uint64_t rng_seed,
                                       uint32_t* support_out, double* values_out, int* on_device);

/* ------------------------------------------------------------------------ */
/* Problem = device-resident instance: operator (sweep description + CSR/CSC
 * materialised on device) + b + tau + planted x*.
 * Replaces: OperatorSpec (linops.hpp:159-206) + finalize (linops.cpp:394-416),
 * ProblemInstance (instance.hpp:36-52), generate_instance (instance.cpp:53-89),
 * build_instance (bench.cpp:253-316).                                         */
typedef struct l1b_problem l1b_problem;

typedef struct {
  uint64_t m, n;
  uint32_t n_right;            /* right stages, in OperatorSpec::right_stages order */
  const int32_t* right_offset; /* 0 or 1 (paired stages only) */
  const double* right_theta;
  uint32_t n_left;
  const int32_t* left_offset;
  const double* left_theta;
  const uint32_t* p1;          /* m-entry map (Pv)[i] = v[map[i]]; NULL = identity */
  const uint32_t* p2;
  const double* sigma;         /* n realised singular values, all > 0 */
} l1b_operator_desc;

enum { L1B_SPECTRUM_UNIFORM_Q = 0, L1B_SPECTRUM_ALTERNATING = 1, L1B_SPECTRUM_EXPLICIT = 2 };
/* SolutionRule::Kind (bench.hpp:25-32): uniform_sparse_solution (OsGen), the
 * spectral one (solution.cpp:77-113, OsGen3) or two values on a uniform support */
enum { L1B_SOLUTION_UNIFORM = 0, L1B_SOLUTION_SPECTRAL = 1, L1B_SOLUTION_TWO_VALUE = 2 };

/* ExperimentConfig + InstanceJob for one job (bench.hpp:16-97). */
typedef struct {
  uint64_t n;
  double m_ratio;            /* m = llround(m_ratio * n), >= 1 */
  uint32_t stages;           /* right stages, offsets (stages-1-i)%2 */
  uint32_t left_stages;
  int permute;               /* seeded P1, P2 */
  int spectrum_kind;
  int q;                     /* uniform: draws in (0, 10^q], + shift */
  double shift;
  double odd_value, even_value;
  const double* sigma_explicit; /* L1B_SPECTRUM_EXPLICIT: n values */
  double gamma;              /* OsGen value bound */
  uint64_t s_divisor;        /* s = max(1, n / s_divisor) */
  double tau;
  double theta;
  uint64_t seed;             /* ExperimentConfig::seed */
  uint64_t job_index;        /* job.seed = mix_seed(seed, job_index) (bench.cpp:237) */
  double fill_bound;         /* FillPolicy::interior bound, 0.9 */
  int lazy_sparse;           /* 1: build the CSR/CSC copy of A only on first sparse use */
  int solution_kind;         /* L1B_SOLUTION_*; 0 = uniform (the default) */
  double s1_fraction;        /* spectral: share of s kept from the small end (0.5) */
  double value_a, value_b;   /* two_value: first half / rest of the support (-1e4, 0.1) */
} l1b_gen_desc;

/* Shard = contiguous block of A's nonempty rows [row_begin, row_end) of a
 * banded instance (identity P1/P2, no left stages: |col - row| <= #stages),
 * holding the matching column block [row_begin, row_end) of A^T.  Local
 * vectors carry `halo` = #stages entries on each side.  NULL shard = the whole
 * operator on one device.  row_end == 0 selects the default even split of
 * [0, n) for (rank, world).                                                  */
typedef struct {
  int rank, world;
  uint64_t row_begin, row_end;
} l1b_shard_desc;

int l1b_generate(int device, const l1b_gen_desc* gen, const l1b_shard_desc* shard,
                 l1b_problem** out);
/* Upload an instance described on the host.  The CSR/CSC copy of A is built
 * on the first call that needs it (sparse products, sparse FISTA, CD, pdNCG). */
int l1b_problem_create(int device, const l1b_operator_desc* op, double tau, const double* b_host,
                       const uint32_t* xstar_support, const double* xstar_values, uint64_t s,
                       l1b_problem** out);
int l1b_problem_free(l1b_problem* p);
/* Build the CSR/CSC copy of A now (otherwise built on first sparse use). */
int l1b_problem_materialize(l1b_problem* p);

typedef struct {
  uint64_t m, n;
  uint64_t m_active;      /* rows [m_active, m) of A are structurally empty */
  uint64_t nnz;           /* nnz(A) (this shard) */
  uint64_t s;             /* |supp x*| */
  double tau, noise_norm, cert_kappa, gram_lmax, f_star;
  uint64_t device_bytes;  /* HBM held by the problem */
  uint64_t row_begin, row_end, col_begin, col_end; /* shard ranges */
  int csr_lanes, csc_lanes; /* lines per warp tile in the SpMV kernels */
  int world, rank;          /* shard of a row-block partition (1, 0 = whole) */
  uint64_t halo;            /* x / r window overhang on each side (= #stages) */
} l1b_problem_info;

int l1b_problem_info_get(const l1b_problem* p, l1b_problem_info* out);
int l1b_problem_get_b(const l1b_problem* p, double* b_host);          /* m */
int l1b_problem_get_sigma(const l1b_problem* p, double* sigma_host);  /* n */
/* Row-block shards of banded operators keep b also on a window of rows around
 * their block ([*lo, *hi); the recomputing FISTA kernel rebuilds r there);
 * b_host (may be NULL) receives hi - lo entries.  *lo == *hi: no window.   */
int l1b_problem_get_b_window(const l1b_problem* p, uint64_t* lo, uint64_t* hi, double* b_host);
/* A new right-hand side for the resident operator (the instance metadata --
 * ||e||, f*, x* -- keeps describing the generated b): b_host holds m entries
 * (a row-block shard: its own rows, as l1b_problem_get_b returns them, plus
 * b_win_host with the window of l1b_problem_get_b_window when it has one).
 * The serving path of bench.py's multi-GPU e2e: operator resident in HBM,
 * b streamed from pinned host memory.                                       */
int l1b_problem_set_rhs(l1b_problem* p, const double* b_host, const double* b_win_host);
/* The sigma entries the problem holds: [*begin, *end) of the global sigma
 * (a row-block shard keeps its window plus the kernels' halos; a whole
 * problem all n).  sigma_host (may be NULL) receives end - begin entries.  */
int l1b_problem_get_sigma_window(const l1b_problem* p, uint64_t* begin, uint64_t* end,
                                 double* sigma_host);
int l1b_problem_get_xstar(const l1b_problem* p, uint32_t* support, double* values);
/* The operator description back (save_instance, serialize.cpp:148-163): stage
 * offsets / angles of the right (right = 1) or left factor (count first, arrays
 * may be NULL), and P1 (which = 1) / P2 (which = 2) as an m-entry map unless
 * *is_identity.                                                             */
int l1b_problem_get_stages(const l1b_problem* p, int right, uint32_t* count, int32_t* offsets,
                           double* thetas);
int l1b_problem_get_perm(const l1b_problem* p, int which, int* is_identity, uint32_t* map);
/* Instance metadata carried by instance files (serialize.cpp:182-219):
 * ||e|| (f* = tau ||x*||_1 + ||e||^2 / 2, instance.cpp:49-51) and cert_kappa. */
int l1b_problem_set_meta(l1b_problem* p, double noise_norm, double cert_kappa);
void* l1b_problem_stream(const l1b_problem* p);  /* cudaStream_t */
int l1b_problem_set_stream(l1b_problem* p, void* stream);

/* ------------------------------------------------------------------------ */
/* Operator products on device vectors.
 * Replace: LinearOperator::apply / apply_transpose (linops.hpp:139-155;
 * OperatorSpec::apply linops.cpp:422-446, apply_transpose :448-473),
 * apply_gram_inverse (:475-490), gram_diagonal (:533-558), row/column
 * (:566-619) via the exported CSR/CSC.                                      */
enum { L1B_PATH_SPARSE = 0, /* CSR (A) / CSC (A^T) SpMV kernels */
       L1B_PATH_SWEEP = 1,  /* matrix-free Givens stage sweeps, one launch per stage */
       L1B_PATH_FUSED = 2   /* matrix-free, all stages fused in one TMA-pipelined kernel
                               (banded operators only: no P1/P2, no left stages) */ };

int l1b_apply(l1b_problem* p, int path, const double* d_x, double* d_y);
int l1b_apply_transpose(l1b_problem* p, int path, const double* d_y, double* d_x);
int l1b_gram_inverse(l1b_problem* p, const double* d_v, double* d_out);
int l1b_gram_diagonal(l1b_problem* p, double* d_out);
/* estimate_gram_lmax (linops.hpp:283, linops.cpp:757-778): power iteration
 * from normal() draws of Rng(seed), products by the matrix-free sweeps */
int l1b_estimate_gram_lmax(l1b_problem* p, uint64_t iters, uint64_t seed, double* out);
/* host buffers: row_ptr[m+1] (rows >= m_active are empty), col[nnz], val[nnz] */
int l1b_export_csr(const l1b_problem* p, uint64_t* row_ptr, uint32_t* col, double* val);
int l1b_export_csc(const l1b_problem* p, uint64_t* col_ptr, uint32_t* row, double* val);

/* The Newton-CG Hessian-vector product on device vectors (smoothed_hessvec,
 * solvers.cpp:188-200; as newton_cg_run's PCG forms it, :536-540):
 * out = A^T (A v) + tau * d2psi_mu(x) .* v.  Whole problems only.          */
int l1b_smoothed_hessvec(l1b_problem* p, double mu, const double* d_x, const double* d_v, double* d_out);
/* tau*||x||_1 + 1/2*||A x - b||^2 (solvers.cpp:145-151). */
int l1b_objective(l1b_problem* p, const double* d_x, double* f_out);

typedef struct {
  double max_support_violation;
  double max_offsupport_violation;
  double threshold;
  int pass;
} l1b_cert;
/* verify_optimality (instance.cpp:175-202) */
int l1b_verify_optimality(l1b_problem* p, double tol, l1b_cert* out);

/* ------------------------------------------------------------------------ */
/* Solvers.  Replace run_solver / fista_run / ista_run / coordinate_descent_run
 * / newton_cg_run (solvers.hpp:106-117); the block-PCDM solver is the C2
 * mapping.                                                  */
enum { L1B_ISTA = 0, L1B_FISTA = 1, L1B_CD = 2, L1B_NEWTON_CG = 3, L1B_PCDM = 4 };
enum { L1B_TARGET_REACHED = 0, L1B_ITER_BUDGET = 1, L1B_TIME_BUDGET = 2 };

/* SolverConfig (solvers.hpp:17-41) */
typedef struct {
  int solver;
  uint64_t max_iters;
  double max_seconds;
  int has_target;
  double target;
  double mu, eta;
  uint64_t pcg_max_iters, ls_max_backtracks;
  double grad_tol_rel;
  double l_fixed;      /* > 0 pins L; else L = sigma_max^2 (LPolicy::spectrum) */
  uint64_t varpi;      /* cd: modelled processors */
  uint64_t omega;      /* cd/pcdm: 0 = measure max row nnz */
  uint64_t seed;
  uint64_t block;      /* pcdm: coordinates per block */
  int op;              /* FISTA/ISTA operator: L1B_OP_AUTO (matrix-free when banded), _SPARSE, _MATRIX_FREE */
  int l_policy;        /* LPolicy (solvers.hpp:15): L1B_L_SPECTRUM, or L1B_L_BACKTRACKING (FISTA / ISTA,
                          unless l_fixed is set: power-iteration seed, halving / doubling; host-led,
                          l1b_solve only) */
  int arith;           /* L1B_ARITH_EXACT (default): every a*b+c rounds twice, as in the
                          reference's x86-64 build -- matrix-free FISTA iterates are the
                          reference's bits; L1B_ARITH_FMA: the matrix-free FISTA kernels of
                          instances with n > 2^20 contract a*b+c into one fused multiply-add
                          (one rounding: <= 1e-12 relative to the reference, not bit-exact).
                          The tile and two-iteration kernels rotate in the scaled form there --
                          cos(theta) [[1, -tan], [tan, 1]] with prod cos carried by sigma (the
                          same operations per entry in both: a sharded run gives the single
                          device's bits); it needs |cos(theta)| >= 1/4 in every stage, else the
                          request is declined (exact arithmetic, L1B_RAN_FMA not set).  Other
                          paths ignore it */
} l1b_solver_cfg;

enum { L1B_OP_AUTO = 0, L1B_OP_SPARSE = 1, L1B_OP_MATRIX_FREE = 2 };
enum { L1B_L_SPECTRUM = 0, L1B_L_BACKTRACKING = 1 };
enum { L1B_ARITH_EXACT = 0, L1B_ARITH_FMA = 1 };

/* SolverConfig's defaults (solvers.hpp:19-38); arith = L1B_ARITH_EXACT unless the
   environment says L1B_ARITH=fma (for callers without a field for it: the drop-in) */
void l1b_solver_cfg_default(l1b_solver_cfg* cfg);

/* TraceSample (solvers.hpp:45-52) */
typedef struct {
  uint64_t iter;
  double elapsed_s;
  double objective;
  uint64_t nnz;
  double matvecs;
  uint64_t extra;
} l1b_sample;

/* SolverTrace scalars (solvers.hpp:54-66) */
typedef struct {
  int status;
  int reached_target;
  double final_objective;
  double elapsed_s;
  double total_matvecs;
  uint64_t total_pcg_iterations;
  uint64_t newton_steps;
  double time_to_target;
  double matvecs_to_target;
  uint64_t n_samples;        /* samples produced (may exceed cap; first cap written) */
  uint64_t iterations;       /* iterations / sweeps / Newton steps executed */
  uint32_t path;             /* L1B_RAN_* flags: which kernels the solve ran (tests assert them) */
} l1b_summary;

/* l1b_summary.path */
enum {
  L1B_RAN_FISTA_SPARSE = 1u << 0,     /* CSR/CSC SpMV kernel pair (k_spmv.cu) */
  L1B_RAN_FISTA_MF_PAIR = 1u << 1,    /* two matrix-free product kernels (k_fused.cu) */
  L1B_RAN_FISTA_STORED = 1u << 2,     /* one matrix-free kernel, stored residuals (k_fused.cu) */
  L1B_RAN_FISTA_RECOMPUTE = 1u << 3,  /* one iteration per launch, residuals recomputed (k_iter_rc.cu) */
  L1B_RAN_FISTA_TWO_ITER = 1u << 4,   /* two iterations per launch (fista_rc2v_kernel) */
  L1B_RAN_FISTA_LOOP = 1u << 5,       /* small instance: chunks of iterations per cooperative launch */
  L1B_RAN_FMA = 1u << 6,              /* the contracted arithmetic (L1B_ARITH_FMA) was applied */
  L1B_RAN_PCDM_PAIR = 1u << 7,        /* pair-local CD / PCDM epochs, device coordinate stream */
  L1B_RAN_PCDM_PLAN = 1u << 8,        /* planned CD / PCDM epochs */
  L1B_RAN_PCDM_DIRECT = 1u << 9,      /* one-CTA CD / PCDM epochs */
  L1B_RAN_PCG_PAIR = 1u << 10,        /* pair-local PCG, one cooperative launch per Newton step */
  L1B_RAN_PCG_LOOP = 1u << 11,        /* CSR/CSC PCG, one cooperative launch per Newton step */
  L1B_RAN_PCG_KERNELS = 1u << 12,     /* CSR/CSC PCG, four kernels per PCG iteration */
  L1B_RAN_HOST_LED = 1u << 13,        /* FISTA / ISTA with LPolicy::backtracking (host-led trials) */
  L1B_RAN_FISTA_TILE = 1u << 14       /* K iterations per launch on chip-resident tiles (fista_tb_kernel) */
};

int l1b_solve(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
              l1b_summary* summary, double* x_host, double* d_x);

/* Stepping session over the device-resident loop (bench / profiling):
 * begin -> step(k) (asynchronous) -> ... -> end.  FISTA / ISTA only.        */
typedef struct l1b_session l1b_session;
int l1b_session_begin(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_session** out);
int l1b_session_step(l1b_session* s, uint64_t iters);
/* Runs iters iterations with CUDA events around each kernel on the problem's
 * stream; ms_out[k] = total milliseconds of kernel k over those iterations
 * (k = 0: A^T r + prox/momentum, 1: A x - b + residual momentum).           */
int l1b_session_profile(l1b_session* s, uint64_t iters, double* ms_out, int n_ms);
int l1b_session_sync(l1b_session* s, int* stopped, uint64_t* iterations);

/* Row-block shards (world >= 1): the caller drives the FISTA loop and does the
 * exchanges and the scalar all-reduce (NCCL through torch.distributed, see
 * paper_1503_03520_b200/distributed.py).  Which protocol a session follows is
 * in l1b_shard_buffers:
 *   matrix-free, recomputing kernels (lagged = 1, the default for 1..4 stages):
 *     begin -> [all-reduce scal, finalize] -> loop { k1 (two iterations when
 *     pairs); x halos (or peer stores); all-reduce scal8 / scal; finalize }
 *     -> flush; all-reduce scal; finalize
 *   stored residuals (single = 1, lagged = 0): loop { k1; x and r halos;
 *     all-reduce scal; finalize }
 *   CSR/CSC two-kernel mode: loop { r_y halo; k1; x halo; k2; all-reduce scal;
 *     finalize }
 *   general operators (general = 1): loop { k1; reduce-scatter g_full; prox;
 *     all-gather x_full; k2; all-reduce scal; finalize }
 * Windows: entry h + j of a window is own column / row row_begin + j; entries
 * [0, h) and [h + own, own + 2h) are the neighbours' boundary values.       */
typedef struct {
  double* x_win;    /* own + 2*halo (two-kernel mode) */
  double* r_y_win;  /* own + 2*halo (two-kernel mode) */
  double* scal;     /* 4 doubles: ||x||_1, nnz(x), #(trial != y), ||r||^2 -- sum over ranks */
  uint64_t own, halo;
  /* single-kernel mode (matrix-free, 1..4 stages): l1b_session_k1 runs iteration
   * j+1 from x_j = x_bufs[j%P], x_{j-1} = x_bufs[(j+P-1)%P] (r: period 3) into
   * x_bufs[(j+1)%P] / r_bufs[(j+1)%3], P = x_nbufs; the caller then exchanges the halos of
   * those two (x_halo / r_halo entries each side); l1b_session_k2 is a no-op.
   * Before the first iteration r_bufs[0] and r_bufs[2] need their halos.
   * lagged = 1 (recomputing kernel, k_iter_rc.cu): no residual buffers
   * (r_bufs null, r_halo 0), only the x halos travel; scal carries ||r_j||^2
   * of the iterate the kernel started from, so each iteration is recorded by
   * the NEXT finalize; after the loop: l1b_session_flush, all-reduce scal,
   * l1b_session_finalize records the last iterate. */
  int single;
  double* x_bufs[4];  /* own + 2*x_halo; x_nbufs of them rotate (x_j = x_bufs[j % x_nbufs]) */
  double* r_bufs[3];  /* own + 2*r_halo */
  uint64_t x_halo, r_halo;
  int lagged;
  int x_nbufs;      /* 3, or 4 when lagged */
  /* pairs = 1 (lagged, default): l1b_session_k1 runs TWO iterations j+1, j+2
   * (x_bufs[(j+1)%4], x_bufs[(j+2)%4]; exchange both halos) and leaves 8 sums
   * in scal8 (all-reduce those, then finalize); the flush still uses scal. */
  int pairs;
  double* scal8;
  /* general = 1: a shard of a non-banded (permuted / left-stage) operator
   * (l1b_generate with permute or left stages): rows of A split, x split by
   * columns.  Per iteration: k1 writes this rank's partial A^T r_y to g_full
   * (n_pad entries); the caller reduce-scatters g_full (rank r keeps entries
   * [r*n_pad/world, ...)); l1b_session_prox updates the own slice of x_full
   * (col_begin, col_count entries); the caller all-gathers x_full; k2; the
   * caller all-reduces scal; finalize.                                      */
  int general;
  double* g_full;
  double* x_full;
  uint64_t n_pad, col_begin, col_count;
} l1b_shard_buffers;
int l1b_session_buffers(l1b_session* s, l1b_shard_buffers* out);
/* Lagged shard sessions: sums ||r||^2 of the last iterate into scal (a no-op
 * for other sessions; single-device sessions flush inside l1b_session_end). */
int l1b_session_flush(l1b_session* s);
/* Peer halos (lagged shards): the kernels store the new x entries within
 * x_halo of the block ends straight into the neighbours' x buffers (over
 * NVLink for other devices), so the caller skips the halo exchange and keeps
 * only the scalar all-reduce (whose completion orders the stores before the
 * neighbours' next kernels).  attach_peers takes the neighbours' x_bufs
 * (4 each, NULL for no neighbour) as pointers valid on this device (same
 * device, or peer access enabled); the IPC pair exchanges them between
 * processes (4 cudaIpcMemHandle_t = 4 x 64 bytes per session).               */
int l1b_session_attach_peers(l1b_session* s, double* const* left_bufs, uint64_t left_row_begin,
                             double* const* right_bufs, uint64_t right_row_begin);
int l1b_session_export_x_ipc(l1b_session* s, void* handles);
int l1b_session_attach_peers_ipc(l1b_session* s, const void* left_handles, uint64_t left_row_begin,
                                 const void* right_handles, uint64_t right_row_begin);
/* General shards: prox / momentum on the own columns from the reduced g.     */
int l1b_session_prox(l1b_session* s);
/* Which FISTA kernels a session runs (bench roofline bookkeeping):
 * bytes per iteration 288n-class CSR/CSC pair, 96n matrix-free pair, 64n
 * stored-residual single kernel, 40n recomputing kernel, 24n two-iteration
 * recomputing kernel (one device), general-shard CSR/CSC.                   */
enum {
  L1B_KMODE_SPARSE = 0,
  L1B_KMODE_MATRIX_FREE_PAIR = 1,
  L1B_KMODE_STORED_RESIDUAL = 2,
  L1B_KMODE_RECOMPUTE = 3,
  L1B_KMODE_RECOMPUTE_TWO = 4,
  L1B_KMODE_GENERAL_SHARD = 5,
  L1B_KMODE_RECOMPUTE_TILE = 6  /* K iterations per launch (fista_tb_kernel); l1b_session_tile_iters gives K */
};
int l1b_session_kernel_mode(l1b_session* s, int* mode);
/* L1B_KMODE_RECOMPUTE_TILE sessions: iterations per launch, entries per tile
 * (span) and entries a tile keeps (valid = span - 2 x the halo erosion of
 * those iterations): HBM bytes per launch = 48 n span / valid.  Other
 * sessions: all three 0.  (No reference counterpart: measurement only.) */
int l1b_session_tile_geometry(l1b_session* s, int* iters, int64_t* span, int64_t* valid);
/* The tile launches l1b_session_step / _profile take for `iters` iterations
 * (each K = 2 mod 4 and at most the session's K, spread evenly: 20 = 10 + 10;
 * fewer than 6 left over go to two-iteration / single launches): up to `cap`
 * launch lengths into ks, their number into *count.  (Measurement only.) */
int l1b_session_tile_plan(l1b_session* s, uint64_t iters, int* ks, int cap, int* count);
/* The same plan without a session, for K = kmax iterations per launch (host arithmetic only). */
int l1b_tile_plan(int kmax, uint64_t iters, int* ks, int cap, int* count);
/* Dense FP64 fma throughput of `device` in TFLOP/s (a probe kernel of
 * independent fma chains; measurement only, no reference counterpart): the
 * denominator of the FP64-bound kernels' roofline in bench.py. */
int l1b_fp64_peak(int device, double* tflops);
int l1b_session_k1(l1b_session* s);
int l1b_session_k2(l1b_session* s);
int l1b_session_finalize(l1b_session* s);
int l1b_session_end(l1b_session* s, l1b_sample* samples, uint64_t cap, l1b_summary* summary,
                    double* x_host);
/* Serving a resident operator: restart the loop from x_0 = 0 (after
 * l1b_problem_set_rhs, say) keeping the session's buffers, peer attachments,
 * communicator and captured graphs; read reports a shard session's trace,
 * summary and own x like l1b_session_end without ending it.                */
int l1b_session_restart(l1b_session* s);
int l1b_session_read(l1b_session* s, l1b_sample* samples, uint64_t cap, l1b_summary* summary,
                     double* x_host);
/* Native shard driver (lagged two-iteration shards, the default protocol of
 * banded 1..4-stage operators): the per-launch loop of distributed.py --
 * k1; x halos by NCCL send / recv (or the kernels' peer stores); all-reduce
 * of the 8 sums; finalize -- issued by the library on the session's stream
 * with its own NCCL communicator, the steady state replayed from a CUDA
 * graph of two launches.  This is the "per-iteration NCCL all-reduce of the
 * partial A^T r" of the north star in its exact sparse form.
 * NCCL is bound at run time (the process's libnccl.so.2).  unique_id: the
 * 128-byte ncclUniqueId of l1b_nccl_get_unique_id on rank 0, broadcast by
 * the caller.  The session's stream must not be the legacy default stream.
 *   attach -> nccl_start -> nccl_steps(launches) ... -> nccl_finish -> end
 * k1_ms (optional): events around every k1 instead of the graph; receives
 * the summed k1 milliseconds of these launches.                            */
int l1b_nccl_get_unique_id(void* id_out);
int l1b_nccl_version(int* version);
int l1b_session_attach_nccl(l1b_session* s, const void* unique_id, int rank, int world);
int l1b_session_nccl_start(l1b_session* s);
int l1b_session_nccl_steps(l1b_session* s, uint64_t launches, int use_graph, double* k1_ms);
int l1b_session_nccl_finish(l1b_session* s);
/* Kernel launches issued by the library since load (all entry points). */
uint64_t l1b_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* L1B_H */
