/*
 * l1oracle.h -- CPU restatement of the reference's l1-least-squares hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1503_03520_b200/,
 * include/) links, loads or calls this code.  It is imported only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, always as the
 * *checker*, never as the thing measured or shipped.
 *
 * Parity pin: every function below cites the reference file:line it restates
 * (paths relative to /root/reference/proj).  The restatement is itself checked
 * against (a) the reference compiled from its own sources into oracle/_ref
 * (oracle/Makefile) and (b) the committed golden vectors in tests/golden/
 * produced from that build (tests/golden/make_golden.py), plus SPEC.md's
 * known answers.
 *
 * Plain C99, no dependencies; compiled with -ffp-contract=off so that every
 * a*b+c rounds twice exactly like the reference's x86-64 -O3 build.
 */
#ifndef L1ORACLE_H
#define L1ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: std::mt19937_64 + helpers (include/l1bench/rng.hpp:14-56) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
} lo_rng;

void lo_rng_seed(lo_rng* r, uint64_t seed);
uint64_t lo_rng_next(lo_rng* r);
uint64_t lo_mix_seed(uint64_t seed, uint64_t salt);
double lo_uniform_unit(lo_rng* r);
double lo_uniform_in(lo_rng* r, double lo, double hi);
uint64_t lo_uniform_index(lo_rng* r, uint64_t n);
void lo_set_index_reject(int s); /* test hook: CD / PCDM redraws with probability ~2^-s */

/* ---- Operator A = P1 * Gtilde * P2 * Sigma * G^T (linops.hpp:159-206) ----
 * Only paired stages (RotationStage::Kind::paired) are restated.           */
typedef struct {
  uint64_t m, n;
  uint32_t n_right, n_left;
  const int32_t* right_offset; /* [n_right] */
  const double* right_theta;   /* [n_right] */
  const int32_t* left_offset;  /* [n_left] */
  const double* left_theta;    /* [n_left] */
  const uint32_t* p1;          /* [m] map, NULL = identity  (Pv)[i] = v[map[i]] */
  const uint32_t* p2;          /* [m] map, NULL = identity */
  const uint32_t* p1_inv;      /* inverse maps (NULL iff map NULL) */
  const uint32_t* p2_inv;
  const double* sigma;         /* [n] realized spectrum */
} lo_op;

void lo_apply_stage(double* v, uint64_t dim, int offset, double theta, int transposed);
void lo_apply(const lo_op* A, const double* x, double* y);            /* y[m] = A x   */
void lo_apply_transpose(const lo_op* A, const double* y, double* x);  /* x[n] = A^T y */
void lo_apply_gram_inverse(const lo_op* A, const double* v, double* out);
void lo_gram_diagonal(const lo_op* A, double* d);
double lo_gram_lmax(const lo_op* A);

/* Fisher-Yates realisation of a seeded permutation (linops.cpp:224-239). */
void lo_permutation_realize(uint64_t n, uint64_t seed, uint32_t* map, uint32_t* inv);
/* Uniform spectrum realisation (linops.cpp:320-331). */
void lo_spectrum_uniform(uint64_t n, double lo, double hi, double shift, uint64_t seed,
                         double* sigma);

/* Streaming windows of the two per-entry generator streams at any length
 * (C5: 2^32 draws, too long to hold): draws [0, count) of Rng(seed) exactly
 * as lo_spectrum_uniform (spectrum = 1: reject u <= lo, + shift;
 * linops.cpp:323-331) or as the l1_subgradient fill before the support signs
 * (spectrum = 0: lo + (hi - lo) u; instance.cpp:33-35), sequentially; draws
 * [wlo, whi) are stored into out, min / max over all draws into vmin / vmax. */
void lo_uniform_stream_window(uint64_t seed, uint64_t count, double lo, double hi, int spectrum,
                              double shift, uint64_t wlo, uint64_t whi, double* out, double* vmin,
                              double* vmax);

/* Sparse row / column via the reference's sparse-accumulator sweeps
 * (linops.cpp:113-192, 566-619).  Returns nnz written (sorted ascending,
 * exact zeros dropped).  ws must come from lo_ws_create(max(m, n)).      */
typedef struct lo_ws lo_ws;
lo_ws* lo_ws_create(uint64_t size);
void lo_ws_free(lo_ws* ws);
uint64_t lo_row(const lo_op* A, uint64_t i, lo_ws* ws, uint32_t* idx, double* val);
uint64_t lo_column(const lo_op* A, uint64_t j, lo_ws* ws, uint32_t* idx, double* val);

/* Full CSR (rows of A) / CSC (columns of A) from lo_row / lo_column.
 * ptr has length dim+1; idx/val capacity cap.  Returns nnz or UINT64_MAX
 * when cap is too small.                                                  */
uint64_t lo_build_csr(const lo_op* A, uint64_t* ptr, uint32_t* idx, double* val, uint64_t cap);
uint64_t lo_build_csc(const lo_op* A, uint64_t* ptr, uint32_t* idx, double* val, uint64_t cap);
/* y = A x through a CSR/CSC held as rows (sequential row dot products). */
void lo_csr_matvec(uint64_t rows, const uint64_t* ptr, const uint32_t* idx, const double* val,
                   const double* x, double* y);

/* ---- Generator (solution.cpp:47-75, instance.cpp:28-89, bench.cpp:253-316) ---- */
/* Floyd sampling + uniform values; support sorted ascending. Returns s.  */
uint64_t lo_uniform_sparse_solution(uint64_t n, uint64_t s, double gamma, lo_rng* rng,
                                    uint32_t* support, double* values);
void lo_l1_subgradient(uint64_t n, const uint32_t* support, const double* values, uint64_t s,
                       double bound, lo_rng* rng, double* g);
/* b = A x* + tau A (A^T A)^{-1} g.  Returns noise_norm. */
double lo_generate_instance(const lo_op* A, double tau, const uint32_t* support,
                            const double* values, uint64_t s, double fill_bound, lo_rng* rng,
                            double* b);

typedef struct {
  double max_support_violation;
  double max_offsupport_violation;
  double threshold;
  int pass;
} lo_cert;
lo_cert lo_verify_optimality(const lo_op* A, double tau, const double* b, const uint32_t* support,
                             const double* values, uint64_t s, double tol);

/* ---- Solvers (solvers.cpp) ---- */
typedef struct {
  uint64_t iter;
  double objective;
  uint64_t nnz;
  double matvecs;
  uint64_t extra;
} lo_sample;

typedef struct {
  int status;          /* 0 target_reached, 1 iter_budget, 2 time_budget (solvers.hpp:24) */
  int reached_target;
  double final_objective;
  double total_matvecs;
  uint64_t total_pcg_iterations;
  uint64_t newton_steps;
  double matvecs_to_target;
  uint64_t n_samples;  /* samples written (<= cap) */
  uint64_t n_samples_total;
} lo_summary;

typedef struct {
  uint64_t max_iters;
  int has_target;
  double target;
  double mu, eta, grad_tol_rel;
  uint64_t pcg_max_iters, ls_max_backtracks;
  double l_fixed;      /* <= 0: spectrum policy */
  uint64_t varpi;
  uint64_t omega;      /* 0: measure */
  uint64_t seed;
  uint64_t block;      /* block PCDM block size */
  int accelerated;     /* fista (1) / ista (0) */
  int backtracking;    /* LPolicy::backtracking (solvers.hpp:15, 31) */
} lo_cfg;

/* estimate_gram_lmax (linops.cpp:757-778): power iteration from normal() draws */
double lo_estimate_gram_lmax(const lo_op* A, uint64_t iters, uint64_t seed);
double lo_normal(lo_rng* r); /* rng.hpp:48-56 */
/* FISTA/ISTA (solvers.cpp:277-382) with LipschitzState (:99-120): spectrum L,
 * l_fixed, or backtracking seeded by the power iteration. x_out[n] may be NULL. */
lo_summary lo_fista(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                    lo_sample* samples, uint64_t cap, double* x_out);
/* Serial randomized CD (solvers.cpp:414-482); columns from a CSC.       */
lo_summary lo_cd(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                 const uint64_t* cptr, const uint32_t* cidx, const double* cval,
                 const uint64_t* rptr, lo_sample* samples, uint64_t cap, double* x_out);
/* Block PCDM restatement of the C2 mapping; no reference
 * counterpart -- defined in DESIGN.md and restated here for the kernel.   */
lo_summary lo_pcdm(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                   const uint64_t* cptr, const uint32_t* cidx, const double* cval,
                   const uint64_t* rptr, const uint32_t* ridx, lo_sample* samples, uint64_t cap,
                   double* x_out);
/* Newton-CG on the pseudo-Huber problem (solvers.cpp:202-264, 487-568). */
lo_summary lo_newton_cg(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                        lo_sample* samples, uint64_t cap, double* x_out);

/* Single PCG solve with hessvec = A^T A v + tau d2psi(x) v (for per-op parity). */
typedef struct {
  uint64_t iterations;
  int converged;
  int negative_curvature;
  double rel_residual;
} lo_pcg_result;
lo_pcg_result lo_pcg_at(const lo_op* A, double tau, double mu, const double* x,
                        const double* rhs, const double* precond, double eta, uint64_t max_iters,
                        double* step);

double lo_soft_threshold(double v, double t);
double lo_cd_damping(uint64_t omega, uint64_t varpi, uint64_t n);
double lo_objective(const lo_op* A, double tau, const double* b, const double* x);

#ifdef __cplusplus
}
#endif
#endif
