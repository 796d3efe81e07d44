// fista.cuh -- device-side FISTA scalar bookkeeping shared by the CSR/CSC
// kernels (k_spmv.cu) and the matrix-free kernels (k_fused.cu).
#pragma once

#include "common.cuh"
#include "kernels.hpp"

namespace l1b {

// t_{k+1} and beta_k of solvers.cpp:349-350 (same operations, same rounding).
__device__ __forceinline__ void fista_momentum(const FistaDev* st, double* t_next, double* beta) {
  const double t = st->t;
  *t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
  *beta = st->accel ? (t - 1.0) / *t_next : 0.0;
}

// Iteration k's record and stop checks (solvers.cpp:366-376 + the loop-head
// checks :312-313): f, trace sample, fixed point / target / iteration budget.
// trace == nullptr: the bookkeeping without the sample store (replicas).
__device__ inline void fista_record(FistaDev* st, FistaSample* trace, uint64_t k, double f,
                                    double nnz, bool fixed, uint64_t ts) {
  st->k = k;
  st->f = f;
  st->nnz = nnz;
  st->last_ts = ts;
  if (!isfinite(f)) {
    st->stop = 1;
    st->status = -1;
    return;
  }
  if (k <= 1000 || k % 10 == 0 || fixed) {
    if (trace && st->n_samples < st->cap) trace[st->n_samples] = FistaSample{k, f, nnz, ts};
    st->n_samples++;
    st->last_sampled = k;
  }
  if (fixed) {
    st->stop = 1;
    st->status = 0;
  } else if (st->has_target && f <= st->target) {
    st->stop = 1;
    st->status = 0;
  } else if (k >= st->max_iters) {
    st->stop = 1;
    st->status = 1;
  }
}

// Bookkeeping after iteration k (scal = l1, nnz, mismatches, ||r||^2 of x_k)
__device__ inline void fista_finalize_device(FistaDev* st, FistaSample* trace) {
  const double f = st->tau * st->scal[0] + 0.5 * (st->scal[3] + st->tail_sq);
  double t_next, beta;
  fista_momentum(st, &t_next, &beta);
  st->beta_y = beta;  // y = trial + beta (trial - x)  (solvers.cpp:349-352)
  if (st->accel) st->t = t_next;
  fista_record(st, trace, st->k + 1, f, st->scal[1], st->scal[2] == 0.0, global_timer_ns());
}

// Lagged bookkeeping after kernel j of the recomputing path: scal = l1, nnz,
// mismatches of x_{j+1} and ||r_j||^2.  Iteration j is recorded first (its l1 /
// nnz / mismatches were stashed by kernel j-1), then -- unless that stopped
// the loop, or this is the flush after the last kernel -- the momentum for
// kernel j+1 (it depends on t only) and x_{j+1}'s sums are stashed.  Same
// values and order of checks as fista_finalize_device, one kernel later.
__device__ inline void fista_finalize_lagged(FistaDev* st, FistaSample* trace, bool flush) {
  if (st->pend_valid) {
    const double f = st->tau * st->pend[0] + 0.5 * (st->scal[3] + st->tail_sq);
    st->pend_valid = 0;
    fista_record(st, trace, st->k + 1, f, st->pend[1], st->pend[2] == 0.0, st->pend_ts);
    if (st->stop) return;
  }
  if (flush) return;
  double t_next, beta;
  fista_momentum(st, &t_next, &beta);
  st->beta_y = beta;
  if (st->accel) st->t = t_next;
  st->pend[0] = st->scal[0];
  st->pend[1] = st->scal[1];
  st->pend[2] = st->scal[2];
  st->pend_ts = global_timer_ns();
  st->pend_valid = 1;
}

// Lagged bookkeeping after a two-iteration kernel (iterations j+1, j+2 from
// x_j, x_{j-1}): records iteration j (stashed sums + ||r_j||^2) and, unless
// that stopped the loop, iteration j+1 (all its sums are in scal8); then the
// momentum for the next kernel and x_{j+2}'s sums are stashed.  The kernel
// itself used beta_y for x_{j+1} and the next step of the t-sequence for
// x_{j+2}; both steps are committed here.  Same values and order of checks as
// two fista_finalize_lagged calls.
__device__ inline void fista_finalize_lagged2(FistaDev* st, FistaSample* trace) {
  const double* q = st->scal8;
  const uint64_t ts = global_timer_ns();
  if (st->pend_valid) {
    const double f = st->tau * st->pend[0] + 0.5 * (q[0] + st->tail_sq);
    st->pend_valid = 0;
    fista_record(st, trace, st->k + 1, f, st->pend[1], st->pend[2] == 0.0, st->pend_ts);
    if (st->stop) return;
  }
  double t_next, beta;
  fista_momentum(st, &t_next, &beta);  // the step the kernel used for x_{j+2}
  st->beta_y = beta;
  if (st->accel) st->t = t_next;
  {
    const double f = st->tau * q[1] + 0.5 * (q[4] + st->tail_sq);
    fista_record(st, trace, st->k + 1, f, q[2], q[3] == 0.0, ts);
    if (st->stop) return;
  }
  fista_momentum(st, &t_next, &beta);
  st->beta_y = beta;
  if (st->accel) st->t = t_next;
  st->pend[0] = q[5];
  st->pend[1] = q[6];
  st->pend[2] = q[7];
  st->pend_ts = ts;
  st->pend_valid = 1;
}

// Lagged bookkeeping after a K-iteration tile kernel (iterations j+1 .. j+K
// from x_j, x_{j-1}): q[4i .. 4i+3] = l1, nnz, mismatches of x_{j+i+1} and
// ||r_{j+i}||^2.  Records iteration j (stashed sums + ||r_j||^2), then j+1 ..
// j+K-1 (each from the previous x's sums and the next r), committing one step
// of the t-sequence after each; x_{j+K}'s sums are stashed.  Same values and
// order of checks as K fista_finalize_lagged calls (K = 2: lagged2).
__device__ inline void fista_finalize_laggedk(FistaDev* st, FistaSample* trace, const double* q, int K) {
  const uint64_t ts = global_timer_ns();
  if (st->pend_valid) {
    const double f = st->tau * st->pend[0] + 0.5 * (q[3] + st->tail_sq);
    st->pend_valid = 0;
    fista_record(st, trace, st->k + 1, f, st->pend[1], st->pend[2] == 0.0, st->pend_ts);
    if (st->stop) return;
  }
  double t_next, beta;
  for (int i = 0; i + 1 < K; ++i) {
    fista_momentum(st, &t_next, &beta);
    st->beta_y = beta;
    if (st->accel) st->t = t_next;
    const double f = st->tau * q[4 * i] + 0.5 * (q[4 * (i + 1) + 3] + st->tail_sq);
    fista_record(st, trace, st->k + 1, f, q[4 * i + 1], q[4 * i + 2] == 0.0, ts);
    if (st->stop) return;
  }
  fista_momentum(st, &t_next, &beta);
  st->beta_y = beta;
  if (st->accel) st->t = t_next;
  st->pend[0] = q[4 * (K - 1)];
  st->pend[1] = q[4 * (K - 1) + 1];
  st->pend[2] = q[4 * (K - 1) + 2];
  st->pend_ts = ts;
  st->pend_valid = 1;
}

}  // namespace l1b
