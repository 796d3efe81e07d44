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

// Bookkeeping after iteration k (solvers.cpp:366-376 + the loop-head checks
// :312-313): f, trace sample, fixed point / target / iteration budget.
__device__ inline void fista_finalize_device(FistaDev* st, FistaSample* trace) {
  const double f = st->tau * st->scal[0] + 0.5 * (st->scal[3] + st->tail_sq);
  const uint64_t k = st->k + 1;
  double t_next, beta;
  fista_momentum(st, &t_next, &beta);
  st->beta_y = beta;  // y = trial + beta (trial - x)  (solvers.cpp:349-352)
  if (st->accel) st->t = t_next;
  st->k = k;
  st->f = f;
  st->nnz = st->scal[1];
  const uint64_t ts = global_timer_ns();
  st->last_ts = ts;
  const bool fixed = st->scal[2] == 0.0;
  if (!isfinite(f)) {
    st->stop = 1;
    st->status = -1;
    return;
  }
  if (k <= 1000 || k % 10 == 0 || fixed) {
    if (st->n_samples < st->cap) trace[st->n_samples] = FistaSample{k, f, st->scal[1], ts};
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

}  // namespace l1b
