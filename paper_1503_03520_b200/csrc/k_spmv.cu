// k_spmv.cu -- fp64 CSR SpMV for A (rows) and A^T (CSC columns) with fused
// solver epilogues, and the FISTA/ISTA device loop (solvers.cpp:277-382).
//
// Kernel shape (HBM-bound, ~0.17 flop/B; no tensor cores -- not a dense
// contraction): one warp per tile of 32 consecutive lines (see spmv_kernel).
// The matrix streams are loaded with the evict-first hint (ld.global.cs) so
// the gathered vector stays L2-resident; each vector element of the epilogue
// is touched exactly once, by a coalesced warp access.  Scalars (||x||_1,
// nnz, ||r||^2, ...) are reduced per block and folded by the last block in a
// fixed order: results are deterministic run to run.
#include <cmath>

#include "common.cuh"
#include "kernels.hpp"
#include "fista.cuh"
#include "spmv.cuh"

namespace l1b {

namespace {

struct EpiStore {
  double* y;
  static constexpr int kVec = 0;
  __host__ __device__ const double* vec(int) const { return nullptr; }
  __device__ bool skip() const { return false; }
  __device__ void start() {}
  __device__ void line(uint64_t i, double s, const double*) { y[i] = s; }
  __device__ void finish() {}
};

// objective (solvers.cpp:145-151): r = A x - b, sum r^2 (+ tail) ...
struct EpiResidualSq {
  const double* b;
  double* partials;
  unsigned int* ticket;
  double* out;
  double acc[1];
  static constexpr int kVec = 1;
  __host__ __device__ const double* vec(int) const { return b; }
  __device__ bool skip() const { return false; }
  __device__ void start() { acc[0] = 0.0; }
  __device__ void line(uint64_t, double s, const double* pv) {
    const double r = s - pv[0];
    acc[0] += r * r;
  }
  __device__ void finish() {
    double tot[1];
    if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
  }
};

// K1 epilogue: grad_j = (A^T r_y)_j  ->  trial = S(y - grad/L, tau/L)
// (solvers.cpp:319-328), fixed-point test against y (:346), momentum on x/y
// (:349-353, :358) and the ||x||_1 / nnz partials of f (:366-369).
// ISTA aliases y == x with beta = 0 (solvers.cpp:362).
struct EpiFistaX {
  double* x;
  double* y;
  FistaDev* st;
  double* partials;
  double inv_l, thr, beta;
  double acc[3];  // ||trial||_1, nnz(trial), #(trial != y)
  static constexpr int kVec = 2;  // y, x at the column
  __host__ __device__ const double* vec(int v) const { return v == 0 ? y : x; }
  __device__ bool skip() const { return *(volatile const int*)&st->stop; }
  __device__ void start() {
    double t_next;
    fista_momentum(st, &t_next, &beta);
    inv_l = 1.0 / st->lval;
    thr = st->tau * inv_l;
    acc[0] = acc[1] = acc[2] = 0.0;
  }
  __device__ void line(uint64_t j, double g, const double* pv) {
    const double yo = pv[0];
    const double xo = pv[1];
    const double tr = soft_threshold(yo - inv_l * g, thr);
    acc[2] += tr != yo ? 1.0 : 0.0;
    y[j] = tr + beta * (tr - xo);
    x[j] = tr;
    acc[0] += fabs(tr);
    acc[1] += tr != 0.0 ? 1.0 : 0.0;
  }
  __device__ void finish() {
    double tot[3];
    if (grid_sum<3>(acc, partials, &st->ticket[0], tot) && threadIdx.x == 0) {
      st->scal[0] = tot[0];
      st->scal[1] = tot[1];
      st->scal[2] = tot[2];
    }
  }
};

// K2 epilogue: r_trial = A trial - b (solvers.cpp:329-330), residual
// momentum r_y = (1+beta) r_trial - beta r_x (:355-357), r_x = r_trial
// (:359), ||r_x||^2 partial; the last block finalises the iteration.
struct EpiFistaR {
  const double* b;
  double* r_x;
  double* r_y;
  FistaDev* st;
  FistaSample* trace;
  double* partials;
  double beta;
  double acc[1];
  static constexpr int kVec = 2;  // b, r_x at the row
  __host__ __device__ const double* vec(int v) const { return v == 0 ? b : r_x; }
  __device__ bool skip() const { return *(volatile const int*)&st->stop; }
  __device__ void start() {
    double t_next;
    fista_momentum(st, &t_next, &beta);
    acc[0] = 0.0;
  }
  __device__ void line(uint64_t i, double s, const double* pv) {
    const double rt = s - pv[0];
    const double rx = pv[1];
    r_y[i] = (1.0 + beta) * rt - beta * rx;
    r_x[i] = rt;
    acc[0] += rt * rt;
  }
  __device__ void finish() {
    double tot[1];
    if (grid_sum<1>(acc, partials, &st->ticket[1], tot) && threadIdx.x == 0) {
      st->scal[3] = tot[0];
      if (!st->defer) fista_finalize_device(st, trace);
    }
  }
};

__device__ void fista_init_finalize(FistaDev* st, FistaSample* trace);

// r_x = r_y = A*0 - b and ||r||^2 (solvers.cpp:294-298, 301-302).
__global__ void fista_init_kernel(const double* __restrict__ b, double* r_x, double* r_y,
                                  uint64_t m, FistaDev* st, FistaSample* trace,
                                  double* partials) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double r = 0.0 - b[i];
    if (r_x) r_x[i] = r;  // null: the recomputing kernel keeps no residual vectors
    if (r_y != r_x) r_y[i] = r;
    acc[0] += r * r;
  }
  double tot[1];
  if (grid_sum<1>(acc, partials, &st->ticket[2], tot) && threadIdx.x == 0) {
    st->scal[3] = tot[0];
    if (!st->defer) fista_init_finalize(st, trace);
  }
}

// f_0, sample 0 and the loop-head checks before the first iteration
__device__ void fista_init_finalize(FistaDev* st, FistaSample* trace) {
  {
    const double f = st->tau * 0.0 + 0.5 * (st->scal[3] + st->init_tail);
    const uint64_t ts = global_timer_ns();
    st->t0_ns = ts;
    st->last_ts = ts;
    st->f = f;
    st->nnz = 0.0;
    st->k = 0;
    if (st->cap > 0) trace[0] = FistaSample{0, f, 0.0, ts};
    st->n_samples = 1;
    st->last_sampled = 0;
    st->initialized = 1;
    if (!isfinite(f)) {
      st->stop = 1;
      st->status = -1;
    } else if (st->has_target && f <= st->target) {
      st->stop = 1;
      st->status = 0;
    } else if (st->max_iters == 0) {
      st->stop = 1;
      st->status = 1;
    }
  }
}

__global__ void fista_finalize_kernel(FistaDev* st, FistaSample* trace) {
  if (st->stop) return;
  if (!st->initialized)
    fista_init_finalize(st, trace);
  else if (st->pair_pending) {
    st->pair_pending = 0;
    fista_finalize_lagged2(st, trace);
  } else if (st->lagged)
    fista_finalize_lagged(st, trace, st->flushing != 0);
  else
    fista_finalize_device(st, trace);
}

__global__ void l1_kernel(const double* __restrict__ x, uint64_t n, double* partials,
                          unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc[0] += fabs(x[i]);
  double tot[1];
  if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
}

__global__ void combine_objective(const double* sc, double tau, double tail_sq, double* f) {
  *f = tau * sc[0] + 0.5 * (sc[1] + tail_sq);
}

}  // namespace

int spmv_grid_max() { return 32 * sm_count(); }

void spmv(const Csr& M, const double* x, double* y, cudaStream_t st) {
  if (M.lines == 0) return;
  launch(M, x, EpiStore{y}, st);
}

void objective(const Csr& A, const double* x, uint64_t n, const double* b, double tau,
               double tail_sq, double* d_f, cudaStream_t st) {
  const int gmax = spmv_grid_max();
  double* scratch = nullptr;  // [l1, rr] + partials
  unsigned int* tickets = nullptr;
  L1B_CUDA(cudaMallocAsync(&scratch, (2 + gmax) * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&tickets, 2 * sizeof(unsigned int), st));
  L1B_CUDA(cudaMemsetAsync(scratch, 0, 2 * sizeof(double), st));
  L1B_CUDA(cudaMemsetAsync(tickets, 0, 2 * sizeof(unsigned int), st));
  l1_kernel<<<grid_for(n), kThreads, 0, st>>>(x, n, scratch + 2, tickets, scratch);
  L1B_LAUNCHED();
  if (A.lines) launch(A, x, EpiResidualSq{b, scratch + 2, tickets + 1, scratch + 1, {0.0}}, st);
  combine_objective<<<1, 1, 0, st>>>(scratch, tau, tail_sq, d_f);
  L1B_LAUNCHED();
  L1B_CUDA(cudaFreeAsync(scratch, st));
  L1B_CUDA(cudaFreeAsync(tickets, st));
}

void fista_init(const FistaBufs& fb, uint64_t m_rows, cudaStream_t st) {
  fista_init_kernel<<<grid_for(m_rows), kThreads, 0, st>>>(fb.b, fb.r_x, fb.r_y, m_rows, fb.st,
                                                           fb.trace, fb.partials);
  L1B_LAUNCHED();
}

void fista_k1(const Csr& At, const FistaBufs& fb, cudaStream_t st) {
  EpiFistaX e{fb.x, fb.y, fb.st, fb.partials, 0.0, 0.0, 0.0, {0.0, 0.0, 0.0}};
  launch(At, fb.r_y_gather, e, st);
}

void fista_k2(const Csr& A, const FistaBufs& fb, cudaStream_t st) {
  EpiFistaR e{fb.b, fb.r_x, fb.r_y, fb.st, fb.trace, fb.partials, 0.0, {0.0}};
  launch(A, fb.x_gather, e, st);
}

// General shards: the prox / momentum half of K1 on the own column slice, once
// the partial A^T r_y of every rank has been reduce-scattered into g (same
// operations as EpiFistaX::line, solvers.cpp:325-352).
__global__ void fista_prox_kernel(const double* __restrict__ g, double* x, double* y, uint64_t cols,
                                  FistaDev* st, double* partials) {
  if (*(volatile const int*)&st->stop) return;
  double t_next, beta;
  fista_momentum(st, &t_next, &beta);
  const double inv_l = 1.0 / st->lval;
  const double thr = st->tau * inv_l;
  double acc[3] = {0.0, 0.0, 0.0};  // ||trial||_1, nnz(trial), #(trial != y)
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < cols;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const double yo = y[j], xo = x[j];
    const double tr = soft_threshold(yo - inv_l * g[j], thr);
    acc[2] += tr != yo ? 1.0 : 0.0;
    y[j] = tr + beta * (tr - xo);
    x[j] = tr;
    acc[0] += fabs(tr);
    acc[1] += tr != 0.0 ? 1.0 : 0.0;
  }
  double tot[3];
  if (grid_sum<3>(acc, partials, &st->ticket[0], tot) && threadIdx.x == 0) {
    st->scal[0] = tot[0];
    st->scal[1] = tot[1];
    st->scal[2] = tot[2];
  }
}

void fista_prox(const double* g, double* x, double* y, uint64_t cols, FistaDev* st,
                double* partials, cudaStream_t stream) {
  fista_prox_kernel<<<grid_for(std::max<uint64_t>(cols, 1)), kThreads, 0, stream>>>(g, x, y, cols, st,
                                                                                  partials);
  L1B_LAUNCHED();
}

void fista_finalize_launch(const FistaBufs& fb, cudaStream_t st) {
  fista_finalize_kernel<<<1, 1, 0, st>>>(fb.st, fb.trace);
  L1B_LAUNCHED();
}

}  // namespace l1b
