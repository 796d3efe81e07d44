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

namespace l1b {

namespace {

// The SpMV skeleton ("row tile per warp"): a warp owns 32 consecutive lines.
//  1. lane l loads ptr[r0+l] and ptr[r0+l+1]: the tile's nonzeros are the
//     contiguous range [ptr[r0], ptr[r0+32]);
//  2. the warp streams that range with coalesced 8 B value / 4 B index loads
//     (U = 8 independent loads per lane in flight, evict-first), gathers x and
//     parks the products in shared memory (padded one slot per 16 to avoid
//     bank conflicts for the 8-entry rows);
//  3. lane l sums its own line's products in ascending index order (the
//     reference's sequential dot order) and runs the epilogue for line r0+l,
//     so every epilogue load/store is a coalesced 256 B warp access.
// Tiles with more than kCap nonzeros are processed in kCap-sized chunks.
// Epi provides: skip(), start(), line(i, value), finish().
constexpr int kCapNnz = 256;
constexpr int kUnroll = 8;

__device__ __forceinline__ int pad(int off) { return off + (off >> 4); }

template <typename PtrT, class Epi>
__global__ void __launch_bounds__(kThreads) spmv_kernel(const PtrT* __restrict__ ptr,
                                                        const uint32_t* __restrict__ idx,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x,
                                                        uint64_t nlines, Epi epi) {
  if (epi.skip()) return;
  epi.start();
  __shared__ double prod_all[kThreads / 32][kCapNnz + kCapNnz / 16];
  const int lane = threadIdx.x & 31;
  double* sp = prod_all[threadIdx.x >> 5];
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t tile = warp; tile * 32 < nlines; tile += nwarps) {
    const uint64_t line = tile * 32 + lane;
    const bool live = line < nlines;
    const PtrT my_s = __ldg(ptr + (live ? line : nlines));
    const PtrT my_e = __ldg(ptr + (live ? line + 1 : nlines));
    const PtrT rs = __shfl_sync(0xffffffffu, my_s, 0);
    const PtrT re = __shfl_sync(0xffffffffu, my_e, 31);
    double sum = 0.0;
    for (PtrT chunk = rs; chunk < re; chunk += kCapNnz) {
      const PtrT cend = min((PtrT)(chunk + kCapNnz), re);
      for (PtrT q0 = chunk + lane; q0 < cend; q0 += 32 * kUnroll) {
        uint32_t ii[kUnroll];
        double vv[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const PtrT q = q0 + 32 * u;
          if (q < cend) {
            ii[u] = __ldcs(idx + q);
            vv[u] = __ldcs(val + q);
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const PtrT q = q0 + 32 * u;
          if (q < cend) sp[pad((int)(q - chunk))] = vv[u] * __ldg(x + ii[u]);
        }
      }
      __syncwarp();
      const PtrT a = max(my_s, chunk), e = min(my_e, cend);
      for (PtrT q = a; q < e; ++q) sum += sp[pad((int)(q - chunk))];
      __syncwarp();
    }
    if (live) epi.line(line, sum);
  }
  epi.finish();
}

struct EpiStore {
  double* y;
  __device__ bool skip() const { return false; }
  __device__ void start() {}
  __device__ void line(uint64_t i, double s) { y[i] = s; }
  __device__ void finish() {}
};

// objective (solvers.cpp:145-151): r = A x - b, sum r^2 (+ tail) ...
struct EpiResidualSq {
  const double* b;
  double* partials;
  unsigned int* ticket;
  double* out;
  double acc[1];
  __device__ bool skip() const { return false; }
  __device__ void start() { acc[0] = 0.0; }
  __device__ void line(uint64_t i, double s) {
    const double r = s - b[i];
    acc[0] += r * r;
  }
  __device__ void finish() {
    double tot[1];
    if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
  }
};

// t_{k+1} and beta_k of solvers.cpp:349-350 (same operations, same rounding).
__device__ __forceinline__ void fista_momentum(const FistaDev* st, double* t_next, double* beta) {
  const double t = st->t;
  *t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
  *beta = st->accel ? (t - 1.0) / *t_next : 0.0;
}

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
  __device__ bool skip() const { return *(volatile const int*)&st->stop; }
  __device__ void start() {
    double t_next;
    fista_momentum(st, &t_next, &beta);
    inv_l = 1.0 / st->lval;
    thr = st->tau * inv_l;
    acc[0] = acc[1] = acc[2] = 0.0;
  }
  __device__ void line(uint64_t j, double g) {
    const double yo = y[j];
    const double xo = x[j];
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

// Bookkeeping after iteration k (solvers.cpp:366-376 + the loop-head checks
// :312-313): f, trace sample, fixed point / target / iteration budget.
__device__ void fista_finalize(FistaDev* st, FistaSample* trace) {
  const double f = st->tau * st->scal[0] + 0.5 * (st->scal[3] + st->tail_sq);
  const uint64_t k = st->k + 1;
  double t_next, beta;
  fista_momentum(st, &t_next, &beta);
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
  __device__ bool skip() const { return *(volatile const int*)&st->stop; }
  __device__ void start() {
    double t_next;
    fista_momentum(st, &t_next, &beta);
    acc[0] = 0.0;
  }
  __device__ void line(uint64_t i, double s) {
    const double rt = s - b[i];
    const double rx = r_x[i];
    r_y[i] = (1.0 + beta) * rt - beta * rx;
    r_x[i] = rt;
    acc[0] += rt * rt;
  }
  __device__ void finish() {
    double tot[1];
    if (grid_sum<1>(acc, partials, &st->ticket[1], tot) && threadIdx.x == 0) {
      st->scal[3] = tot[0];
      fista_finalize(st, trace);
    }
  }
};

// r_x = r_y = A*0 - b, f_0 (solvers.cpp:294-298, 301-302) and the loop-head
// checks before the first iteration.
__global__ void fista_init_kernel(const double* __restrict__ b, double* r_x, double* r_y,
                                  uint64_t m, FistaDev* st, FistaSample* trace,
                                  double* partials) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double r = 0.0 - b[i];
    r_x[i] = r;
    if (r_y != r_x) r_y[i] = r;
    acc[0] += r * r;
  }
  double tot[1];
  if (grid_sum<1>(acc, partials, &st->ticket[2], tot) && threadIdx.x == 0) {
    const double f = st->tau * 0.0 + 0.5 * tot[0];
    const uint64_t ts = global_timer_ns();
    st->t0_ns = ts;
    st->last_ts = ts;
    st->f = f;
    st->nnz = 0.0;
    st->k = 0;
    if (st->cap > 0) trace[0] = FistaSample{0, f, 0.0, ts};
    st->n_samples = 1;
    st->last_sampled = 0;
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

// ---------------------------------------------------------------------------
// dispatch over the pointer width

template <class Epi, typename PtrT>
void launch_p(const Csr& M, const double* x, const Epi& epi, cudaStream_t st) {
  static int grid_cap = 0;
  if (!grid_cap) {
    int per_sm = 0;
    L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_kernel<PtrT, Epi>, kThreads, 0));
    grid_cap = std::max(1, per_sm) * sm_count();
  }
  const uint64_t tiles = (M.lines + 31) / 32;
  const uint64_t blocks = (tiles + (kThreads / 32) - 1) / (kThreads / 32);
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)grid_cap));
  spmv_kernel<PtrT, Epi><<<grid, kThreads, 0, st>>>((const PtrT*)M.ptr, M.idx, M.val, x, M.lines, epi);
  L1B_LAUNCHED();
}

template <class Epi>
void launch(const Csr& M, const double* x, const Epi& epi, cudaStream_t st) {
  if (M.ptr32)
    launch_p<Epi, uint32_t>(M, x, epi, st);
  else
    launch_p<Epi, uint64_t>(M, x, epi, st);
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
  launch(At, fb.r_y, e, st);
}

void fista_k2(const Csr& A, const FistaBufs& fb, cudaStream_t st) {
  EpiFistaR e{fb.b, fb.r_x, fb.r_y, fb.st, fb.trace, fb.partials, 0.0, {0.0}};
  launch(A, fb.x, e, st);
}

}  // namespace l1b
