// k_ncg.cu -- Newton-CG on the pseudo-Huber smoothed problem (pdNCG, C3):
// newton_cg_run + pcg_solve (solvers.cpp:159-264, 487-568) on device.
//
// Per Newton step (host loop, one sync per step):
//   grad kernel  (CSC):  grad = A^T r + tau x/sqrt(mu^2+x^2), d2psi, precond,
//                        partials of ||x||_1, nnz, psi, ||grad||^2
//   PCG (device loop, four kernels per iteration, no host round trip):
//     Ka (CSR)  hav = A p
//     Kb (CSC)  hp  = A^T hav + tau d2psi p, p.hp -> alpha / breakdown
//     Kc        step += alpha p, r -= alpha hp, ||r||^2 and r.z partials ->
//               best / convergence / beta
//     Kd        best = step (if improved), p = z + beta p
//   ad = A step (CSR), slope = grad.step, then Armijo backtracking with
//   eight trial steps per pass (one fused reduction kernel for all eight).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "guard.hpp"
#include "solvers.hpp"
#include "spmv.cuh"

namespace l1b {

namespace {

constexpr int kLs = 8;  // trial steps evaluated per line-search pass

struct NcgDev {
  double tau, mu;
  // grad pass
  double l1, nnz, psi, gg;
  // PCG state (solvers.cpp:211-264)
  double rz, php, alpha, beta, rn, best_norm, rhs_norm, eta, rr_pcg, rz_next;
  uint64_t iterations, max_iters;
  int done, converged, negcurv, error, improved, pad;
  unsigned int ticket[4];
  double ls[2 * kLs];  // psi(x + a s), ||r + a ad||^2 per trial
  double slope;
};

// -- grad pass (solvers.cpp:522-529) ---------------------------------------
struct EpiGrad {
  const double* x;
  const double* gram;
  double* grad;
  double* d2psi;
  double* precond;
  NcgDev* st;
  double* partials;
  double tau, mu;
  double acc[4];  // ||x||_1, nnz(x), psi(x), ||grad||^2
  static constexpr int kVec = 2;  // x, diag(A^T A) at the column
  __host__ __device__ const double* vec(int v) const { return v == 0 ? x : gram; }
  __device__ bool skip() const { return false; }
  __device__ void start() {
    tau = st->tau;
    mu = st->mu;
    acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
  }
  __device__ void line(uint64_t j, double g, const double* pv) {
    const double xj = pv[0];
    const double q = mu * mu + xj * xj;
    const double root = sqrt(q);
    const double gj = g + tau * xj / root;
    const double d = mu * mu / (q * root);
    grad[j] = gj;
    d2psi[j] = d;
    precond[j] = tau * d + pv[1];
    acc[0] += fabs(xj);
    acc[1] += xj != 0.0 ? 1.0 : 0.0;
    acc[2] += root - mu;  // pseudo_huber term (solvers.cpp:162)
    acc[3] += gj * gj;
  }
  __device__ void finish() {
    double tot[4];
    if (grid_sum<4>(acc, partials, &st->ticket[0], tot) && threadIdx.x == 0) {
      st->l1 = tot[0];
      st->nnz = tot[1];
      st->psi = tot[2];
      st->gg = tot[3];
    }
  }
};

// -- PCG ----------------------------------------------------------------------
// r = rhs = -grad, z = r / precond, p = z, step = best = 0, rz = r.z
__global__ void pcg_init_kernel(const double* __restrict__ grad, const double* __restrict__ pre,
                                double* r, double* p, double* step, double* best, uint64_t n,
                                NcgDev* st, double* partials) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double ri = -grad[i];
    const double zi = ri / pre[i];
    r[i] = ri;
    p[i] = zi;
    step[i] = 0.0;
    best[i] = 0.0;
    acc[0] += ri * zi;
  }
  double tot[1];
  if (grid_sum<1>(acc, partials, &st->ticket[1], tot) && threadIdx.x == 0) {
    st->rz = tot[0];
    st->iterations = 0;
    st->best_norm = st->rhs_norm;
    st->done = st->rhs_norm == 0.0 || st->max_iters == 0;
    st->converged = st->rhs_norm == 0.0;
    st->negcurv = 0;
    st->error = 0;
    st->improved = 0;
  }
}

struct EpiHav {  // Ka: hav = A p
  double* hav;
  const NcgDev* st;
  static constexpr int kVec = 0;
  __host__ __device__ const double* vec(int) const { return nullptr; }
  __device__ bool skip() const { return *(volatile const int*)&st->done; }
  __device__ void start() {}
  __device__ void line(uint64_t i, double s, const double*) { hav[i] = s; }
  __device__ void finish() {}
};

struct EpiHp {  // Kb: hp = A^T hav + tau d2psi p  (solvers.cpp:537-541), p.hp
  const double* p;
  const double* d2psi;
  double* hp;
  NcgDev* st;
  double* partials;
  double tau;
  double acc[1];
  static constexpr int kVec = 2;  // p, d2psi at the column
  __host__ __device__ const double* vec(int v) const { return v == 0 ? p : d2psi; }
  __device__ bool skip() const { return *(volatile const int*)&st->done; }
  __device__ void start() {
    tau = st->tau;
    acc[0] = 0.0;
  }
  __device__ void line(uint64_t j, double g, const double* pv) {
    const double pj = pv[0];
    const double h = g + tau * pv[1] * pj;
    hp[j] = h;
    acc[0] += pj * h;
  }
  __device__ void finish() {
    double tot[1];
    if (grid_sum<1>(acc, partials, &st->ticket[2], tot) && threadIdx.x == 0) {
      const double php = tot[0];  // solvers.cpp:231-237
      st->php = php;
      if (!(php > 0.0)) {
        if (!isfinite(php)) st->error = 1;
        st->negcurv = 1;
        st->done = 1;
      } else {
        st->alpha = st->rz / php;
      }
    }
  }
};

// Kc: step += alpha p; r -= alpha hp (:238-241); ||r||, best, convergence;
// r.z for the next direction (:255-258)
__global__ void pcg_update_kernel(const double* __restrict__ p, const double* __restrict__ hp,
                                  const double* __restrict__ pre, double* step, double* r,
                                  uint64_t n, NcgDev* st, double* partials) {
  if (*(volatile int*)&st->done) return;
  const double alpha = st->alpha;
  double acc[2] = {0.0, 0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    step[i] += alpha * p[i];
    const double ri = r[i] - alpha * hp[i];
    r[i] = ri;
    acc[0] += ri * ri;
    acc[1] += ri * (ri / pre[i]);
  }
  double tot[2];
  if (grid_sum<2>(acc, partials, &st->ticket[3], tot) && threadIdx.x == 0) {
    const double rn = sqrt(tot[0]);
    st->iterations += 1;
    st->rn = rn;
    st->improved = 0;
    if (!isfinite(rn)) {
      st->error = 2;
      st->done = 1;
      return;
    }
    if (rn < st->best_norm) {
      st->best_norm = rn;
      st->improved = 1;
    }
    if (rn <= st->eta * st->rhs_norm) {
      st->converged = 1;
      st->done = 1;
      return;
    }
    st->rz_next = tot[1];
    st->beta = tot[1] / st->rz;
    st->rz = tot[1];
    if (st->iterations >= st->max_iters) st->done = 1;
  }
}

// Kd: best = step when improved (:245-248); p = z + beta p (:259).  Safe to
// re-run after the solve stopped: the copy is idempotent (step no longer
// changes) and p only moves while !done; the last block clears `improved` so
// trailing launches of a chunk return immediately.
__global__ void pcg_direction_kernel(const double* __restrict__ r, const double* __restrict__ pre,
                                     const double* __restrict__ step, double* p, double* best,
                                     uint64_t n, NcgDev* st, unsigned int* ticket) {
  const int improved = *(volatile int*)&st->improved;
  const bool more = !*(volatile int*)&st->done;
  if (!improved && !more) return;
  const double beta = st->beta;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (improved) best[i] = step[i];
    if (more) p[i] = r[i] / pre[i] + beta * p[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
      st->improved = 0;
      *ticket = 0u;
    }
  }
}

// -- PCG in one cooperative launch (small / medium n) -------------------------
// At C3 (n = 2^19) the four PCG kernels run 10-20 us each while the data of
// an iteration (~40 MB) sits in L2: the iteration is latency-bound.  This
// kernel runs the whole pcg_solve loop with four grid barriers per iteration;
// every block folds the per-block partials itself (same order everywhere, so
// all blocks take identical decisions) and block 0 writes the state back.
// Per-element formulas and line sums (ascending, from 0.0) are those of
// Ka..Kd; only the grouping of the three dot products differs.
struct PcgArgs {
  const void* a_ptr;
  const uint32_t* a_idx;
  const double* a_val;
  uint64_t a_lines;
  const void* t_ptr;
  const uint32_t* t_idx;
  const double* t_val;
  uint64_t n;
  const double *pre, *d2psi;
  double *p, *hav, *hp, *r, *step, *best;
  NcgDev* st;
  double* partials;  // >= 6 x grid doubles
  double* p2;        // second direction buffer (n)
};

template <int NS>
__device__ __forceinline__ void fold_partials(const double* partials, double (&tot)[NS]) {
#pragma unroll
  for (int k = 0; k < NS; ++k) tot[k] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NS; ++k) tot[k] += __ldcg(&partials[(size_t)b * NS + k]);
  }
  block_sum<NS>(tot);
  __shared__ double bc[NS];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) bc[k] = tot[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NS; ++k) tot[k] = bc[k];
  __syncthreads();
}

// sum_q val[q] * f(idx[q]) over [q0, q1), ascending from 0.0 (the SpMV line
// sum); K >= q1 - q0: all index / value loads are issued before the gathers
template <int K, typename PtrT, class F>
__device__ __forceinline__ double line_sum(PtrT q0, PtrT q1, const uint32_t* __restrict__ idx,
                                           const double* __restrict__ val, F f) {
  if constexpr (K == 0) {
    double sum = 0.0;
    for (PtrT q = q0; q < q1; ++q) sum += val[q] * f(idx[q]);
    return sum;
  } else {
    uint32_t c[K];
    double v[K], g[K];
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const bool in = q0 + e < q1;
      c[e] = in ? idx[q0 + e] : 0u;
      v[e] = in ? val[q0 + e] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < K; ++e) g[e] = q0 + e < q1 ? f(c[e]) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int e = 0; e < K; ++e)
      if (q0 + e < q1) sum += v[e] * g[e];
    return sum;
  }
}

template <typename PtrT, int K = 0>
__global__ void __launch_bounds__(kThreads) pcg_loop_kernel(PcgArgs P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  NcgDev* st = P.st;
  const PtrT* ap = static_cast<const PtrT*>(P.a_ptr);
  const PtrT* tp = static_cast<const PtrT*>(P.t_ptr);
  const uint64_t gsz = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const double tau = st->tau, eta = st->eta, rhs_norm = st->rhs_norm;
  const uint64_t max_iters = st->max_iters;
  double rz = st->rz, best_norm = st->best_norm, php = 0.0, alpha = 0.0, beta = 0.0, rn = 0.0;
  int done = st->done, converged = st->converged, negcurv = 0, error = 0, improved = 0;
  uint64_t it = 0;
  // p_k in pc; Kd of iteration k-1 (best copy, p_k = z + beta p_{k-1}) is folded
  // into Ka of iteration k: A p_k gathers p_k = r/pre + beta p_{k-1} on the fly
  // (the same operations as the stored p_k) while the owners write it to pn.
  // Two partial buffers (p.hp / the r sums) so that one fold needs no barrier.
  double* pc = P.p;
  double* pn = P.p2;
  double* part_b = P.partials;
  double* part_c = P.partials + 4 * (size_t)gridDim.x;
  bool first = true;
  while (!done) {
    if (first) {  // Ka: hav = A p_0
      for (uint64_t i = t0; i < P.a_lines; i += gsz)
        P.hav[i] = line_sum<K>(ap[i], ap[i + 1], P.a_idx, P.a_val,
                               [&](uint32_t c) { return __ldcg(pc + c); });
    } else {  // Kd of the last iteration + Ka
      for (uint64_t i = t0; i < P.n; i += gsz) {
        if (improved) P.best[i] = P.step[i];  // (:245-248)
        pn[i] = P.r[i] / P.pre[i] + beta * pc[i];  // p = z + beta p (:259)
      }
      for (uint64_t i = t0; i < P.a_lines; i += gsz)
        P.hav[i] = line_sum<K>(ap[i], ap[i + 1], P.a_idx, P.a_val, [&](uint32_t c) {
          return __ldcg(P.r + c) / P.pre[c] + beta * __ldcg(pc + c);
        });
      double* t = pc;
      pc = pn;
      pn = t;
    }
    first = false;
    grid.sync();
    // Kb: hp = A^T hav + tau d2psi p (solvers.cpp:537-541), p.hp
    {
      double acc[1] = {0.0};
      for (uint64_t j = t0; j < P.n; j += gsz) {
        const double g = line_sum<K>(tp[j], tp[j + 1], P.t_idx, P.t_val,
                                     [&](uint32_t c) { return __ldcg(P.hav + c); });
        const double pj = pc[j];
        const double h = g + tau * P.d2psi[j] * pj;
        P.hp[j] = h;
        acc[0] += pj * h;
      }
      block_sum<1>(acc);
      if (threadIdx.x == 0) part_b[blockIdx.x] = acc[0];
    }
    grid.sync();
    {
      double tot[1];
      fold_partials<1>(part_b, tot);
      php = tot[0];  // solvers.cpp:231-237
    }
    improved = 0;
    if (!(php > 0.0)) {
      if (!isfinite(php)) error = 1;
      negcurv = 1;
      done = 1;
      break;
    }
    alpha = rz / php;
    // Kc: step += alpha p; r -= alpha hp (:238-241); ||r||^2, r.z
    {
      double acc[2] = {0.0, 0.0};
      for (uint64_t i = t0; i < P.n; i += gsz) {
        P.step[i] += alpha * pc[i];
        const double ri = P.r[i] - alpha * P.hp[i];
        P.r[i] = ri;
        acc[0] += ri * ri;
        acc[1] += ri * (ri / P.pre[i]);
      }
      block_sum<2>(acc);
      if (threadIdx.x == 0) {
        part_c[(size_t)blockIdx.x * 2] = acc[0];
        part_c[(size_t)blockIdx.x * 2 + 1] = acc[1];
      }
    }
    grid.sync();
    double tot[2];
    fold_partials<2>(part_c, tot);
    rn = sqrt(tot[0]);
    ++it;
    if (!isfinite(rn)) {
      error = 2;
      done = 1;
      break;
    }
    if (rn < best_norm) {
      best_norm = rn;
      improved = 1;
    }
    if (rn <= eta * rhs_norm) {
      converged = 1;
      done = 1;
    } else {
      beta = tot[1] / rz;
      rz = tot[1];
      if (it >= max_iters) done = 1;
    }
  }
  // Kd of the last iteration: the best-iterate copy only
  if (improved)
    for (uint64_t i = t0; i < P.n; i += gsz) P.best[i] = P.step[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rz = rz;
    st->php = php;
    st->alpha = alpha;
    st->beta = beta;
    st->rn = rn;
    st->best_norm = best_norm;
    st->iterations = it;
    st->done = 1;
    st->converged = converged;
    st->negcurv = negcurv;
    st->error = error;
    st->improved = 0;
  }
}

// -- PCG for one right stage (C1-C3's operators): pair-local products --------
// With a single Givens stage, no left stages and identity permutations,
// A p = Sigma G^T p (rows >= n empty) and A^T A p = G Sigma Sigma G^T p act on
// disjoint pairs (a, a + 1), a = 2u - offset: the Hessian-vector product of a
// pair needs only that pair.  Each thread owns P pairs for the whole solve and
// keeps p, r, step and hp in registers; an iteration is the pair-local
// hessvec (the reference's own sweep arithmetic: OperatorSpec::apply /
// apply_transpose, linops.cpp:422-473) and two grid-wide sums (p.hp, then
// ||r||^2 and r.z), i.e. two grid barriers instead of three, with no gathers.
struct PcgPairArgs {
  uint64_t n;
  int off;
  double c, s;
  const double *sigma, *pre, *d2psi;
  const double *p, *r;  // p_0, r_0 (pcg_init_kernel)
  double *step, *best;
  NcgDev* st;
  double* partials;  // >= 3 x grid doubles
};

// The Hessian-vector product of one pair (a, a + 1) of a single-stage
// operator (solvers.cpp:536-540 with OperatorSpec::apply / apply_transpose,
// linops.cpp:422-473): w = G Sigma^T Sigma G^T v, h = w + tau d2psi v.
// pair = both entries exist (else the lone entry is not rotated).
__device__ __forceinline__ void pair_hessvec(double v0, double v1, bool pair, double c, double s, double s0,
                                             double s1, double d0, double d1, double tau, double& h0,
                                             double& h1) {
  double u0 = v0, u1 = v1;
  if (pair) rotate_pair(u0, u1, c, s, true);  // G^T v
  double w0 = s0 * (s0 * u0), w1 = s1 * (s1 * u1);  // Sigma^T (Sigma G^T v)
  if (pair) rotate_pair(w0, w1, c, s, false);      // G (...)
  h0 = w0 + tau * d0 * v0;
  h1 = w1 + tau * d1 * v1;
}

// d2psi of the pseudo-Huber term, as the gradient pass forms it (EpiGrad)
__device__ __forceinline__ double huber_d2(double xj, double mu) {
  const double q = mu * mu + xj * xj;
  const double root = sqrt(q);
  return mu * mu / (q * root);
}

// l1b_smoothed_hessvec, single-stage operators: one thread per pair
__global__ void hessvec_pair_kernel(uint64_t n, int off, double c, double s, const double* __restrict__ sigma,
                                    const double* __restrict__ x, const double* __restrict__ v, double mu,
                                    double tau, double* __restrict__ out) {
  const uint64_t U = (n + 2) / 2;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < U;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t a = 2 * (int64_t)u - off;
    const bool va = a >= 0 && a < (int64_t)n, vb = a + 1 >= 0 && a + 1 < (int64_t)n;
    const double v0 = va ? v[a] : 0.0, v1 = vb ? v[a + 1] : 0.0;
    const double d0 = va ? huber_d2(x[a], mu) : 0.0, d1 = vb ? huber_d2(x[a + 1], mu) : 0.0;
    double h0, h1;
    pair_hessvec(v0, v1, va && vb, c, s, va ? sigma[a] : 0.0, vb ? sigma[a + 1] : 0.0, d0, d1, tau, h0, h1);
    if (va) out[a] = h0;
    if (vb) out[a + 1] = h1;
  }
}

// l1b_smoothed_hessvec, other operators: out = A^T (A v) (sweeps) + tau d2psi v
__global__ void hessvec_diag_kernel(uint64_t n, const double* __restrict__ x, const double* __restrict__ v,
                                    double mu, double tau, double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] += tau * huber_d2(x[i], mu) * v[i];
}

template <int P, int BT = kThreads>
__global__ void __launch_bounds__(BT) pcg_pair_kernel(PcgPairArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  // sigma, d2psi, precond of the thread's entries, constant during the solve:
  // thread-private slots of shared memory ([k][e][thread]: conflict-free)
  extern __shared__ double cst[];
  double* c_sig = cst;
  double* c_d2 = cst + 2 * P * BT;
  double* c_pre = cst + 4 * P * BT;
  NcgDev* st = A.st;
  const int64_t n = (int64_t)A.n;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t g0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const int tid = threadIdx.x;
  const double c = A.c, s = A.s;
  const double tau = st->tau, eta = st->eta, rhs_norm = st->rhs_norm;
  const uint64_t max_iters = st->max_iters;
  double rz = st->rz, best_norm = st->best_norm, php = 0.0, alpha = 0.0, beta = 0.0, rn = 0.0;
  int done = st->done, converged = st->converged, negcurv = 0, error = 0;
  uint64_t it = 0;
  double p[P][2], r[P][2], stp[P][2], hp[P][2];
  int64_t a[P];
  bool va[P], vb[P];
  auto slot = [&](int k, int e) { return (2 * k + e) * BT + tid; };
#pragma unroll
  for (int k = 0; k < P; ++k) {
    a[k] = 2 * (int64_t)(g0 + (uint64_t)k * T) - A.off;
    va[k] = a[k] >= 0 && a[k] < n;
    vb[k] = a[k] + 1 >= 0 && a[k] + 1 < n;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool v = e == 0 ? va[k] : vb[k];
      const int64_t i = a[k] + e;
      p[k][e] = v ? A.p[i] : 0.0;
      r[k][e] = v ? A.r[i] : 0.0;
      stp[k][e] = 0.0;  // step_0 = 0 (pcg_init_kernel)
      c_sig[slot(k, e)] = v ? A.sigma[i] : 0.0;
      c_d2[slot(k, e)] = v ? A.d2psi[i] : 0.0;
      c_pre[slot(k, e)] = v ? A.pre[i] : 1.0;
    }
  }
  double* part_b = A.partials;
  double* part_c = A.partials + (size_t)gridDim.x;
  while (!done) {
    // hessvec (solvers.cpp:536-540): hav = A p, hp = A^T hav + tau d2psi p; p.hp
    double acc[1] = {0.0};
#pragma unroll
    for (int k = 0; k < P; ++k) {
      pair_hessvec(p[k][0], p[k][1], va[k] && vb[k], c, s, c_sig[slot(k, 0)], c_sig[slot(k, 1)],
                   c_d2[slot(k, 0)], c_d2[slot(k, 1)], tau, hp[k][0], hp[k][1]);
      if (va[k]) acc[0] += p[k][0] * hp[k][0];
      if (vb[k]) acc[0] += p[k][1] * hp[k][1];
    }
    block_sum<1>(acc);
    if (tid == 0) part_b[blockIdx.x] = acc[0];
    grid.sync();
    {
      double tot[1];
      fold_partials<1>(part_b, tot);
      php = tot[0];  // solvers.cpp:231-237
    }
    if (!(php > 0.0)) {
      if (!isfinite(php)) error = 1;
      negcurv = 1;
      break;
    }
    alpha = rz / php;
    // step += alpha p; r -= alpha hp (:238-241); ||r||^2 and r.z, z = r / pre
    // kept for the direction update
    double acc2[2] = {0.0, 0.0};
    double z[P][2];
#pragma unroll
    for (int k = 0; k < P; ++k) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        stp[k][e] += alpha * p[k][e];
        const double ri = r[k][e] - alpha * hp[k][e];
        r[k][e] = ri;
        z[k][e] = ri / c_pre[slot(k, e)];
        if (e == 0 ? va[k] : vb[k]) {
          acc2[0] += ri * ri;
          acc2[1] += ri * z[k][e];
        }
      }
    }
    block_sum<2>(acc2);
    if (tid == 0) {
      part_c[(size_t)blockIdx.x * 2] = acc2[0];
      part_c[(size_t)blockIdx.x * 2 + 1] = acc2[1];
    }
    grid.sync();
    double tot[2];
    fold_partials<2>(part_c, tot);
    rn = sqrt(tot[0]);
    ++it;
    if (!isfinite(rn)) {
      error = 2;
      break;
    }
    if (rn < best_norm) {  // best = step (:245-248)
      best_norm = rn;
#pragma unroll
      for (int k = 0; k < P; ++k) {
        if (va[k]) A.best[a[k]] = stp[k][0];
        if (vb[k]) A.best[a[k] + 1] = stp[k][1];
      }
    }
    if (rn <= eta * rhs_norm) {
      converged = 1;
      break;
    }
    beta = tot[1] / rz;  // (:255-259)
    rz = tot[1];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      p[k][0] = z[k][0] + beta * p[k][0];
      p[k][1] = z[k][1] + beta * p[k][1];
    }
    if (it >= max_iters) break;
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    if (va[k]) A.step[a[k]] = stp[k][0];
    if (vb[k]) A.step[a[k] + 1] = stp[k][1];
  }
  if (blockIdx.x == 0 && tid == 0) {
    st->rz = rz;
    st->php = php;
    st->alpha = alpha;
    st->beta = beta;
    st->rn = rn;
    st->best_norm = best_norm;
    st->iterations = it;
    st->done = 1;
    st->converged = converged;
    st->negcurv = negcurv;
    st->error = error;
    st->improved = 0;
  }
}

template <int P, int BT = kThreads>
constexpr int pair_smem() {
  return 6 * P * BT * (int)sizeof(double);
}

// pairs per thread and grid of the pair-local PCG loop for n entries (0: the
// operator or n does not fit; L1B_PCG_PAIR=0 disables it)
struct PairPlan {
  int P = 0, grid = 0, bt = kThreads;
};
template <int P, int BT = kThreads>
int pair_capacity() {
  static const int cap = [] {
    int per_sm = 0;
    if (cudaFuncSetAttribute(pcg_pair_kernel<P, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             pair_smem<P, BT>()) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_pair_kernel<P, BT>, BT, pair_smem<P, BT>()) !=
            cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return per_sm * sm_count();
  }();
  return cap;
}
bool e_persist_on() {
  const char* e = getenv("L1B_PERSIST");
  return !(e && e[0] == '0');
}
PairPlan pcg_pair_plan(const ProblemView& v) {
  PairPlan pl;
  const char* e = getenv("L1B_PCG_PAIR");
  if (e && e[0] == '0') return pl;
  const OpView* op = v.op;
  if (!op || v.shard || op->right.count != 1 || op->left.count != 0 || op->p1 || op->p2 || v.m < v.n)
    return pl;
  const uint64_t units = (v.n + 2) / 2;
  auto try_p = [&](int P, int cap, int bt = kThreads) {
    const uint64_t per = (uint64_t)P * bt;
    const uint64_t g = (units + per - 1) / per;
    if (!pl.P && cap > 0 && g <= (uint64_t)cap) {
      pl.P = P;
      pl.grid = (int)g;
      pl.bt = bt;
    }
  };
  // four pairs per thread: 512-thread CTAs (one per SM, fewer partials per
  // barrier; C3 42.3 -> 39.7 ms against 256-thread CTAs)
  try_p(1, pair_capacity<1>());
  try_p(2, pair_capacity<2>());
  try_p(4, pair_capacity<4, 512>(), 512);
  try_p(8, pair_capacity<8>());
  return pl;
}

// grid of the cooperative PCG loop (0: not applicable -> the four-kernel loop)
template <typename PtrT, int K>
int pcg_loop_grid() {
  static const int cap = [] {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_loop_kernel<PtrT, K>, kThreads, 0) !=
        cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    // all co-resident CTAs (measured at C3: 1/2/4/8 per SM -> 49/31/27/27 us per
    // PCG iteration)
    return std::min(per_sm * sm_count(), spmv_grid_max());
  }();
  return cap;
}

// -- line search (solvers.cpp:551-560): eight trials per pass ---------------
__global__ void ls_eval_kernel(const double* __restrict__ x, const double* __restrict__ s,
                               const double* __restrict__ r, const double* __restrict__ ad,
                               uint64_t n, uint64_t m_act, double alpha0, NcgDev* st,
                               double* partials, unsigned int* ticket) {
  double acc[2 * kLs];
#pragma unroll
  for (int k = 0; k < 2 * kLs; ++k) acc[k] = 0.0;
  const double mu = st->mu;
  const uint64_t lim = n > m_act ? n : m_act;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lim;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double a = alpha0;
    if (i < n) {
      const double xi = x[i], si = s[i];
#pragma unroll
      for (int k = 0; k < kLs; ++k) {
        const double xt = xi + a * si;  // x_trial (:554)
        acc[k] += sqrt(mu * mu + xt * xt) - mu;
        a *= 0.5;
      }
    }
    a = alpha0;
    if (i < m_act) {
      const double ri = r[i], di = ad[i];
#pragma unroll
      for (int k = 0; k < kLs; ++k) {
        const double rt = ri + a * di;  // r_trial (:555)
        acc[kLs + k] += rt * rt;
        a *= 0.5;
      }
    }
  }
  double tot[2 * kLs];
  if (grid_sum<2 * kLs>(acc, partials, ticket, tot) && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 2 * kLs; ++k) st->ls[k] = tot[k];
  }
}

__global__ void ls_accept_kernel(double* x, const double* __restrict__ s, double* r,
                                 const double* __restrict__ ad, uint64_t n, uint64_t m_act,
                                 double alpha) {
  const uint64_t lim = n > m_act ? n : m_act;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lim;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < n) x[i] = x[i] + alpha * s[i];
    if (i < m_act) r[i] = r[i] + alpha * ad[i];
  }
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, uint64_t n,
                           double* partials, unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc[0] += a[i] * b[i];
  double tot[1];
  if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
}

__global__ void neg_residual_kernel(const double* __restrict__ b, double* r, uint64_t m) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    r[i] = 0.0 - b[i];
}

}  // namespace

void run_newton_cg(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
                   l1b_summary* sum, double* x_host, double* d_x) {
  const ProblemView v = problem_view(p);
  const uint64_t n = v.n, m = v.m, ma = v.A.lines;
  const double tau = v.tau, mu = cfg->mu;
  cudaStream_t st = v.stream;
  const double* gram = problem_gram(p);
  std::vector<void*> bufs;
  auto alloc = [&](auto** ptr, size_t bytes) {
    L1B_CUDA(cudaMalloc((void**)ptr, std::max<size_t>(bytes, 8)));
    bufs.push_back((void*)*ptr);
  };
  double *x, *r, *grad, *d2psi, *pre, *ad, *hav, *rp, *pp, *pp2, *hp, *step, *best, *partials, *scal;
  unsigned int* tickets;
  NcgDev* dst;
  NcgDev* h = nullptr;
  std::vector<l1b_sample> out;
  auto fail = [&]() {
    cudaStreamSynchronize(st);
    for (void* q : bufs) cudaFree(q);
    if (h) cudaFreeHost(h);
  };
  try {
    alloc(&x, n * 8);
    alloc(&r, m * 8);
    alloc(&grad, n * 8);
    alloc(&d2psi, n * 8);
    alloc(&pre, n * 8);
    alloc(&ad, m * 8);
    alloc(&hav, m * 8);
    alloc(&rp, n * 8);
    alloc(&pp, n * 8);
    alloc(&pp2, n * 8);
    alloc(&hp, n * 8);
    alloc(&step, n * 8);
    alloc(&best, n * 8);
    alloc(&partials, (size_t)spmv_grid_max() * 2 * kLs * 8);
    alloc(&scal, 8 * 8);
    alloc(&tickets, 8 * 4);
    alloc(&dst, sizeof(NcgDev));
    L1B_CUDA(cudaMallocHost(&h, sizeof(NcgDev)));
    L1B_CUDA(cudaMemsetAsync(tickets, 0, 8 * 4, st));
    L1B_CUDA(cudaMemsetAsync(x, 0, n * 8, st));
    L1B_CUDA(cudaMemsetAsync(ad, 0, m * 8, st));
    std::memset(h, 0, sizeof(NcgDev));
    h->tau = tau;
    h->mu = mu;
    h->eta = cfg->eta;
    h->max_iters = cfg->pcg_max_iters;
    L1B_CUDA(cudaMemcpyAsync(dst, h, sizeof(NcgDev), cudaMemcpyHostToDevice, st));
    // cooperative PCG loop for small / medium n (L1B_PERSIST=0: four kernels)
    int coop_grid = 0, pcg_k = 0;
    {
      const char* e = getenv("L1B_PERSIST");
      if (!(e && e[0] == '0') && n <= (1ull << 21) && v.A.ptr32 == v.At.ptr32) {
        // lines of <= 2 / 4 entries (1 / 2 stages): unrolled gathers
        const uint64_t lmax = std::max<uint64_t>(v.max_row_nnz, v.max_col_nnz);
        pcg_k = lmax <= 2 ? 2 : lmax <= 4 ? 4 : 0;
        if (v.A.ptr32)
          coop_grid = pcg_k == 2 ? pcg_loop_grid<uint32_t, 2>() : pcg_k == 4 ? pcg_loop_grid<uint32_t, 4>()
                                                                            : pcg_loop_grid<uint32_t, 0>();
        else
          coop_grid = pcg_k == 2 ? pcg_loop_grid<uint64_t, 2>() : pcg_k == 4 ? pcg_loop_grid<uint64_t, 4>()
                                                                            : pcg_loop_grid<uint64_t, 0>();
      }
    }
    const PairPlan pair = (e_persist_on() ? pcg_pair_plan(v) : PairPlan{});
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] {
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    uint64_t mv = 0;  // CountingOperator
    // grad_tol = grad_tol_rel * max(1, ||A^T b||) (solvers.cpp:498-500)
    spmv(v.At, v.b, grad, st);
    ++mv;
    dot_kernel<<<grid_for(n), kThreads, 0, st>>>(grad, grad, n, partials, tickets + 4, scal);
    L1B_LAUNCHED();
    double atb_sq = 0.0;
    L1B_CUDA(cudaMemcpyAsync(&atb_sq, scal, 8, cudaMemcpyDeviceToHost, st));
    // r = A*0 - b (:503-505)
    neg_residual_kernel<<<grid_for(m), kThreads, 0, st>>>(v.b, r, m);
    L1B_LAUNCHED();
    ++mv;
    dot_kernel<<<grid_for(ma), kThreads, 0, st>>>(r, r, ma, partials, tickets + 4, scal + 1);
    L1B_LAUNCHED();
    double rr = 0.0;
    L1B_CUDA(cudaMemcpyAsync(&rr, scal + 1, 8, cudaMemcpyDeviceToHost, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    rr += v.tail_sq;
    const double grad_tol = cfg->grad_tol_rel * std::max(1.0, std::sqrt(atb_sq));
    int status = L1B_ITER_BUDGET;
    uint64_t newton = 0, last_pcg = 0, total_pcg = 0;
    bool reached = false;
    double time_to = INFINITY, mv_to = INFINITY, f_last = NAN;
    while (true) {
      // grad pass: also yields ||x||_1, nnz, psi for f_true / f_smooth
      launch(v.At, r, EpiGrad{x, gram, grad, d2psi, pre, dst, partials, 0, 0, {0, 0, 0, 0}}, st);
      L1B_CUDA(cudaMemcpyAsync(h, dst, sizeof(NcgDev), cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
      ++mv;
      const double f_true = tau * h->l1 + 0.5 * rr;  // :515
      if (!std::isfinite(f_true))
        throw std::runtime_error("newton_cg: objective diverged to a non-finite value");
      l1b_sample smp{newton, elapsed(), f_true, (uint64_t)h->nnz, (double)(mv - 1), last_pcg};
      out.push_back(smp);
      f_last = f_true;
      if (!reached && cfg->has_target && f_true <= cfg->target) {
        reached = true;
        time_to = smp.elapsed_s;
        mv_to = smp.matvecs;
      }
      if (cfg->has_target && f_true <= cfg->target) {
        status = L1B_TARGET_REACHED;
        break;
      }
      const double f_smooth = tau * h->psi + 0.5 * rr;  // :521
      if (std::sqrt(h->gg) <= grad_tol) {
        status = L1B_TARGET_REACHED;
        break;
      }
      if (newton >= cfg->max_iters) {
        status = L1B_ITER_BUDGET;
        break;
      }
      if (elapsed() > cfg->max_seconds) {
        status = L1B_TIME_BUDGET;
        break;
      }
      ++newton;
      // ---- PCG (solvers.cpp:202-264) on device
      h->rhs_norm = std::sqrt(h->gg);
      L1B_CUDA(cudaMemcpyAsync(&dst->rhs_norm, &h->rhs_norm, 8, cudaMemcpyHostToDevice, st));
      pcg_init_kernel<<<grid_for(n), kThreads, 0, st>>>(grad, pre, rp, pp, step, best, n, dst, partials);
      L1B_LAUNCHED();
      uint64_t launched = 0, chunk = 4;
      if (pair.P) {  // single stage: pair-local products, one cooperative launch
        PcgPairArgs pa{n, v.op->right.offset[0], v.op->right.c[0], v.op->right.s[0], v.op->sigma, pre, d2psi,
                       pp, rp, step, best, dst, partials};
        void* args[] = {&pa};
        const bool wide = pair.bt == 512;
        const void* fn = wide            ? (const void*)pcg_pair_kernel<4, 512>
                         : pair.P == 1   ? (const void*)pcg_pair_kernel<1>
                         : pair.P == 2   ? (const void*)pcg_pair_kernel<2>
                         : pair.P == 4   ? (const void*)pcg_pair_kernel<4>
                                         : (const void*)pcg_pair_kernel<8>;
        const int smem = wide            ? pair_smem<4, 512>()
                         : pair.P == 1   ? pair_smem<1>()
                         : pair.P == 2   ? pair_smem<2>()
                         : pair.P == 4   ? pair_smem<4>()
                                         : pair_smem<8>();
        L1B_CUDA(cudaLaunchCooperativeKernel(fn, dim3(pair.grid), dim3(pair.bt), args, smem, st));
        L1B_LAUNCHED();
        launched = cfg->pcg_max_iters;
      } else if (coop_grid > 0) {  // the whole solve in one cooperative launch
        PcgArgs pa{v.A.ptr, v.A.idx, v.A.val, v.A.lines, v.At.ptr, v.At.idx, v.At.val, n,
                   pre, d2psi, pp, hav, hp, rp, step, best, dst, partials, pp2};
        void* args[] = {&pa};
        const void* fn =
            v.A.ptr32 ? (pcg_k == 2   ? (const void*)pcg_loop_kernel<uint32_t, 2>
                         : pcg_k == 4 ? (const void*)pcg_loop_kernel<uint32_t, 4>
                                      : (const void*)pcg_loop_kernel<uint32_t, 0>)
                      : (pcg_k == 2   ? (const void*)pcg_loop_kernel<uint64_t, 2>
                         : pcg_k == 4 ? (const void*)pcg_loop_kernel<uint64_t, 4>
                                      : (const void*)pcg_loop_kernel<uint64_t, 0>);
        L1B_CUDA(cudaLaunchCooperativeKernel(fn, dim3(coop_grid), dim3(kThreads), args, 0, st));
        L1B_LAUNCHED();
        launched = cfg->pcg_max_iters;  // skip the four-kernel loop
      }
      while (launched < cfg->pcg_max_iters) {
        const uint64_t k = std::min<uint64_t>(chunk, cfg->pcg_max_iters - launched);
        for (uint64_t it = 0; it < k; ++it) {
          launch(v.A, pp, EpiHav{hav, dst}, st);
          launch(v.At, hav, EpiHp{pp, d2psi, hp, dst, partials, 0.0, {0.0}}, st);
          pcg_update_kernel<<<grid_for(n), kThreads, 0, st>>>(pp, hp, pre, step, rp, n, dst, partials);
          L1B_LAUNCHED();
          pcg_direction_kernel<<<grid_for(n), kThreads, 0, st>>>(rp, pre, step, pp, best, n, dst, tickets + 6);
          L1B_LAUNCHED();
        }
        launched += k;
        L1B_CUDA(cudaMemcpyAsync(h, dst, sizeof(NcgDev), cudaMemcpyDeviceToHost, st));
        L1B_CUDA(cudaStreamSynchronize(st));
        if (h->done) break;
        chunk = std::min<uint64_t>(chunk * 2, 64);
      }
      L1B_CUDA(cudaMemcpyAsync(h, dst, sizeof(NcgDev), cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
      if (h->error == 1) throw std::runtime_error("pcg_solve: breakdown, non-finite curvature");
      if (h->error == 2) throw std::runtime_error("pcg_solve: breakdown, non-finite residual");
      const uint64_t pcg_it = h->iterations;
      mv += 2 * pcg_it;
      last_pcg = pcg_it;
      total_pcg += pcg_it;
      // converged -> the current step; otherwise the best iterate (:250-263)
      double* s = (h->converged && !h->negcurv) ? step : best;
      if (h->rhs_norm == 0.0) s = step;
      // ad = A s (:546), slope = grad.s (:547)
      spmv(v.A, s, ad, st);
      ++mv;
      dot_kernel<<<grid_for(n), kThreads, 0, st>>>(grad, s, n, partials, tickets + 4, scal + 2);
      L1B_LAUNCHED();
      double slope = 0.0;
      L1B_CUDA(cudaMemcpyAsync(&slope, scal + 2, 8, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
      // Armijo backtracking (:551-560), the last trial accepted at the cap
      double alpha = 1.0, alpha0 = 1.0, rr_acc = rr;
      uint64_t bt = 0;
      bool accepted = false;
      while (!accepted) {
        ls_eval_kernel<<<grid_for(std::max(n, ma)), kThreads, 0, st>>>(x, s, r, ad, n, ma, alpha0, dst,
                                                                      partials, tickets + 5);
        L1B_LAUNCHED();
        L1B_CUDA(cudaMemcpyAsync(h, dst, sizeof(NcgDev), cudaMemcpyDeviceToHost, st));
        L1B_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < kLs; ++k) {
          const double rrt = h->ls[kLs + k] + v.tail_sq;
          const double f_trial = tau * h->ls[k] + 0.5 * rrt;
          if (f_trial <= f_smooth + 1e-4 * alpha * slope || bt >= cfg->ls_max_backtracks) {
            accepted = true;
            rr_acc = rrt;
            break;
          }
          alpha *= 0.5;
          ++bt;
        }
        alpha0 = alpha;
      }
      ls_accept_kernel<<<grid_for(std::max(n, ma)), kThreads, 0, st>>>(x, s, r, ad, n, ma, alpha);
      L1B_LAUNCHED();
      rr = rr_acc;
    }
    std::memset(sum, 0, sizeof(*sum));
    sum->path = pair.P ? L1B_RAN_PCG_PAIR : coop_grid > 0 ? L1B_RAN_PCG_LOOP : L1B_RAN_PCG_KERNELS;
    for (size_t q = 0; q < out.size() && samples; ++q)
      if (q < cap) samples[q] = out[q];
    if (x_host) L1B_CUDA(cudaMemcpyAsync(x_host, x, n * 8, cudaMemcpyDeviceToHost, st));
    if (d_x) L1B_CUDA(cudaMemcpyAsync(d_x, x, n * 8, cudaMemcpyDeviceToDevice, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    sum->status = status;
    sum->reached_target = reached;
    sum->time_to_target = time_to;
    sum->matvecs_to_target = mv_to;
    sum->final_objective = f_last;
    sum->elapsed_s = elapsed();
    sum->total_matvecs = (double)mv;
    sum->total_pcg_iterations = total_pcg;
    sum->newton_steps = newton;
    sum->n_samples = out.size();
    sum->iterations = newton;
    if (status == L1B_TARGET_REACHED && !reached) {
      sum->reached_target = 1;
      sum->time_to_target = sum->elapsed_s;
      sum->matvecs_to_target = sum->total_matvecs;
    }
  } catch (...) {
    fail();
    throw;
  }
  fail();
}

// The Newton-CG Hessian-vector product at x (l1b_smoothed_hessvec): the
// pair-local arithmetic of pcg_pair_kernel for single-stage operators, the
// reference's sweeps (+ the same d2psi epilogue) otherwise.
void smoothed_hessvec(l1b_problem* p, double mu, const double* x, const double* v, double* out) {
  const ProblemView pv = problem_view(p, false);
  if (pv.shard) throw Unsupported("smoothed_hessvec: whole problems only");
  if (!(mu > 0.0)) throw InvalidArgument("pseudo_huber: mu must be positive");
  const OpView* op = pv.op;
  cudaStream_t st = pv.stream;
  if (op->right.count == 1 && op->left.count == 0 && !op->p1 && !op->p2 && pv.m >= pv.n) {
    hessvec_pair_kernel<<<grid_for((pv.n + 2) / 2), kThreads, 0, st>>>(
        pv.n, op->right.offset[0], op->right.c[0], op->right.s[0], op->sigma, x, v, mu, pv.tau, out);
    L1B_LAUNCHED();
  } else {
    double* av = nullptr;
    L1B_CUDA(cudaMallocAsync((void**)&av, pv.m * sizeof(double), st));
    sweep_apply(*op, v, av, st);
    sweep_apply_transpose(*op, av, out, st);
    hessvec_diag_kernel<<<grid_for(pv.n), kThreads, 0, st>>>(pv.n, x, v, mu, pv.tau, out);
    L1B_LAUNCHED();
    L1B_CUDA(cudaFreeAsync(av, st));
  }
  L1B_CUDA(cudaStreamSynchronize(st));
}

}  // namespace l1b

extern "C" int l1b_smoothed_hessvec(l1b_problem* p, double mu, const double* d_x, const double* d_v,
                                    double* d_out) {
  return l1b::guard([&] {
    if (!p || !d_x || !d_v || !d_out) throw l1b::InvalidArgument("null argument");
    l1b::smoothed_hessvec(p, mu, d_x, d_v, d_out);
  });
}
