// k_bt.cu -- FISTA / ISTA with LPolicy::backtracking (solvers.cpp:99-120,
// 277-382): L seeded by the power iteration estimate_gram_lmax
// (linops.cpp:757-778), halved at every iteration and doubled until the
// quadratic upper bound holds.  The Lipschitz search is a data-dependent loop
// with one decision per trial, so this driver is host-led: per trial one
// prox kernel (the trial point and the sums the test needs), the matrix-free
// product (k_sweep.cu: the reference's own apply, bit for bit) and one
// residual kernel, then one 8-byte-vector read-back.  Element-wise arithmetic
// is the reference's; the sums are grid reductions (not left-to-right), which
// the test's 1e-12 relative slack absorbs.
#include <chrono>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "../../include/l1b.h"
#include "common.cuh"
#include "kernels.hpp"
#include "solvers.hpp"

namespace l1b {
namespace {

constexpr int kBtSums = 8;

// sum_i a_i * b_i (a == b: a sum of squares)
__global__ void bt_dot_kernel(const double* __restrict__ a, const double* __restrict__ b, uint64_t n,
                              double* partials, unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc[0] += a[i] * b[i];
  double tot[1];
  if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
}

// v /= s (estimate_gram_lmax's normalisation: a division, as in the reference)
__global__ void bt_div_kernel(double* v, uint64_t n, double s) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] /= s;
}

// trial = S(base - grad / L, tau / L) (solvers.cpp:325-328) and, for the
// bound test (:333-340) and the record: sum grad.d, sum d^2 (d = trial - base),
// #(trial != base), ||trial||_1, nnz(trial)
__global__ void bt_prox_kernel(const double* __restrict__ base, const double* __restrict__ grad,
                               double* __restrict__ trial, uint64_t n, double inv_l, double thr,
                               double* partials, unsigned int* ticket, double* out) {
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double bi = base[i], gi = grad[i];
    const double t = soft_threshold(bi - inv_l * gi, thr);
    trial[i] = t;
    const double d = t - bi;
    acc[0] += gi * d;
    acc[1] += d * d;
    acc[2] += t != bi ? 1.0 : 0.0;
    acc[3] += fabs(t);
    acc[4] += t != 0.0 ? 1.0 : 0.0;
  }
  double tot[5];
  if (grid_sum<5>(acc, partials, ticket, tot) && threadIdx.x == 0)
    for (int k = 0; k < 5; ++k) out[k] = tot[k];
}

// r -= b (:329-330) and sum r^2
__global__ void bt_resid_kernel(double* __restrict__ r, const double* __restrict__ b, uint64_t m,
                                double* partials, unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double ri = r[i] - b[i];
    r[i] = ri;
    acc[0] += ri * ri;
  }
  double tot[1];
  if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
}

// y = trial + beta (trial - x) (:351-353); r_y = (1 + beta) r_trial - beta r_x (:355-357)
__global__ void bt_momentum_kernel(const double* __restrict__ trial, const double* __restrict__ x,
                                   double* __restrict__ y, uint64_t n,
                                   const double* __restrict__ r_trial, const double* __restrict__ r_x,
                                   double* __restrict__ r_y, uint64_t m, double beta) {
  const uint64_t lim = n > m ? n : m;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lim;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < n) y[i] = trial[i] + beta * (trial[i] - x[i]);
    if (i < m) r_y[i] = (1.0 + beta) * r_trial[i] - beta * r_x[i];
  }
}

// rng.hpp:48-56 on the host (std::log / std::cos of the same libm as the reference)
double normal_draw(std::mt19937_64& r) {
  double u1;
  do {
    u1 = static_cast<double>(r() >> 11) * 0x1.0p-53;
  } while (u1 <= 0.0);
  const double u2 = static_cast<double>(r() >> 11) * 0x1.0p-53;
  constexpr double two_pi = 6.283185307179586476925286766559;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
}

struct BtScratch {
  double* partials = nullptr;
  unsigned int* tickets = nullptr;
  double* out = nullptr;  // kBtSums
  double* h = nullptr;    // pinned copy
  int grid = 0;
};

}  // namespace

// estimate_gram_lmax (linops.cpp:757-778): v from normal() draws of Rng(seed)
// (host, same libm), then `iters` rounds of v /= ||v||; w = A^T A v;
// lambda = v.w; v <-> w, with the reference's matrix-free products
double estimate_gram_lmax_device(const OpView& op, uint64_t m, uint64_t n, uint64_t iters, uint64_t seed,
                                 cudaStream_t st) {
  std::mt19937_64 rng(seed);
  std::vector<double> hv(n);
  for (auto& q : hv) q = normal_draw(rng);
  double *v = nullptr, *w = nullptr, *av = nullptr, *scratch = nullptr;
  unsigned int* ticket = nullptr;
  const int grid = grid_for(n);
  L1B_CUDA(cudaMallocAsync(&v, n * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&w, n * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&av, m * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&scratch, (grid + 1) * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&ticket, sizeof(unsigned int), st));
  L1B_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  L1B_CUDA(cudaMemcpyAsync(v, hv.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  auto dot = [&](const double* a, const double* b) {
    bt_dot_kernel<<<grid, kThreads, 0, st>>>(a, b, n, scratch + 1, ticket, scratch);
    L1B_LAUNCHED();
    double h = 0.0;
    L1B_CUDA(cudaMemcpyAsync(&h, scratch, sizeof(double), cudaMemcpyDeviceToHost, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    return h;
  };
  double lambda = 0.0;
  for (uint64_t it = 0; it < iters; ++it) {
    const double norm = std::sqrt(dot(v, v));
    if (norm == 0.0) break;
    bt_div_kernel<<<grid, kThreads, 0, st>>>(v, n, norm);
    L1B_LAUNCHED();
    sweep_apply(op, v, av, st);
    sweep_apply_transpose(op, av, w, st);
    lambda = dot(v, w);
    std::swap(v, w);
  }
  for (void* q : {(void*)v, (void*)w, (void*)av, (void*)scratch, (void*)ticket}) L1B_CUDA(cudaFreeAsync(q, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  return lambda;
}

void run_fista_backtracking(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
                            l1b_summary* sum, double* x_host, double* d_x) {
  const ProblemView v = problem_view(p, false);
  const OpView& op = *v.op;
  const uint64_t n = v.n, m = v.m;
  const double tau = v.tau;
  const bool accel = cfg->solver == L1B_FISTA;
  const char* name = accel ? "fista" : "ista";
  cudaStream_t st = v.stream;
  std::vector<void*> bufs;
  auto alloc = [&](double** q, uint64_t cnt) {
    L1B_CUDA(cudaMalloc((void**)q, std::max<uint64_t>(cnt, 1) * sizeof(double)));
    bufs.push_back(*q);
  };
  BtScratch S;
  S.grid = grid_for(std::max(n, m));
  double *x, *y, *grad, *trial, *r_x, *r_y, *r_trial;
  try {
    alloc(&x, n);
    alloc(&y, n);
    alloc(&grad, n);
    alloc(&trial, n);
    alloc(&r_x, m);
    alloc(&r_y, m);
    alloc(&r_trial, m);
    alloc(&S.partials, (uint64_t)S.grid * kBtSums);
    alloc(&S.out, kBtSums);
    L1B_CUDA(cudaMalloc(&S.tickets, 4 * sizeof(unsigned int)));
    bufs.push_back(S.tickets);
    L1B_CUDA(cudaMemsetAsync(S.tickets, 0, 4 * sizeof(unsigned int), st));
    L1B_CUDA(cudaMallocHost(&S.h, kBtSums * sizeof(double)));
    auto fetch = [&](int k) {
      L1B_CUDA(cudaMemcpyAsync(S.h, S.out, k * sizeof(double), cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
    };
    auto dot = [&](const double* a, const double* b, uint64_t len) {
      bt_dot_kernel<<<grid_for(len), kThreads, 0, st>>>(a, b, len, S.partials, S.tickets, S.out);
      L1B_LAUNCHED();
      fetch(1);
      return S.h[0];
    };
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };

    // LipschitzState (solvers.cpp:103-119): l_fixed wins; else the power iteration
    double lval = 0.0;
    bool bt = false;
    if (cfg->l_fixed > 0.0) {
      lval = cfg->l_fixed;
    } else {
      bt = true;
      const double est = estimate_gram_lmax_device(op, v.m, v.n, 30, l1b_mix_seed(cfg->seed, 0x4c6d6178ULL), st);
      lval = est > 0.0 ? est : 1.0;
    }
    const double lcap = lval * 0x1p60;

    std::vector<l1b_sample> out;
    double mv = 0.0;
    bool reached = false;
    double time_to = INFINITY, mv_to = INFINITY;
    auto sample = [&](uint64_t k, double f, double nnz, uint64_t extra) {
      l1b_sample s{k, elapsed(), f, (uint64_t)nnz, mv, extra};
      out.push_back(s);
      if (cfg->has_target && !reached && f <= cfg->target) {
        reached = true;
        time_to = s.elapsed_s;
        mv_to = s.matvecs;
      }
    };
    // x = 0; r_x = A x - b (:290-295)
    L1B_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), st));
    sweep_apply(op, x, r_x, st);
    mv += 1;
    bt_resid_kernel<<<S.grid, kThreads, 0, st>>>(r_x, v.b, m, S.partials, S.tickets, S.out);
    L1B_LAUNCHED();
    fetch(1);
    double f = 0.5 * S.h[0];
    if (!std::isfinite(f)) throw std::runtime_error(std::string(name) + ": objective diverged to a non-finite value");
    sample(0, f, 0.0, 0);
    L1B_CUDA(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    L1B_CUDA(cudaMemcpyAsync(r_y, r_x, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    double t_mom = 1.0;
    int status = L1B_ITER_BUDGET;
    uint64_t k = 0, last_sampled = 0;
    double nnz = 0.0;
    while (true) {
      if (cfg->has_target && f <= cfg->target) {
        status = L1B_TARGET_REACHED;
        break;
      }
      if (k >= cfg->max_iters) {
        status = L1B_ITER_BUDGET;
        break;
      }
      if (elapsed() > cfg->max_seconds) {
        status = L1B_TIME_BUDGET;
        break;
      }
      ++k;
      const double* base = accel ? y : x;
      const double* r_base = accel ? r_y : r_x;
      sweep_apply_transpose(op, r_base, grad, st);
      mv += 1;
      const double g_base = 0.5 * dot(r_base, r_base, m);
      if (bt) lval = std::max(lval * 0.5, 1e-12);
      uint64_t backtracks = 0;
      double sums[6];
      while (true) {  // :324-343
        const double inv_l = 1.0 / lval;
        bt_prox_kernel<<<grid_for(n), kThreads, 0, st>>>(base, grad, trial, n, inv_l, tau * inv_l, S.partials,
                                                         S.tickets + 1, S.out);
        L1B_LAUNCHED();
        sweep_apply(op, trial, r_trial, st);
        mv += 1;
        bt_resid_kernel<<<S.grid, kThreads, 0, st>>>(r_trial, v.b, m, S.partials + (uint64_t)S.grid * 5,
                                                     S.tickets + 2, S.out + 5);
        L1B_LAUNCHED();
        fetch(6);
        std::memcpy(sums, S.h, sizeof(sums));
        if (!bt) break;
        const double lhs = 0.5 * sums[5];
        double quad = g_base + sums[0];
        quad += 0.5 * lval * sums[1];
        if (lhs <= quad + 1e-12 * (std::abs(lhs) + std::abs(quad)) || lval >= lcap) break;
        lval *= 2.0;
        ++backtracks;
      }
      const bool fixed_point = sums[2] == 0.0;  // trial == base (:346)
      if (accel) {
        const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t_mom * t_mom));
        const double beta = (t_mom - 1.0) / t_next;
        bt_momentum_kernel<<<S.grid, kThreads, 0, st>>>(trial, x, y, n, r_trial, r_x, r_y, m, beta);
        L1B_LAUNCHED();
        t_mom = t_next;
      }
      std::swap(x, trial);  // x = trial; r_x = r_trial
      std::swap(r_x, r_trial);
      f = tau * sums[3] + 0.5 * sums[5];
      nnz = sums[4];
      if (!std::isfinite(f)) throw std::runtime_error(std::string(name) + ": objective diverged to a non-finite value");
      if (k <= 1000 || k % 10 == 0 || fixed_point) {
        sample(k, f, nnz, backtracks);
        last_sampled = k;
      }
      if (fixed_point) {
        status = L1B_TARGET_REACHED;
        break;
      }
    }
    if (last_sampled != k) sample(k, f, nnz, 0);
    std::memset(sum, 0, sizeof(*sum));
    sum->path = L1B_RAN_HOST_LED;
    for (size_t q = 0; q < out.size() && samples; ++q)
      if (q < cap) samples[q] = out[q];
    if (x_host) L1B_CUDA(cudaMemcpyAsync(x_host, x, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (d_x) L1B_CUDA(cudaMemcpyAsync(d_x, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    sum->status = status;
    sum->reached_target = reached;
    sum->time_to_target = time_to;
    sum->matvecs_to_target = mv_to;
    sum->final_objective = f;
    sum->elapsed_s = elapsed();
    sum->total_matvecs = mv;
    sum->n_samples = out.size();
    sum->iterations = k;
    if (status == L1B_TARGET_REACHED && !reached) {
      sum->reached_target = 1;
      sum->time_to_target = sum->elapsed_s;
      sum->matvecs_to_target = sum->total_matvecs;
    }
  } catch (...) {
    cudaStreamSynchronize(st);
    for (void* q : bufs) cudaFree(q);
    if (S.h) cudaFreeHost(S.h);
    throw;
  }
  for (void* q : bufs) cudaFree(q);
  cudaFreeHost(S.h);
}

}  // namespace l1b
