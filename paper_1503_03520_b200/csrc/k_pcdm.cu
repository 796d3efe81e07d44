// k_pcdm.cu -- randomised (block) coordinate descent on device.
//
// L1B_PCDM: block PCDM, the C2 mapping of SURVEY.md 8(d): an epoch is
//   floor(n/B) blocks of B distinct coordinates drawn from the
//   uniform_index(rng, n) stream (duplicates inside a block redrawn); all B
//   coordinates of a block take the CD model step of solvers.cpp:457-461
//   against the same residual (one thread each, B "processors"), beta =
//   cd_damping(omega, B, n); the block's residual update adds
//   delta_c * A(rho, c) into r(rho) in ascending column order c.
// L1B_CD: the reference's serial sampler (solvers.cpp:414-482) is the B = 1
//   case with beta = cd_damping(omega, varpi, n); it replays the reference's
//   updates bit for bit (same stream, same column values, same order).
//
// One CTA runs a whole epoch (the blocks are sequentially dependent; the
// parallelism of PCDM is B).  Ownership of each touched residual row goes to
// the smallest column of the block that touches it with a non-zero step, so
// every row is updated by exactly one thread in a fixed order: no atomics,
// deterministic.  After each epoch r = A x - b is refreshed with the
// matrix-free sweeps (solvers.cpp:472-474, bit-exact with OperatorSpec::apply)
// and f, the sample and the stop tests run on device.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "solvers.hpp"
#include "kernels.hpp"

namespace l1b {

namespace {

struct CdDev {
  double tau, beta, target, tail_sq, f;
  uint64_t epoch, max_epochs, n_samples, cap, t0_ns, last_ts;
  int stop, status, has_target, pad;
  unsigned int ticket[4];
  double scal[4];  // rr, l1, nnz
  unsigned long long applied, colops;  // of the running epoch
};

struct CdSample {
  uint64_t epoch;
  double f, nnz, applied, colops;
  uint64_t ts;
};

template <typename CP, typename RP>
__global__ void __launch_bounds__(1024) cd_epoch_kernel(
    const uint32_t* __restrict__ coords, uint64_t nblocks, int B, const CP* __restrict__ cptr,
    const uint32_t* __restrict__ crow, const double* __restrict__ cval,
    const RP* __restrict__ rptr, const uint32_t* __restrict__ rcol,
    const double* __restrict__ lips, double* x, double* r, uint32_t* stamp, double* delta,
    uint32_t stamp_base, CdDev* st) {
  if (*(volatile int*)&st->stop) return;
  const double beta = st->beta, tau = st->tau;
  const int t = threadIdx.x;
  unsigned long long applied = 0, colops = 0;
  for (uint64_t blk = 0; blk < nblocks; ++blk) {
    const uint32_t sid = stamp_base + (uint32_t)blk + 1u;
    uint32_t i = 0;
    double d = 0.0;
    if (t < B) {
      i = coords[blk * (uint64_t)B + t];
      const double li = lips[i];
      if (li != 0.0) {  // zero columns are skipped (solvers.cpp:455)
        double gi = 0.0;
        for (CP p = cptr[i]; p < cptr[i + 1]; ++p) gi += cval[p] * r[crow[p]];
        ++colops;
        const double scale = beta * li;
        const double xi = x[i];
        const double xn = soft_threshold(xi - gi / scale, tau / scale);
        d = xn - xi;
        if (d != 0.0) {
          x[i] = xn;
          ++applied;
          ++colops;
        }
      }
      delta[i] = d;
      stamp[i] = sid;
    }
    __syncthreads();
    if (t < B && d != 0.0) {
      for (CP p = cptr[i]; p < cptr[i + 1]; ++p) {
        const uint32_t rho = crow[p];
        // owner = smallest block column with a non-zero step touching rho
        bool owner = true;
        for (RP q = rptr[rho]; q < rptr[rho + 1]; ++q) {
          const uint32_t c = rcol[q];
          if (c >= i) break;
          if (stamp[c] == sid && delta[c] != 0.0) {
            owner = false;
            break;
          }
        }
        if (!owner) continue;
        double acc = r[rho];
        for (RP q = rptr[rho]; q < rptr[rho + 1]; ++q) {
          const uint32_t c = rcol[q];
          if (stamp[c] != sid) continue;
          const double dc = delta[c];
          if (dc == 0.0) continue;
          double v = 0.0;  // A(rho, c) as stored in column c (solvers.cpp:465)
          for (CP pc = cptr[c]; pc < cptr[c + 1]; ++pc)
            if (crow[pc] == rho) {
              v = cval[pc];
              break;
            }
          acc += dc * v;
        }
        r[rho] = acc;
      }
    }
    __syncthreads();
  }
  // epoch counters
  __shared__ unsigned long long s_app, s_col;
  if (t == 0) s_app = s_col = 0;
  __syncthreads();
  atomicAdd(&s_app, applied);
  atomicAdd(&s_col, colops);
  __syncthreads();
  if (t == 0) {
    st->applied = s_app;
    st->colops = s_col;
  }
}

// ---------------------------------------------------------------------------
// Planned epochs (columns of <= KC and rows of <= KR entries: k <= 2 stages,
// C2).  The epoch kernel above walks the CSC / CSR and the stamp / delta
// arrays through L2 for every block: ~8 dependent round trips per block.  The
// static part of that walk (column entries, and for each touched row its
// columns with A(rho, c) as stored in column c) only depends on the drawn
// coordinates, so one parallel pass per chunk writes it as a per-slot record
// (structure of arrays); the epoch kernel then prefetches the next block's
// records, reads r and x once per block, and resolves "which block columns
// moved" through a shared-memory hash of (column -> delta).  Same operations
// in the same order as cd_epoch_kernel: identical iterates.
struct Plan {
  uint32_t* i;   // coordinate
  double* l;     // L_i
  uint32_t* nc;  // column length
  uint32_t* row; // [KC][S] column rows (ascending)
  double* val;   // [KC][S] column values
  uint32_t* nr;  // [KC][S] row lengths
  uint32_t* rc;  // [KC][KR][S] row columns (ascending)
  double* rv;    // [KC][KR][S] A(row, col) as stored in the column
  uint64_t S;    // slots (stride of the per-entry arrays)
};

template <int KC, int KR, typename CP, typename RP>
__global__ void cd_plan_kernel(const uint32_t* __restrict__ coords, uint64_t count,
                               const CP* __restrict__ cptr, const uint32_t* __restrict__ crow,
                               const double* __restrict__ cval, const RP* __restrict__ rptr,
                               const uint32_t* __restrict__ rcol, const double* __restrict__ lips,
                               Plan P) {
  const uint64_t S = P.S;
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < count;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = coords[s];
    P.i[s] = i;
    P.l[s] = lips[i];
    uint32_t e = 0;
    for (CP p = cptr[i]; p < cptr[i + 1] && e < KC; ++p, ++e) {
      const uint32_t rho = crow[p];
      P.row[e * S + s] = rho;
      P.val[e * S + s] = cval[p];
      uint32_t f = 0;
      for (RP q = rptr[rho]; q < rptr[rho + 1] && f < KR; ++q, ++f) {
        const uint32_t c = rcol[q];
        double v = 0.0;
        for (CP pc = cptr[c]; pc < cptr[c + 1]; ++pc)
          if (crow[pc] == rho) {
            v = cval[pc];
            break;
          }
        P.rc[((uint64_t)e * KR + f) * S + s] = c;
        P.rv[((uint64_t)e * KR + f) * S + s] = v;
      }
      P.nr[e * S + s] = f;
    }
    P.nc[s] = e;
  }
}

constexpr int kHash = 1024;  // >= 2 B: the planned path takes B <= 512
constexpr uint32_t kEmpty = 0xffffffffu;

__device__ __forceinline__ uint32_t hslot(uint32_t c) { return (c * 2654435761u) >> 22; }  // 10 bits

__device__ __forceinline__ void h_insert(uint32_t* keys, double* vals, uint32_t c, double d) {
  uint32_t h = hslot(c);
  while (atomicCAS(&keys[h], kEmpty, c) != kEmpty) h = (h + 1) & (kHash - 1);
  vals[h] = d;
}
__device__ __forceinline__ double h_find(const uint32_t* keys, const double* vals, uint32_t c) {
  uint32_t h = hslot(c);
  for (;;) {
    const uint32_t k = keys[h];
    if (k == c) return vals[h];
    if (k == kEmpty) return 0.0;
    h = (h + 1) & (kHash - 1);
  }
}

template <int KC, int KR>
struct Rec {
  uint32_t i, nc, row[KC], nr[KC], rc[KC][KR];
  double l, val[KC], rv[KC][KR];
};

template <int KC, int KR>
__device__ __forceinline__ void load_rec(const Plan& P, uint64_t s, Rec<KC, KR>& R) {
  const uint64_t S = P.S;
  R.i = P.i[s];
  R.l = P.l[s];
  R.nc = P.nc[s];
#pragma unroll
  for (int e = 0; e < KC; ++e) {
    R.row[e] = P.row[e * S + s];
    R.val[e] = P.val[e * S + s];
    R.nr[e] = P.nr[e * S + s];
#pragma unroll
    for (int f = 0; f < KR; ++f) {
      R.rc[e][f] = P.rc[((uint64_t)e * KR + f) * S + s];
      R.rv[e][f] = P.rv[((uint64_t)e * KR + f) * S + s];
    }
  }
}

template <int KC, int KR>
__global__ void __launch_bounds__(512) cd_epoch_plan_kernel(Plan P, uint64_t slot0, uint64_t nblocks,
                                                             int B, double* x, double* r, CdDev* st) {
  if (*(volatile int*)&st->stop) return;
  __shared__ uint32_t keys[2][kHash];
  __shared__ double vals[2][kHash];
  const double beta = st->beta, tau = st->tau;
  const int t = threadIdx.x;
  for (int k = t; k < 2 * kHash; k += blockDim.x) (&keys[0][0])[k] = kEmpty;
  unsigned long long applied = 0, colops = 0;
  Rec<KC, KR> cur, nxt;
  if (t < B && nblocks) load_rec(P, slot0 + t, cur);
  __syncthreads();
  for (uint64_t blk = 0; blk < nblocks; ++blk) {
    const int T = (int)(blk & 1);
    if (t < B && blk + 1 < nblocks) load_rec(P, slot0 + (blk + 1) * (uint64_t)B + t, nxt);
    double d = 0.0, rval[KC];
    if (t < B && cur.l != 0.0) {  // zero columns are skipped (solvers.cpp:455)
      const uint32_t i = cur.i;
#pragma unroll
      for (int e = 0; e < KC; ++e) rval[e] = e < (int)cur.nc ? __ldcg(r + cur.row[e]) : 0.0;
      const double xi = __ldcg(x + i);
      double gi = 0.0;
#pragma unroll
      for (int e = 0; e < KC; ++e)
        if (e < (int)cur.nc) gi += cur.val[e] * rval[e];
      ++colops;
      const double scale = beta * cur.l;
      const double xn = soft_threshold(xi - gi / scale, tau / scale);
      d = xn - xi;
      if (d != 0.0) {
        x[i] = xn;
        ++applied;
        ++colops;
        h_insert(keys[T], vals[T], i, d);
      }
    }
    __syncthreads();
    if (d != 0.0) {
      const uint32_t i = cur.i;
#pragma unroll
      for (int e = 0; e < KC; ++e) {
        if (e >= (int)cur.nc) break;
        // owner = smallest block column with a non-zero step touching the row
        bool owner = true;
#pragma unroll
        for (int f = 0; f < KR; ++f) {
          if (f >= (int)cur.nr[e]) break;
          const uint32_t c = cur.rc[e][f];
          if (c >= i) break;
          if (h_find(keys[T], vals[T], c) != 0.0) {
            owner = false;
            break;
          }
        }
        if (!owner) continue;
        double acc = rval[e];
#pragma unroll
        for (int f = 0; f < KR; ++f) {
          if (f >= (int)cur.nr[e]) break;
          const uint32_t c = cur.rc[e][f];
          const double dc = c == i ? d : h_find(keys[T], vals[T], c);
          if (dc == 0.0) continue;
          acc += dc * cur.rv[e][f];
        }
        r[cur.row[e]] = acc;
      }
    }
    // the other table was last used by block blk - 1 (done) and is next used
    // by block blk + 1 (after the barrier below)
    for (int k = t; k < kHash; k += blockDim.x) keys[T ^ 1][k] = kEmpty;
    __syncthreads();
    if (t < B) cur = nxt;
  }
  __shared__ unsigned long long s_app, s_col;
  if (t == 0) s_app = s_col = 0;
  __syncthreads();
  atomicAdd(&s_app, applied);
  atomicAdd(&s_col, colops);
  __syncthreads();
  if (t == 0) {
    st->applied = s_app;
    st->colops = s_col;
  }
}

// r -= b after the matrix-free refresh r = A x (solvers.cpp:473-474): the
// sweep path is the reference's own OperatorSpec::apply, so the residual (and
// hence every later coordinate decision) matches the reference bit for bit.
__global__ void cd_refresh_finish(const double* __restrict__ b, double* r, uint64_t m, CdDev* st,
                                  double* partials) {
  if (*(volatile int*)&st->stop) return;
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = r[i] - b[i];
    r[i] = v;
    acc[0] += v * v;
  }
  double tot[1];
  if (grid_sum<1>(acc, partials, &st->ticket[0], tot) && threadIdx.x == 0) st->scal[0] = tot[0];
}

__device__ void cd_record(CdDev* st, CdSample* trace, uint64_t e, double f, double nnz,
                          double applied, double colops, uint64_t ts) {
  if (st->n_samples < st->cap) trace[st->n_samples] = CdSample{e, f, nnz, applied, colops, ts};
  st->n_samples++;
}

// ||x||_1, nnz(x) + finalisation of the epoch (solvers.cpp:475-477, 445-447)
__global__ void cd_stats_kernel(const double* __restrict__ x, uint64_t n, CdDev* st,
                                CdSample* trace, double* partials, int init) {
  if (!init && *(volatile int*)&st->stop) return;
  double acc[2] = {0.0, 0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    acc[0] += fabs(v);
    acc[1] += v != 0.0 ? 1.0 : 0.0;
  }
  double tot[2];
  if (grid_sum<2>(acc, partials, &st->ticket[1], tot) && threadIdx.x == 0) {
    const double f = st->tau * tot[0] + 0.5 * st->scal[0];
    const uint64_t ts = global_timer_ns();
    if (init) {
      st->t0_ns = ts;
      st->epoch = 0;
      cd_record(st, trace, 0, f, tot[1], 0.0, 0.0, ts);
    } else {
      st->epoch += 1;
      cd_record(st, trace, st->epoch, f, tot[1], (double)st->applied, (double)st->colops, ts);
    }
    st->f = f;
    st->last_ts = ts;
    if (!isfinite(f)) {
      st->stop = 1;
      st->status = -1;
    } else if (st->has_target && f <= st->target) {
      st->stop = 1;
      st->status = 0;
    } else if (st->epoch >= st->max_epochs) {
      st->stop = 1;
      st->status = 1;
    }
  }
}

// r = A*0 - b over all m rows (solvers.cpp:436-437) and ||r||^2
__global__ void cd_init_residual(const double* __restrict__ b, double* r, uint64_t m,
                                 CdDev* st, double* partials) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = 0.0 - b[i];
    r[i] = v;
    acc[0] += v * v;
  }
  double tot[1];
  if (grid_sum<1>(acc, partials, &st->ticket[0], tot) && threadIdx.x == 0) st->scal[0] = tot[0];
}

template <typename CP, typename RP>
void launch_epoch(const ProblemView& v, const uint32_t* coords, uint64_t nblocks, int B,
                  const double* lips, double* x, double* r, uint32_t* stamp, double* delta,
                  uint32_t stamp_base, CdDev* st) {
  const int threads = std::min(1024, std::max(32, (B + 31) / 32 * 32));
  cd_epoch_kernel<CP, RP><<<1, threads, 0, v.stream>>>(
      coords, nblocks, B, (const CP*)v.At.ptr, v.At.idx, v.At.val, (const RP*)v.A.ptr, v.A.idx,
      lips, x, r, stamp, delta, stamp_base, st);
  L1B_LAUNCHED();
}

template <int KC, int KR>
void plan_and_run(const ProblemView& v, const uint32_t* coords, uint64_t count, const double* lips,
                  Plan P, cudaStream_t st) {
  const int grid = grid_for(count);
  if (v.At.ptr32 && v.A.ptr32)
    cd_plan_kernel<KC, KR, uint32_t, uint32_t><<<grid, kThreads, 0, st>>>(
        coords, count, (const uint32_t*)v.At.ptr, v.At.idx, v.At.val, (const uint32_t*)v.A.ptr,
        v.A.idx, lips, P);
  else if (v.At.ptr32)
    cd_plan_kernel<KC, KR, uint32_t, uint64_t><<<grid, kThreads, 0, st>>>(
        coords, count, (const uint32_t*)v.At.ptr, v.At.idx, v.At.val, (const uint64_t*)v.A.ptr,
        v.A.idx, lips, P);
  else if (v.A.ptr32)
    cd_plan_kernel<KC, KR, uint64_t, uint32_t><<<grid, kThreads, 0, st>>>(
        coords, count, (const uint64_t*)v.At.ptr, v.At.idx, v.At.val, (const uint32_t*)v.A.ptr,
        v.A.idx, lips, P);
  else
    cd_plan_kernel<KC, KR, uint64_t, uint64_t><<<grid, kThreads, 0, st>>>(
        coords, count, (const uint64_t*)v.At.ptr, v.At.idx, v.At.val, (const uint64_t*)v.A.ptr,
        v.A.idx, lips, P);
  L1B_LAUNCHED();
}

uint64_t uniform_index(std::mt19937_64& g, uint64_t n) {  // rng.hpp:37-45
  const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = g();
  } while (x >= lim);
  return x % n;
}

double cd_damping(uint64_t omega, uint64_t varpi, uint64_t n) {  // solvers.cpp:266-270
  if (n <= 1 || varpi <= 1) return 1.0;
  return 1.0 + static_cast<double>(omega - 1) * static_cast<double>(varpi - 1) /
                   static_cast<double>(n - 1);
}

}  // namespace

void run_pcdm(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
              l1b_summary* sum, double* x_host, double* d_x) {
  const ProblemView v = problem_view(p);
  const bool serial = cfg->solver == L1B_CD;
  const char* name = serial ? "cd" : "pcdm";
  const uint64_t n = v.n;
  if (v.m > (1ull << 32) || n > (1ull << 32)) throw Unsupported("cd: dimensions above 2^32");
  const uint64_t B = serial ? 1 : std::min<uint64_t>(cfg->block ? cfg->block : 256, n);
  if (B > 1024) throw Unsupported("pcdm: at most 1024 coordinates per block");
  uint64_t omega = 1;
  if (!serial || cfg->varpi > 1)  // solvers.cpp:424-427 (PCDM always models B processors)
    omega = cfg->omega ? cfg->omega : std::min<uint64_t>(std::max<uint64_t>(1, v.max_row_nnz), n);
  const double beta = serial ? cd_damping(omega, cfg->varpi, n) : cd_damping(omega, B, n);
  const uint64_t per_epoch = serial ? n : n / B;  // blocks per epoch
  const double* lips = problem_gram(p);
  cudaStream_t st = v.stream;

  double *x = nullptr, *r = nullptr, *delta = nullptr, *partials = nullptr;
  // planned epochs for short columns / rows (k <= 2 stages); L1B_PCDM_PLAN=0: off
  int plan_k = 0;
  {
    const char* e = getenv("L1B_PCDM_PLAN");
    if (!(e && e[0] == '0') && v.max_col_nnz <= 4 && v.max_row_nnz <= 4 && B <= 512)
      plan_k = (v.max_col_nnz <= 2 && v.max_row_nnz <= 2) ? 2 : 4;
  }
  Plan plan{};
  uint32_t *stamp = nullptr, *d_coords = nullptr;
  CdDev* dst = nullptr;
  CdSample* trace = nullptr;
  const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(16, (1ull << 26) / std::max<uint64_t>(1, per_epoch * B)));
  const uint64_t tcap = std::min<uint64_t>(cfg->max_iters + 2, 1ull << 22);
  std::vector<void*> bufs;
  auto alloc = [&](auto** ptr, size_t bytes) {
    L1B_CUDA(cudaMalloc((void**)ptr, std::max<size_t>(bytes, 8)));
    bufs.push_back((void*)*ptr);
  };
  uint32_t* h_coords = nullptr;  // two chunk buffers: generate one while the other uploads
  CdDev* h_st = nullptr;
  cudaEvent_t uploaded[2] = {nullptr, nullptr};
  try {
    alloc(&x, n * 8);
    alloc(&r, v.m * 8);
    alloc(&delta, n * 8);
    alloc(&stamp, n * 4);
    alloc(&partials, (size_t)spmv_grid_max() * 4 * 8);
    alloc(&d_coords, 2 * chunk * per_epoch * B * 4);
    if (plan_k) {
      const uint64_t S = chunk * per_epoch * B, K = (uint64_t)plan_k;
      plan.S = S;
      alloc(&plan.i, S * 4);
      alloc(&plan.l, S * 8);
      alloc(&plan.nc, S * 4);
      alloc(&plan.row, K * S * 4);
      alloc(&plan.val, K * S * 8);
      alloc(&plan.nr, K * S * 4);
      alloc(&plan.rc, K * K * S * 4);
      alloc(&plan.rv, K * K * S * 8);
    }
    alloc(&dst, sizeof(CdDev));
    alloc(&trace, tcap * sizeof(CdSample));
    L1B_CUDA(cudaMallocHost(&h_coords, 2 * chunk * per_epoch * B * 4));
    for (auto& e : uploaded) L1B_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    L1B_CUDA(cudaMallocHost(&h_st, sizeof(CdDev)));
    L1B_CUDA(cudaMemsetAsync(x, 0, n * 8, st));
    L1B_CUDA(cudaMemsetAsync(stamp, 0, n * 4, st));
    CdDev h;
    std::memset(&h, 0, sizeof(h));
    h.tau = v.tau;
    h.beta = beta;
    h.target = cfg->target;
    h.has_target = cfg->has_target ? 1 : 0;
    h.tail_sq = v.tail_sq;
    h.max_epochs = cfg->max_iters;
    h.cap = tcap;
    *h_st = h;
    L1B_CUDA(cudaMemcpyAsync(dst, h_st, sizeof(CdDev), cudaMemcpyHostToDevice, st));
    const auto t0 = std::chrono::steady_clock::now();
    cd_init_residual<<<grid_for(v.m), kThreads, 0, st>>>(v.b, r, v.m, dst, partials);
    L1B_LAUNCHED();
    cd_stats_kernel<<<grid_for(n), kThreads, 0, st>>>(x, n, dst, trace, partials, 1);
    L1B_LAUNCHED();
    std::mt19937_64 rng(cfg->seed);  // Rng rng = make_rng(cfg.seed) (solvers.cpp:430)
    std::vector<uint64_t> seen(serial ? 0 : n, 0);
    uint64_t draw_block = 0, launched = 0;
    uint32_t stamp_base = 0;
    bool time_out = false;
    // coordinate stream (host: mt19937_64 is sequential), one chunk of epochs
    // at a time into buffer `slot`; the next chunk is drawn while the device
    // runs this one, so the host RNG is off the critical path
    auto draw = [&](uint64_t ep, int slot) {
      uint32_t* out = h_coords + (uint64_t)slot * chunk * per_epoch * B;
      uint64_t k = 0;
      for (uint64_t e = 0; e < ep; ++e)
        for (uint64_t bl = 0; bl < per_epoch; ++bl) {
          ++draw_block;
          for (uint64_t t = 0; t < B; ++t) {
            uint64_t i;
            if (serial) {
              i = uniform_index(rng, n);
            } else {
              do {
                i = uniform_index(rng, n);
              } while (seen[i] == draw_block);
              seen[i] = draw_block;
            }
            out[k++] = (uint32_t)i;
          }
        }
      return k;
    };
    int slot = 0;
    uint64_t ep = std::min<uint64_t>(chunk, cfg->max_iters);
    uint64_t k = ep ? draw(ep, slot) : 0;
    while (launched < cfg->max_iters) {
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > cfg->max_seconds) {
        time_out = true;
        break;
      }
      L1B_CUDA(cudaMemcpyAsync(d_coords + (uint64_t)slot * chunk * per_epoch * B,
                               h_coords + (uint64_t)slot * chunk * per_epoch * B, k * 4,
                               cudaMemcpyHostToDevice, st));
      L1B_CUDA(cudaEventRecord(uploaded[slot], st));
      if (plan_k == 2)
        plan_and_run<2, 2>(v, d_coords + (uint64_t)slot * chunk * per_epoch * B, k, lips, plan, st);
      else if (plan_k == 4)
        plan_and_run<4, 4>(v, d_coords + (uint64_t)slot * chunk * per_epoch * B, k, lips, plan, st);
      for (uint64_t e = 0; e < ep; ++e) {
        const uint32_t* c = d_coords + (slot * chunk + e) * per_epoch * B;
        const int threads = std::min(1024, std::max(32, (int)(B + 31) / 32 * 32));
        if (plan_k == 2) {
          cd_epoch_plan_kernel<2, 2><<<1, threads, 0, st>>>(plan, e * per_epoch * B, per_epoch, (int)B,
                                                            x, r, dst);
          L1B_LAUNCHED();
        } else if (plan_k == 4) {
          cd_epoch_plan_kernel<4, 4><<<1, threads, 0, st>>>(plan, e * per_epoch * B, per_epoch, (int)B,
                                                            x, r, dst);
          L1B_LAUNCHED();
        } else if (v.At.ptr32 && v.A.ptr32)
          launch_epoch<uint32_t, uint32_t>(v, c, per_epoch, (int)B, lips, x, r, stamp, delta, stamp_base, dst);
        else if (v.At.ptr32)
          launch_epoch<uint32_t, uint64_t>(v, c, per_epoch, (int)B, lips, x, r, stamp, delta, stamp_base, dst);
        else if (v.A.ptr32)
          launch_epoch<uint64_t, uint32_t>(v, c, per_epoch, (int)B, lips, x, r, stamp, delta, stamp_base, dst);
        else
          launch_epoch<uint64_t, uint64_t>(v, c, per_epoch, (int)B, lips, x, r, stamp, delta, stamp_base, dst);
        stamp_base += (uint32_t)per_epoch;
        sweep_apply(*v.op, x, r, st);
        cd_refresh_finish<<<grid_for(v.m), kThreads, 0, st>>>(v.b, r, v.m, dst, partials);
        L1B_LAUNCHED();
        cd_stats_kernel<<<grid_for(n), kThreads, 0, st>>>(x, n, dst, trace, partials, 0);
        L1B_LAUNCHED();
      }
      launched += ep;
      L1B_CUDA(cudaMemcpyAsync(h_st, dst, sizeof(CdDev), cudaMemcpyDeviceToHost, st));
      // draw the next chunk while the device works (its buffer's last upload
      // must have left the host first)
      const uint64_t ep_next = std::min<uint64_t>(chunk, cfg->max_iters - launched);
      slot ^= 1;
      if (ep_next) {
        L1B_CUDA(cudaEventSynchronize(uploaded[slot]));
        k = draw(ep_next, slot);
      }
      L1B_CUDA(cudaStreamSynchronize(st));
      if (h_st->stop) break;
      ep = ep_next;
    }
    L1B_CUDA(cudaMemcpyAsync(h_st, dst, sizeof(CdDev), cudaMemcpyDeviceToHost, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    const CdDev hs = *h_st;
    if (hs.status < 0)
      throw std::runtime_error(std::string(name) + ": objective diverged to a non-finite value");
    const uint64_t kept = std::min<uint64_t>(hs.n_samples, tcap);
    std::vector<CdSample> tr(kept);
    if (kept) L1B_CUDA(cudaMemcpyAsync(tr.data(), trace, kept * sizeof(CdSample), cudaMemcpyDeviceToHost, st));
    if (x_host) L1B_CUDA(cudaMemcpyAsync(x_host, x, n * 8, cudaMemcpyDeviceToHost, st));
    if (d_x) L1B_CUDA(cudaMemcpyAsync(d_x, x, n * 8, cudaMemcpyDeviceToDevice, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    std::memset(sum, 0, sizeof(*sum));
    sum->status = hs.stop ? hs.status : (time_out ? L1B_TIME_BUDGET : L1B_ITER_BUDGET);
    sum->time_to_target = INFINITY;
    sum->matvecs_to_target = INFINITY;
    sum->final_objective = NAN;
    uint64_t mvc = 1;   // CountingOperator::count_ (initial apply, :436)
    double mvf = 0.0;   // CountingOperator::fractional_ (:470)
    for (size_t q = 0; q < tr.size(); ++q) {
      if (q > 0) {
        mvf += tr[q].colops / static_cast<double>(n);
        mvc += 1;  // refresh apply (:473)
      }
      l1b_sample o;
      o.iter = tr[q].epoch;
      o.elapsed_s = (double)(tr[q].ts - hs.t0_ns) * 1e-9;
      o.objective = tr[q].f;
      o.nnz = (uint64_t)tr[q].nnz;
      o.matvecs = static_cast<double>(mvc) + mvf;
      o.extra = (uint64_t)tr[q].applied;
      if (samples && q < cap) samples[q] = o;
      sum->final_objective = o.objective;
      if (!sum->reached_target && cfg->has_target && o.objective <= cfg->target) {
        sum->reached_target = 1;
        sum->time_to_target = o.elapsed_s;
        sum->matvecs_to_target = o.matvecs;
      }
    }
    sum->n_samples = hs.n_samples;
    sum->iterations = hs.epoch;
    sum->elapsed_s = (double)(hs.last_ts - hs.t0_ns) * 1e-9;
    sum->total_matvecs = static_cast<double>(mvc) + mvf;
    if (sum->status == L1B_TARGET_REACHED && !sum->reached_target) {
      sum->reached_target = 1;
      sum->time_to_target = sum->elapsed_s;
      sum->matvecs_to_target = sum->total_matvecs;
    }
  } catch (...) {
    cudaStreamSynchronize(st);
    for (void* q : bufs) cudaFree(q);
    if (h_coords) cudaFreeHost(h_coords);
    if (h_st) cudaFreeHost(h_st);
    for (auto e : uploaded)
      if (e) cudaEventDestroy(e);
    throw;
  }
  cudaStreamSynchronize(st);
  for (void* q : bufs) cudaFree(q);
  cudaFreeHost(h_coords);
  cudaFreeHost(h_st);
  for (auto e : uploaded) cudaEventDestroy(e);
}

}  // namespace l1b
