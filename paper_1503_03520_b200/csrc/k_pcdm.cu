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

#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>

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

// ---------------------------------------------------------------------------
// Pair-local epochs (one right stage, no left stages, identity permutations:
// C2's operator).  Column i of A = Sigma G^T e_i touches only the rows of
// i's rotation pair (a, a + 1), a = 2u - offset, and row a / a + 1 only the
// columns of that pair: a block step of coordinate i reads and writes nothing
// outside its pair.  An epoch therefore splits into independent per-pair
// sequences -- for each block in draw order, the block's members of the pair
// (one or both) take the step of cd_epoch_kernel against the pair's residual
// rows as they stood at the block's start, then the rows get
// r + sum_c delta_c A(rho, c) in ascending column order -- and so does the
// refresh r = A x - b (the one-stage sweep of OperatorSpec::apply on the
// pair).  One thread keeps its pair's x, r, sigma, b, L and column values in
// registers for the whole launch; the only grid-wide step per epoch is the
// objective (one grid barrier).  Identical operations to cd_epoch_kernel:
// identical iterates.
//
// The block draws come from the device (mt_stream_indices) in four steps per
// chunk of epochs:
//   cd_prevd_kernel   distance from each stream position back to the
//                     previous draw of the same coordinate (<= W) -- a draw
//                     is redrawn iff that previous draw lies in its block;
//   cd_cand_*         the positions with such a previous draw within W
//                     (~ W/n of them), compacted in stream order; the host
//                     walks them to the block starts (s_{b+1} = s_b + B +
//                     #redrawn in the block: sequential, ~1 candidate per
//                     block, tens of microseconds per 100 epochs at C2);
//   cd_scatter_kernel each kept draw -> an event (block << 1 | member) in
//                     its pair's bucket of the epoch;
//   cd_pair_kernel    the epochs.
constexpr uint16_t kPrevRej = 0xffff;
constexpr int kEvCap = 16;  // events per pair and epoch (Poisson(2B/n * ...) tail: overflow -> direct path)

__global__ void cd_prevd_kernel(const uint32_t* __restrict__ idx, uint64_t L, int W,
                                uint16_t* __restrict__ prevd) {
  extern __shared__ uint32_t tile[];  // [W + blockDim.x]
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x;
  for (int k = threadIdx.x; k < W + (int)blockDim.x; k += blockDim.x) {
    const int64_t q = (int64_t)t0 - W + k;
    tile[k] = (q >= 0 && (uint64_t)q < L) ? idx[q] : 0xffffffffu;
  }
  __syncthreads();
  const uint64_t q = t0 + threadIdx.x;
  if (q >= L) return;
  const uint32_t v = tile[W + threadIdx.x];
  uint16_t d = 0;
  if (v == 0xffffffffu) {
    d = kPrevRej;
  } else {
    const int lim = (int)((uint64_t)W < q ? (uint64_t)W : q);
    for (int k = 1; k <= lim; ++k)
      if (tile[W + threadIdx.x - k] == v) {
        d = (uint16_t)k;
        break;
      }
  }
  prevd[q] = d;
}

// Candidates: the positions whose previous draw of the same coordinate lies
// within W (or that the reference redraws outright), in stream order, packed
// (q << 16 | distance).  Tiles of kCandTile positions: count, scan, write.
constexpr int kCandTile = 4096;
constexpr int kCandPer = kCandTile / kThreads;

__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t* total) {
  __shared__ uint64_t warp_tot[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    uint64_t t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;  // inclusive
  }
  __syncthreads();
  const uint64_t before = (w ? warp_tot[w - 1] : 0) + x - v;
  *total = warp_tot[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(kThreads) cd_cand_count(const uint16_t* __restrict__ prevd, uint64_t L,
                                                          uint32_t* tile_cnt) {
  const uint64_t q0 = blockIdx.x * (uint64_t)kCandTile + (uint64_t)threadIdx.x * kCandPer;
  uint32_t c = 0;
  for (int k = 0; k < kCandPer; ++k) c += (q0 + k < L && prevd[q0 + k] != 0) ? 1u : 0u;
  double v[1] = {(double)c};
  block_sum<1>(v);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = (uint32_t)v[0];
}

__global__ void __launch_bounds__(kThreads) cd_cand_write(const uint16_t* __restrict__ prevd, uint64_t L,
                                                          const uint32_t* __restrict__ tile_off,
                                                          uint64_t* __restrict__ cand) {
  const uint64_t q0 = blockIdx.x * (uint64_t)kCandTile + (uint64_t)threadIdx.x * kCandPer;
  uint32_t c = 0;
  for (int k = 0; k < kCandPer; ++k) c += (q0 + k < L && prevd[q0 + k] != 0) ? 1u : 0u;
  uint64_t tot;
  uint64_t o = tile_off[blockIdx.x] + block_exclusive_scan(c, &tot);
  for (int k = 0; k < kCandPer; ++k) {
    const uint64_t q = q0 + k;
    if (q < L) {
      const uint16_t d = prevd[q];
      if (d != 0) cand[o++] = (q << 16) | d;
    }
  }
}

__global__ void cd_iota_kernel(uint64_t* s, uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    s[i] = i;
}

__global__ void cd_scatter_kernel(const uint32_t* __restrict__ idx, const uint16_t* __restrict__ prevd,
                                  const uint64_t* __restrict__ s, uint64_t nb, uint64_t per_epoch,
                                  int off, uint64_t U, uint32_t* cnt, uint32_t* ev, int* flag) {
  const uint64_t end = s[nb];
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < end;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint16_t d = prevd[q];
    if (d == kPrevRej) continue;
    uint64_t lo = 0, hi = nb;  // block b: s[b] <= q < s[b + 1]
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) >> 1;
      if (s[mid] <= q) lo = mid;
      else hi = mid;
    }
    if (d != 0 && (uint64_t)d <= q - s[lo]) continue;  // redrawn
    const uint64_t e = lo / per_epoch, bl = lo % per_epoch;
    const uint64_t i = idx[q] + (uint64_t)off;
    const uint64_t u = i >> 1;
    const uint32_t slot = atomicAdd(&cnt[e * U + u], 1u);
    if (slot < (uint32_t)kEvCap) ev[(e * kEvCap + slot) * U + u] = (uint32_t)(bl << 1) | (uint32_t)(i & 1);
    else atomicOr(flag, 4);
  }
}

struct CdPairArgs {
  uint64_t n, m, U;
  int off, ptr32;
  double c, s;
  const double *sigma, *b, *lips;
  const void* cptr;
  const uint32_t* crow;
  const double* cval;
  double *x, *r;
  const uint32_t *cnt, *ev;
  uint64_t epochs;  // of this launch
  CdDev* st;
  CdSample* trace;
  double* partials;  // 2 x grid x 5
};

// the objective of an epoch from the blocks' partials (fixed order: every
// caller folds identically) and cd_stats_kernel's bookkeeping
__device__ __forceinline__ void epoch_objective(const double* part, unsigned nblocks, double tau, double& f,
                                                double& nnz, double& applied, double& colops) {
  double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (unsigned q = threadIdx.x; q < nblocks; q += blockDim.x) {
#pragma unroll
    for (int w = 0; w < 5; ++w) tot[w] += __ldcg(&part[(size_t)q * 5 + w]);
  }
  block_sum<5>(tot);
  __shared__ double bc[5];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < 5; ++w) bc[w] = tot[w];
  }
  __syncthreads();
  f = tau * bc[0] + 0.5 * bc[2];
  nnz = bc[1];
  applied = bc[3];
  colops = bc[4];
  __syncthreads();
}

// stop: 0 = go on, 1 = target, 2 = non-finite, 3 = epoch budget
__device__ __forceinline__ void epoch_record(CdDev* st, CdSample* trace, uint64_t epoch, double f, double nnz,
                                             double applied, double colops, int stop) {
  const uint64_t ts = global_timer_ns();
  st->epoch = epoch;
  st->applied = (unsigned long long)applied;
  st->colops = (unsigned long long)colops;
  cd_record(st, trace, epoch, f, nnz, applied, colops, ts);
  st->f = f;
  st->last_ts = ts;
  if (stop) {
    st->stop = 1;
    st->status = stop == 2 ? -1 : stop == 1 ? 0 : 1;
  }
}

// !SYNC launches: the samples of its epochs, in order (one CTA)
__global__ void cd_pair_fold(const double* partials, unsigned nblocks, uint64_t epochs, CdDev* st,
                             CdSample* trace) {
  if (*(volatile int*)&st->stop) return;
  const uint64_t epoch0 = st->epoch, max_epochs = st->max_epochs;
  const double tau = st->tau;
  for (uint64_t ep = 0; ep < epochs; ++ep) {
    double f, nnz, applied, colops;
    epoch_objective(partials + (size_t)ep * nblocks * 5, nblocks, tau, f, nnz, applied, colops);
    const uint64_t epoch = epoch0 + ep + 1;
    const int stop = !isfinite(f) ? 2 : epoch >= max_epochs ? 3 : 0;
    if (threadIdx.x == 0) epoch_record(st, trace, epoch, f, nnz, applied, colops, stop);
    if (stop) break;
  }
}

// SYNC: a grid barrier per epoch, the objective and the stop test in the
// kernel (runs with a target).  !SYNC: epochs back to back, each block's
// partials kept per epoch; cd_pair_fold records the samples afterwards (no
// target: only the epoch budget or a non-finite objective stops a run, and the
// budget is the launch's epoch count).
constexpr int kPairThreads = 128;  // more SMs, one warp per sub-partition (the epoch is a latency chain)
template <int P, bool SYNC>
__global__ void __launch_bounds__(kPairThreads) cd_pair_kernel(CdPairArgs A) {
  namespace cg = cooperative_groups;
  CdDev* st = A.st;
  if (*(volatile int*)&st->stop) return;
  const double beta = st->beta, tau = st->tau;
  const uint64_t epoch0 = st->epoch, max_epochs = st->max_epochs;
  const int has_target = st->has_target;
  const double target = st->target;
  const int64_t n = (int64_t)A.n;
  const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t g0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const double c = A.c, s = A.s;
  // per pair: members e = 0, 1 (coordinates a + e), column entries (row member, value)
  double x[P][2], r[P][2], sig[P][2], bb[P][2], li[P][2], cv[P][2][2];
  int cr[P][2][2], nc[P][2];
  bool va[P][2];
  int64_t a[P];
  bool live[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const uint64_t u = g0 + (uint64_t)k * T;
    live[k] = u < A.U;
    a[k] = 2 * (int64_t)u - A.off;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t i = a[k] + e;
      va[k][e] = live[k] && i >= 0 && i < n;
      x[k][e] = va[k][e] ? A.x[i] : 0.0;
      r[k][e] = va[k][e] ? A.r[i] : 0.0;
      sig[k][e] = va[k][e] ? A.sigma[i] : 0.0;
      bb[k][e] = va[k][e] ? A.b[i] : 0.0;
      li[k][e] = va[k][e] ? A.lips[i] : 0.0;
      nc[k][e] = 0;
      cr[k][e][0] = cr[k][e][1] = 0;
      cv[k][e][0] = cv[k][e][1] = 0.0;
      if (va[k][e]) {
        const uint64_t p0 = A.ptr32 ? ((const uint32_t*)A.cptr)[i] : ((const uint64_t*)A.cptr)[i];
        const uint64_t p1 = A.ptr32 ? ((const uint32_t*)A.cptr)[i + 1] : ((const uint64_t*)A.cptr)[i + 1];
        int q = 0;
        for (uint64_t p = p0; p < p1 && q < 2; ++p, ++q) {
          cr[k][e][q] = (int)((int64_t)A.crow[p] - a[k]);  // 0 or 1
          cv[k][e][q] = A.cval[p];
        }
        nc[k][e] = q;
      }
    }
  }
  // rows [n, m) stay 0 - b (empty rows): their ||r||^2 share, once
  double tail = 0.0;
  for (uint64_t i = (uint64_t)n + g0; i < A.m; i += T) tail += A.r[i] * A.r[i];
  // the bucket count and first kPre events of the next epoch are loaded one
  // epoch ahead (independent of the running epoch)
  constexpr int kPre = 4;
  uint32_t pc[P], pk[P][kPre];
  auto prefetch = [&](uint64_t ep) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const uint64_t u = g0 + (uint64_t)k * T;
      pc[k] = 0;
      if (!live[k] || ep >= A.epochs) continue;
      pc[k] = __ldcg(&A.cnt[ep * A.U + u]);
#pragma unroll
      for (int j = 0; j < kPre; ++j) pk[k][j] = __ldcg(&A.ev[(ep * kEvCap + j) * A.U + u]);
    }
  };
  prefetch(0);
  for (uint64_t ep = 0; ep < A.epochs; ++ep) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // ||x||_1, nnz, ||r||^2, applied, colops
    uint32_t cur_c[P], cur_k[P][kPre];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      cur_c[k] = pc[k];
#pragma unroll
      for (int j = 0; j < kPre; ++j) cur_k[k][j] = pk[k][j];
    }
    prefetch(ep + 1);
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (!live[k]) continue;
      const uint64_t u = g0 + (uint64_t)k * T;
      const int cnt = min((int)cur_c[k], kEvCap);
      uint32_t key[kEvCap];
      for (int j = 0; j < cnt; ++j) {
        const uint32_t v = j < kPre ? cur_k[k][j] : __ldcg(&A.ev[(ep * kEvCap + j) * A.U + u]);
        int q = j;  // insertion sort: ascending (block, member)
        while (q > 0 && key[q - 1] > v) {
          key[q] = key[q - 1];
          --q;
        }
        key[q] = v;
      }
      int j = 0;
      while (j < cnt) {
        const uint32_t bl = key[j] >> 1;
        int in = 0;  // bit e: member e steps in this block
        while (j < cnt && (key[j] >> 1) == bl) in |= 1 << (key[j++] & 1);
        const double r0 = r[k][0], r1 = r[k][1];  // the block's residual
        double d[2] = {0.0, 0.0};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (!((in >> e) & 1) || li[k][e] == 0.0) continue;  // zero columns are skipped (solvers.cpp:455)
          double gi = 0.0;
          for (int q = 0; q < nc[k][e]; ++q) gi += cv[k][e][q] * (cr[k][e][q] ? r1 : r0);
          acc[4] += 1.0;
          const double scale = beta * li[k][e];
          const double xi = x[k][e];
          const double xn = soft_threshold(xi - gi / scale, tau / scale);
          d[e] = xn - xi;
          if (d[e] != 0.0) {
            x[k][e] = xn;
            acc[3] += 1.0;
            acc[4] += 1.0;
          }
        }
        // rows: r + sum over the pair's columns (ascending) with a step of delta_c A(rho, c)
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          double v = f ? r1 : r0;
          bool any = false;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (d[e] == 0.0) continue;
            for (int q = 0; q < nc[k][e]; ++q)
              if (cr[k][e][q] == f) {
                v += d[e] * cv[k][e][q];
                any = true;
              }
          }
          if (any) r[k][f] = v;
        }
      }
      // refresh r = A x - b on the pair's rows (solvers.cpp:472-474: apply, then - b)
      double v0 = x[k][0], v1 = x[k][1];
      if (va[k][0] && va[k][1]) rotate_pair(v0, v1, c, s, true);
      const double y0 = sig[k][0] * v0, y1 = sig[k][1] * v1;
      r[k][0] = y0 - bb[k][0];
      r[k][1] = y1 - bb[k][1];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (!va[k][e]) continue;
        acc[0] += fabs(x[k][e]);
        acc[1] += x[k][e] != 0.0 ? 1.0 : 0.0;
        acc[2] += r[k][e] * r[k][e];
      }
    }
    acc[2] += tail;
    block_sum<5>(acc);
    double* part = A.partials + (size_t)(SYNC ? (ep & 1) : ep) * gridDim.x * 5;
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < 5; ++q) part[(size_t)blockIdx.x * 5 + q] = acc[q];
    }
    if constexpr (!SYNC) continue;
    cg::this_grid().sync();
    double f, nnz, applied, colops;
    epoch_objective(part, gridDim.x, tau, f, nnz, applied, colops);
    const uint64_t epoch = epoch0 + ep + 1;
    const int stop = !isfinite(f) ? 2 : (has_target && f <= target) ? 1 : epoch >= max_epochs ? 3 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) epoch_record(st, A.trace, epoch, f, nnz, applied, colops, stop);
    if (stop) break;
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (!va[k][e]) continue;
      A.x[a[k] + e] = x[k][e];
      A.r[a[k] + e] = r[k][e];
    }
  }
}

template <int P>
int cd_pair_capacity() {
  static const int cap = [] {
    int per_sm = 0, per_sm2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cd_pair_kernel<P, true>, kPairThreads, 0) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, cd_pair_kernel<P, false>, kPairThreads, 0) !=
            cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return std::min(per_sm, per_sm2) * sm_count();
  }();
  return cap;
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


// The pair-local path (see cd_pair_kernel): 1 = ran (state in x / r / dst),
// 0 = not applicable, -1 = handed over mid-run (the caller restarts on the
// direct path; only on an event-bucket or look-back overflow).
template <typename Start>
int pair_epochs(const ProblemView& v, const l1b_solver_cfg* cfg, uint64_t B, uint64_t per_epoch,
                const double* lips, double* x, double* r, CdDev* dst, CdSample* trace, CdDev* h_st,
                Start&& start, const std::chrono::steady_clock::time_point& t0, uint64_t& launched,
                bool& time_out) {
  const char* env = getenv("L1B_PCDM_PAIR");
  if (env && env[0] == '0') return 0;
  const OpView* op = v.op;
  const uint64_t n = v.n;
  if (!op || v.shard || op->right.count != 1 || op->left.count != 0 || op->p1 || op->p2 || v.m < n ||
      v.max_col_nnz > 2 || v.max_row_nnz > 2 || n >= (1ull << 30) || n < 4 * B || !v.At.ptr || !v.b)
    return 0;
  const uint64_t U = (n + 2) / 2;
  int P = 0, grid = 0;
  const void* fn = nullptr;
  auto try_p = [&](int p, int cap, const void* f) {
    const uint64_t g = (U + (uint64_t)p * kPairThreads - 1) / ((uint64_t)p * kPairThreads);
    if (!P && cap > 0 && g <= (uint64_t)cap) {
      P = p;
      grid = (int)g;
      fn = f;
    }
  };
  // with a target the objective is tested every epoch inside the kernel (grid
  // barrier); without one the epochs run back to back
  const bool sync = cfg->has_target != 0;
  try_p(1, cd_pair_capacity<1>(), sync ? (const void*)cd_pair_kernel<1, true> : (const void*)cd_pair_kernel<1, false>);
  try_p(2, cd_pair_capacity<2>(), sync ? (const void*)cd_pair_kernel<2, true> : (const void*)cd_pair_kernel<2, false>);
  try_p(4, cd_pair_capacity<4>(), sync ? (const void*)cd_pair_kernel<4, true> : (const void*)cd_pair_kernel<4, false>);
  if (!P) return 0;
  cudaStream_t st = v.stream;
  // chunks of ~2^19 draws: the stream for the next chunk is drawn (side stream,
  // one SM) while the current chunk's walk and epochs run
  const uint64_t E_max = std::max<uint64_t>(1, std::min<uint64_t>(cfg->max_iters, (1ull << 19) / (per_epoch * B)));
  auto margin = [&](uint64_t T) { return T * B / n + 4096; };  // ~2x the expected redraws (B / 2n per draw)
  const uint64_t cap_raw = 2 * (E_max * per_epoch * B + margin(E_max * per_epoch * B));  // one chunk
  const uint64_t G = cap_raw / 2;  // draws per generator launch
  // stream buffer: the whole run when it fits in 2^25 draws, else rewound
  const uint64_t run_draws = cfg->max_iters * per_epoch * B;
  const uint64_t scap = std::min<uint64_t>(run_draws + margin(run_draws) + 2 * cap_raw, (1ull << 25) + 2 * cap_raw);
  // look-back: a block is B kept draws plus ~B^2 / 2n redraws; W bounds its
  // length (a longer block hands the run to the direct path)
  // (B = 1, serial CD: a block never redraws; no look-back, only rejected raw
  // draws become candidates)
  const int W = (int)(B + 64 + 4 * ((B * B + 2 * n - 1) / (2 * n)));
  const int W_prev = B == 1 ? 0 : W;
  std::vector<void*> bufs;
  auto alloc = [&](auto** ptr, size_t bytes) {  // out of memory: hand the run to the direct path
    const cudaError_t e = cudaMalloc((void**)ptr, std::max<size_t>(bytes, 8));
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw Unsupported("pcdm pairs: device memory");
    }
    L1B_CUDA(e);
    bufs.push_back((void*)*ptr);
  };
  int rc = 1;
  int* h_flag = nullptr;
  uint64_t* h_starts_pinned = nullptr;
  cudaStream_t gs = nullptr;  // generator stream
  // stream positions relative to S[cur]: [0, gen_end) drawn (or queued on
  // gs), the chunk starts at pos; pieces = (end, event) of each launch, dropped
  // (event destroyed) once the chunk walk has moved past them
  std::vector<std::pair<uint64_t, cudaEvent_t>> pieces;
  try {
    uint32_t* S[2] = {nullptr, nullptr};
    uint16_t* prevd;
    uint64_t *sarr, *win, *words;
    uint32_t *cnt, *ev;
    int* flag;
    double* part;
    uint32_t* tile_cnt;
    uint64_t* cand;
    void* scan_tmp;
    size_t scan_bytes = 0;
    std::vector<uint64_t> h_cand;
    alloc(&S[0], (scap + 312) * 4);  // + one generator round of slack
    alloc(&prevd, (cap_raw + 312) * 2);
    alloc(&sarr, (E_max * per_epoch + 1) * 8);
    alloc(&cnt, E_max * U * 4);
    alloc(&ev, E_max * kEvCap * U * 4);
    alloc(&win, 312 * 8);
    alloc(&words, (G + 312) * 8);
    alloc(&flag, 16);
    alloc(&part, (size_t)(sync ? 2 : E_max) * grid * 5 * 8);
    const uint64_t max_tiles = (cap_raw + 312 + kCandTile - 1) / kCandTile;
    alloc(&tile_cnt, (max_tiles + 1) * 4);
    alloc(&cand, (cap_raw + 312) * 8);
    L1B_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, tile_cnt, tile_cnt, (int)(max_tiles + 1), st));
    alloc(&scan_tmp, scan_bytes);
    L1B_CUDA(cudaMallocHost(&h_starts_pinned, (E_max * per_epoch + 1) * 8));
    L1B_CUDA(cudaMallocHost(&h_flag, 16));
    L1B_CUDA(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
    {
      uint64_t w[312];
      mt_seed_state(cfg->seed, w);  // Rng rng = make_rng(cfg.seed) (solvers.cpp:430)
      L1B_CUDA(cudaMemcpyAsync(win, w, sizeof(w), cudaMemcpyHostToDevice, st));
      L1B_CUDA(cudaStreamSynchronize(st));
    }
    auto new_event = [&]() {
      cudaEvent_t e;
      L1B_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      return e;
    };
    auto drop_pieces = [&](uint64_t upto) {  // events of launches ending at or before upto
      size_t k = 0;
      while (k < pieces.size() && pieces[k].first <= upto) cudaEventDestroy(pieces[k++].second);
      pieces.erase(pieces.begin(), pieces.begin() + k);
    };
    start();  // x = 0, r = -b, epoch-0 sample: the solve's clock starts here
    {
      cudaEvent_t e = new_event();
      pieces.emplace_back(0, e);
      L1B_CUDA(cudaEventRecord(e, st));
      L1B_CUDA(cudaStreamWaitEvent(gs, e, 0));
    }
    CdPairArgs a;
    a.n = n;
    a.m = v.m;
    a.U = U;
    a.off = op->right.offset[0];
    a.ptr32 = v.At.ptr32 ? 1 : 0;
    a.c = op->right.c[0];
    a.s = op->right.s[0];
    a.sigma = op->sigma;
    a.b = v.b;
    a.lips = lips;
    a.cptr = v.At.ptr;
    a.crow = v.At.idx;
    a.cval = v.At.val;
    a.x = x;
    a.r = r;
    a.cnt = cnt;
    a.ev = ev;
    a.st = dst;
    a.trace = trace;
    a.partials = part;
    int cur = 0;
    uint64_t pos = 0, gen_end = 0;
    auto gen_to = [&](uint64_t upto) {
      while (gen_end < upto && gen_end + G <= scap) {
        gen_end += mt_stream_indices(win, G, n, S[cur] + gen_end, words, gs);
        cudaEvent_t e = new_event();
        L1B_CUDA(cudaEventRecord(e, gs));
        pieces.emplace_back(gen_end, e);
      }
    };
    auto wait_for = [&](uint64_t upto) {  // st waits until [0, upto) is drawn
      for (auto& pc : pieces)
        if (pc.first >= upto) {
          L1B_CUDA(cudaStreamWaitEvent(st, pc.second, 0));
          return;
        }
      throw Unsupported("pcdm pairs: stream buffer");
    };
    while (launched < cfg->max_iters) {
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > cfg->max_seconds) {
        time_out = true;
        break;
      }
      const uint64_t E = std::min<uint64_t>(E_max, cfg->max_iters - launched);
      const uint64_t nb = E * per_epoch, T = nb * B;
      uint64_t need = T + margin(T);
      if (pos + need + G > scap) {  // rewind: the undrawn tail moves to the front of the other buffer
        L1B_CUDA(cudaStreamSynchronize(gs));
        if (!S[cur ^ 1]) alloc(&S[cur ^ 1], (scap + 312) * 4);
        L1B_CUDA(cudaMemcpyAsync(S[cur ^ 1], S[cur] + pos, (gen_end - pos) * 4, cudaMemcpyDeviceToDevice, st));
        L1B_CUDA(cudaStreamSynchronize(st));
        cur ^= 1;
        gen_end -= pos;
        pos = 0;
        drop_pieces(~0ull);
        pieces.emplace_back(gen_end, new_event());
        L1B_CUDA(cudaEventRecord(pieces.back().second, st));
      }
      uint32_t* idx = S[cur] + pos;
      uint64_t have = 0;
      for (;;) {
        if (need > cap_raw) throw Unsupported("pcdm pairs: chunk buffer");
        gen_to(pos + need + G);  // this chunk's draws and one launch ahead
        wait_for(pos + need);
        have = need;
        cd_prevd_kernel<<<(unsigned)((have + kThreads - 1) / kThreads), kThreads, (W + kThreads) * 4, st>>>(
            idx, have, W_prev, prevd);
        L1B_LAUNCHED();
        const uint64_t tiles = (have + kCandTile - 1) / kCandTile;
        cd_cand_count<<<(unsigned)tiles, kThreads, 0, st>>>(prevd, have, tile_cnt);
        L1B_LAUNCHED();
        L1B_CUDA(cudaMemsetAsync(tile_cnt + tiles, 0, 4, st));
        size_t tb = scan_bytes;
        L1B_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, tb, tile_cnt, tile_cnt, (int)(tiles + 1), st));
        cd_cand_write<<<(unsigned)tiles, kThreads, 0, st>>>(prevd, have, tile_cnt, cand);
        L1B_LAUNCHED();
        uint32_t ncand = 0;
        L1B_CUDA(cudaMemcpyAsync(h_flag, tile_cnt + tiles, 4, cudaMemcpyDeviceToHost, st));
        L1B_CUDA(cudaStreamSynchronize(st));
        ncand = (uint32_t)h_flag[0];
        h_cand.resize(ncand);
        if (ncand)
          L1B_CUDA(cudaMemcpyAsync(h_cand.data(), cand, (size_t)ncand * 8, cudaMemcpyDeviceToHost, st));
        L1B_CUDA(cudaStreamSynchronize(st));
        // block starts: a draw is redrawn iff its previous draw lies inside its block
        if (B == 1 && ncand == 0) {  // serial CD without a rejected draw: block b starts at b
          if (nb + 1 > have) {
            need = have + have / 2;
            continue;
          }
          cd_iota_kernel<<<grid_for(nb + 1), kThreads, 0, st>>>(sarr, nb + 1);
          L1B_LAUNCHED();
          h_starts_pinned[nb] = nb;
          break;
        }
        bool short_stream = false;
        uint64_t sb = 0, j = 0;
        for (uint64_t blk = 0; blk < nb; ++blk) {
          h_starts_pinned[blk] = sb;
          uint64_t e = sb + B;
          while (j < ncand && (h_cand[j] >> 16) < e) {
            const uint64_t q = h_cand[j] >> 16, d = h_cand[j] & 0xffff;
            if (d == kPrevRej || q - d >= sb) ++e;
            ++j;
          }
          if (e - sb > (uint64_t)W) throw Unsupported("pcdm pairs: block longer than the look-back");
          if (e > have) {
            short_stream = true;
            break;
          }
          sb = e;
        }
        if (short_stream) {  // more redraws than the margin: wait for more draws and walk again
          need = have + have / 2;
          continue;
        }
        h_starts_pinned[nb] = sb;
        L1B_CUDA(cudaMemcpyAsync(sarr, h_starts_pinned, (nb + 1) * 8, cudaMemcpyHostToDevice, st));
        break;
      }
      L1B_CUDA(cudaMemsetAsync(flag, 0, 4, st));
      L1B_CUDA(cudaMemsetAsync(cnt, 0, E * U * 4, st));
      cd_scatter_kernel<<<grid_for(T), kThreads, 0, st>>>(idx, prevd, sarr, nb, per_epoch, a.off, U, cnt, ev,
                                                        flag);
      L1B_LAUNCHED();
      a.epochs = E;
      void* args[] = {&a};
      if (sync) {
        L1B_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kPairThreads), args, 0, st));
        L1B_LAUNCHED();
      } else {
        L1B_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kPairThreads), args, 0, st));
        L1B_LAUNCHED();
        cd_pair_fold<<<1, kPairThreads, 0, st>>>(part, (unsigned)grid, E, dst, trace);
        L1B_LAUNCHED();
      }
      const uint64_t used = h_starts_pinned[nb];
      L1B_CUDA(cudaMemcpyAsync(h_flag, flag, 4, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaMemcpyAsync(h_st, dst, sizeof(CdDev), cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
      if (*h_flag & 4) throw Unsupported("pcdm pairs: event bucket");
      pos += used;  // the draws past the chunk's last block open the next chunk
      drop_pieces(pos);
      launched += E;
      if (h_st->stop) break;
    }
  } catch (const Unsupported&) {
    rc = -1;
  } catch (...) {
    cudaStreamSynchronize(st);
    if (gs) cudaStreamSynchronize(gs);
    if (gs) cudaStreamDestroy(gs);
    for (auto& pc : pieces) cudaEventDestroy(pc.second);
    for (void* q : bufs) cudaFree(q);
    if (h_flag) cudaFreeHost(h_flag);
    if (h_starts_pinned) cudaFreeHost(h_starts_pinned);
    throw;
  }
  cudaStreamSynchronize(st);
  if (gs) cudaStreamSynchronize(gs);
  if (gs) cudaStreamDestroy(gs);
  for (auto& pc : pieces) cudaEventDestroy(pc.second);
  for (void* q : bufs) cudaFree(q);
  if (h_flag) cudaFreeHost(h_flag);
  if (h_starts_pinned) cudaFreeHost(h_starts_pinned);
  return rc;
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
    CdDev h;
    std::memset(&h, 0, sizeof(h));
    h.tau = v.tau;
    h.beta = beta;
    h.target = cfg->target;
    h.has_target = cfg->has_target ? 1 : 0;
    h.tail_sq = v.tail_sq;
    h.max_epochs = cfg->max_iters;
    h.cap = tcap;
    // x = 0, r = A 0 - b, the epoch-0 sample (also the restart of the direct
    // path when the pair-local one hands over)
    auto init_state = [&]() {
      L1B_CUDA(cudaMemsetAsync(x, 0, n * 8, st));
      L1B_CUDA(cudaMemsetAsync(stamp, 0, n * 4, st));
      *h_st = h;
      L1B_CUDA(cudaMemcpyAsync(dst, h_st, sizeof(CdDev), cudaMemcpyHostToDevice, st));
      cd_init_residual<<<grid_for(v.m), kThreads, 0, st>>>(v.b, r, v.m, dst, partials);
      L1B_LAUNCHED();
      cd_stats_kernel<<<grid_for(n), kThreads, 0, st>>>(x, n, dst, trace, partials, 1);
      L1B_LAUNCHED();
    };
    auto t0 = std::chrono::steady_clock::now();
    auto start = [&]() {
      t0 = std::chrono::steady_clock::now();
      init_state();
    };
    uint64_t launched = 0;
    bool time_out = false;
    // the pair-local path allocates its buffers, then calls start()
    const int pair_mode = pair_epochs(v, cfg, B, per_epoch, lips, x, r, dst, trace, h_st, start, t0, launched,
                                      time_out);
    if (pair_mode <= 0) {  // not applicable, or handed over (a bucket / the look-back overflowed)
      L1B_CUDA(cudaStreamSynchronize(st));
      launched = 0;
      time_out = false;
      start();
    }
    std::mt19937_64 rng(cfg->seed);  // Rng rng = make_rng(cfg.seed) (solvers.cpp:430)
    std::vector<uint64_t> seen(serial ? 0 : n, 0);
    uint64_t draw_block = 0;
    uint32_t stamp_base = 0;
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
    uint64_t ep = pair_mode > 0 ? 0 : std::min<uint64_t>(chunk, cfg->max_iters);
    uint64_t k = ep ? draw(ep, slot) : 0;
    while (pair_mode <= 0 && launched < cfg->max_iters) {
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
    sum->path = pair_mode > 0 ? L1B_RAN_PCDM_PAIR : plan_k ? L1B_RAN_PCDM_PLAN : L1B_RAN_PCDM_DIRECT;
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
