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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <random>
#include <vector>

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
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

// The same look-back from a stable radix sort of (coordinate, position): in
// sorted order the previous entry with the same key is the previous draw of
// that coordinate.  key = coordinate, n for the reference's redraw marker.
__global__ void cd_key_kernel(const uint32_t* __restrict__ idx, uint64_t L, uint32_t n,
                              uint32_t* __restrict__ key, uint32_t* __restrict__ pos) {
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < L; q += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = idx[q];
    key[q] = v == 0xffffffffu ? n : v;
    pos[q] = (uint32_t)q;
  }
}

__global__ void cd_prevd_sorted_kernel(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ spos,
                                       uint64_t L, uint32_t n, int W, uint16_t* __restrict__ prevd) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < L; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = skey[i], q = spos[i];
    uint16_t d = 0;
    if (k == n) {
      d = kPrevRej;
    } else if (i > 0 && skey[i - 1] == k) {
      const uint32_t dist = q - spos[i - 1];
      if (dist <= (uint32_t)W) d = (uint16_t)dist;
    }
    prevd[q] = d;
  }
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

// ---- the walk to the block starts, on the device --------------------------
// Block b spans [s_b, s_{b+1}): B kept draws plus the redrawn ones; candidate q
// (its coordinate's previous draw d back) is redrawn in the block starting at s
// iff d == kPrevRej or q - d >= s (rng.hpp:37-45 + the distinct-coordinate
// rule of block PCDM).  The walk is sequential by definition, but through a
// segment of kSegLen draws starting at S it depends only on the entry phase p =
// (first block start >= S) - S, which lies in [0, W) since no block is longer
// than W: F_S(p) = (exit phase, blocks started in the segment).  Every
// (segment, phase) pair is walked at once (cd_seg_walk_kernel), the F are
// composed up a binary tree (cd_seg_compose_kernel), each segment finds its
// entry phase and block offset by descending the tree and re-walks itself to
// write its block starts (cd_seg_emit_kernel).  No host round trip.
constexpr uint64_t kSegLen = 4096;
// one thread per item (these kernels are not grid-stride loops, unlike grid_for's users)
inline unsigned blocks_for(uint64_t items) { return (unsigned)((items + kThreads - 1) / kThreads); }

// walk from block start s to the first block start >= lim; out[base + t] = the
// starts with base + t <= out_max (out may be null).  False: a block longer than W.
// Candidates j0 .. j0 + ns - 1 come from the shared-memory copy sm.
__device__ __forceinline__ bool walk_blocks(const uint64_t* __restrict__ cand, uint64_t ncand,
                                            const uint64_t* sm, uint64_t j0, uint64_t ns, uint64_t& j,
                                            uint64_t& s, uint64_t lim, uint64_t B, uint64_t W, uint32_t& cnt,
                                            uint64_t* out, uint64_t base, uint64_t out_max) {
  auto get = [&](uint64_t k) { return k - j0 < ns ? sm[k - j0] : cand[k]; };
  while (s < lim) {
    while (j < ncand && (get(j) >> 16) < s) ++j;
    if (out && base + cnt <= out_max) out[base + cnt] = s;
    uint64_t e = s + B;
    while (j < ncand) {
      const uint64_t c = get(j), q = c >> 16, d = c & 0xffff;
      if (q >= e) break;
      if (d == kPrevRej || q - d >= s) ++e;
      ++j;
    }
    if (e - s > W) return false;
    s = e;
    ++cnt;
  }
  return true;
}

// a segment's candidates (from its first one on, at most kSegCand) into smem
constexpr int kSegCand = 1024;
// (a segment's walks read candidates below S + L + W < S + 2L: up to the first
// one of segment seg + 2)
__device__ __forceinline__ uint64_t stage_candidates(const uint64_t* __restrict__ cand, uint64_t ncand,
                                                     const uint64_t* __restrict__ seg_first, uint64_t seg,
                                                     uint64_t nseg, uint64_t* sm, int tid, int nthreads) {
  const uint64_t j0 = seg_first[seg], j1 = seg + 2 < nseg ? seg_first[seg + 2] : ncand;
  const uint64_t ns = j1 - j0 < (uint64_t)kSegCand ? j1 - j0 : (uint64_t)kSegCand;
  for (uint64_t t = tid; t < ns; t += nthreads) sm[t] = cand[j0 + t];
  return ns;
}

__device__ __forceinline__ uint64_t cand_lower_bound(const uint64_t* __restrict__ cand, uint64_t ncand,
                                                     uint64_t pos) {
  uint64_t lo = 0, hi = ncand;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if ((cand[mid] >> 16) < pos) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void cd_seg_first_kernel(const uint64_t* __restrict__ cand, const uint32_t* ncand_p, uint64_t nseg,
                                    uint64_t* __restrict__ seg_first) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < nseg) seg_first[i] = cand_lower_bound(cand, *ncand_p, i * kSegLen);
}

// F[seg * W + p] = exit phase | blocks << 32: one CTA per segment, thread p
// walks from phase p (the segment's candidates staged in shared memory)
__global__ void cd_seg_walk_kernel(const uint64_t* __restrict__ cand, const uint32_t* ncand_p,
                                   const uint64_t* __restrict__ seg_first, uint64_t nseg, uint64_t B, uint64_t W,
                                   uint64_t* __restrict__ F, int* flag) {
  __shared__ uint64_t sm[kSegCand];
  const uint64_t seg = blockIdx.x, p = threadIdx.x;
  const uint64_t ncand = *ncand_p, j0 = seg_first[seg];
  const uint64_t ns = stage_candidates(cand, ncand, seg_first, seg, nseg, sm, threadIdx.x, blockDim.x);
  __syncthreads();
  const uint64_t lim = (seg + 1) * kSegLen;
  for (uint64_t ph = p; ph < W; ph += blockDim.x) {
    uint64_t s = seg * kSegLen + ph, j = j0;
    uint32_t cnt = 0;
    if (!walk_blocks(cand, ncand, sm, j0, ns, j, s, lim, B, W, cnt, nullptr, 0, 0)) {
      atomicOr(flag, 16);  // the run is handed over; keep the tree's indices in range
      F[seg * W + ph] = 0;
      continue;
    }
    F[seg * W + ph] = (s - lim) | ((uint64_t)cnt << 32);
  }
}

// parent node i of level l+1 = child 2i, then child 2i + 1 (when it exists).
// A CTA composes kComposeLevels levels of the subtree over 2^kComposeLevels
// nodes of level l0 (level by level, barriers between): 3 launches for ~1000
// segments instead of one per level.
constexpr int kComposeLevels = 4;
struct LevelTab {
  uint64_t off[40], cnt[40];
};
__global__ void cd_seg_compose_kernel(uint64_t* __restrict__ lv, LevelTab tab, int l0, int l1, uint64_t W) {
  for (int l = l0; l < l1; ++l) {
    const uint64_t n_child = tab.cnt[l], n_par = tab.cnt[l + 1];
    const uint64_t span = 1ull << (l + 1 - l0);  // parents of this CTA at level l + 1
    const uint64_t first = (uint64_t)blockIdx.x << (kComposeLevels - (l + 1 - l0));
    const uint64_t* child = lv + tab.off[l];
    uint64_t* parent = lv + tab.off[l + 1];
    const uint64_t count = (kComposeLevels >= (l + 1 - l0) ? (1ull << (kComposeLevels - (l + 1 - l0))) : 1) * W;
    (void)span;
    for (uint64_t t = threadIdx.x; t < count; t += blockDim.x) {
      const uint64_t i = first + t / W, p = t % W;
      if (i >= n_par) continue;
      const uint64_t a = child[(2 * i) * W + p];
      if (2 * i + 1 >= n_child) {
        parent[i * W + p] = a;
        continue;
      }
      const uint64_t b = child[(2 * i + 1) * W + (a & 0xffffffffull)];
      parent[i * W + p] = (b & 0xffffffffull) | (((a >> 32) + (b >> 32)) << 32);
    }
    __syncthreads();  // (the next level reads this one's nodes, written by this CTA)
  }
}

// segment i (one warp each): entry (phase, block offset) from the root down (a
// right child enters where its left sibling exits), then its block starts into
// starts[] (entries <= nb; starts[nb] = the end of the chunk's last block)
__global__ void __launch_bounds__(128) cd_seg_emit_kernel(const uint64_t* __restrict__ cand, const uint32_t* ncand_p,
                                   const uint64_t* __restrict__ seg_first, const uint64_t* __restrict__ levels,
                                   const uint64_t* __restrict__ level_off, int nlevels, uint64_t nseg, uint64_t B,
                                   uint64_t W, uint64_t nb, uint64_t* __restrict__ starts) {
  __shared__ uint64_t smem[4][kSegCand];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t i = blockIdx.x * 4ull + w;
  if (i >= nseg) return;
  const uint64_t ncand = *ncand_p, j0 = seg_first[i];
  const uint64_t ns = stage_candidates(cand, ncand, seg_first, i, nseg, smem[w], lane, 32);
  __syncwarp();
  if (lane) return;
  uint64_t p = 0, off = 0;
  for (int l = nlevels - 2; l >= 0; --l) {
    const uint64_t c = i >> l;
    if (c & 1) {
      const uint64_t v = levels[level_off[l] + (c - 1) * W + p];
      off += v >> 32;
      p = v & 0xffffffffull;
    }
  }
  if (off > nb) return;
  uint64_t s = i * kSegLen + p, j = j0;
  uint32_t cnt = 0;
  walk_blocks(cand, ncand, smem[w], j0, ns, j, s, (i + 1) * kSegLen, B, W, cnt, starts, off, nb);
}

// B = 1 (serial CD): no look-back, a block is the rejected raw draws before
// one kept draw: s_{b+1} = (position of kept draw b) + 1 = b + k + 1, k = the
// rejected positions before it (~never: p = n / 2^64 per draw)
__global__ void cd_b1_starts_kernel(const uint64_t* __restrict__ cand, const uint32_t* ncand_p, uint64_t nb,
                                    uint64_t* __restrict__ starts) {
  const uint64_t nc = *ncand_p;
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b <= nb; b += (uint64_t)gridDim.x * blockDim.x) {
    if (b == 0) {
      starts[0] = 0;
      continue;
    }
    uint64_t k = 0;
    while (k < nc && (cand[k] >> 16) <= (b - 1) + k) ++k;
    starts[b] = b + k;
  }
}

__global__ void cd_iota_kernel(uint64_t* s, uint64_t count) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
    s[i] = i;
}

// `lanes` (1 or 32) threads per block b: its draws are [s[b], s[b + 1]); a
// draw is redrawn iff its previous draw of the same coordinate lies in the block
__global__ void cd_scatter_kernel(const uint32_t* __restrict__ idx, const uint16_t* __restrict__ prevd,
                                  const uint64_t* __restrict__ s, uint64_t nb, uint64_t per_epoch,
                                  int off, uint64_t U, int lanes, uint32_t* cnt, uint32_t* ev, int* flag,
                                  uint64_t have) {
  const uint64_t groups = ((uint64_t)gridDim.x * blockDim.x) / lanes;
  const int lane = lanes == 1 ? 0 : (threadIdx.x & 31);
  const uint64_t lim = s[nb] < have ? s[nb] : have;  // (a failed walk is handed over after the launch)
  for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / lanes; b < nb; b += groups) {
    const uint64_t s0 = min(s[b], lim), s1 = min(s[b + 1], lim);
    const uint64_t e = b / per_epoch, bl = b % per_epoch;
    for (uint64_t q = s0 + lane; q < s1; q += lanes) {
      const uint16_t d = prevd[q];
      if (d == kPrevRej) continue;
      if (d != 0 && (uint64_t)d <= q - s0) continue;  // redrawn
      const uint64_t i = idx[q] + (uint64_t)off;
      const uint64_t u = i >> 1;
      const uint32_t slot = atomicAdd(&cnt[e * U + u], 1u);
      if (slot < (uint32_t)kEvCap) ev[(e * kEvCap + slot) * U + u] = (uint32_t)(bl << 1) | (uint32_t)(i & 1);
      else atomicOr(flag, 4);
    }
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
  const unsigned long long* mask;  // event masks (MW > 0)
  uint64_t epochs;  // of this launch
  CdDev* st;
  CdSample* trace;
  double* partials;  // (SYNC: 2, else epochs) x warps x 5
};

// the objective of an epoch from the blocks' partials, folded by ONE warp in a
// fixed order (lane-strided sums, then a shuffle tree; lane 0's result): every
// caller -- the SYNC epoch kernel's warp 0, the fold kernel's warp per epoch --
// reduces identically, so a run with a target records the same bits as one
// without.  Returns f, nnz, applied, colops in every lane.
template <bool CG = true>
__device__ __forceinline__ void epoch_objective_warp(const double* part, unsigned nblocks, double tau,
                                                     double& f, double& nnz, double& applied,
                                                     double& colops) {
  const int lane = threadIdx.x & 31;
  double tot[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (unsigned q0 = lane; q0 < nblocks; q0 += 128) {  // rows q0, q0 + 32, ..: loads first, sums in order
    double v[4][5];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int w = 0; w < 5; ++w) {
        const double* a = &part[(size_t)(q0 + 32 * j) * 5 + w];
        v[j][w] = q0 + 32 * j < nblocks ? (CG ? __ldcg(a) : *a) : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (q0 + 32 * j < nblocks)
#pragma unroll
        for (int w = 0; w < 5; ++w) tot[w] += v[j][w];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int w = 0; w < 5; ++w) tot[w] += __shfl_down_sync(0xffffffffu, tot[w], o);
  }
#pragma unroll
  for (int w = 0; w < 5; ++w) tot[w] = __shfl_sync(0xffffffffu, tot[w], 0);
  f = tau * tot[0] + 0.5 * tot[2];
  nnz = tot[1];
  applied = tot[3];
  colops = tot[4];
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

// !SYNC launches: the samples of its epochs, in order -- a warp folds each
// epoch and writes its sample (all SMs); the last CTA to finish (threadfence +
// ticket) finds the first stopping epoch and writes the loop state.  The sample
// count of epoch ep is n_samples + ep: a record loop has no other state.
constexpr int kFoldMax = 256;  // epochs per launch (the chunk's E <= this)
__global__ void cd_pair_fold(const double* partials, unsigned nblocks, uint64_t epochs, CdDev* st,
                             CdSample* trace, double* vals, unsigned* ticket) {
  if (*(volatile int*)&st->stop) return;
  const uint64_t ep = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t epoch0 = st->epoch, max_epochs = st->max_epochs, cap = st->cap, ns0 = st->n_samples;
  if (ep < epochs) {
    double f, nnz, applied, colops;
    epoch_objective_warp<false>(partials + (size_t)ep * nblocks * 5, nblocks, st->tau, f, nnz, applied, colops);
    if ((threadIdx.x & 31) == 0) {
      vals[ep * 4 + 0] = f;
      vals[ep * 4 + 1] = nnz;
      vals[ep * 4 + 2] = applied;
      vals[ep * 4 + 3] = colops;
      const uint64_t slot = ns0 + ep;  // (samples after a stopping epoch lie past n_samples: never read)
      if (slot < cap) trace[slot] = CdSample{epoch0 + ep + 1, f, nnz, applied, colops, global_timer_ns()};
    }
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the first epoch that stops the run: non-finite objective or the epoch budget
  __shared__ unsigned long long first;
  if (threadIdx.x == 0) first = epochs;
  __syncthreads();
  for (uint64_t e = threadIdx.x; e < epochs; e += blockDim.x) {
    const double f = __ldcg(&vals[e * 4]);
    if (!isfinite(f) || epoch0 + e + 1 >= max_epochs) atomicMin(&first, (unsigned long long)e);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t lastep = first < epochs ? first : epochs - 1;
  const double f = __ldcg(&vals[lastep * 4]);
  st->n_samples = ns0 + lastep + 1;
  st->epoch = epoch0 + lastep + 1;
  st->applied = (unsigned long long)__ldcg(&vals[lastep * 4 + 2]);
  st->colops = (unsigned long long)__ldcg(&vals[lastep * 4 + 3]);
  st->f = f;
  st->last_ts = global_timer_ns();
  if (first < epochs) {
    st->stop = 1;
    st->status = !isfinite(f) ? -1 : 1;
  }
  *ticket = 0;  // ready for the next launch
}

constexpr int kPairThreads = 128;  // more SMs, one warp per sub-partition (the epoch is a latency chain)

// Event masks (the default when an epoch has at most 64 MW blocks, C2: 128):
// bit bl of mask[e][member][bl >> 6][u] = member `member` of pair u steps in
// block bl of epoch e.  Ascending set bits are the pair's events in block
// order: no per-pair sort, no event list.  MW = 0: the event lists (cnt / ev).
__global__ void cd_mask_scatter_kernel(const uint32_t* __restrict__ idx, const uint16_t* __restrict__ prevd,
                                       const uint64_t* __restrict__ s, uint64_t nb, uint64_t per_epoch,
                                       int off, uint64_t U, int MW, unsigned long long* __restrict__ mask,
                                       uint64_t have) {
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t lim = s[nb] < have ? s[nb] : have;  // (a failed walk is handed over after the launch)
  for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; b < nb; b += warps) {
    const uint64_t s0 = min(s[b], lim), s1 = min(s[b + 1], lim);
    const uint64_t e = b / per_epoch, bl = b % per_epoch;
    for (uint64_t q = s0 + lane; q < s1; q += 32) {
      const uint16_t d = prevd[q];
      if (d == kPrevRej) continue;
      if (d != 0 && (uint64_t)d <= q - s0) continue;  // redrawn
      const uint64_t i = idx[q] + (uint64_t)off;
      const uint64_t u = i >> 1, mem = i & 1;
      atomicOr(&mask[((e * 2 + mem) * MW + (bl >> 6)) * U + u], 1ull << (bl & 63));
    }
  }
}

// sum of 5 doubles over the warp, lane 0 (fixed order)
__device__ __forceinline__ void warp_sum5(double* v) {
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int w = 0; w < 5; ++w) v[w] += __shfl_down_sync(0xffffffffu, v[w], o);
}

// SYNC: a grid barrier per epoch, the objective and the stop test in the
// kernel (runs with a target).  !SYNC: epochs back to back, each WARP's
// partials kept per epoch (no block barrier: warps run their epochs
// independently); cd_pair_fold records the samples afterwards (no target: only
// the epoch budget or a non-finite objective stops a run, and the budget is
// the launch's epoch count).
template <int P, bool SYNC, int MW>
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
  const unsigned nwarps = (unsigned)(T >> 5), gwarp = (unsigned)(g0 >> 5);
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
  // the step's scale beta L_i and threshold tau / (beta L_i) (solvers.cpp:457-458),
  // the same operations on the same operands as every step recomputes them
  double sc[P][2], th[P][2];
#pragma unroll
  for (int k = 0; k < P; ++k)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      sc[k][e] = beta * li[k][e];
      th[k][e] = tau / sc[k][e];
    }
  // rows [n, m) stay 0 - b (empty rows): their ||r||^2 share, once
  double tail = 0.0;
  for (uint64_t i = (uint64_t)n + g0; i < A.m; i += T) tail += A.r[i] * A.r[i];
  double acc[5];  // ||x||_1, nnz, ||r||^2, applied, colops of the running epoch
  // one block of pair k: the members in `in` step against the block's residual
  // rows, then the rows take r + sum_c delta_c A(rho, c) in ascending column order
  auto block_step = [&](int k, int in) {
    const double r0 = r[k][0], r1 = r[k][1];
    double d[2] = {0.0, 0.0};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (!((in >> e) & 1) || li[k][e] == 0.0) continue;  // zero columns are skipped (solvers.cpp:455)
      double gi = 0.0;
      for (int q = 0; q < nc[k][e]; ++q) gi += cv[k][e][q] * (cr[k][e][q] ? r1 : r0);
      acc[4] += 1.0;
      const double xi = x[k][e];
      const double xn = soft_threshold(xi - gi / sc[k][e], th[k][e]);
      d[e] = xn - xi;
      if (d[e] != 0.0) {
        x[k][e] = xn;
        acc[3] += 1.0;
        acc[4] += 1.0;
      }
    }
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
  };
  // one member e alone in its block (the common case: a block holds B of n
  // coordinates): block_step(k, 1 << e) with the member picked by selects, so a
  // warp runs one FP64 division per event instead of both members' code
  auto one_step = [&](int k, int e) {
    const double lie = e ? li[k][1] : li[k][0];
    if (lie == 0.0) return;  // zero columns are skipped (solvers.cpp:455)
    const double r0 = r[k][0], r1 = r[k][1];
    const int nce = e ? nc[k][1] : nc[k][0];
    const int c0 = e ? cr[k][1][0] : cr[k][0][0], c1 = e ? cr[k][1][1] : cr[k][0][1];
    const double v0 = e ? cv[k][1][0] : cv[k][0][0], v1 = e ? cv[k][1][1] : cv[k][0][1];
    double gi = 0.0;
    if (nce > 0) gi += v0 * (c0 ? r1 : r0);
    if (nce > 1) gi += v1 * (c1 ? r1 : r0);
    acc[4] += 1.0;
    const double xi = e ? x[k][1] : x[k][0];
    const double xn = soft_threshold(xi - gi / (e ? sc[k][1] : sc[k][0]), e ? th[k][1] : th[k][0]);
    const double d = xn - xi;
    if (d == 0.0) return;
    if (e) x[k][1] = xn;
    else x[k][0] = xn;
    acc[3] += 1.0;
    acc[4] += 1.0;
    double w0 = r0, w1 = r1;
    bool a0 = false, a1 = false;
    if (nce > 0) {
      if (c0) { w1 += d * v0; a1 = true; } else { w0 += d * v0; a0 = true; }
    }
    if (nce > 1) {
      if (c1) { w1 += d * v1; a1 = true; } else { w0 += d * v1; a0 = true; }
    }
    if (a0) r[k][0] = w0;
    if (a1) r[k][1] = w1;
  };
  auto step = [&](int k, int in) {
    if (in == 3) block_step(k, 3);
    else one_step(k, in >> 1);
  };
  // MW > 0: the masks are loaded two epochs ahead; MW == 0: the bucket count
  // and first kPre events one epoch ahead
  constexpr int kPre = 4;
  constexpr int NM = MW > 0 ? 2 * MW : 1;
  // mask mode: a 3-epoch ring in shared memory filled by cp.async two epochs
  // ahead (no registers held by pending loads)
  __shared__ __align__(16) unsigned long long mring[MW > 0 ? 3 : 1][kPairThreads][MW > 0 ? P * NM : 1];
  auto issue_masks = [&](uint64_t ep) {
    if constexpr (MW > 0) {
      if (ep < A.epochs) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
          if (!live[k]) continue;
          const uint64_t u = g0 + (uint64_t)k * T;
#pragma unroll
          for (int w = 0; w < NM; ++w) {
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&mring[ep % 3][threadIdx.x][k * NM + w]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa),
                         "l"(&A.mask[(ep * NM + w) * A.U + u]));
          }
        }
      }
      asm volatile("cp.async.commit_group;");
    }
  };
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
  if constexpr (MW > 0) {
    issue_masks(0);
    issue_masks(1);
  } else {
    prefetch(0);
  }
  for (uint64_t ep = 0; ep < A.epochs; ++ep) {
#pragma unroll
    for (int w = 0; w < 5; ++w) acc[w] = 0.0;
    unsigned long long cur_m[P][NM];
    uint32_t cur_c[P], cur_k[P][kPre];
    if constexpr (MW > 0) {
      issue_masks(ep + 2);
      asm volatile("cp.async.wait_group 2;" ::: "memory");  // epoch ep's group has landed
#pragma unroll
      for (int k = 0; k < P; ++k)
#pragma unroll
        for (int w = 0; w < NM; ++w) cur_m[k][w] = live[k] ? mring[ep % 3][threadIdx.x][k * NM + w] : 0ull;
    } else {
#pragma unroll
      for (int k = 0; k < P; ++k) {
        cur_c[k] = pc[k];
#pragma unroll
        for (int j = 0; j < kPre; ++j) cur_k[k][j] = pk[k][j];
      }
      prefetch(ep + 1);
    }
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (!live[k]) continue;
      if constexpr (MW > 0) {
        // member masks m0 = cur_m[k][0 .. MW), m1 = cur_m[k][MW .. 2 MW): set
        // bits of their union in ascending order = the pair's blocks
#pragma unroll
        for (int w = 0; w < MW; ++w) {
          unsigned long long m0 = cur_m[k][w], m1 = cur_m[k][MW + w], both = m0 | m1;
          while (both) {
            const unsigned long long bit = both & (~both + 1ull);
            both ^= bit;
            step(k, ((m0 & bit) ? 1 : 0) | ((m1 & bit) ? 2 : 0));
          }
        }
      } else {
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
          step(k, in);
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
    warp_sum5(acc);
    double* part = A.partials + (size_t)(SYNC ? (ep & 1) : ep) * nwarps * 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
      for (int q = 0; q < 5; ++q) part[(size_t)gwarp * 5 + q] = acc[q];
    }
    if constexpr (!SYNC) continue;
    cg::this_grid().sync();
    __shared__ double fo[4];
    if (threadIdx.x < 32) {
      double f, nnz, applied, colops;
      epoch_objective_warp(part, nwarps, tau, f, nnz, applied, colops);
      if (threadIdx.x == 0) {
        fo[0] = f;
        fo[1] = nnz;
        fo[2] = applied;
        fo[3] = colops;
      }
    }
    __syncthreads();
    const double f = fo[0], nnz = fo[1], applied = fo[2], colops = fo[3];
    __syncthreads();
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

template <int P, int MW>
int cd_pair_capacity() {
  static const int cap = [] {
    int per_sm = 0, per_sm2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cd_pair_kernel<P, true, MW>, kPairThreads, 0) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, cd_pair_kernel<P, false, MW>, kPairThreads, 0) !=
            cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return std::min(per_sm, per_sm2) * sm_count();
  }();
  return cap;
}

template <int MW>
void pick_pair_kernel(bool sync, const std::function<void(int, int, const void*)>& try_p) {
  auto fn = [&](auto pc) -> const void* {
    constexpr int Pk = decltype(pc)::value;
    return sync ? (const void*)cd_pair_kernel<Pk, true, MW> : (const void*)cd_pair_kernel<Pk, false, MW>;
  };
  try_p(1, cd_pair_capacity<1, MW>(), fn(std::integral_constant<int, 1>()));
  try_p(2, cd_pair_capacity<2, MW>(), fn(std::integral_constant<int, 2>()));
  if constexpr (MW == 0) try_p(4, cd_pair_capacity<4, MW>(), fn(std::integral_constant<int, 4>()));
}

uint64_t uniform_index(std::mt19937_64& g, uint64_t n) {  // rng.hpp:37-45
  const uint64_t lim = coord_index_limit(n);
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


// Page-locked host staging kept per thread and grown on demand: a solve does
// not pay cudaMallocHost (milliseconds for megabytes) after the first.
template <class T>
T* pinned_scratch(int slot, size_t count) {
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    ~Buf() {
      if (p) cudaFreeHost(p);
    }
  };
  thread_local Buf bufs[4];
  Buf& b = bufs[slot];
  const size_t want = std::max<size_t>(count * sizeof(T), 64);
  if (b.bytes < want) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.bytes = 0;
    L1B_CUDA(cudaMallocHost(&b.p, want + want / 2));
    b.bytes = want + want / 2;
  }
  return static_cast<T*>(b.p);
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
  // barrier); without one the epochs run back to back.  Epochs of at most 256
  // blocks take event masks (MW words per member), longer ones event lists.
  const bool sync = cfg->has_target != 0;
  int mw = per_epoch <= 128 ? 2 : 0;
  if (mw) pick_pair_kernel<2>(sync, try_p);
  if (!P) {  // (mask kernels take at most 2 pairs per thread)
    mw = 0;
    pick_pair_kernel<0>(sync, try_p);
  }
  if (!P) return 0;
  const uint64_t nwarps = (uint64_t)grid * (kPairThreads / 32);
  cudaStream_t st = v.stream;
  // chunks of up to ~2^22 draws (C2's 100 epochs: one chunk): the stream for the
  // next chunk is drawn (side stream, jump-started chunks on all SMs) while the
  // current chunk's walk and epochs run
  const uint64_t E_max = std::max<uint64_t>(
      1, std::min<uint64_t>(std::min<uint64_t>(cfg->max_iters, kFoldMax), (1ull << 22) / (per_epoch * B)));
  // rejected raw draws per kept one: < n / 2^64 with the reference's limit,
  // ~2^-s under the L1B_TEST_INDEX_REJECT hook
  const double p_rej = (double)(UINT64_MAX - coord_index_limit(n)) * 0x1p-64;
  const double rej = p_rej / (1.0 - p_rej);
  auto margin = [&](uint64_t T) {  // ~2x the expected redraws (B / 2n per draw, plus rejections)
    return T * B / n + (uint64_t)(2.0 * rej * (double)T) + 4096;
  };
  const uint64_t cap_raw = 2 * (E_max * per_epoch * B + margin(E_max * per_epoch * B));  // one chunk
  const uint64_t G = cap_raw / 2;  // draws per generator launch
  // stream buffer: the whole run when it fits in 2^25 draws, else rewound
  const uint64_t run_draws = cfg->max_iters * per_epoch * B;
  const uint64_t scap = std::min<uint64_t>(run_draws + margin(run_draws) + 2 * cap_raw, (1ull << 25) + 2 * cap_raw);
  // look-back: a block is B kept draws plus ~B^2 / 2n redraws; W bounds its
  // length (a longer block hands the run to the direct path)
  // (B = 1, serial CD: a block never redraws; no look-back, only rejected raw
  // draws become candidates)
  const int W = (int)(B + 64 + 4 * ((B * B + 2 * n - 1) / (2 * n)) + (uint64_t)(4.0 * rej * (double)B));
  const int W_prev = B == 1 ? 0 : W;
  std::vector<void*> bufs;
  cudaStream_t st0 = v.stream;
  keep_pool(v.device);
  // stream-ordered pool (kept cached): no cudaMalloc after the first solve;
  // out of memory hands the run to the direct path
  auto alloc = [&](auto** ptr, size_t bytes) {
    const cudaError_t e = cudaMallocAsync((void**)ptr, std::max<size_t>(bytes, 8), st0);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw Unsupported("pcdm pairs: device memory");
    }
    L1B_CUDA(e);
    bufs.push_back((void*)*ptr);
  };
  // L1B_PCDM_TRACE=1: host-side phase times on stderr
  const bool tracing = getenv("L1B_PCDM_TRACE") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto ptrace = [&](const char* what) {
    if (!tracing) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[pcdm pairs] %-20s %8.1f us\n", what, std::chrono::duration<double, std::micro>(now - tprev).count());
    tprev = now;
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
    alloc(&S[0], (scap + 312) * 4);  // + one generator round of slack
    alloc(&prevd, (cap_raw + 312) * 2);
    alloc(&sarr, (E_max * per_epoch + 1) * 8);
    alloc(&cnt, E_max * U * 4);
    alloc(&ev, E_max * kEvCap * U * 4);
    alloc(&win, 312 * 8);
    alloc(&words, (G + 312) * 8);
    alloc(&flag, 16);
    alloc(&part, (size_t)(sync ? 2 : E_max) * nwarps * 5 * 8);
    double* fvals = nullptr;
    alloc(&fvals, (size_t)E_max * 4 * 8 + 16);
    unsigned* fticket = reinterpret_cast<unsigned*>(fvals + E_max * 4);
    L1B_CUDA(cudaMemsetAsync(fticket, 0, 8, st0));
    unsigned long long* mask = nullptr;
    if (mw) alloc(&mask, (size_t)E_max * 2 * mw * U * 8);
    const uint64_t max_tiles = (cap_raw + 312 + kCandTile - 1) / kCandTile;
    alloc(&tile_cnt, (max_tiles + 1) * 4);
    alloc(&cand, (cap_raw + 312) * 8);
    L1B_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, tile_cnt, tile_cnt, (int)(max_tiles + 1), st));
    // look-back by a stable sort of (coordinate, position) (blocks of B > 1)
    const int key_bits = 64 - __builtin_clzll((unsigned long long)n);  // keys 0 .. n
    uint32_t *key = nullptr, *pos_in = nullptr, *skey = nullptr, *spos = nullptr;
    size_t sort_bytes = 0;
    if (W_prev > 0) {
      alloc(&key, (cap_raw + 312) * 4);
      alloc(&pos_in, (cap_raw + 312) * 4);
      alloc(&skey, (cap_raw + 312) * 4);
      alloc(&spos, (cap_raw + 312) * 4);
      L1B_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, key, skey, pos_in, spos,
                                               (int)(cap_raw + 312), 0, key_bits, st));
    }
    alloc(&scan_tmp, std::max(scan_bytes, sort_bytes));
    h_starts_pinned = pinned_scratch<uint64_t>(0, 64);  // [0]: the chunk's end, [1..]: level offsets
    h_flag = pinned_scratch<int>(1, 4);
    uint64_t* h_lvoff = h_starts_pinned + 1;
    // the device walk: segment heads, the phase maps of every tree level
    const uint64_t max_seg = (cap_raw + 312 + kSegLen - 1) / kSegLen;
    uint64_t *seg_first = nullptr, *seg_lv = nullptr, *lvoff = nullptr;
    alloc(&seg_first, max_seg * 8);
    alloc(&seg_lv, (2 * max_seg + 64) * (uint64_t)W * 8);
    alloc(&lvoff, 64 * 8);
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
    ptrace("set up");
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
    a.mask = mask;
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
      // draws the rest of the run can consume (blocks + expected redraws, x2 margin)
      const uint64_t rest = (cfg->max_iters - launched) * per_epoch * B;
      const uint64_t total_bound = pos + rest + margin(rest);
      for (;;) {
        if (need > cap_raw) throw Unsupported("pcdm pairs: chunk buffer");
        // this chunk's draws, and one launch ahead while the run can still use it
        gen_to(std::max(pos + need, std::min(pos + need + G, total_bound)));
        wait_for(pos + need);
        have = need;
        if (W_prev > 0) {
          cd_key_kernel<<<grid_for(have), kThreads, 0, st>>>(idx, have, (uint32_t)n, key, pos_in);
          L1B_LAUNCHED();
          size_t sb = sort_bytes;
          L1B_CUDA(cub::DeviceRadixSort::SortPairs(scan_tmp, sb, key, skey, pos_in, spos, (int)have, 0, key_bits,
                                                   st));
          cd_prevd_sorted_kernel<<<grid_for(have), kThreads, 0, st>>>(skey, spos, have, (uint32_t)n, W_prev,
                                                                      prevd);
          L1B_LAUNCHED();
        } else {
          cd_prevd_kernel<<<(unsigned)((have + kThreads - 1) / kThreads), kThreads, (W + kThreads) * 4, st>>>(
              idx, have, W_prev, prevd);
          L1B_LAUNCHED();
        }
        const uint64_t tiles = (have + kCandTile - 1) / kCandTile;
        cd_cand_count<<<(unsigned)tiles, kThreads, 0, st>>>(prevd, have, tile_cnt);
        L1B_LAUNCHED();
        L1B_CUDA(cudaMemsetAsync(tile_cnt + tiles, 0, 4, st));
        size_t tb = scan_bytes;
        L1B_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, tb, tile_cnt, tile_cnt, (int)(tiles + 1), st));
        cd_cand_write<<<(unsigned)tiles, kThreads, 0, st>>>(prevd, have, tile_cnt, cand);
        L1B_LAUNCHED();
        // block starts on the device (no host round trip); a stream too short
        // for nb blocks leaves starts[nb] at ~0 and hands the run over below
        const uint64_t nseg = (have + kSegLen - 1) / kSegLen;
        const uint32_t* ncand_d = tile_cnt + tiles;
        L1B_CUDA(cudaMemsetAsync(flag, 0, 4, st));
        L1B_CUDA(cudaMemsetAsync(sarr + nb, 0xff, 8, st));
        if (B == 1) {
          cd_b1_starts_kernel<<<grid_for(nb + 1), kThreads, 0, st>>>(cand, ncand_d, nb, sarr);
          L1B_LAUNCHED();
          break;
        }
        cd_seg_first_kernel<<<blocks_for(nseg), kThreads, 0, st>>>(cand, ncand_d, nseg, seg_first);
        L1B_LAUNCHED();
        cd_seg_walk_kernel<<<(unsigned)nseg, (unsigned)std::min(1024, (W + 31) / 32 * 32), 0, st>>>(cand, ncand_d, seg_first,
                                                                                      nseg, B, W, seg_lv, flag);
        L1B_LAUNCHED();
        int nlevels = 1;
        {
          LevelTab tab;
          uint64_t n_l = nseg, o = 0;
          tab.off[0] = 0;
          tab.cnt[0] = nseg;
          h_lvoff[0] = 0;
          while (n_l > 1) {  // level sizes and offsets
            o += n_l * W;
            n_l = (n_l + 1) / 2;
            if (nlevels >= 40) throw Unsupported("pcdm pairs: walk tree depth");
            tab.off[nlevels] = o;
            tab.cnt[nlevels] = n_l;
            h_lvoff[nlevels++] = o;
          }
          for (int l0 = 0; l0 + 1 < nlevels; l0 += kComposeLevels) {
            const int l1 = std::min(nlevels - 1, l0 + kComposeLevels);
            const uint64_t groups = (tab.cnt[l0] + (1ull << kComposeLevels) - 1) >> kComposeLevels;
            cd_seg_compose_kernel<<<(unsigned)groups, 512, 0, st>>>(seg_lv, tab, l0, l1, W);
            L1B_LAUNCHED();
          }
          L1B_CUDA(cudaMemcpyAsync(lvoff, h_lvoff, nlevels * 8, cudaMemcpyHostToDevice, st));
        }
        cd_seg_emit_kernel<<<(unsigned)((nseg + 3) / 4), 128, 0, st>>>(cand, ncand_d, seg_first, seg_lv, lvoff,
                                                                     nlevels, nseg, B, W, nb, sarr);
        L1B_LAUNCHED();
        ptrace("walk queued");
        if (getenv("L1B_PCDM_WALK_CHECK")) {  // the device walk against the sequential one (tests)
          uint32_t nc = 0;
          L1B_CUDA(cudaMemcpyAsync(&nc, ncand_d, 4, cudaMemcpyDeviceToHost, st));
          L1B_CUDA(cudaStreamSynchronize(st));
          std::vector<uint64_t> hc(nc), dev(nb + 1);
          if (nc) L1B_CUDA(cudaMemcpy(hc.data(), cand, (size_t)nc * 8, cudaMemcpyDeviceToHost));
          L1B_CUDA(cudaMemcpy(dev.data(), sarr, (nb + 1) * 8, cudaMemcpyDeviceToHost));
          uint64_t sb = 0, j = 0;
          for (uint64_t blk = 0; blk <= nb; ++blk) {
            if (dev[blk] != sb) {
              fprintf(stderr, "[pcdm pairs] walk mismatch at block %llu: device %llu, host %llu\n",
                      (unsigned long long)blk, (unsigned long long)dev[blk], (unsigned long long)sb);
              throw std::runtime_error("pcdm pairs: device walk differs from the sequential walk");
            }
            uint64_t e = sb + B;
            while (j < nc && (hc[j] >> 16) < e) {
              const uint64_t q = hc[j] >> 16, d = hc[j] & 0xffff;
              if (d == kPrevRej || q - d >= sb) ++e;
              ++j;
            }
            sb = e;
          }
        }
        break;
      }
      if (mw) {
        L1B_CUDA(cudaMemsetAsync(mask, 0, (size_t)E * 2 * mw * U * 8, st));
        cd_mask_scatter_kernel<<<grid_for(nb * 32), kThreads, 0, st>>>(idx, prevd, sarr, nb, per_epoch, a.off, U,
                                                                      mw, mask, have);
      } else {
        L1B_CUDA(cudaMemsetAsync(cnt, 0, E * U * 4, st));
        const int lanes = B >= 32 ? 32 : 1;  // per block
        cd_scatter_kernel<<<grid_for(nb * lanes), kThreads, 0, st>>>(idx, prevd, sarr, nb, per_epoch, a.off, U,
                                                                    lanes, cnt, ev, flag, have);
      }
      L1B_LAUNCHED();
      a.epochs = E;
      void* args[] = {&a};
      if (sync) {
        L1B_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kPairThreads), args, 0, st));
        L1B_LAUNCHED();
      } else {
        L1B_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kPairThreads), args, 0, st));
        L1B_LAUNCHED();
        cd_pair_fold<<<(unsigned)((E + 3) / 4), 128, 0, st>>>(part, (unsigned)nwarps, E, dst, trace, fvals,
                                                             fticket);
        L1B_LAUNCHED();
      }
      L1B_CUDA(cudaMemcpyAsync(h_flag, flag, 4, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaMemcpyAsync(h_starts_pinned, sarr + nb, 8, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaMemcpyAsync(h_st, dst, sizeof(CdDev), cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
      ptrace("epochs done");
      const uint64_t used = h_starts_pinned[0];
      if (*h_flag & 4) throw Unsupported("pcdm pairs: event bucket");
      if (*h_flag & 16) throw Unsupported("pcdm pairs: block longer than the look-back");
      if (used > have) throw Unsupported("pcdm pairs: stream shorter than the chunk's blocks");
      pos += used;  // the draws past the chunk's last block open the next chunk
      drop_pieces(pos);
      launched += E;
      if (h_st->stop) break;
    }
  } catch (const Unsupported& e) {
    rc = -1;
    if (tracing) fprintf(stderr, "[pcdm pairs] declined: %s\n", e.what());
  } catch (...) {
    cudaStreamSynchronize(st);
    if (gs) cudaStreamSynchronize(gs);
    if (gs) cudaStreamDestroy(gs);
    for (auto& pc : pieces) cudaEventDestroy(pc.second);
    for (void* q : bufs) cudaFreeAsync(q, st0);
    throw;
  }
  cudaStreamSynchronize(st);
  if (gs) cudaStreamSynchronize(gs);
  if (gs) cudaStreamDestroy(gs);
  for (auto& pc : pieces) cudaEventDestroy(pc.second);
  for (void* q : bufs) cudaFreeAsync(q, st0);
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
  keep_pool(v.device);
  auto alloc = [&](auto** ptr, size_t bytes) {  // stream-ordered pool, kept cached
    L1B_CUDA(cudaMallocAsync((void**)ptr, std::max<size_t>(bytes, 8), st));
    bufs.push_back((void*)*ptr);
  };
  uint32_t* h_coords = nullptr;  // two chunk buffers: generate one while the other uploads
  CdDev* h_st = nullptr;
  cudaEvent_t uploaded[2] = {nullptr, nullptr};
  // the direct path's buffers (host draws, planned or direct epochs): only when
  // the pair-local path does not run
  auto alloc_direct = [&]() {
    alloc(&delta, n * 8);
    alloc(&stamp, n * 4);
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
    h_coords = pinned_scratch<uint32_t>(3, 2 * chunk * per_epoch * B);
    for (auto& e : uploaded) L1B_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  };
  try {
    alloc(&x, n * 8);
    alloc(&r, v.m * 8);
    alloc(&partials, (size_t)spmv_grid_max() * 4 * 8);
    alloc(&dst, sizeof(CdDev));
    alloc(&trace, tcap * sizeof(CdSample));
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
      if (stamp) L1B_CUDA(cudaMemsetAsync(stamp, 0, n * 4, st));
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
      alloc_direct();
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
    for (void* q : bufs) cudaFreeAsync(q, st);
    if (h_st) cudaFreeHost(h_st);
    for (auto e : uploaded)
      if (e) cudaEventDestroy(e);
    throw;
  }
  for (void* q : bufs) cudaFreeAsync(q, st);
  cudaStreamSynchronize(st);
  cudaFreeHost(h_st);
  for (auto e : uploaded)
    if (e) cudaEventDestroy(e);
}

}  // namespace l1b
