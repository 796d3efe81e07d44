// One FISTA iteration per kernel, matrix-free, with the residuals RECOMPUTED
// instead of stored (banded operators, 1..4 right stages).
//
// The reference keeps r_x = A x - b and r_y = A y - b as vectors
// (solvers.cpp:311-377).  The single-kernel path in k_fused.cu stores r_k and
// reads r_k, r_{k-1} back: 64n bytes per iteration.  Here r_k and r_{k-1} are
// rebuilt from x_k and x_{k-1} with the very operations that produced them
// (sigma .* (G^T x) - b, identical operands and order => identical bits), so
// an iteration streams only x_k, x_{k-1}, sigma, b and writes x_{k+1}:
// 40n bytes.  The extra Givens work runs on registers:
//
//   * a warp holds a window of 128 consecutive entries, 4 per lane (one
//     256-bit load per array and lane, a warp load = 1 KiB contiguous);
//   * a stage whose pairs start on even entries is lane-local; an odd stage
//     rotates (v1, v2) in the lane, and the pair straddling lanes l, l+1 is
//     rotated by lane l (neighbour's entry in by one shuffle, the right output
//     back by another) -- every rotation is done exactly once;
//   * per iteration the chain runs three times (r_k and r_{k-1} side by side,
//     then g = G u); each of the two runs in series invalidates S entries at
//     both window ends, so the window carries a halo of H3 >= 2S entries per
//     side and owns the middle 128 - 2 H3 (112 for 3-4 stages);
//   * ||r_{k+1}||^2 is not formed here: the next kernel sums ||r_k||^2 from the
//     r_k it rebuilds anyway, and the objective is recorded one kernel late
//     (fista_finalize_lagged; a flush launch records the last iterate);
//   * no shared memory and no block barriers in the loop: warps stream their
//     segments independently, with the next segment's loads in flight while
//     the current one computes.
//
// Per segment (own entries [a, a + OWN), window [a - H3, a + OWN + H3)):
//   r_k     = sigma .* (G^T x_k)     - b          (solvers.cpp:357, linops.cpp:433)
//   r_{k-1} = sigma .* (G^T x_{k-1}) - b
//   u       = sigma .* ((1 + beta) r_k - beta r_{k-1})        (r_y, then A^T's sigma)
//   g       = G u                                              (A^T r_y)
//   y       = x_k + beta (x_k - x_{k-1});  trial = S(y - g/L, tau/L)   (:325-336)
//   own:      x_{k+1} = trial; ||x_{k+1}||_1, nnz, #(trial != y); ||r_k||^2
//
// Kernels in this file:
//   fista_rc_kernel      one iteration per launch (shards with L1B_RC2=0, odd
//                        remainders, the flush that records the last iterate)
//   fista_rc2v_kernel    TWO iterations per launch, V entries per lane (the
//                        default, V = 8: 24n bytes per iteration)
//   fista_rc_persistent  up to a chunk of iterations in one cooperative
//                        launch (small instances, n <= 2^20)
//   fista_pair_cluster   single-stage instances (n <= 16384): pair-local
//                        products, state in registers, an 8-CTA cluster for
//                        the whole chunk
#include "common.cuh"
#include "fista.cuh"
#include "kernels.hpp"

#include <cooperative_groups.h>
#include <cstdlib>

#ifndef TB_WARPS
#define TB_WARPS 8
#endif

namespace l1b {
namespace {

constexpr int kRcThreads = 256;
constexpr int kRcWarps = kRcThreads / 32;
constexpr int kWin = 128;  // window entries per warp (4 per lane)
constexpr unsigned kFull = 0xffffffffu;

template <int S>
struct RcGeom {
  // halo: two chains in series (r = sigma G^T x - b, then g = G u) each spoil S
  // entries per window end; 32-byte aligned
  static constexpr int H3 = (2 * S + 3) / 4 * 4;
  static constexpr int OWN = kWin - 2 * H3;
};

struct RcArgs {
  int64_t n, lo, hi;
  StageTab right;
  const double* sigma;  // global index
  IterBufs b;           // x_k, x_km1, x_next, b by global index (r_* unused)
  // row-block shards with attached peers: the new x entries within ph of the
  // block ends are also stored straight into the neighbours' x windows
  // (global-index views; [0]: x_{k+1}, [1]: x_{k+2}) -- the halo exchange
  // rides on the kernel's own stores over NVLink instead of NCCL send / recv
  PeerViews peers;
};

template <int V>
__device__ __forceinline__ void peer_store(const RcArgs& A, int which, int64_t e0,
                                           const bool (&mine)[V], const double (&v)[V]) {
  if (!A.peers.on) return;
  const int64_t lo = A.lo, hi = A.hi, ph = A.peers.halo;
  if (e0 >= lo + ph && e0 + V <= hi - ph) return;
  double* l = A.peers.left[which];
  double* r = A.peers.right[which];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int64_t g = e0 + i;
    if (!mine[i]) continue;
    if (l && g < lo + ph) l[g] = v[i];
    if (r && g >= hi - ph) r[g] = v[i];
  }
}

__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
// x in the persistent kernel: written by other SMs between grid barriers -> L2 (.cg)
__device__ __forceinline__ void ld4cg(const double* p, double (&v)[4]) {
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double (&v)[4]) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]),
               "d"(v[3])
               : "memory");
}

struct Seg {
  double xk[4], xm[4], sg[4], bb[4];
};

// window group [e, e+4) of every input; entries outside [lim_lo, lim_hi) read 0.
// COH: x is read through L2 (the persistent kernel rewrites it between barriers).
template <bool COH = false>
__device__ __forceinline__ void load_seg(const RcArgs& A, int64_t e, bool full, int64_t lim_lo,
                                         int64_t lim_hi, Seg& s) {
  if (full) {
    if (COH) {
      ld4cg(A.b.x_k + e, s.xk);
      ld4cg(A.b.x_km1 + e, s.xm);
    } else {
      ld4(A.b.x_k + e, s.xk);
      ld4(A.b.x_km1 + e, s.xm);
    }
    ld4(A.sigma + e, s.sg);
    ld4(A.b.b + e, s.bb);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool in = e + i >= lim_lo && e + i < lim_hi;
      s.xk[i] = in ? (COH ? __ldcg(A.b.x_k + e + i) : A.b.x_k[e + i]) : 0.0;
      s.xm[i] = in ? (COH ? __ldcg(A.b.x_km1 + e + i) : A.b.x_km1[e + i]) : 0.0;
      s.sg[i] = in ? A.sigma[e + i] : 0.0;
      s.bb[i] = in ? A.b.b[e + i] : 0.0;
    }
  }
}

// All S stages on the warp's window; v holds entries [e0, e0+4) (e0 = 0 mod 4).
// Stage pairs (p, p+1), p = offset (mod 2), p >= offset, p + 1 < n
// (linops.cpp:46-60); INTERIOR: the window is away from both ends, every pair
// exists.  Entries within S of a window end come out wrong (their partners
// live outside the window) and are never used.
// PAR >= 0: bit s is the parity of stage s's offset, fixed at compile time
// (the generator's alternating offsets); PAR < 0: read from the table.
template <int S, bool TR, bool INTERIOR, int K, int PAR, bool F = false>
__device__ __forceinline__ void wchain(double (&v)[K][4], int64_t e0, int64_t n,
                                       const StageTab& tab) {
  // F: the scaled form of the contracted arithmetic (rot_scaled; the caller's
  // sigma carries prod cos(theta), entries a stage leaves unpaired take
  // 1 / cos(theta)) -- wchainv's operations at 4 entries per lane
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int s = TR ? k : S - 1 - k;  // A x: forward, transposed; A^T: reverse, plain
    const int o = tab.offset[s];
    const double c = F ? tab.tn[s] : tab.c[s], sn = F ? tab.ic[s] : tab.s[s];
    const int par = PAR >= 0 ? (PAR >> s) & 1 : (o & 1);
    auto pair = [&](double& a, double& b, bool ok) {
      if (F) {
        if (ok) rot_scaled(a, b, c, TR);
        else a *= sn, b *= sn;
      } else if (ok) {
        rotate_pair(a, b, c, sn, TR);
      }
    };
    if (par == 0) {
      const bool p0 = INTERIOR || (e0 >= o && e0 + 1 < n);
      const bool p2 = INTERIOR || (e0 + 2 >= o && e0 + 3 < n);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        pair(v[q][0], v[q][1], p0);
        pair(v[q][2], v[q][3], p2);
      }
    } else {
      // the pair straddling lanes l, l+1 is rotated once, by lane l, which
      // hands the right output back through a second shuffle
      double right[K], back[K];
#pragma unroll
      for (int q = 0; q < K; ++q) right[q] = __shfl_down_sync(kFull, v[q][0], 1);  // lane+1's first entry
      const bool p1 = INTERIOR || (e0 + 1 >= o && e0 + 2 < n);
      const bool p3 = INTERIOR || (e0 + 3 >= o && e0 + 4 < n);
      const bool pm = INTERIOR || (e0 - 1 >= o && e0 < n);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        double a = v[q][3], b = right[q];
        if (F) {
          if (p3) rot_scaled(a, b, c, TR);
          else a *= sn;
        } else if (p3) {
          rotate_pair(a, b, c, sn, TR);
        }
        v[q][3] = a;
        back[q] = b;
      }
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const double b = __shfl_up_sync(kFull, back[q], 1);  // lane-1's right output
        if (pm) v[q][0] = b;
        else if (F) v[q][0] *= sn;
      }
#pragma unroll
      for (int q = 0; q < K; ++q) pair(v[q][1], v[q][2], p1);
    }
  }
}

// Per-thread sums over the segments a thread sees
struct Acc {
  double l1 = 0.0, rr = 0.0;  // ||x_{k+1}||_1, ||r_k||^2 (own entries)
  unsigned nz = 0, mism = 0;  // nnz(x_{k+1}), #(trial != y)
};

// soft_threshold (solvers.cpp:153-157) with selects instead of branches (same values)
__device__ __forceinline__ double shrink(double v, double t) {
  const double a = v - t, c = v + t;
  return v > t ? a : (v < -t ? c : 0.0);
}

// One segment.  FAST: the window is away from both ends of [0, n) and of the
// shard's x windows and the segment owns OWN full entries, so every pair
// exists and a lane's four entries are either all own (lane_own) or all halo.
// FLUSH: only ||r_k||^2 of the own rows (the objective of the last iterate).
// SMEM: x_next is shared memory (generic stores instead of 256-bit global ones).
template <int S, bool FAST, bool FLUSH, int PAR, bool SMEM = false, bool F = false>
__device__ __forceinline__ void segment(const RcArgs& A, const Seg& d, int64_t w0, int lane,
                                        bool lane_own, double beta, double inv_l, double thr,
                                        Acc& acc) {
  using G = RcGeom<S>;
  const int64_t n = A.n;
  const int64_t e0 = w0 + 4 * lane;
  bool mine[4];
  if (FAST) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mine[i] = lane_own;
  } else {
    // own entries of this segment: [w0 + H3, min(w0 + H3 + OWN, hi))
    const int64_t own_lo = w0 + G::H3, own_hi = min(own_lo + G::OWN, A.hi);
#pragma unroll
    for (int i = 0; i < 4; ++i) mine[i] = e0 + i >= own_lo && e0 + i < own_hi;
  }
  constexpr int K = FLUSH ? 1 : 2;
  double t[K][4];  // G^T x_k and G^T x_{k-1}, side by side (independent chains)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    t[0][i] = d.xk[i];
    if (!FLUSH) t[K - 1][i] = d.xm[i];
  }
  wchain<S, true, FAST, K, PAR, F>(t, e0, n, A.right);
  double g[1][4], rr = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double rk = mul_sub<F>(d.sg[i], t[0][i], d.bb[i]);
    if (mine[i]) rr = F ? __fma_rn(rk, rk, rr) : rr + rk * rk;  // ||r_k||^2: x_k's objective, recorded one kernel late
    if (!FLUSH) {
      const double rm = mul_sub<F>(d.sg[i], t[K - 1][i], d.bb[i]);
      g[0][i] = d.sg[i] * mul_sub<F>(1.0 + beta, rk, beta * rm);
    }
  }
  acc.rr += rr;
  if (FLUSH) return;
  wchain<S, false, FAST, 1, PAR, F>(g, e0, n, A.right);
  double tr[4], l1 = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double y = F ? __fma_rn(beta, d.xk[i] - d.xm[i], d.xk[i]) : d.xk[i] + beta * (d.xk[i] - d.xm[i]);
    tr[i] = shrink(F ? __fma_rn(-inv_l, g[0][i], y) : y - inv_l * g[0][i], thr);
    l1 += mine[i] ? fabs(tr[i]) : 0.0;
    acc.nz += (unsigned)(mine[i] & (tr[i] != 0.0));
    acc.mism += (unsigned)(mine[i] & (tr[i] != y));
  }
  acc.l1 += l1;
  if (!SMEM) peer_store<4>(A, 0, e0, mine, tr);
  if (SMEM) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (mine[i]) A.b.x_next[e0 + i] = tr[i];
  } else if (FAST) {
    if (lane_own) st4(A.b.x_next + e0, tr);
  } else if (mine[0] && mine[3]) {
    st4(A.b.x_next + e0, tr);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (mine[i]) A.b.x_next[e0 + i] = tr[i];
  }
}

// Warps stream segments q = warp_id, warp_id + #warps, ...; the next segment's
// loads are issued before the current one computes.
template <int S, int MB, bool FLUSH = false, int PAR = -1, bool F = false>
__global__ void __launch_bounds__(kRcThreads, MB) fista_rc_kernel(RcArgs A) {
  using G = RcGeom<S>;
  FistaDev* st = A.b.st;
  if (*(volatile int*)&st->stop) return;
  const double beta = st->beta_y;  // forms y_k, r_y from the last two iterates
  const double inv_l = 1.0 / st->lval;
  const double thr = st->tau * inv_l;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool lane_own = 4 * lane >= G::H3 && 4 * lane < G::H3 + G::OWN;
  const int64_t n = A.n, lo = A.lo, hi = A.hi;
  // loads stay inside [0, n) and inside the x windows [lo - H3, hi + H3)
  const int64_t lim_lo = max((int64_t)0, lo - G::H3), lim_hi = min(n, hi + G::H3);
  const int64_t nseg = (hi - lo + G::OWN - 1) / G::OWN;
  // segments of one block are consecutive (their halos meet in L1/L2)
  const int64_t stride = (int64_t)gridDim.x * kRcWarps;
  Acc acc;

  auto w0_of = [&](int64_t q) { return lo + q * G::OWN - G::H3; };
  auto full_of = [&](int64_t w0) { return w0 >= lim_lo && w0 + kWin <= lim_hi; };
  auto load = [&](int64_t q, Seg& d) {
    const int64_t w0 = w0_of(q);
    load_seg(A, w0 + 4 * lane, full_of(w0), lim_lo, lim_hi, d);
  };
  // fast segments q in [q_lo, q_hi): the window lies inside the loadable range
  // and [2, n - 1) -- every pair touching it exists (p >= w0 - 1 >= 1 >= offset,
  // p + 1 <= w0 + kWin < n) -- and all OWN entries are inside [lo, hi)
  const int64_t base = lo - G::H3;  // w0 of segment 0
  const int64_t w_min = max((int64_t)2, lim_lo), w_max = min(lim_hi, n - 1) - kWin;
  const int64_t q_lo = w_min <= base ? 0 : (w_min - base + G::OWN - 1) / G::OWN;
  const int64_t q_hi = w_max < base ? 0 : min((w_max - base) / G::OWN + 1, (hi - lo) / G::OWN);
  auto run = [&](int64_t q, const Seg& d) {
    const int64_t w0 = w0_of(q);
    if (q >= q_lo && q < q_hi)
      segment<S, true, FLUSH, PAR, false, F>(A, d, w0, lane, lane_own, beta, inv_l, thr, acc);
    else
      segment<S, false, FLUSH, PAR, false, F>(A, d, w0, lane, lane_own, beta, inv_l, thr, acc);
  };
  Seg sa, sb;
  int64_t q = (int64_t)blockIdx.x * kRcWarps + warp;
  if (q < nseg) load(q, sa);
  // (measured slower: a two-way unrolled ping-pong without the copy -- code
  // size; an extra L2 bulk prefetch of the segment after next)
  for (; q < nseg; q += stride) {
    if (q + stride < nseg) load(q + stride, sb);
    run(q, sa);
    sa = sb;
  }
  if (A.peers.on) __threadfence_system();  // peer stores performed before the kernel ends
  double sums[4] = {acc.l1, (double)acc.nz, (double)acc.mism, acc.rr};
  double tot[4];
  if (grid_sum<4>(sums, A.b.partials, &st->ticket[0], tot) && threadIdx.x == 0) {
    st->scal[0] = tot[0];
    st->scal[1] = tot[1];
    st->scal[2] = tot[2];
    st->scal[3] = tot[3];
    if (FLUSH) st->flushing = 1;
    if (!st->defer) fista_finalize_lagged(st, A.b.trace, FLUSH);  // shards: after the all-reduce
  }
}

// ---------------------------------------------------------------------------
// Two iterations per kernel (temporal blocking).  x_{k+1} is formed on the
// whole window and kept in registers; the second iteration rebuilds only
// r_{k+1} (r_k is reused) and writes x_{k+2}: x_k, x_{k-1}, sigma, b read once
// and x_{k+1}, x_{k+2} written -- 48n bytes per two iterations (24n each
// instead of 40n).  Four chain runs in series spoil 4S entries per window end
// (halo 16 for 3-4 stages, 96 own entries of 128); five chain runs per two
// iterations.  Per entry the operations are those of segment(): identical
// iterates.
struct Acc2 {
  double rr0 = 0.0, l1a = 0.0, rr1 = 0.0, l1b = 0.0;  // ||r_k||^2, ||x_{k+1}||_1, ||r_{k+1}||^2, ||x_{k+2}||_1
  unsigned nza = 0, misa = 0, nzb = 0, misb = 0;
};

struct Rc2Out {
  double* x1;  // x_{k+1}
  double* x2;  // x_{k+2}
};

// ---------------------------------------------------------------------------
// The two-iteration kernel with V entries per lane (window 32 V): the halo
// (>= 4S, a multiple of V) is a smaller share of a wider window -- fewer
// rotations per own entry, more registers per thread.
template <int S, bool TR, bool INTERIOR, int K, int PAR, int V, bool F, bool SC = false, bool SYM = false>
__device__ __forceinline__ void wchainv(double (&v)[K][V], int64_t e0, int64_t n,
                                        const StageTab& tab) {
  // SC (= F): the scaled form of the contracted arithmetic -- every pair takes
  // [[1, -tan], [tan, 1]] and the caller's sigma carries prod cos(theta); an
  // entry a stage leaves unpaired (the ends of [0, n)) takes 1 / cos(theta).
  static_assert(SC == F, "contracted arithmetic <=> scaled form");
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int s = TR ? k : S - 1 - k;
    const int o = tab.offset[s];
    const double c = SC ? tab.tn[s] : tab.c[s];
    const double sn = SC ? tab.ic[s] : tab.s[s];
    const int par = PAR >= 0 ? (PAR >> s) & 1 : (o & 1);
    if (par == 0) {
#pragma unroll
      for (int p = 0; p < V; p += 2) {
        const bool ok = INTERIOR || (e0 + p >= o && e0 + p + 1 < n);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          if (SC) {
            if (ok) rot_scaled(v[q][p], v[q][p + 1], c, TR);
            else v[q][p] *= sn, v[q][p + 1] *= sn;
          } else if (ok) {
            rot<F>(v[q][p], v[q][p + 1], c, sn, TR);
          }
        }
      }
    } else {
      if (SYM && (SC || !F)) {
        // the pair straddling lanes l, l+1: each output of a rotation is a
        // function of the pair alone, so lane l forms the left output from its
        // neighbour's first entry and lane l+1 the right output from its
        // neighbour's last one -- the same operations as rotating the pair on
        // one lane (the same bits), one shuffle deep instead of shuffle ->
        // rotation -> shuffle back
        const bool pr = INTERIOR || (e0 + V - 1 >= o && e0 + V < n);
        const bool pl = INTERIOR || (e0 - 1 >= o && e0 < n);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const double right = __shfl_down_sync(kFull, v[q][0], 1);
          const double left = __shfl_up_sync(kFull, v[q][V - 1], 1);
          const double a = v[q][V - 1], b = v[q][0];
          if (SC) {
            v[q][V - 1] = pr ? __fma_rn(TR ? c : -c, right, a) : a * sn;
            v[q][0] = pl ? __fma_rn(TR ? -c : c, left, b) : b * sn;
          } else {  // rotate_pair's two outputs (linops.cpp:20-30)
            if (pr) v[q][V - 1] = TR ? c * a + sn * right : c * a - sn * right;
            if (pl) v[q][0] = TR ? -sn * left + c * b : sn * left + c * b;
          }
        }
      } else {
        // the pair straddling lanes l, l+1 is rotated once, by lane l, which
        // hands the right output back (one rotation fewer per lane and odd stage
        // than rotating it on both sides)
        double right[K], back[K];
#pragma unroll
        for (int q = 0; q < K; ++q) right[q] = __shfl_down_sync(kFull, v[q][0], 1);
        const bool pr = INTERIOR || (e0 + V - 1 >= o && e0 + V < n);
        const bool pl = INTERIOR || (e0 - 1 >= o && e0 < n);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          double a = v[q][V - 1], b = right[q];
          if (SC) {
            if (pr) rot_scaled(a, b, c, TR);
            else a *= sn;
          } else if (pr) {
            rot<F>(a, b, c, sn, TR);
          }
          v[q][V - 1] = a;
          back[q] = b;
        }
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const double b = __shfl_up_sync(kFull, back[q], 1);
          if (pl) v[q][0] = b;
          else if (SC) v[q][0] *= sn;
        }
      }
#pragma unroll
      for (int p = 1; p + 1 < V; p += 2) {
        const bool ok = INTERIOR || (e0 + p >= o && e0 + p + 1 < n);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          if (SC) {
            if (ok) rot_scaled(v[q][p], v[q][p + 1], c, TR);
            else v[q][p] *= sn, v[q][p + 1] *= sn;
          } else if (ok) {
            rot<F>(v[q][p], v[q][p + 1], c, sn, TR);
          }
        }
      }
    }
  }
}

template <int S, int V>
struct RcGeomV {
  static constexpr int W = 32 * V;
  static constexpr int H3 = (4 * S + V - 1) / V * V;
  static constexpr int OWN = W - 2 * H3;
};

template <int V>
struct SegV {
  double xk[V], xm[V], sg[V], bb[V];
};

template <int V>
__device__ __forceinline__ void ldv(const double* p, double (&v)[V]) {
  if (V % 4 == 0) {
#pragma unroll
    for (int j = 0; j < V; j += 4) {
      double t[4];
      ld4(p + j, t);
      v[j] = t[0], v[j + 1] = t[1], v[j + 2] = t[2], v[j + 3] = t[3];
    }
  } else {
#pragma unroll
    for (int j = 0; j < V; j += 2) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p + j));
      v[j] = t.x, v[j + 1] = t.y;
    }
  }
}

template <int V>
__device__ __forceinline__ void load_segv(const RcArgs& A, int64_t e, bool full, int64_t lim_lo,
                                          int64_t lim_hi, SegV<V>& s) {
  if (full) {
    ldv<V>(A.b.x_k + e, s.xk);
    ldv<V>(A.b.x_km1 + e, s.xm);
    ldv<V>(A.sigma + e, s.sg);
    ldv<V>(A.b.b + e, s.bb);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const bool in = e + i >= lim_lo && e + i < lim_hi;
      s.xk[i] = in ? A.b.x_k[e + i] : 0.0;
      s.xm[i] = in ? A.b.x_km1[e + i] : 0.0;
      s.sg[i] = in ? A.sigma[e + i] : 0.0;
      s.bb[i] = in ? A.b.b[e + i] : 0.0;
    }
  }
}

template <bool FAST, int V>
__device__ __forceinline__ void store_ownv(double* dst, int64_t e0, const bool (&mine)[V],
                                           bool lane_own, const double (&v)[V]) {
  if (FAST) {
    if (lane_own) {
      if (V % 4 == 0) {
#pragma unroll
        for (int j = 0; j < V; j += 4) {
          const double t[4] = {v[j], v[j + 1], v[j + 2], v[j + 3]};
          st4(dst + e0 + j, t);
        }
      } else {
#pragma unroll
        for (int j = 0; j < V; j += 2)
          *reinterpret_cast<double2*>(dst + e0 + j) = make_double2(v[j], v[j + 1]);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i)
      if (mine[i]) dst[e0 + i] = v[i];
  }
}

template <int S, bool FAST, int PAR, int V, bool F>
__device__ __forceinline__ void segment2v(const RcArgs& A, const Rc2Out& O, const SegV<V>& d,
                                          int64_t w0, int lane, bool lane_own, double beta_a,
                                          double beta_b, double inv_l, double thr, Acc2& acc) {
  using G = RcGeomV<S, V>;
  const int64_t n = A.n;
  const int64_t e0 = w0 + V * lane;
  bool mine[V];
  if (FAST) {
#pragma unroll
    for (int i = 0; i < V; ++i) mine[i] = lane_own;
  } else {
    const int64_t own_lo = w0 + G::H3, own_hi = min(own_lo + G::OWN, A.hi);
#pragma unroll
    for (int i = 0; i < V; ++i) mine[i] = e0 + i >= own_lo && e0 + i < own_hi;
  }
  double t[2][V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    t[0][i] = d.xk[i];
    t[1][i] = d.xm[i];
  }
  // (F: the scaled form, A.sigma = sigma * prod cos(theta) -- the tile kernel's
  // operations entry for entry, so the two kernels agree bit for bit)
  wchainv<S, true, FAST, 2, PAR, V, F, F>(t, e0, n, A.right);
  double rk[V], g[1][V], rr = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    rk[i] = mul_sub<F>(d.sg[i], t[0][i], d.bb[i]);
    if (mine[i]) rr = F ? __fma_rn(rk[i], rk[i], rr) : rr + rk[i] * rk[i];
    const double rm = mul_sub<F>(d.sg[i], t[1][i], d.bb[i]);
    g[0][i] = d.sg[i] * mul_sub<F>(1.0 + beta_a, rk[i], beta_a * rm);
  }
  acc.rr0 += rr;
  wchainv<S, false, FAST, 1, PAR, V, F, F>(g, e0, n, A.right);
  double x1[1][V], l1 = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const double y = F ? __fma_rn(beta_a, d.xk[i] - d.xm[i], d.xk[i]) : d.xk[i] + beta_a * (d.xk[i] - d.xm[i]);
    // (the FP64 compares of shrink() here; the tile kernel takes the same values from the
    // bit patterns, soft_threshold_bits -- measured neutral in this kernel: 1996 vs 2002 iter/s)
    double v = shrink(F ? __fma_rn(-inv_l, g[0][i], y) : y - inv_l * g[0][i], thr);
    l1 += mine[i] ? fabs(v) : 0.0;
    acc.nza += (unsigned)(mine[i] & (v != 0.0));
    acc.misa += (unsigned)(mine[i] & (v != y));
    if (!FAST && (e0 + i < 0 || e0 + i >= n)) v = 0.0;
    x1[0][i] = v;
  }
  acc.l1a += l1;
  store_ownv<FAST, V>(O.x1, e0, mine, lane_own, x1[0]);
  peer_store<V>(A, 0, e0, mine, x1[0]);
  double t1[1][V];
#pragma unroll
  for (int i = 0; i < V; ++i) t1[0][i] = x1[0][i];
  wchainv<S, true, FAST, 1, PAR, V, F, F>(t1, e0, n, A.right);
  double rr1 = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const double r1 = mul_sub<F>(d.sg[i], t1[0][i], d.bb[i]);
    if (mine[i]) rr1 = F ? __fma_rn(r1, r1, rr1) : rr1 + r1 * r1;
    g[0][i] = d.sg[i] * mul_sub<F>(1.0 + beta_b, r1, beta_b * rk[i]);
  }
  acc.rr1 += rr1;
  wchainv<S, false, FAST, 1, PAR, V, F, F>(g, e0, n, A.right);
  double x2[V], l1b = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const double y = F ? __fma_rn(beta_b, x1[0][i] - d.xk[i], x1[0][i]) : x1[0][i] + beta_b * (x1[0][i] - d.xk[i]);
    x2[i] = shrink(F ? __fma_rn(-inv_l, g[0][i], y) : y - inv_l * g[0][i], thr);
    l1b += mine[i] ? fabs(x2[i]) : 0.0;
    acc.nzb += (unsigned)(mine[i] & (x2[i] != 0.0));
    acc.misb += (unsigned)(mine[i] & (x2[i] != y));
  }
  acc.l1b += l1b;
  store_ownv<FAST, V>(O.x2, e0, mine, lane_own, x2);
  peer_store<V>(A, 1, e0, mine, x2);
}

template <int S, int MB, int PAR, int V, bool PF, bool F>
__global__ void __launch_bounds__(kRcThreads, MB) fista_rc2v_kernel(RcArgs A, Rc2Out O) {
  using G = RcGeomV<S, V>;
  FistaDev* st = A.b.st;
  if (*(volatile int*)&st->stop) return;
  const double beta_a = st->beta_y;
  double t_next, beta_b;
  fista_momentum(st, &t_next, &beta_b);
  const double inv_l = 1.0 / st->lval;
  const double thr = st->tau * inv_l;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool lane_own = V * lane >= G::H3 && V * lane < G::H3 + G::OWN;
  const int64_t n = A.n, lo = A.lo, hi = A.hi;
  const int64_t lim_lo = max((int64_t)0, lo - G::H3), lim_hi = min(n, hi + G::H3);
  const int64_t nseg = (hi - lo + G::OWN - 1) / G::OWN;
  const int64_t stride = (int64_t)gridDim.x * kRcWarps;
  Acc2 acc;
  auto w0_of = [&](int64_t q) { return lo + q * G::OWN - G::H3; };
  auto full_of = [&](int64_t w0) { return w0 >= lim_lo && w0 + G::W <= lim_hi; };
  const int64_t base = lo - G::H3;
  const int64_t w_min = max((int64_t)2, lim_lo), w_max = min(lim_hi, n - 1) - G::W;
  const int64_t q_lo = w_min <= base ? 0 : (w_min - base + G::OWN - 1) / G::OWN;
  const int64_t q_hi = w_max < base ? 0 : min((w_max - base) / G::OWN + 1, (hi - lo) / G::OWN);
  SegV<V> sa, sb;
  int64_t q = (int64_t)blockIdx.x * kRcWarps + warp;
  if (q < nseg) load_segv<V>(A, w0_of(q) + V * lane, full_of(w0_of(q)), lim_lo, lim_hi, sa);
  for (; q < nseg; q += stride) {
    if (PF && q + stride < nseg) {
      const int64_t w1 = w0_of(q + stride);
      load_segv<V>(A, w1 + V * lane, full_of(w1), lim_lo, lim_hi, sb);
    }
    if (q >= q_lo && q < q_hi)
      segment2v<S, true, PAR, V, F>(A, O, sa, w0_of(q), lane, lane_own, beta_a, beta_b, inv_l, thr, acc);
    else
      segment2v<S, false, PAR, V, F>(A, O, sa, w0_of(q), lane, lane_own, beta_a, beta_b, inv_l, thr, acc);
    if (PF) {
      sa = sb;
    } else if (q + stride < nseg) {
      const int64_t w1 = w0_of(q + stride);
      load_segv<V>(A, w1 + V * lane, full_of(w1), lim_lo, lim_hi, sa);
    }
  }
  if (A.peers.on) __threadfence_system();  // peer stores performed before the kernel ends
  double sums[8] = {acc.rr0, acc.l1a, (double)acc.nza, (double)acc.misa,
                    acc.rr1, acc.l1b, (double)acc.nzb, (double)acc.misb};
  double tot[8];
  if (grid_sum<8>(sums, A.b.partials, &st->ticket[0], tot) && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) st->scal8[k] = tot[k];
    if (st->defer)
      st->pair_pending = 1;  // shards: recorded by the finalize after the all-reduce
    else
      fista_finalize_lagged2(st, A.b.trace);
  }
}

// Small instances (C1: n = 2^12, a few warps of work per iteration): the
// per-kernel cost is launch + grid-reduction latency, not bandwidth.  One
// cooperative launch then runs up to `iters` iterations back to back, with
// two grid barriers per iteration (after the sums; after block 0 recorded the
// iteration), the x buffers rotating as in the one-kernel-per-iteration loop.
// Same segment code => same iterates.
struct RcPArgs {
  RcArgs a;          // a.b.x_* unused: X[] rotate
  double* X[4];      // global-index views of the four x buffers
  uint64_t j0, iters;
};

template <int S, int PAR>
__global__ void __launch_bounds__(kRcThreads, 2) fista_rc_persistent(RcPArgs P) {
  namespace cg = cooperative_groups;
  using G = RcGeom<S>;
  cg::grid_group grid = cg::this_grid();
  RcArgs A = P.a;
  FistaDev* st = A.b.st;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool lane_own = 4 * lane >= G::H3 && 4 * lane < G::H3 + G::OWN;
  const int64_t n = A.n, lo = A.lo, hi = A.hi;
  const int64_t lim_lo = max((int64_t)0, lo - G::H3), lim_hi = min(n, hi + G::H3);
  const int64_t nseg = (hi - lo + G::OWN - 1) / G::OWN;
  const int64_t stride = (int64_t)gridDim.x * kRcWarps;
  const int64_t base = lo - G::H3;
  const int64_t w_min = max((int64_t)2, lim_lo), w_max = min(lim_hi, n - 1) - kWin;
  const int64_t q_lo = w_min <= base ? 0 : (w_min - base + G::OWN - 1) / G::OWN;
  const int64_t q_hi = w_max < base ? 0 : min((w_max - base) / G::OWN + 1, (hi - lo) / G::OWN);
  for (uint64_t it = 0; it < P.iters; ++it) {
    if (*(volatile int*)&st->stop) break;  // uniform: read after the last barrier
    const uint64_t j = P.j0 + it;
    A.b.x_k = P.X[j % 4];
    A.b.x_km1 = P.X[(j + 3) % 4];
    A.b.x_next = P.X[(j + 1) % 4];
    const double beta = __ldcg(&st->beta_y);
    const double inv_l = 1.0 / __ldcg(&st->lval);
    const double thr = __ldcg(&st->tau) * inv_l;
    Acc acc;
    for (int64_t q = (int64_t)blockIdx.x * kRcWarps + warp; q < nseg; q += stride) {
      const int64_t w0 = base + q * G::OWN;
      Seg d;
      load_seg<true>(A, w0 + 4 * lane, w0 >= lim_lo && w0 + kWin <= lim_hi, lim_lo, lim_hi, d);
      if (q >= q_lo && q < q_hi)
        segment<S, true, false, PAR>(A, d, w0, lane, lane_own, beta, inv_l, thr, acc);
      else
        segment<S, false, false, PAR>(A, d, w0, lane, lane_own, beta, inv_l, thr, acc);
    }
    double sums[4] = {acc.l1, (double)acc.nz, (double)acc.mism, acc.rr};
    block_sum<4>(sums);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) A.b.partials[(size_t)blockIdx.x * 4 + k] = sums[k];
    }
    grid.sync();
    if (blockIdx.x == 0) {  // fixed-order fold of the block partials, then the record
      double tot[4] = {0.0, 0.0, 0.0, 0.0};
      for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
        for (int k = 0; k < 4; ++k) tot[k] += __ldcg(&A.b.partials[(size_t)b * 4 + k]);
      }
      block_sum<4>(tot);
      if (threadIdx.x == 0) {
        st->scal[0] = tot[0];
        st->scal[1] = tot[1];
        st->scal[2] = tot[2];
        st->scal[3] = tot[3];
        fista_finalize_lagged(st, A.b.trace, false);
      }
    }
    grid.sync();
  }
}

// co-resident CTAs of a kernel, once per process (the first query also loads
// the kernel's module: fista_rc_prepare calls it before the timed loop)
template <auto K>
int grid_cap_of() {
  static const int cap = [] {
    int per_sm = 0;
    L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K, kRcThreads, 0));
    return std::min(std::max(1, per_sm) * sm_count(), spmv_grid_max());
  }();
  return cap;
}

// Small instances that fit in shared memory (C1: n = 2^12): ONE CTA of 32
// warps runs the chunk with sigma, b and the four x buffers resident in shared
// memory (zero-padded by H3 on both sides) and the FISTA state in a shared
// copy of FistaDev: an iteration costs block barriers and shared-memory
// traffic only.  Same segment code, same bookkeeping => the same iterates.
constexpr int kSmallThreads = 512;

template <int S>
struct SmallGeom {
  static constexpr int P = RcGeom<S>::H3;  // padding on both sides (entries)
};

__host__ __device__ inline uint64_t small_stride(uint64_t n, int pad) {
  return (n + 2 * (uint64_t)pad + 3) / 4 * 4;
}

template <int S, int PAR>
__global__ void __launch_bounds__(kSmallThreads, 1) fista_rc_small(RcPArgs P) {
  using G = RcGeom<S>;
  extern __shared__ __align__(16) double sm[];
  __shared__ FistaDev sst;
  const RcArgs& A0 = P.a;
  const int64_t n = A0.n;
  const int pad = SmallGeom<S>::P;
  const uint64_t N = small_stride((uint64_t)n, pad);
  double* s_sig = sm;
  double* s_b = sm + N;
  double* s_x[4] = {sm + 2 * N, sm + 3 * N, sm + 4 * N, sm + 5 * N};
  const int t = threadIdx.x;
  if (t == 0) sst = *A0.b.st;
  for (uint64_t q = t; q < N; q += blockDim.x) {
    const int64_t g = (int64_t)q - pad;
    const bool in = g >= 0 && g < n;
    s_sig[q] = in ? A0.sigma[g] : 0.0;
    s_b[q] = in ? A0.b.b[g] : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s_x[k][q] = in ? P.X[k][g] : 0.0;
  }
  __syncthreads();
  const int lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
  const bool lane_own = 4 * lane >= G::H3 && 4 * lane < G::H3 + G::OWN;
  const int64_t nseg = (n + G::OWN - 1) / G::OWN;
  RcArgs A = A0;
  A.lo = 0;
  A.hi = n;
  A.sigma = s_sig + pad;  // global-index views of the padded arrays
  A.b.b = s_b + pad;
  for (uint64_t it = 0; it < P.iters; ++it) {
    if (sst.stop) break;  // uniform: read after the last barrier
    const uint64_t j = P.j0 + it;
    A.b.x_k = s_x[j % 4] + pad;
    A.b.x_km1 = s_x[(j + 3) % 4] + pad;
    A.b.x_next = s_x[(j + 1) % 4] + pad;
    const double beta = sst.beta_y;
    const double inv_l = 1.0 / sst.lval;
    const double thr = sst.tau * inv_l;
    Acc acc;
    for (int64_t q = warp; q < nseg; q += nwarps) {
      const int64_t w0 = q * G::OWN - G::H3;
      const int64_t e = w0 + 4 * lane;  // window entries read from the padded arrays
      Seg d;
      const bool inpad = e >= -pad && e + 4 <= n + pad;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t g = e + i;
        const bool ok = inpad || (g >= -pad && g < n + pad);
        d.xk[i] = ok ? A.b.x_k[g] : 0.0;
        d.xm[i] = ok ? A.b.x_km1[g] : 0.0;
        d.sg[i] = ok ? A.sigma[g] : 0.0;
        d.bb[i] = ok ? A.b.b[g] : 0.0;
      }
      const bool fast = w0 >= 2 && w0 + kWin < n && w0 + G::H3 + G::OWN <= n;
      if (fast)
        segment<S, true, false, PAR, true>(A, d, w0, lane, lane_own, beta, inv_l, thr, acc);
      else
        segment<S, false, false, PAR, true>(A, d, w0, lane, lane_own, beta, inv_l, thr, acc);
    }
    double sums[4] = {acc.l1, (double)acc.nz, (double)acc.mism, acc.rr};
    block_sum<4>(sums);  // (ends with a barrier: every x_{k+1} entry is written)
    if (t == 0) {
      sst.scal[0] = sums[0];
      sst.scal[1] = sums[1];
      sst.scal[2] = sums[2];
      sst.scal[3] = sums[3];
      fista_finalize_lagged(&sst, A0.b.trace, false);
    }
    __syncthreads();
  }
  for (uint64_t q = t; q < (uint64_t)n; q += blockDim.x) {
#pragma unroll
    for (int k = 0; k < 4; ++k) P.X[k][q] = s_x[k][q + pad];
  }
  if (t == 0) *A0.b.st = sst;
}

template <int S, int PAR>
bool launch_rc_small(const RcPArgs& p, cudaStream_t st) {
  const size_t bytes = 6 * small_stride(p.a.n, SmallGeom<S>::P) * sizeof(double);
  static int max_dyn = -1;
  if (max_dyn < 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    max_dyn = std::max(0, optin - (int)sizeof(FistaDev) - 1024);
    L1B_CUDA(cudaFuncSetAttribute(fista_rc_small<S, PAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  max_dyn));
  }
  if (bytes > (size_t)max_dyn) return false;
  fista_rc_small<S, PAR><<<1, kSmallThreads, bytes, st>>>(p);
  L1B_LAUNCHED();
  return true;
}

// Small single-stage instances (C1: n = 2^12, one Givens stage): every
// product is pair-local -- A x = Sigma G^T x and G u act on disjoint pairs
// (a, a + 1), a = 2u - offset -- so one CTA runs the chunk with each thread
// owning up to P pairs for the whole chunk: x_k, x_{k-1}, r_k, r_{k-1} in
// registers, sigma and b in thread-private shared memory.  An iteration is the
// segment arithmetic of the window kernels restricted to a pair (same
// operations, same order => the same iterates): g = G (sigma ((1 + beta) r_k
// - beta r_{k-1})), the prox, then r_{k+1} = sigma G^T x_{k+1} - b for the
// next iteration (one rotation each way per pair), and one block reduction
// for the lagged bookkeeping (fista_finalize_lagged, as fista_rc_small).
constexpr int kPairThreads = 512;

__device__ __forceinline__ void pair_residual(double x0, double x1, bool pair, double c, double s,
                                              double s0, double s1, double b0, double b1, double& r0,
                                              double& r1) {
  if (pair) rotate_pair(x0, x1, c, s, true);  // G^T x (linops.cpp:428)
  r0 = s0 * x0 - b0;                          // Sigma (.) - b
  r1 = s1 * x1 - b1;
}

// Single-stage instances, pair-local: with one Givens stage every product acts
// on disjoint pairs, so a thread keeps its pairs' x_k, x_{k-1}, r_k, r_{k-1}
// in registers for a whole chunk of iterations, on a cluster of kClusterCtas
// CTAs (one per SM).  The reduction goes
// through distributed shared memory with ONE cluster barrier per iteration:
// every CTA stores its four block sums into every CTA (double-buffered by
// iteration parity), and after the barrier each CTA folds the eight partials
// in rank order and runs the lagged bookkeeping on its own copy of the FISTA
// state -- identical inputs, identical decisions; only CTA 0 writes the trace
// and the state back.
constexpr int kClusterCtas = 8;

template <int P>
__global__ void __launch_bounds__(kPairThreads, 1) fista_pair_cluster(RcPArgs Pa, int off) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ FistaDev sst;                     // every CTA: its replica of the state
  __shared__ double part[2][kClusterCtas][4];  // block sums of every CTA, by parity
  __shared__ double bc[2];                     // (stop, beta_y) of the replica
  extern __shared__ double cs[];
  const RcArgs& A = Pa.a;
  const int64_t n = A.n;
  const int t = threadIdx.x, T = blockDim.x;
  const int rank = (int)cluster.block_rank();
  const double c = A.right.c[0], s = A.right.s[0];
  double* c_sig = cs;
  double* c_b = cs + 2 * P * T;
  auto slot = [&](int k, int e) { return (2 * k + e) * T + t; };
  if (t == 0) {
    sst = *A.b.st;
    bc[0] = sst.stop ? 1.0 : 0.0;
    bc[1] = sst.beta_y;
  }
  const double inv_l = 1.0 / A.b.st->lval;
  const double thr = A.b.st->tau * inv_l;
  int64_t a[P];
  bool va[P], vb[P];
  double xk[P][2], xm[P][2], rk[P][2], rm[P][2];
  const uint64_t j0 = Pa.j0;
  const double* X0 = Pa.X[j0 % 4];
  const double* X1 = Pa.X[(j0 + 3) % 4];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    a[k] = 2 * (int64_t)(rank * T + t + k * kClusterCtas * T) - off;
    va[k] = a[k] >= 0 && a[k] < n;
    vb[k] = a[k] + 1 >= 0 && a[k] + 1 < n;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool v = e == 0 ? va[k] : vb[k];
      const int64_t i = a[k] + e;
      c_sig[slot(k, e)] = v ? A.sigma[i] : 0.0;
      c_b[slot(k, e)] = v ? A.b.b[i] : 0.0;
      xk[k][e] = v ? X0[i] : 0.0;
      xm[k][e] = v ? X1[i] : 0.0;
    }
    const bool pair = va[k] && vb[k];
    const double s0 = c_sig[slot(k, 0)], s1 = c_sig[slot(k, 1)];
    const double b0 = c_b[slot(k, 0)], b1 = c_b[slot(k, 1)];
    pair_residual(xk[k][0], xk[k][1], pair, c, s, s0, s1, b0, b1, rk[k][0], rk[k][1]);
    pair_residual(xm[k][0], xm[k][1], pair, c, s, s0, s1, b0, b1, rm[k][0], rm[k][1]);
  }
  __syncthreads();
  uint64_t done = 0;
  for (; done < Pa.iters; ++done) {
    if (bc[0] != 0.0) break;  // every replica took the same decision
    const double beta = bc[1];
    double l1 = 0.0, rr = 0.0;
    unsigned nz = 0, mism = 0;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const bool pair = va[k] && vb[k];
      const double s0 = c_sig[slot(k, 0)], s1 = c_sig[slot(k, 1)];
      if (va[k]) rr += rk[k][0] * rk[k][0];
      if (vb[k]) rr += rk[k][1] * rk[k][1];
      double g0 = s0 * ((1.0 + beta) * rk[k][0] - beta * rm[k][0]);
      double g1 = s1 * ((1.0 + beta) * rk[k][1] - beta * rm[k][1]);
      if (pair) rotate_pair(g0, g1, c, s, false);
      double tr[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool v = e == 0 ? va[k] : vb[k];
        const double y = xk[k][e] + beta * (xk[k][e] - xm[k][e]);
        const double v_ = shrink(y - inv_l * (e == 0 ? g0 : g1), thr);
        tr[e] = v ? v_ : 0.0;
        if (v) {
          l1 += fabs(v_);
          nz += v_ != 0.0;
          mism += v_ != y;
        }
      }
      double n0, n1;
      pair_residual(tr[0], tr[1], pair, c, s, s0, s1, c_b[slot(k, 0)], c_b[slot(k, 1)], n0, n1);
      xm[k][0] = xk[k][0];
      xm[k][1] = xk[k][1];
      xk[k][0] = tr[0];
      xk[k][1] = tr[1];
      rm[k][0] = rk[k][0];
      rm[k][1] = rk[k][1];
      rk[k][0] = n0;
      rk[k][1] = n1;
    }
    double sums[4] = {l1, (double)nz, (double)mism, rr};
    block_sum<4>(sums);
    const int par = (int)(done & 1);
    if (t < kClusterCtas) {  // thread r stores this CTA's sums into CTA r
      double* dst = cluster.map_shared_rank(&part[par][rank][0], t);
      // thread 0 holds the block sums; the others read them from shared memory
      dst[0] = __shfl_sync(0xffu, sums[0], 0);
      dst[1] = __shfl_sync(0xffu, sums[1], 0);
      dst[2] = __shfl_sync(0xffu, sums[2], 0);
      dst[3] = __shfl_sync(0xffu, sums[3], 0);
    }
    cluster.sync();
    if (t == 0) {
      double tot[4] = {0.0, 0.0, 0.0, 0.0};
      for (int r = 0; r < kClusterCtas; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) tot[q] += part[par][r][q];
#pragma unroll
      for (int q = 0; q < 4; ++q) sst.scal[q] = tot[q];
      fista_finalize_lagged(&sst, rank == 0 ? A.b.trace : nullptr, false);
      bc[0] = sst.stop ? 1.0 : 0.0;
      bc[1] = sst.beta_y;
    }
    __syncthreads();
  }
  double* Xk = Pa.X[(j0 + done) % 4];
  double* Xm = Pa.X[(j0 + done + 3) % 4];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    if (va[k]) {
      Xk[a[k]] = xk[k][0];
      Xm[a[k]] = xm[k][0];
    }
    if (vb[k]) {
      Xk[a[k] + 1] = xk[k][1];
      Xm[a[k] + 1] = xm[k][1];
    }
  }
  // no CTA may exit while others could still store into its shared memory
  cluster.sync();
  if (rank == 0 && t == 0) *A.b.st = sst;
}

template <int P>
void launch_pair_cluster_p(const RcPArgs& p, int threads, int off, cudaStream_t st) {
  const int bytes = 4 * P * threads * (int)sizeof(double);
  L1B_CUDA(cudaFuncSetAttribute(fista_pair_cluster<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterCtas);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClusterCtas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  L1B_CUDA(cudaLaunchKernelEx(&cfg, fista_pair_cluster<P>, p, off));
  L1B_LAUNCHED();
}

// single-stage instances: a cluster of 8 CTAs for at most 2 x 8 x 512 pairs
// (n <= 16384); offset 1 needs n / 2 + 1 pairs.  L1B_PAIR_SMALL=0 keeps the
// window kernel (the cross-check).
bool launch_pair_small(const RcPArgs& p, const StageTab& right, cudaStream_t st) {
  const char* e = getenv("L1B_PAIR_SMALL");
  if (e && e[0] == '0') return false;
  if (right.count != 1) return false;
  const int off = right.offset[0];
  const uint64_t n = (uint64_t)p.a.n;
  const uint64_t units = off ? n / 2 + 1 : (n + 1) / 2;
  for (int P : {1, 2}) {
    const uint64_t thr = (units + (uint64_t)P * kClusterCtas - 1) / ((uint64_t)P * kClusterCtas);
    if (thr > (uint64_t)kPairThreads) continue;
    const int threads = (int)std::max<uint64_t>(32, (thr + 31) / 32 * 32);
    if (P == 1) launch_pair_cluster_p<1>(p, threads, off, st);
    if (P == 2) launch_pair_cluster_p<2>(p, threads, off, st);
    return true;
  }
  return false;
}

template <int S, int PAR>
void launch_rc_persistent(const RcPArgs& p, cudaStream_t st) {
  const int grid_cap = grid_cap_of<fista_rc_persistent<S, PAR>>();
  using G = RcGeom<S>;
  const int64_t nseg = (p.a.hi - p.a.lo + G::OWN - 1) / G::OWN;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nseg + kRcWarps - 1) / kRcWarps, grid_cap));
  RcPArgs a = p;
  void* args[] = {&a};
  L1B_CUDA(cudaLaunchCooperativeKernel((const void*)fista_rc_persistent<S, PAR>, dim3(grid),
                                       dim3(kRcThreads), args, 0, st));
  L1B_LAUNCHED();
}

template <int S, int MB, bool FLUSH, int PAR, bool F>
void launch_rc_v(const RcArgs& a, cudaStream_t st) {
  using G = RcGeom<S>;
  const int grid_cap = grid_cap_of<fista_rc_kernel<S, MB, FLUSH, PAR, F>>();
  const int64_t nseg = (a.hi - a.lo + G::OWN - 1) / G::OWN;
  const int64_t blocks = (nseg + kRcWarps - 1) / kRcWarps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, grid_cap));
  fista_rc_kernel<S, MB, FLUSH, PAR, F><<<grid, kRcThreads, 0, st>>>(a);
  L1B_LAUNCHED();
}

// The two-iteration kernel: 8 entries per lane with the next segment's loads
// in flight, 1 CTA of 8 warps per SM (255 registers in the exact build).
// Measured at C4 (iter/s, exact arithmetic): this shape 1843; 6 per lane 1682;
// 8 per lane without prefetch 1466; 4 per lane, 2 CTAs/SM 1468 (those shapes
// were dropped in round 2).
constexpr int kRc2V = 8;
template <int S, int PAR, bool F>
void launch_rc2(const RcArgs& a, const Rc2Out& o, cudaStream_t st) {
  using G = RcGeomV<S, kRc2V>;
  const int grid_cap = grid_cap_of<fista_rc2v_kernel<S, 1, PAR, kRc2V, true, F>>();
  const int64_t nseg = (a.hi - a.lo + G::OWN - 1) / G::OWN;
  const int64_t blocks = (nseg + kRcWarps - 1) / kRcWarps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, grid_cap));
  fista_rc2v_kernel<S, 1, PAR, kRc2V, true, F><<<grid, kRcThreads, 0, st>>>(a, o);
  L1B_LAUNCHED();
}

// offsets (S-1-s) % 2, the generator's alternating stages (bench.cpp:270)
template <int S>
constexpr int canon_par() {
  int m = 0;
  for (int s = 0; s < S; ++s) m |= ((S - 1 - s) & 1) << s;
  return m;
}
template <int S>
bool is_canon(const StageTab& t) {
  for (int s = 0; s < S; ++s)
    if ((t.offset[s] & 1) != ((S - 1 - s) & 1)) return false;
  return true;
}

// one iteration per launch, 2 CTAs/SM (measured: 1 CTA/SM slower)
template <int S, bool F>
void launch_rc(const RcArgs& a, cudaStream_t st) {
  if (is_canon<S>(a.right)) return launch_rc_v<S, 2, false, canon_par<S>(), F>(a, st);
  launch_rc_v<S, 2, false, -1, F>(a, st);
}

template <int S, bool F>
void launch_rc_flush(const RcArgs& a, cudaStream_t st) {
  launch_rc_v<S, 2, true, -1, F>(a, st);  // once per solve: the generic stage table
}

// ---------------------------------------------------------------------------
// K iterations per launch: tiles of the line advanced K iterations on chip.
//
// A CTA of kTbWarps warps takes a tile of SPAN = kTbWarps * OWN consecutive
// entries; warp w holds the window [s0 + w OWN - H, s0 + (w+1) OWN + H) in
// registers (8 entries per lane: lane 0 / 31 are the halos, lanes 1..30 own),
// sigma and b of the window in shared memory.  One iteration:
//   r_k = sigma .* (G^T x_k) - b on the window (r_{k-1} is the previous
//   iteration's r_k, kept in registers: two chain runs per iteration, against
//   the two-iteration kernel's 2.5), u = sigma .* ((1+beta) r_k - beta r_{k-1}),
//   g = G u, x_{k+1} on the own lanes; then every warp hands its first / last
//   8 own entries to its neighbours through shared memory (one block barrier).
// The tile's two outermost halos are never refreshed: their wrong values creep
// inwards by 2S entries per iteration, so only the middle VALID = SPAN - 2E
// entries (E >= 2S (K-1)) of a tile are kept; consecutive tiles overlap by 2E.
// HBM: x_k, x_{k-1}, sigma, b read once and two x written per K iterations,
// 48n (1 + 2E / VALID) bytes per launch -- the FP64 pipe bounds the kernel.
// Per entry the operations are segment2v's: identical iterates.  CTAs are
// persistent (one per SM), tiles strided by the grid; the per-iteration sums
// are accumulated per warp in shared memory and folded in a fixed order.
#ifndef TB_V
#define TB_V 8  // entries per lane
#endif
constexpr int kTbWarps = TB_WARPS, kTbThreads = 32 * kTbWarps, kTbV = TB_V;
// contracted arithmetic: rotations in the scaled form, as in the other two
// kernels.  Exact arithmetic: each lane forms its own output of a straddling
// pair (one shuffle deep, +0.5 %; the scaled form measured 1 % slower that way
// and shuffles the rotated value back instead).
constexpr bool kTbScaled = true, kTbSym = true, kTbSymF = false;
constexpr int kTbCtas = (kTbV <= 8 ? 512 : 256) / kTbThreads;  // resident CTAs per SM (128 registers per thread at 8 entries per lane)
template <int S>
struct TbGeom {
  static constexpr int W = 32 * kTbV;
  static constexpr int H = kTbV;  // one lane per side; >= 2S for S <= 4
  static constexpr int OWN = W - 2 * H;
  static constexpr int SPAN = kTbWarps * OWN;
  static_assert(2 * S <= H, "halo narrower than two chain runs");
};
constexpr int tb_erosion(int S, int K) { return (2 * S * (K - 1) + kTbV - 1) / kTbV * kTbV; }

struct TbArgs {
  int64_t n;
  StageTab right;
  const double* sigma;
  const double* b;
  const double* x_k;
  const double* x_km1;
  double* out1;  // x_{k+K-1}
  double* out2;  // x_{k+K}
  FistaDev* st;
  FistaSample* trace;
  double* partials;  // gridDim.x * 4K per-CTA sums, then the 4K totals
  int64_t valid, ntiles;
  int K, E, replay;
};

struct TbSmem {
  double2 sb[kTbWarps][kTbV][32];  // (sigma, b) by [warp][entry][lane]: one 128-bit load, conflict-free
  double xch[2][2][kTbWarps][kTbV];  // [iteration parity][first / last own lane][warp][entry]
  double2 lane_acc[kTbKMax][kTbWarps][32];  // per lane and iteration: (||x_{k+1}||_1, ||r_k||^2), one 128-bit access
  double cnt[kTbWarps][kTbKMax][2];           // per warp and iteration: nnz, mismatches
  double beta[kTbKMax];
  double inv_l, thr;
  int last;
};

// One iteration on the warp's window.  xc = x_k (window, halos current);
// xo = x_{k-1} on entry (own lanes), x_{k+1} on exit; rp = r_{k-1} on entry,
// r_k on exit (both valid on the own entries +- S).
// STORE: 0 = an iteration that stores no iterate (it < K - 2), -1 = decided
// from it (the first and the last iterations of a tile).
template <int S, int PAR, bool F, bool INTERIOR, bool FIRST, int STORE = -1>
__device__ __forceinline__ void tb_step(const TbArgs& A, TbSmem& sm, int it, int64_t e0, int lane,
                                        int warp, bool lane_valid, const double (&xc)[kTbV],
                                        double (&xo)[kTbV], double (&rp)[kTbV], unsigned& nx) {
  constexpr int V = kTbV;
  constexpr int KC = FIRST ? 2 : 1;
  const int64_t n = A.n;
  const double bt = sm.beta[it], bt1 = 1.0 + bt;
  double t[KC][V];
#pragma unroll
  for (int i = 0; i < V; ++i) {
    t[0][i] = xc[i];
    if (FIRST) t[KC - 1][i] = xo[i];
  }
  wchainv<S, true, INTERIOR, KC, PAR, V, F, F && kTbScaled, F ? kTbSymF : kTbSym>(t, e0, n, A.right);
  double g[1][V], rr = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const double2 q = sm.sb[warp][i][lane];
    const double sg = q.x, bb = q.y;
    const double rk = mul_sub<F>(sg, t[0][i], bb);
    rr = F ? __fma_rn(rk, rk, rr) : rr + rk * rk;
    const double rm = FIRST ? mul_sub<F>(sg, t[KC - 1][i], bb) : rp[i];
    g[0][i] = sg * mul_sub<F>(bt1, rk, bt * rm);
    rp[i] = rk;
  }
  wchainv<S, false, INTERIOR, 1, PAR, V, F, F && kTbScaled, F ? kTbSymF : kTbSym>(g, e0, n, A.right);
  const double inv_l = sm.inv_l, thr = sm.thr;
  double l1 = 0.0;
  unsigned nz = 0, mis = 0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const double y = F ? __fma_rn(bt, xc[i] - xo[i], xc[i]) : xc[i] + bt * (xc[i] - xo[i]);
    const double z = F ? __fma_rn(-inv_l, g[0][i], y) : y - inv_l * g[0][i];
    // soft_threshold and (trial != y) on the bit patterns (neither x nor y is
    // ever -0: a difference of equal doubles is +0, and so is +0 + -0): five
    // FP64 instructions of the shrink and its counters become integer ones
    bool nzp;
    double v = soft_threshold_bits(z, thr, nzp);
    l1 += fabs(v);
    nz += nzp ? 1u : 0u;
    mis = differing_bits(mis, v, y);  // (only mis != 0 matters: the fixed-point check)
    if (!INTERIOR && (e0 + i < 0 || e0 + i >= n)) v = 0.0;
    xo[i] = v;
  }
  const int K = A.K;
  double* dst = STORE == 0 ? nullptr : it == K - 1 ? A.out2 : (it == K - 2 && !A.replay) ? A.out1 : nullptr;
  if (STORE != 0 && dst && lane_valid) {
    if (INTERIOR || e0 + V <= n) {
#pragma unroll
      for (int j = 0; j < V; j += 4) {
        const double a[4] = {xo[j], xo[j + 1], xo[j + 2], xo[j + 3]};
        st4(dst + e0 + j, a);
      }
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i)
        if (e0 + i < n) dst[e0 + i] = xo[i];
    }
  }
  if (lane_valid) {
    double2 acc = sm.lane_acc[it][warp][lane];
    acc.x += l1;
    acc.y += rr;
    sm.lane_acc[it][warp][lane] = acc;
  }
  nz = __reduce_add_sync(kFull, lane_valid ? nz : 0u);
  mis = __any_sync(kFull, lane_valid && mis != 0u) ? 1u : 0u;
  if (lane == 0) {
    sm.cnt[warp][it][0] += (double)nz;
    sm.cnt[warp][it][1] += (double)mis;
  }
  if (it + 1 < K) {
    // halo exchange for the next iteration (slot parity alternates: one
    // block barrier per exchange)
    const int p = nx & 1;
    ++nx;
    // (one store / load sequence for both sides: the side picks the address)
    if (lane == 1 || lane == 30) {
      double* d = &sm.xch[p][lane == 30 ? 1 : 0][warp][0];
#pragma unroll
      for (int i = 0; i < V; i += 2) *reinterpret_cast<double2*>(d + i) = make_double2(xo[i], xo[i + 1]);
    }
    __syncthreads();
    if ((lane == 0 && warp > 0) || (lane == 31 && warp + 1 < kTbWarps)) {
      const double* q = lane == 0 ? &sm.xch[p][1][warp - 1][0] : &sm.xch[p][0][warp + 1][0];
#pragma unroll
      for (int i = 0; i < V; i += 2) {
        const double2 w = *reinterpret_cast<const double2*>(q + i);
        xo[i] = w.x, xo[i + 1] = w.y;
      }
    }
  }
}

template <int S, int PAR, bool F, bool INTERIOR>
__device__ __forceinline__ void tb_tile(const TbArgs& A, TbSmem& sm, int64_t t0, int lane, int warp,
                                        unsigned& nx) {
  using G = TbGeom<S>;
  constexpr int V = kTbV;
  const int64_t n = A.n;
  const int64_t w0 = t0 - A.E + (int64_t)warp * G::OWN - G::H;
  const int64_t e0 = w0 + V * lane;
  // validity is per lane: t0, VALID, E, OWN and H are multiples of V, so a
  // tile's kept range starts and ends on lane boundaries; entries past n are
  // zero in every array and contribute nothing to the sums
  const bool lane_valid = lane >= 1 && lane <= 30 && e0 >= t0 && e0 + V <= t0 + A.valid && e0 < n;
  double xa[V], xb[V], rp[V];  // x_k / x_{k-1} ping-pong: no register copies between iterations
  {
    double sg[V], bb[V];
    if (w0 >= 0 && w0 + G::W <= n) {
      ldv<V>(A.x_k + e0, xa);
      ldv<V>(A.x_km1 + e0, xb);
      ldv<V>(A.sigma + e0, sg);
      ldv<V>(A.b + e0, bb);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const bool in = e0 + i >= 0 && e0 + i < n;
        xa[i] = in ? A.x_k[e0 + i] : 0.0;
        xb[i] = in ? A.x_km1[e0 + i] : 0.0;
        sg[i] = in ? A.sigma[e0 + i] : 0.0;
        bb[i] = in ? A.b[e0 + i] : 0.0;
      }
    }
    // (contracted arithmetic: A.sigma is sigma * prod cos(theta), the factor
    // the scaled rotations leave out -- r = (sigma C) (M^T x) - b and
    // u = (sigma C) w, so G u = M (sigma C w); problem_sigma_scaled)
#pragma unroll
    for (int i = 0; i < V; ++i) sm.sb[warp][i][lane] = make_double2(sg[i], bb[i]);
  }
  {
    // this CTA's next tile: its four input lines pulled into L2 now, K
    // iterations before they are loaded (64 B per lane and array)
    const int64_t en = e0 + (int64_t)gridDim.x * A.valid;
    if (en >= 0 && en + V <= n) {
#pragma unroll
      for (int j = 0; j < V; j += 8) {
        prefetch_l2(A.x_k + en + j);
        prefetch_l2(A.x_km1 + en + j);
        prefetch_l2(A.sigma + en + j);
        prefetch_l2(A.b + en + j);
      }
    }
  }
  __syncwarp();
  const int K = A.K;
  tb_step<S, PAR, F, INTERIOR, true>(A, sm, 0, e0, lane, warp, lane_valid, xa, xb, rp, nx);  // x_{k+1} in xb
  // iterations 1 .. K-3 store nothing (their instantiation carries no store
  // logic); the last two (and whatever a replay's K leaves) decide from `it`
  int it = 1;
  for (; it + 3 < K; it += 2) {
    tb_step<S, PAR, F, INTERIOR, false, 0>(A, sm, it, e0, lane, warp, lane_valid, xb, xa, rp, nx);
    tb_step<S, PAR, F, INTERIOR, false, 0>(A, sm, it + 1, e0, lane, warp, lane_valid, xa, xb, rp, nx);
  }
  for (; it < K; ++it) {
    if (it & 1)
      tb_step<S, PAR, F, INTERIOR, false>(A, sm, it, e0, lane, warp, lane_valid, xb, xa, rp, nx);
    else
      tb_step<S, PAR, F, INTERIOR, false>(A, sm, it, e0, lane, warp, lane_valid, xa, xb, rp, nx);
  }
}

template <int S, int PAR, bool F>
__global__ void __launch_bounds__(kTbThreads, kTbCtas) fista_tb_kernel(TbArgs A) {
  using G = TbGeom<S>;
  extern __shared__ __align__(16) unsigned char tb_raw[];
  TbSmem& sm = *reinterpret_cast<TbSmem*>(tb_raw);
  FistaDev* st = A.st;
  if (!A.replay && *(volatile int*)&st->stop) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = A.K;
  if (threadIdx.x == 0) {
    // beta of each iteration: beta_y, then the t-sequence (fista_momentum)
    double t = A.replay ? st->snap_t : st->t;
    sm.beta[0] = A.replay ? st->snap_beta : st->beta_y;
    if (!A.replay && blockIdx.x == 0) {
      st->snap_t = st->t;
      st->snap_beta = st->beta_y;
    }
    for (int i = 1; i < K; ++i) {
      const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
      sm.beta[i] = st->accel ? (t - 1.0) / tn : 0.0;
      t = tn;
    }
    sm.inv_l = 1.0 / st->lval;
    sm.thr = st->tau * sm.inv_l;
  }
  for (int q = threadIdx.x; q < kTbKMax * 2 * kTbWarps * 32; q += kTbThreads) (&sm.lane_acc[0][0][0].x)[q] = 0.0;
  for (int q = threadIdx.x; q < kTbWarps * kTbKMax * 2; q += kTbThreads) (&sm.cnt[0][0][0])[q] = 0.0;
  __syncthreads();
  unsigned nx = 0;  // exchanges so far (the same count in every warp)
  for (int64_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const int64_t t0 = tile * A.valid;
    const int64_t s_lo = t0 - A.E - G::H, s_hi = t0 - A.E + G::SPAN + G::H;
    if (s_lo >= 2 && s_hi <= A.n - 1)
      tb_tile<S, PAR, F, true>(A, sm, t0, lane, warp, nx);
    else
      tb_tile<S, PAR, F, false>(A, sm, t0, lane, warp, nx);
  }
  __syncthreads();
  double* part = A.partials;
  for (int q = threadIdx.x; q < 4 * K; q += kTbThreads) {  // fixed order: warps, then lanes
    const int i = q >> 2, c = q & 3;
    double s = 0.0;
    if (c == 1 || c == 2) {
      for (int w = 0; w < kTbWarps; ++w) s += sm.cnt[w][i][c - 1];
    } else {
      for (int w = 0; w < kTbWarps; ++w)
        for (int l = 0; l < 32; ++l) {
          const double2 a = sm.lane_acc[i][w][l];
          s += c == 0 ? a.x : a.y;
        }
    }
    part[(size_t)blockIdx.x * 4 * K + q] = s;
  }
  if (A.replay) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sm.last = atomicAdd(&st->ticket[0], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  double* tot = part + (size_t)gridDim.x * 4 * K;
  for (int q = threadIdx.x; q < 4 * K; q += kTbThreads) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(&part[(size_t)b * 4 * K + q]);
    tot[q] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->ticket[0] = 0u;
    fista_finalize_laggedk(st, A.trace, tot, K);
  }
}

template <int S, int PAR, bool F>
int tb_grid_cap() {
  static const int cap = [] {
    L1B_CUDA(cudaFuncSetAttribute(fista_tb_kernel<S, PAR, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(TbSmem)));
    int per_sm = 0;
    L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fista_tb_kernel<S, PAR, F>, kTbThreads,
                                                           sizeof(TbSmem)));
    return std::max(1, per_sm) * sm_count();
  }();
  return cap;
}

template <int S, int PAR, bool F>
void launch_tb(TbArgs a, cudaStream_t st) {
  using G = TbGeom<S>;
  a.E = tb_erosion(S, a.K);
  a.valid = G::SPAN - 2 * a.E;
  a.ntiles = (a.n + a.valid - 1) / a.valid;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, tb_grid_cap<S, PAR, F>()));
  fista_tb_kernel<S, PAR, F><<<grid, kTbThreads, sizeof(TbSmem), st>>>(a);
  L1B_LAUNCHED();
}

template <int S, bool F>
void launch_rc2_s(const RcArgs& a, const Rc2Out& o, cudaStream_t st) {
  if (is_canon<S>(a.right)) return launch_rc2<S, canon_par<S>(), F>(a, o, st);
  launch_rc2<S, -1, F>(a, o, st);
}

template <int S, bool F>
void launch_tb_s(const TbArgs& a, cudaStream_t st) {
  if (is_canon<S>(a.right)) return launch_tb<S, canon_par<S>(), F>(a, st);
  launch_tb<S, -1, F>(a, st);
}

}  // namespace

template <int S, bool F>
void prepare_s(const StageTab& t) {
  if (is_canon<S>(t)) {
    grid_cap_of<fista_rc_kernel<S, 2, false, canon_par<S>(), F>>();
    grid_cap_of<fista_rc2v_kernel<S, 1, canon_par<S>(), kRc2V, true, F>>();
    if (!F) grid_cap_of<fista_rc_persistent<S, canon_par<S>()>>();
  } else {
    grid_cap_of<fista_rc_kernel<S, 2, false, -1, F>>();
    grid_cap_of<fista_rc2v_kernel<S, 1, -1, kRc2V, true, F>>();
    if (!F) grid_cap_of<fista_rc_persistent<S, -1>>();
  }
  grid_cap_of<fista_rc_kernel<S, 2, true, -1, F>>();
  if (is_canon<S>(t))
    tb_grid_cap<S, canon_par<S>(), F>();
  else
    tb_grid_cap<S, -1, F>();
}

void fista_rc_prepare(const OpView& op, bool fma) {
  switch (op.right.count * 2 + (fma ? 1 : 0)) {
    case 2: return prepare_s<1, false>(op.right);
    case 3: return prepare_s<1, true>(op.right);
    case 4: return prepare_s<2, false>(op.right);
    case 5: return prepare_s<2, true>(op.right);
    case 6: return prepare_s<3, false>(op.right);
    case 7: return prepare_s<3, true>(op.right);
    case 8: return prepare_s<4, false>(op.right);
    case 9: return prepare_s<4, true>(op.right);
    default: return;
  }
}

bool small_enabled() {  // L1B_SMALL=0: the cooperative multi-CTA loop for every size
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("L1B_SMALL");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

void fista_rc_loop(const OpView& op, const IterBufs& ib, double* const X[4], uint64_t j0,
                   uint64_t iters, uint64_t lo, uint64_t hi, cudaStream_t st) {
  if (lo % 4 != 0) throw std::invalid_argument("fista_rc_loop: block start must be a multiple of 4");
  RcPArgs p;
  p.a.n = (int64_t)op.n;
  p.a.lo = (int64_t)lo;
  p.a.hi = (int64_t)hi;
  p.a.right = op.right;
  p.a.sigma = op.sigma;
  p.a.b = ib;
  for (int q = 0; q < 4; ++q) p.X[q] = X[q];
  p.j0 = j0;
  p.iters = iters;
  if (lo == 0 && hi == op.n && small_enabled()) {  // one CTA, everything in shared memory
    if (launch_pair_small(p, op.right, st)) return;
    bool done = false;
    switch (op.right.count) {
      case 1: done = is_canon<1>(op.right) ? launch_rc_small<1, canon_par<1>()>(p, st) : launch_rc_small<1, -1>(p, st); break;
      case 2: done = is_canon<2>(op.right) ? launch_rc_small<2, canon_par<2>()>(p, st) : launch_rc_small<2, -1>(p, st); break;
      case 3: done = is_canon<3>(op.right) ? launch_rc_small<3, canon_par<3>()>(p, st) : launch_rc_small<3, -1>(p, st); break;
      case 4: done = is_canon<4>(op.right) ? launch_rc_small<4, canon_par<4>()>(p, st) : launch_rc_small<4, -1>(p, st); break;
      default: break;
    }
    if (done) return;
  }
  switch (op.right.count) {
    case 1: return is_canon<1>(op.right) ? launch_rc_persistent<1, canon_par<1>()>(p, st) : launch_rc_persistent<1, -1>(p, st);
    case 2: return is_canon<2>(op.right) ? launch_rc_persistent<2, canon_par<2>()>(p, st) : launch_rc_persistent<2, -1>(p, st);
    case 3: return is_canon<3>(op.right) ? launch_rc_persistent<3, canon_par<3>()>(p, st) : launch_rc_persistent<3, -1>(p, st);
    case 4: return is_canon<4>(op.right) ? launch_rc_persistent<4, canon_par<4>()>(p, st) : launch_rc_persistent<4, -1>(p, st);
    default: throw Unsupported("recomputing FISTA kernel: 1..4 stages");
  }
}

void fista_rc_iter2(const OpView& op, const IterBufs& ib, double* x_next2, uint64_t lo, uint64_t hi,
                    cudaStream_t st, const PeerViews& peers, bool fma) {
  if (lo % 4 != 0) throw std::invalid_argument("fista_rc_iter2: block start must be a multiple of 4");
  RcArgs a;
  a.n = (int64_t)op.n;
  a.lo = (int64_t)lo;
  a.hi = (int64_t)hi;
  a.right = op.right;
  a.sigma = op.sigma;
  a.b = ib;
  a.peers = peers;
  const Rc2Out o{ib.x_next, x_next2};
  switch (op.right.count * 2 + (fma ? 1 : 0)) {
    case 2: return launch_rc2_s<1, false>(a, o, st);
    case 3: return launch_rc2_s<1, true>(a, o, st);
    case 4: return launch_rc2_s<2, false>(a, o, st);
    case 5: return launch_rc2_s<2, true>(a, o, st);
    case 6: return launch_rc2_s<3, false>(a, o, st);
    case 7: return launch_rc2_s<3, true>(a, o, st);
    case 8: return launch_rc2_s<4, false>(a, o, st);
    case 9: return launch_rc2_s<4, true>(a, o, st);
    default: throw Unsupported("recomputing FISTA kernel: 1..4 stages");
  }
}

void fista_rc_iterk(const OpView& op, const IterBufs& ib, double* out1, double* out2, int K, bool replay,
                    double* tb, cudaStream_t st, bool fma) {
  if (K < 1 || K > kTbKMax) throw std::invalid_argument("fista_rc_iterk: K out of range");
  TbArgs a;
  a.n = (int64_t)op.n;
  a.right = op.right;
  a.sigma = op.sigma;
  a.b = ib.b;
  a.x_k = ib.x_k;
  a.x_km1 = ib.x_km1;
  a.out1 = out1;
  a.out2 = out2;
  a.st = ib.st;
  a.trace = ib.trace;
  a.partials = tb;
  a.K = K;
  a.replay = replay ? 1 : 0;
  switch (op.right.count * 2 + (fma ? 1 : 0)) {
    case 2: return launch_tb_s<1, false>(a, st);
    case 3: return launch_tb_s<1, true>(a, st);
    case 4: return launch_tb_s<2, false>(a, st);
    case 5: return launch_tb_s<2, true>(a, st);
    case 6: return launch_tb_s<3, false>(a, st);
    case 7: return launch_tb_s<3, true>(a, st);
    case 8: return launch_tb_s<4, false>(a, st);
    case 9: return launch_tb_s<4, true>(a, st);
    default: throw Unsupported("recomputing FISTA kernel: 1..4 stages");
  }
}

void fista_tb_geometry(int stages, int K, int64_t* span, int64_t* valid) {
  *span = TbGeom<4>::SPAN;  // (the tile shape does not depend on S)
  *valid = *span - 2 * tb_erosion(stages, K);
}

uint64_t fista_tb_scratch() { return (uint64_t)(4 * sm_count() + 1) * 4 * kTbKMax; }

// the tile kernel above 2^20 entries (smaller instances run whole chunks of
// iterations in one cooperative launch); L1B_TB=0 switches it off
// (read per session: tests switch it; L1B_TB=2 takes the tile kernel at any n)
bool tb_enabled(uint64_t n, int stages) {
  const char* e = getenv("L1B_TB");
  if (stages < 1 || stages > 4 || (e && e[0] == '0')) return false;
  return (e && e[0] == '2') || n > (1ull << 20);  // (<= 2^20: fista_rc_loop)
}

// iterations per tile launch (L1B_TB_K, read per session): K = 2 (mod 4)
// keeps the x rotation of the two-iteration kernel (a launch from x_j writes
// X[(j+K-1) % 4], X[(j+K) % 4], never its inputs X[j % 4], X[(j-1) % 4])
int tb_iters() {
  const char* e = getenv("L1B_TB_K");
  const int k = e ? atoi(e) : 14;  // (C4: 14 -> 2119 iter/s, 10 -> 2112, 6 -> less)
  return (k < 2 || k > kTbKMax || k % 4 != 2) ? 14 : k;
}

int fista_rc2_halo(int stages) {
  switch (stages) {
    case 1: return RcGeomV<1, kRc2V>::H3;
    case 2: return RcGeomV<2, kRc2V>::H3;
    case 3: return RcGeomV<3, kRc2V>::H3;
    case 4: return RcGeomV<4, kRc2V>::H3;
    default: throw Unsupported("recomputing FISTA kernel: 1..4 stages");
  }
}

int fista_rc_halo(int stages) {
  switch (stages) {
    case 1: return RcGeom<1>::H3;
    case 2: return RcGeom<2>::H3;
    case 3: return RcGeom<3>::H3;
    case 4: return RcGeom<4>::H3;
    default: throw Unsupported("recomputing FISTA kernel: 1..4 stages");
  }
}

void fista_rc_iter(const OpView& op, const IterBufs& ib, uint64_t lo, uint64_t hi,
                   cudaStream_t st, bool flush, const PeerViews& peers, bool fma) {
  if (lo % 4 != 0) throw std::invalid_argument("fista_rc_iter: block start must be a multiple of 4");
  RcArgs a;
  a.n = (int64_t)op.n;
  a.lo = (int64_t)lo;
  a.hi = (int64_t)hi;
  a.right = op.right;
  a.sigma = op.sigma;
  a.b = ib;
  a.peers = peers;
  const int S = (int)op.right.count;
  if (S < 1 || S > 4) throw Unsupported("recomputing FISTA kernel: 1..4 stages");
  switch ((S - 1) * 4 + (flush ? 2 : 0) + (fma ? 1 : 0)) {
    case 0: return launch_rc<1, false>(a, st);
    case 1: return launch_rc<1, true>(a, st);
    case 2: return launch_rc_flush<1, false>(a, st);
    case 3: return launch_rc_flush<1, true>(a, st);
    case 4: return launch_rc<2, false>(a, st);
    case 5: return launch_rc<2, true>(a, st);
    case 6: return launch_rc_flush<2, false>(a, st);
    case 7: return launch_rc_flush<2, true>(a, st);
    case 8: return launch_rc<3, false>(a, st);
    case 9: return launch_rc<3, true>(a, st);
    case 10: return launch_rc_flush<3, false>(a, st);
    case 11: return launch_rc_flush<3, true>(a, st);
    case 12: return launch_rc<4, false>(a, st);
    case 13: return launch_rc<4, true>(a, st);
    case 14: return launch_rc_flush<4, false>(a, st);
    default: return launch_rc_flush<4, true>(a, st);
  }
}

}  // namespace l1b
