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
//     rotates (v1, v2) in the lane and the pairs straddling lanes through one
//     shuffle each way -- every rotation is done exactly once, no redundant
//     cone work;
//   * per iteration the chain runs four times (r_k, r_{k-1}, g = G u,
//     r_{k+1}); each run invalidates S entries at both window ends, so the
//     window carries a halo of H3 >= 3S entries per side and owns the middle
//     128 - 2 H3 (104 for 3-4 stages);
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
//   own:      x_{k+1} = trial; ||x||_1, nnz, #(trial != y)
//   r_{k+1} = sigma .* (G^T trial) - b  -> ||r_{k+1}||^2 on the own rows
#include "common.cuh"
#include "fista.cuh"
#include "kernels.hpp"

#include <cstdlib>

namespace l1b {
namespace {

constexpr int kRcThreads = 256;
constexpr int kRcWarps = kRcThreads / 32;
constexpr int kWin = 128;  // window entries per warp (4 per lane)
constexpr unsigned kFull = 0xffffffffu;

template <int S>
struct RcGeom {
  static constexpr int H3 = (3 * S + 3) / 4 * 4;  // halo: >= 3S, 32-byte aligned
  static constexpr int OWN = kWin - 2 * H3;
};

struct RcArgs {
  int64_t n, lo, hi;
  StageTab right;
  const double* sigma;  // global index
  IterBufs b;           // x_k, x_km1, x_next, b by global index (r_* unused)
};

__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
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

// window group [e, e+4) of every input; entries outside [lim_lo, lim_hi) read 0
__device__ __forceinline__ void load_seg(const RcArgs& A, int64_t e, bool full, int64_t lim_lo,
                                         int64_t lim_hi, Seg& s) {
  if (full) {
    ld4(A.b.x_k + e, s.xk);
    ld4(A.b.x_km1 + e, s.xm);
    ld4(A.sigma + e, s.sg);
    ld4(A.b.b + e, s.bb);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool in = e + i >= lim_lo && e + i < lim_hi;
      s.xk[i] = in ? A.b.x_k[e + i] : 0.0;
      s.xm[i] = in ? A.b.x_km1[e + i] : 0.0;
      s.sg[i] = in ? A.sigma[e + i] : 0.0;
      s.bb[i] = in ? A.b.b[e + i] : 0.0;
    }
  }
}

// the same group from a TMA-filled shared-memory slot [x_k | x_km1 | sigma | b]
__device__ __forceinline__ void load_seg_smem(const double* slot, int lane, Seg& s) {
  const double2* p = reinterpret_cast<const double2*>(slot) + 2 * lane;
  double2 a, b;
  a = p[0], b = p[1];
  s.xk[0] = a.x, s.xk[1] = a.y, s.xk[2] = b.x, s.xk[3] = b.y;
  a = p[kWin / 2], b = p[kWin / 2 + 1];
  s.xm[0] = a.x, s.xm[1] = a.y, s.xm[2] = b.x, s.xm[3] = b.y;
  a = p[kWin], b = p[kWin + 1];
  s.sg[0] = a.x, s.sg[1] = a.y, s.sg[2] = b.x, s.sg[3] = b.y;
  a = p[3 * kWin / 2], b = p[3 * kWin / 2 + 1];
  s.bb[0] = a.x, s.bb[1] = a.y, s.bb[2] = b.x, s.bb[3] = b.y;
}

// All S stages on the warp's window; v holds entries [e0, e0+4) (e0 = 0 mod 4).
// Stage pairs (p, p+1), p = offset (mod 2), p >= offset, p + 1 < n
// (linops.cpp:46-60); INTERIOR: the window is away from both ends, every pair
// exists.  Entries within S of a window end come out wrong (their partners
// live outside the window) and are never used.
template <int S, bool TR, bool INTERIOR, int K>
__device__ __forceinline__ void wchain(double (&v)[K][4], int64_t e0, int64_t n,
                                       const StageTab& tab) {
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int s = TR ? k : S - 1 - k;  // A x: forward, transposed; A^T: reverse, plain
    const int o = tab.offset[s];
    const double c = tab.c[s], sn = tab.s[s];
    if ((o & 1) == 0) {
      const bool p0 = INTERIOR || (e0 >= o && e0 + 1 < n);
      const bool p2 = INTERIOR || (e0 + 2 >= o && e0 + 3 < n);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if (p0) rotate_pair(v[q][0], v[q][1], c, sn, TR);
        if (p2) rotate_pair(v[q][2], v[q][3], c, sn, TR);
      }
    } else {
      double right[K], left[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        right[q] = __shfl_down_sync(kFull, v[q][0], 1);  // lane+1's first entry
        left[q] = __shfl_up_sync(kFull, v[q][3], 1);     // lane-1's last entry
      }
      const bool p1 = INTERIOR || (e0 + 1 >= o && e0 + 2 < n);
      const bool p3 = INTERIOR || (e0 + 3 >= o && e0 + 4 < n);
      const bool pm = INTERIOR || (e0 - 1 >= o && e0 < n);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if (p1) rotate_pair(v[q][1], v[q][2], c, sn, TR);
        if (p3) {
          double a = v[q][3], b = right[q];
          rotate_pair(a, b, c, sn, TR);
          v[q][3] = a;
        }
        if (pm) {
          double a = left[q], b = v[q][0];
          rotate_pair(a, b, c, sn, TR);
          v[q][0] = b;
        }
      }
    }
  }
}

// FLUSH: only ||r_k||^2 of the own rows (the objective of the last iterate)
template <int S, bool INTERIOR, bool FLUSH>
__device__ __forceinline__ void segment(const RcArgs& A, const Seg& d, int64_t w0, int lane,
                                        double beta, double inv_l, double thr, double (&acc)[4]) {
  using G = RcGeom<S>;
  const int64_t n = A.n;
  const int64_t e0 = w0 + 4 * lane;
  // own entries of this segment: [w0 + H3, min(w0 + H3 + OWN, hi))
  const int64_t own_lo = w0 + G::H3, own_hi = min(own_lo + G::OWN, A.hi);
  bool mine[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) mine[i] = e0 + i >= own_lo && e0 + i < own_hi;
  constexpr int K = FLUSH ? 1 : 2;
  double t[K][4];  // G^T x_k and G^T x_{k-1}, side by side (independent chains)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    t[0][i] = d.xk[i];
    if (!FLUSH) t[K - 1][i] = d.xm[i];
  }
  wchain<S, true, INTERIOR, K>(t, e0, n, A.right);
  double g[1][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double rk = d.sg[i] * t[0][i] - d.bb[i];
    if (mine[i]) acc[3] += rk * rk;  // ||r_k||^2: x_k's objective, recorded one kernel late
    if (!FLUSH) {
      const double rm = d.sg[i] * t[K - 1][i] - d.bb[i];
      g[0][i] = d.sg[i] * ((1.0 + beta) * rk - beta * rm);
    }
  }
  if (FLUSH) return;
  wchain<S, false, INTERIOR, 1>(g, e0, n, A.right);
  double tr[4];
  unsigned nz = 0, mism = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double y = d.xk[i] + beta * (d.xk[i] - d.xm[i]);
    tr[i] = soft_threshold(y - inv_l * g[0][i], thr);
    if (mine[i]) {
      acc[0] += fabs(tr[i]);
      nz += tr[i] != 0.0;
      mism += tr[i] != y;
    }
  }
  acc[1] += (double)nz;
  acc[2] += (double)mism;
  if (mine[0] && mine[3]) {
    st4(A.b.x_next + e0, tr);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (mine[i]) A.b.x_next[e0 + i] = tr[i];
  }
}

template <int S, int MB, int PF, int kD = 2, bool FLUSH = false>
__global__ void __launch_bounds__(kRcThreads, MB) fista_rc_kernel(RcArgs A) {
  using G = RcGeom<S>;
  FistaDev* st = A.b.st;
  if (*(volatile int*)&st->stop) return;
  const double beta = st->beta_y;  // forms y_k, r_y from the last two iterates
  const double inv_l = 1.0 / st->lval;
  const double thr = st->tau * inv_l;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = A.n, lo = A.lo, hi = A.hi;
  // loads stay inside [0, n) and inside the x windows [lo - H3, hi + H3)
  const int64_t lim_lo = max((int64_t)0, lo - G::H3), lim_hi = min(n, hi + G::H3);
  const int64_t nseg = (hi - lo + G::OWN - 1) / G::OWN;
  // segments of one block are consecutive (their halos meet in L1/L2)
  const int64_t stride = (int64_t)gridDim.x * kRcWarps;
  int64_t sgi = (int64_t)blockIdx.x * kRcWarps + warp;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // ||x||_1, nnz, #(trial != y), ||r||^2

  auto w0_of = [&](int64_t q) { return lo + q * G::OWN - G::H3; };
  auto full_of = [&](int64_t w0) { return w0 >= lim_lo && w0 + kWin <= lim_hi; };
  Seg cur, nxt;
  if (PF == 4) {
    // per-warp ring of kD slots, each one segment of the four inputs (4 KiB),
    // filled by bulk copies (lane 0) kD - 1 segments ahead of the compute
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int kSlot = 4 * kWin * 8;
    unsigned char* ring = smem + (size_t)warp * kD * kSlot;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kRcWarps * kD * kSlot) + warp * kD;
    if (lane == 0) {
      for (int q = 0; q < kD; ++q) mbar_init(&bars[q], 1);
      fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int64_t q, int slot) {  // lane 0
      const int64_t w = w0_of(q);
      if (q >= nseg || !full_of(w)) return;
      unsigned char* d = ring + slot * kSlot;
      mbar_arrive_expect_tx(&bars[slot], kSlot);
      bulk_g2s(d, A.b.x_k + w, kWin * 8, &bars[slot]);
      bulk_g2s(d + kWin * 8, A.b.x_km1 + w, kWin * 8, &bars[slot]);
      bulk_g2s(d + 2 * kWin * 8, A.sigma + w, kWin * 8, &bars[slot]);
      bulk_g2s(d + 3 * kWin * 8, A.b.b + w, kWin * 8, &bars[slot]);
    };
    if (lane == 0)
      for (int q = 0; q < kD - 1; ++q) issue(sgi + q * stride, q);
    uint32_t phase = 0;  // bit q: parity of slot q's next completion
    int slot = 0;
    for (int64_t i = 0; sgi < nseg; sgi += stride, ++i) {
      const int64_t w0 = w0_of(sgi);
      if (lane == 0) issue(sgi + (kD - 1) * stride, (slot + kD - 1) % kD);
      const bool full = full_of(w0);
      if (full) {
        mbar_wait(&bars[slot], (phase >> slot) & 1);
        phase ^= 1u << slot;
        load_seg_smem(reinterpret_cast<const double*>(ring + slot * kSlot), lane, cur);
      } else {
        load_seg(A, w0 + 4 * lane, false, lim_lo, lim_hi, cur);
      }
      const bool interior = full && w0 >= 2 && w0 + kWin < n;
      if (interior)
        segment<S, true, FLUSH>(A, cur, w0, lane, beta, inv_l, thr, acc);
      else
        segment<S, false, FLUSH>(A, cur, w0, lane, beta, inv_l, thr, acc);
      __syncwarp();  // the slot's reads are done before it is refilled
      if (lane == 0) fence_proxy_async();
      slot = (slot + 1) % kD;
    }
  } else {
    if (sgi < nseg) {
      const int64_t w0 = w0_of(sgi);
      load_seg(A, w0 + 4 * lane, full_of(w0), lim_lo, lim_hi, cur);
    }
    for (; sgi < nseg; sgi += stride) {
      const int64_t w0 = w0_of(sgi);
      if (PF != 1) {
        if (sgi != (int64_t)blockIdx.x * kRcWarps + warp)
          load_seg(A, w0 + 4 * lane, full_of(w0), lim_lo, lim_hi, cur);
        if (PF >= 2 && lane < 4) {  // bulk L2 prefetch of a later segment (no registers held)
          const int64_t q = sgi + (PF - 1) * stride;
          if (q < nseg && full_of(w0_of(q))) {
            const double* base = lane == 0 ? A.b.x_k : lane == 1 ? A.b.x_km1 : lane == 2 ? A.sigma : A.b.b;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + w0_of(q)),
                         "r"(kWin * 8)
                         : "memory");
          }
        }
      } else if (sgi + stride < nseg) {  // next segment's loads in flight during this one
        const int64_t w1 = w0_of(sgi + stride);
        load_seg(A, w1 + 4 * lane, full_of(w1), lim_lo, lim_hi, nxt);
      }
      // every pair touching the window exists: p >= w0 - 1 >= 1 >= offset, p + 1 <= w0 + kWin < n
      const bool interior = full_of(w0) && w0 >= 2 && w0 + kWin < n;
      if (interior)
        segment<S, true, FLUSH>(A, cur, w0, lane, beta, inv_l, thr, acc);
      else
        segment<S, false, FLUSH>(A, cur, w0, lane, beta, inv_l, thr, acc);
      if (PF == 1) cur = nxt;
    }
  }
  double tot[4];
  if (grid_sum<4>(acc, A.b.partials, &st->ticket[0], tot) && threadIdx.x == 0) {
    st->scal[0] = tot[0];
    st->scal[1] = tot[1];
    st->scal[2] = tot[2];
    st->scal[3] = tot[3];
    fista_finalize_lagged(st, A.b.trace, FLUSH);
  }
}

template <int S, int MB, int PF, int kD = 2, bool FLUSH = false>
void launch_rc_v(const RcArgs& a, cudaStream_t st) {
  using G = RcGeom<S>;
  static int grid_cap = 0;
  const size_t smem = PF == 4 ? (size_t)kRcWarps * kD * (4 * kWin * 8 + 8) : 0;
  if (!grid_cap) {
    if (smem)
      L1B_CUDA(cudaFuncSetAttribute(fista_rc_kernel<S, MB, PF, kD, FLUSH>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fista_rc_kernel<S, MB, PF, kD, FLUSH>,
                                                          kRcThreads, smem));
    grid_cap = std::min(std::max(1, per_sm) * sm_count(), spmv_grid_max());
  }
  const int64_t nseg = (a.hi - a.lo + G::OWN - 1) / G::OWN;
  const int64_t blocks = (nseg + kRcWarps - 1) / kRcWarps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(blocks, grid_cap));
  fista_rc_kernel<S, MB, PF, kD, FLUSH><<<grid, kRcThreads, smem, st>>>(a);
  L1B_LAUNCHED();
}

// min CTAs/SM x register prefetch of the next segment; L1B_RC_VARIANT picks (tuning runs)
int rc_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("L1B_RC_VARIANT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int S>
void launch_rc(const RcArgs& a, cudaStream_t st) {
  switch (rc_variant()) {
    case 1: return launch_rc_v<S, 3, 0>(a, st);
    case 2: return launch_rc_v<S, 3, 2>(a, st);
    case 3: return launch_rc_v<S, 3, 3>(a, st);
    case 4: return launch_rc_v<S, 2, 2>(a, st);
    case 5: return launch_rc_v<S, 3, 4, 2>(a, st);
    case 6: return launch_rc_v<S, 2, 4, 3>(a, st);
    case 7: return launch_rc_v<S, 2, 4, 2>(a, st);
    default: return launch_rc_v<S, 2, 1>(a, st);
  }
}

template <int S>
void launch_rc_flush(const RcArgs& a, cudaStream_t st) {
  launch_rc_v<S, 2, 0, 2, true>(a, st);
}

}  // namespace

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
                   cudaStream_t st, bool flush) {
  if (lo % 4 != 0) throw std::invalid_argument("fista_rc_iter: block start must be a multiple of 4");
  RcArgs a;
  a.n = (int64_t)op.n;
  a.lo = (int64_t)lo;
  a.hi = (int64_t)hi;
  a.right = op.right;
  a.sigma = op.sigma;
  a.b = ib;
  switch (op.right.count * 2 + (flush ? 1 : 0)) {
    case 2: return launch_rc<1>(a, st);
    case 3: return launch_rc_flush<1>(a, st);
    case 4: return launch_rc<2>(a, st);
    case 5: return launch_rc_flush<2>(a, st);
    case 6: return launch_rc<3>(a, st);
    case 7: return launch_rc_flush<3>(a, st);
    case 8: return launch_rc<4>(a, st);
    case 9: return launch_rc_flush<4>(a, st);
    default: throw Unsupported("recomputing FISTA kernel: 1..4 stages");
  }
}

}  // namespace l1b
