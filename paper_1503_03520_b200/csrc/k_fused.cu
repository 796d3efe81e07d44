// k_fused.cu -- matrix-free FISTA for banded operators.
//
// For identity P1/P2 and no left stages, A = Sigma G^T (rows >= n empty) with
// G = S_0 S_1 ... S_{k-1} the product of the right stages (linops.cpp:422-473):
//   A x    = sigma .* (S_{k-1}^T ... S_0^T x)              (stages forward, transposed)
//   A^T r  = S_0 (S_1 ( ... S_{k-1} (sigma .* r[0:n])))     (stages reverse, plain)
// Each product is one kernel: a tile of T = 1024 entries plus a k-entry halo
// on each side is streamed into shared memory by TMA bulk copies (3-stage
// mbarrier ring, as in spmv.cuh), the k stages are applied in shared memory
// (one pass per stage, every pair rotated exactly once, in the reference's
// stage order and rounding), and the fused FISTA epilogue consumes the valid
// centre.  The operation sequence per entry is the reference's own, so the
// products -- and therefore the FISTA iterates -- are bit-identical to
// OperatorSpec::apply / apply_transpose; only the reduction order of f
// differs.  HBM traffic per iteration: 48n + 48n bytes (K1: r_y, sigma, y, x
// r/w; K2: x, sigma, b, r_x r/w, r_y w) versus 288n for the CSR/CSC path.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "fista.cuh"
#include "kernels.hpp"

namespace l1b {

namespace {

constexpr int kT = 1024;      // tile entries
constexpr int kFThreads = 256;
constexpr int kHaloMax = 16;  // >= #stages, even
constexpr int kFStages = 3;

constexpr size_t round16(size_t b) { return (b + 15) / 16 * 16; }

struct FusedLayout {
  static constexpr size_t win = kT + 2 * kHaloMax + 2;  // swept window (+ rounding slack)
  static constexpr size_t win_bytes = round16(win * 8);
  static constexpr size_t vec_bytes = round16((kT + 2) * 8);
  // slot: [work window][sigma window][vec0][vec1]
  static constexpr size_t slot_bytes = 2 * win_bytes + 2 * vec_bytes;
  static constexpr size_t bars_off = kFStages * slot_bytes;
  static constexpr size_t total = bars_off + kFStages * 8;
};

struct FusedArgs {
  uint64_t n;
  uint64_t lo, hi;  // lines produced: global [lo, hi) (a shard's own range)
  int halo;  // even, >= #stages
  StageTab right;
  const double* sigma;  // n (+2 slack)
  // K1 (transpose): in = r_y; vec0 = y, vec1 = x; writes x, y
  // K2 (forward):   in = x;   vec0 = b, vec1 = r_x; writes r_x, r_y
  // every pointer is indexed by GLOBAL entry (pre-offset by the caller)
  const double* in;
  const double* vec0;
  const double* vec1;
  double* out0;
  double* out1;
  FistaDev* st;
  FistaSample* trace;
  double* partials;
  int mode;  // 0: plain product into out0, 1: FISTA epilogue
};

// pairs (p, p+1), p = off (mod 2), p+1 < min(w1, n), p >= w0 -- applied to
// buf[p - w0]; one pass of the stage.  With `sig` (first pass of A^T r), the
// entries are first scaled by sigma (linops.cpp:460) as they are loaded --
// the same two roundings as a separate pass -- and the entries no pair of
// this stage covers are scaled by the threads at the two ends.
__device__ __forceinline__ void sweep_stage(double* buf, uint64_t w0, uint64_t w1, uint64_t n,
                                            int off, double c, double s, bool transposed,
                                            const double* sig = nullptr) {
  const uint64_t first = w0 > (uint64_t)off ? w0 + ((w0 - off) & 1) : (uint64_t)off;
  const uint64_t last = min(w1, n);
  const int npairs = last >= first + 2 ? (int)((last - first) / 2) : 0;
  for (int q = threadIdx.x; q < npairs; q += blockDim.x) {
    const uint64_t k = first + 2 * (uint64_t)q - w0;
    double a = buf[k], b = buf[k + 1];
    if (sig) {
      a = sig[k] * a;
      b = sig[k + 1] * b;
    }
    rotate_pair(a, b, c, s, transposed);
    buf[k] = a;
    buf[k + 1] = b;
  }
  if (sig) {
    const uint64_t covered_end = npairs ? first + 2 * (uint64_t)npairs : w0;
    const uint64_t lead_end = npairs ? first : w1;
    for (uint64_t p = w0 + threadIdx.x; p < lead_end; p += blockDim.x) buf[p - w0] = sig[p - w0] * buf[p - w0];
    if (npairs)
      for (uint64_t p = covered_end + threadIdx.x; p < w1; p += blockDim.x)
        buf[p - w0] = sig[p - w0] * buf[p - w0];
  }
}

template <bool kTranspose>
__global__ void __launch_bounds__(kFThreads, 2) fused_kernel(FusedArgs A) {
  if (A.mode == 1 && *(volatile int*)&A.st->stop) return;
  using L = FusedLayout;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bars_off);
  const int t = threadIdx.x;
  const uint64_t n = A.n;
  const uint64_t H = (uint64_t)A.halo;
  const uint64_t ntiles = (A.hi - A.lo + kT - 1) / kT;
  const uint64_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  // FISTA scalars (solvers.cpp:322-358)
  double beta = 0.0, inv_l = 0.0, thr = 0.0, tau = 0.0;
  if (A.mode == 1) {
    const double tm = A.st->t;
    const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * tm * tm));
    beta = A.st->accel ? (tm - 1.0) / t_next : 0.0;
    inv_l = 1.0 / A.st->lval;
    tau = A.st->tau;
    thr = tau * inv_l;
  }
  double acc[3] = {0.0, 0.0, 0.0};

  if (t == 0) {
    for (int s = 0; s < kFStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto window = [&](uint64_t k, uint64_t* t0, uint64_t* te, uint64_t* w0, uint64_t* w1) {
    *t0 = A.lo + (blockIdx.x + k * gridDim.x) * (uint64_t)kT;
    *te = min(*t0 + kT, A.hi);
    *w0 = *t0 > H ? *t0 - H : 0;
    *w1 = min(n, *te + H);
  };
  auto issue = [&](uint64_t k) {
    uint64_t t0, te, w0, w1;
    window(k, &t0, &te, &w0, &w1);
    unsigned char* slot = smem + (k % kFStages) * L::slot_bytes;
    double* s_in = reinterpret_cast<double*>(slot);
    double* s_sig = reinterpret_cast<double*>(slot + L::win_bytes);
    double* s_v0 = reinterpret_cast<double*>(slot + 2 * L::win_bytes);
    double* s_v1 = reinterpret_cast<double*>(slot + 2 * L::win_bytes + L::vec_bytes);
    const uint32_t win_b = (uint32_t)(((w1 - w0) + 1) & ~1ull) * 8u;  // even count: 16 B multiple
    const uint32_t own_b = (uint32_t)(((te - t0) + 1) & ~1ull) * 8u;
    uint32_t tx = win_b + (kTranspose ? win_b : own_b);
    if (A.mode == 1) tx += 2 * own_b;
    uint64_t* bar = &bars[k % kFStages];
    mbar_arrive_expect_tx(bar, tx);
    bulk_g2s(s_in, A.in + w0, win_b, bar);
    if (kTranspose)
      bulk_g2s(s_sig, A.sigma + w0, win_b, bar);  // sigma multiplies before the sweep
    else
      bulk_g2s(s_sig, A.sigma + t0, own_b, bar);  // ... after it
    if (A.mode == 1) {
      bulk_g2s(s_v0, A.vec0 + t0, own_b, bar);
      bulk_g2s(s_v1, A.vec1 + t0, own_b, bar);
    }
  };

  if (t == 0)
    for (uint64_t k = 0; k + 1 < (uint64_t)kFStages && k < mine; ++k) issue(k);

  for (uint64_t k = 0; k < mine; ++k) {
    if (t == 0 && k + kFStages - 1 < mine) {
      fence_proxy_async();
      issue(k + kFStages - 1);
    }
    uint64_t t0, te, w0, w1;
    window(k, &t0, &te, &w0, &w1);
    unsigned char* slot = smem + (k % kFStages) * L::slot_bytes;
    double* s_in = reinterpret_cast<double*>(slot);
    const double* s_sig = reinterpret_cast<const double*>(slot + L::win_bytes);
    const double* s_v0 = reinterpret_cast<const double*>(slot + 2 * L::win_bytes);
    const double* s_v1 = reinterpret_cast<const double*>(slot + 2 * L::win_bytes + L::vec_bytes);
    mbar_wait(&bars[k % kFStages], (uint32_t)((k / kFStages) & 1));
    const int wlen = (int)(w1 - w0);
    if (kTranspose) {
      // v[j] = sigma[j] * r[j] (linops.cpp:460), then G = S_0 ... S_{k-1}: reverse, plain
      if (A.right.count == 0) {
        for (int q = t; q < wlen; q += kFThreads) s_in[q] = s_sig[q] * s_in[q];
        __syncthreads();
      }
      for (int s = A.right.count - 1; s >= 0; --s) {
        sweep_stage(s_in, w0, w1, n, A.right.offset[s], A.right.c[s], A.right.s[s], false,
                    s == A.right.count - 1 ? s_sig : nullptr);
        __syncthreads();
      }
    } else {
      // G^T x: stages forward, transposed (linops.cpp:429)
      for (int s = 0; s < A.right.count; ++s) {
        sweep_stage(s_in, w0, w1, n, A.right.offset[s], A.right.c[s], A.right.s[s], true);
        __syncthreads();
      }
    }
    const int own = (int)(te - t0), off = (int)(t0 - w0);
    for (int q = t; q < own; q += kFThreads) {
      const uint64_t j = t0 + q;
      if (kTranspose) {
        const double g = s_in[off + q];
        if (A.mode == 0) {
          A.out0[j] = g;
        } else {  // EpiFistaX of k_spmv.cu
          const double yo = s_v0[q], xo = s_v1[q];
          const double tr = soft_threshold(yo - inv_l * g, thr);
          acc[2] += tr != yo ? 1.0 : 0.0;
          A.out0[j] = tr + beta * (tr - xo);  // y
          A.out1[j] = tr;                     // x
          acc[0] += fabs(tr);
          acc[1] += tr != 0.0 ? 1.0 : 0.0;
        }
      } else {
        const double ax = s_sig[q] * s_in[off + q];  // t[i] = sigma[i] * v[i] (linops.cpp:433)
        if (A.mode == 0) {
          A.out0[j] = ax;
        } else {  // EpiFistaR of k_spmv.cu
          const double rt = ax - s_v0[q];
          const double rx = s_v1[q];
          A.out1[j] = (1.0 + beta) * rt - beta * rx;  // r_y
          A.out0[j] = rt;                             // r_x
          acc[0] += rt * rt;
        }
      }
    }
    __syncthreads();
  }
  if (A.mode == 1) {
    if (kTranspose) {
      double tot[3];
      if (grid_sum<3>(acc, A.partials, &A.st->ticket[0], tot) && t == 0) {
        A.st->scal[0] = tot[0];
        A.st->scal[1] = tot[1];
        A.st->scal[2] = tot[2];
      }
    } else {
      double a1[1] = {acc[0]}, tot[1];
      if (grid_sum<1>(a1, A.partials, &A.st->ticket[1], tot) && t == 0) {
        A.st->scal[3] = tot[0];
        if (!A.st->defer) fista_finalize_device(A.st, A.trace);
      }
    }
  }
}

template <bool kTranspose>
void launch_fused(const FusedArgs& a, cudaStream_t st) {
  using L = FusedLayout;
  static int grid_cap = 0;
  if (!grid_cap) {
    L1B_CUDA(cudaFuncSetAttribute(fused_kernel<kTranspose>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::total));
    int per_sm = 0;
    L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<kTranspose>,
                                                          kFThreads, L::total));
    grid_cap = std::max(1, per_sm) * sm_count();
  }
  const uint64_t tiles = (a.hi - a.lo + kT - 1) / kT;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)grid_cap));
  fused_kernel<kTranspose><<<grid, kFThreads, L::total, st>>>(a);
  L1B_LAUNCHED();
}

FusedArgs base_args(const OpView& op) {
  if (op.right.count > kHaloMax) throw Unsupported("fused operator: more than 16 stages");
  FusedArgs a{};
  a.n = op.n;
  a.lo = 0;
  a.hi = op.n;
  a.halo = (op.right.count + 1) & ~1;
  a.right = op.right;
  a.sigma = op.sigma;
  return a;
}

}  // namespace

bool fused_supported(const OpView& op) {
  return !op.p1 && !op.p2 && op.left.count == 0 && op.right.count <= kHaloMax;
}

void fused_apply(const OpView& op, const double* x, double* y, cudaStream_t st) {
  FusedArgs a = base_args(op);
  a.in = x;
  a.out0 = y;
  a.mode = 0;
  launch_fused<false>(a, st);
}

void fused_apply_transpose(const OpView& op, const double* r, double* g, cudaStream_t st) {
  FusedArgs a = base_args(op);
  a.in = r;
  a.out0 = g;
  a.mode = 0;
  launch_fused<true>(a, st);
}

// global-index view of an own-range array that starts at global index `first`
template <class T>
T* at_global(T* p, int64_t first) {
  return p - first;
}

void fista_fused_k1(const OpView& op, const FistaBufs& fb, cudaStream_t st) {
  FusedArgs a = base_args(op);
  a.lo = fb.lo;
  a.hi = fb.hi;
  const int64_t lo = (int64_t)fb.lo;
  a.in = at_global(fb.r_y_gather, fb.gather_base);
  a.vec0 = at_global(fb.y, lo);
  a.vec1 = at_global(fb.x, lo);
  a.out0 = at_global(fb.y, lo);
  a.out1 = at_global(fb.x, lo);
  a.st = fb.st;
  a.trace = fb.trace;
  a.partials = fb.partials;
  a.mode = 1;
  launch_fused<true>(a, st);
}

void fista_fused_k2(const OpView& op, const FistaBufs& fb, cudaStream_t st) {
  FusedArgs a = base_args(op);
  a.lo = fb.lo;
  a.hi = fb.hi;
  const int64_t lo = (int64_t)fb.lo;
  a.in = at_global(fb.x_gather, fb.gather_base);
  a.vec0 = at_global(fb.b, lo);
  a.vec1 = at_global(fb.r_x, lo);
  a.out0 = at_global(fb.r_x, lo);
  a.out1 = at_global(fb.r_y, lo);
  a.st = fb.st;
  a.trace = fb.trace;
  a.partials = fb.partials;
  a.mode = 1;
  launch_fused<false>(a, st);
}

// ---------------------------------------------------------------------------
// One kernel per FISTA iteration (banded operators, one device).
//
// Iteration k+1 needs only the last two iterates: y_k = x_k + beta (x_k -
// x_{k-1}) and r_y = (1 + beta) r_k - beta r_{k-1} are formed on the fly
// (solvers.cpp:349-357, same operations), so y and r_y are never stored and
// x / r rotate through three buffers (a tile's halo reads of x_k, x_{k-1}
// never meet another tile's writes of x_{k+1}).  Per tile [t0, te):
//   r windows [t0-2H, te+2H):  u = sigma .* r_y ; g = G u        (A^T r_y)
//   x windows [t0-H, te+H):    trial = S(y - g/L, tau/L); own -> x_{k+1}
//   own rows:                  r_{k+1} = sigma .* (G^T trial) - b
// HBM per iteration: x_k, x_{k-1}, r_k, r_{k-1}, sigma, b read + x_{k+1},
// r_{k+1} written = 64n bytes (96n for the two-kernel pair, 288n for CSR/CSC).
namespace {

constexpr int kTI = 1024;     // tile entries
template <int kIStages>
struct IterLayoutT {
  static constexpr size_t rwin = kTI + 4 * kHaloMax + 2;
  static constexpr size_t xwin = kTI + 2 * kHaloMax + 2;
  // whole 128-byte rows: the chain inputs are stored swizzled within rows
  static constexpr size_t rwin_b = (rwin * 8 + 127) / 128 * 128;
  static constexpr size_t xwin_b = (xwin * 8 + 127) / 128 * 128;
  static constexpr size_t own_b = round16((kTI + 2) * 8);
  // slot: r_k | r_km1 | sigma (r window) | x_k | x_km1 (x window) | b (own)
  static constexpr size_t off_rkm1 = rwin_b;
  static constexpr size_t off_sig = 2 * rwin_b;
  static constexpr size_t off_xk = 3 * rwin_b;
  static constexpr size_t off_xkm1 = 3 * rwin_b + xwin_b;
  static constexpr size_t off_b = 3 * rwin_b + 2 * xwin_b;
  static constexpr size_t slot_bytes = off_b + own_b;
  static constexpr size_t bars_off = kIStages * slot_bytes;
  static constexpr size_t total = bars_off + kIStages * 8;
};

struct IterArgs {
  uint64_t n;
  uint64_t lo, hi;  // own rows == columns [lo, hi) (a shard's block; [0, n) on one device)
  int halo;
  StageTab right;
  const double* sigma;
  IterBufs b;
};

// All S stages of one product for NO consecutive outputs [P, P+NO), in
// registers: the window [P-S, P+NO+S) of the input is loaded, every pair of
// every stage that lies inside the window is rotated, and the NO centre
// entries -- whose dependency cones fit the window -- come out exactly as in
// the reference's full-vector sweeps.  No barrier between stages.  The pair
// parity of a stage is warp-uniform (P is a multiple of NO for every thread),
// so away from the global ends the pairs are a fixed unrolled set.
// Chain inputs (u, trial) are written by lane-contiguous passes into a
// swizzled layout: 16-byte chunk c of each 128-byte row r sits at c ^ (r & 7),
// so that the chains' per-thread windows (lane stride 32 bytes) hit all 32
// banks in every 16-byte load instead of half of them.
__device__ __forceinline__ int swz_chunk(int c) { return (c & ~7) | ((c ^ (c >> 3)) & 7); }
__device__ __forceinline__ int swz(int e) { return (swz_chunk(e >> 1) << 1) | (e & 1); }
struct LoadSwz {
  const double* w;
  int e0;  // logical index of window entry 0
  __device__ __forceinline__ double operator()(int q) const { return w[swz(e0 + q)]; }
  __device__ __forceinline__ double2 pair(int q) const {  // e0 even
    return reinterpret_cast<const double2*>(w)[swz_chunk((e0 >> 1) + q)];
  }
};
template <int S, int NO, bool TR, bool INTERIOR, class Load>
__device__ __forceinline__ void chain(const Load& ld, int64_t g0, int64_t n, const StageTab& tab,
                                      double (&out)[NO]) {
  constexpr int W = 2 * S + NO;
  double v[W];
  if ((S & 1) == 0) {  // window starts on an even smem index: 16-byte loads
#pragma unroll
    for (int q = 0; q < W / 2; ++q) {
      const double2 d = ld.pair(q);
      v[2 * q] = d.x;
      v[2 * q + 1] = d.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < W; ++q) v[q] = ld(q);
  }
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int s = TR ? k : S - 1 - k;  // A x: forward, transposed; A^T: reverse, plain
    const int o = tab.offset[s];
    const double c = tab.c[s], sn = tab.s[s];
    // g0 has the parity of S (tiles start on even entries, chains on multiples of NO)
    const int par = (S + o) & 1;
    if (INTERIOR) {  // tile away from both ends: every pair start p >= 1 >= offset, p+1 < n
      if (par == 0) {
#pragma unroll
        for (int l = 0; l + 1 < W; l += 2) rotate_pair(v[l], v[l + 1], c, sn, TR);
      } else {
#pragma unroll
        for (int l = 1; l + 1 < W; l += 2) rotate_pair(v[l], v[l + 1], c, sn, TR);
      }
    } else {
#pragma unroll
      for (int l = 0; l + 1 < W; ++l) {
        const int64_t p = g0 + l;
        if ((l & 1) == par && p >= o && p + 1 < n) rotate_pair(v[l], v[l + 1], c, sn, TR);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < NO; ++e) out[e] = v[S + e];
}

constexpr int kNO = 4;  // outputs per thread and chain

template <int S, int kIStages, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) fista_iter_kernel(IterArgs A) {
  FistaDev* st = A.b.st;
  if (*(volatile int*)&st->stop) return;
  using L = IterLayoutT<kIStages>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bars_off);
  const int t = threadIdx.x;
  const int64_t n = (int64_t)A.n;
  constexpr int64_t H = (S + 1) & ~1;  // window overhang (even)
  constexpr int64_t TT = kTI - 2 * H;    // tile: the x window is exactly kNO * kThreads entries
  const uint64_t ntiles = (A.hi - A.lo + TT - 1) / TT;
  const uint64_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const double beta = st->beta_y;  // forms y_k, r_y from the last two iterates
  const double inv_l = 1.0 / st->lval;
  const double thr = st->tau * inv_l;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // ||x||_1, nnz, #(trial != y), ||r||^2

  if (t == 0) {
    for (int s = 0; s < kIStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // tile [t0, te); r window [t0 - 2H, te + 2H) and x window [t0 - H, te + H),
  // both kept on their unclipped grid in shared memory (entries outside
  // [0, n) are zero-filled and never rotated)
  auto tile0 = [&](uint64_t k) {
    return (int64_t)(A.lo + (blockIdx.x + k * gridDim.x) * (uint64_t)TT);
  };
  auto even_bytes = [](int64_t len) { return (uint32_t)((len + 1) & ~1ll) * 8u; };
  auto issue = [&](uint64_t k) {
    const int64_t t0 = tile0(k), te = min(t0 + TT, (int64_t)A.hi);
    const int64_t r0 = max(t0 - 2 * H, (int64_t)0), r1 = min(n, te + 2 * H);
    const int64_t x0 = max(t0 - H, (int64_t)0), x1 = min(n, te + H);
    unsigned char* slot = smem + (k % kIStages) * L::slot_bytes;
    // smem index 0 <-> global t0 - 2H (r) / t0 - H (x)
    const int64_t rs = r0 - (t0 - 2 * H), xs = x0 - (t0 - H);
    const uint32_t rb = even_bytes(r1 - r0), xb = even_bytes(x1 - x0), ob = even_bytes(te - t0);
    uint64_t* bar = &bars[k % kIStages];
    mbar_arrive_expect_tx(bar, 3 * rb + 2 * xb + ob);
    bulk_g2s(slot + rs * 8, A.b.r_k + r0, rb, bar);
    bulk_g2s(slot + L::off_rkm1 + rs * 8, A.b.r_km1 + r0, rb, bar);
    bulk_g2s(slot + L::off_sig + rs * 8, A.sigma + r0, rb, bar);
    bulk_g2s(slot + L::off_xk + xs * 8, A.b.x_k + x0, xb, bar);
    bulk_g2s(slot + L::off_xkm1 + xs * 8, A.b.x_km1 + x0, xb, bar);
    bulk_g2s(slot + L::off_b, A.b.b + t0, ob, bar);
  };

  // zero the out-of-range margins of both slots once (they are never written by TMA)
  for (int q = t; q < (int)(kIStages * L::slot_bytes / 8); q += kThreads)
    reinterpret_cast<double*>(smem)[q] = 0.0;
  __syncthreads();
  if (t == 0) {
    fence_proxy_async();
    for (uint64_t k = 0; k + 1 < (uint64_t)kIStages && k < mine; ++k) issue(k);
  }

  for (uint64_t k = 0; k < mine; ++k) {
    if (t == 0 && k + kIStages - 1 < mine) {
      fence_proxy_async();
      issue(k + kIStages - 1);
    }
    const int64_t t0 = tile0(k), te = min(t0 + TT, (int64_t)A.hi);
    const int64_t gx = t0 - H;  // global index of x smem entry 0 (r windows start at t0 - 2H)
    unsigned char* slot = smem + (k % kIStages) * L::slot_bytes;
    double* s_r = reinterpret_cast<double*>(slot);  // r_k -> sigma .* r_y
    const double* s_rm = reinterpret_cast<const double*>(slot + L::off_rkm1);
    const double* s_sig = reinterpret_cast<const double*>(slot + L::off_sig);
    double* s_x = reinterpret_cast<double*>(slot + L::off_xk);     // x_k -> y
    double* s_tr = reinterpret_cast<double*>(slot + L::off_xkm1);  // x_{k-1} -> trial
    const double* s_b = reinterpret_cast<const double*>(slot + L::off_b);
    mbar_wait(&bars[k % kIStages], (uint32_t)((k / kIStages) & 1));
    const int rlen = (int)(te - t0 + 4 * H), xlen = (int)(te - t0 + 2 * H);
    const bool interior = t0 - 2 * H >= 1 && te + 2 * H <= n;  // tile-uniform
    // Shared-memory traffic is the limiter here: per-element work runs with
    // consecutive threads on consecutive entries (2 wavefronts per warp
    // access); only the register chains read per-thread windows.
    // 0. u = sigma .* r_y, r_y = (1 + beta) r_k - beta r_{k-1}: in place of r_k,
    //    swizzled (rows lie inside one warp's 32 entries: read all, then write)
    for (int q0 = 0; q0 < rlen; q0 += kThreads) {
      const int q = q0 + t;
      double u = 0.0;
      if (q < rlen) u = s_sig[q] * ((1.0 + beta) * s_r[q] - beta * s_rm[q]);
      __syncwarp();
      if (q < rlen) s_r[swz(q)] = u;
    }
    __syncthreads();
    // 1. g = G u on the x window: kNO entries per thread, all stages in registers;
    //    g parked (swizzled) in the now free r_{k-1} buffer at x-window positions
    double* s_g = const_cast<double*>(s_rm);
    for (int q = kNO * t; q < xlen; q += kNO * kThreads) {
      double g[kNO];
      const LoadSwz ld{s_r, q + (int)H - S};
      if (interior)
        chain<S, kNO, false, true>(ld, gx + q - S, n, A.right, g);
      else
        chain<S, kNO, false, false>(ld, gx + q - S, n, A.right, g);
      reinterpret_cast<double2*>(s_g)[swz_chunk(q >> 1)] = make_double2(g[0], g[1]);
      reinterpret_cast<double2*>(s_g)[swz_chunk((q >> 1) + 1)] = make_double2(g[2], g[3]);
    }
    __syncthreads();
    // 2. y = x_k + beta (x_k - x_{k-1}); trial = S(y - g/L, tau/L); own -> x_{k+1};
    //    trial in place of x_{k-1}, swizzled
    for (int q0 = 0; q0 < xlen; q0 += kThreads) {
      const int q = q0 + t;
      double tr = 0.0;
      if (q < xlen) {
        const double xk = s_x[q];
        const double y = xk + beta * (xk - s_tr[q]);
        tr = soft_threshold(y - inv_l * s_g[swz(q)], thr);
        const int64_t j = gx + q;
        if (j >= t0 && j < te) {
          A.b.x_next[j] = tr;
          acc[0] += fabs(tr);
          acc[1] += tr != 0.0 ? 1.0 : 0.0;
          acc[2] += tr != y ? 1.0 : 0.0;
        }
        if (j < 0 || j >= n) tr = 0.0;
      }
      __syncwarp();
      if (q < xlen) s_tr[swz(q)] = tr;
    }
    __syncthreads();
    // 3. r_{k+1} = sigma .* (G^T trial) - b on the own rows
    const int own = (int)(te - t0);
    for (int q = kNO * t; q < own; q += kNO * kThreads) {
      double av[kNO];
      const LoadSwz ld{s_tr, q + (int)H - S};
      if (interior)
        chain<S, kNO, true, true>(ld, t0 + q - S, n, A.right, av);
      else
        chain<S, kNO, true, false>(ld, t0 + q - S, n, A.right, av);
      const double2 sg0 = reinterpret_cast<const double2*>(s_sig + 2 * H + q)[0];
      const double2 sg1 = reinterpret_cast<const double2*>(s_sig + 2 * H + q)[1];
      const double2 b0 = reinterpret_cast<const double2*>(s_b + q)[0];
      const double2 b1 = reinterpret_cast<const double2*>(s_b + q)[1];
      const double rt[kNO] = {sg0.x * av[0] - b0.x, sg0.y * av[1] - b0.y, sg1.x * av[2] - b1.x,
                              sg1.y * av[3] - b1.y};
      if (q + kNO <= own) {
        double2* dst = reinterpret_cast<double2*>(A.b.r_next + t0 + q);
        dst[0] = make_double2(rt[0], rt[1]);
        dst[1] = make_double2(rt[2], rt[3]);
#pragma unroll
        for (int e = 0; e < kNO; ++e) acc[3] += rt[e] * rt[e];
      } else {
#pragma unroll
        for (int e = 0; e < kNO; ++e)
          if (e < own - q) {
            A.b.r_next[t0 + q + e] = rt[e];
            acc[3] += rt[e] * rt[e];
          }
      }
    }
    __syncthreads();
  }
  double tot[4];
  if (grid_sum<4>(acc, A.b.partials, &st->ticket[0], tot) && t == 0) {
    st->scal[0] = tot[0];
    st->scal[1] = tot[1];
    st->scal[2] = tot[2];
    st->scal[3] = tot[3];
    if (!st->defer) fista_finalize_device(st, A.b.trace);
  }
}

template <int S, int ST, int MB>
void launch_iter_v(const IterArgs& a, cudaStream_t st) {
  using L = IterLayoutT<ST>;
  static int grid_cap = 0;
  if (!grid_cap) {
    L1B_CUDA(cudaFuncSetAttribute(fista_iter_kernel<S, ST, MB>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::total));
    int per_sm = 0;
    L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fista_iter_kernel<S, ST, MB>,
                                                          kThreads, L::total));
    grid_cap = std::max(1, per_sm) * sm_count();
  }
  constexpr uint64_t TT = kTI - 2 * ((S + 1) & ~1);
  const uint64_t tiles = (a.hi - a.lo + TT - 1) / TT;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)grid_cap));
  fista_iter_kernel<S, ST, MB><<<grid, kThreads, L::total, st>>>(a);
  L1B_LAUNCHED();
}

// pipeline depth 2 x 2 CTAs/SM (measured best of 3/4/5 x 1..4)
template <int S>
void launch_iter(const IterArgs& a, cudaStream_t st) {
  launch_iter_v<S, 2, 2>(a, st);
}

}  // namespace

bool fused_iter_supported(const OpView& op) {
  return fused_supported(op) && op.right.count >= 1 && op.right.count <= 4;
}

void fista_fused_iter(const OpView& op, const IterBufs& ib, uint64_t lo, uint64_t hi,
                      cudaStream_t st) {
  IterArgs a;
  a.n = op.n;
  a.lo = lo;
  a.hi = hi;
  a.halo = (op.right.count + 1) & ~1;
  a.right = op.right;
  a.sigma = op.sigma;
  a.b = ib;
  switch (op.right.count) {
    case 1: return launch_iter<1>(a, st);
    case 2: return launch_iter<2>(a, st);
    case 3: return launch_iter<3>(a, st);
    case 4: return launch_iter<4>(a, st);
    default: throw Unsupported("single-kernel FISTA: 1..4 stages");
  }
}

}  // namespace l1b
