// spmv.cuh -- the fp64 CSR SpMV skeleton shared by every solver kernel
// (k_spmv.cu FISTA, k_ncg.cu Newton-CG/PCG, k_pcdm.cu refresh): a template
// over the pointer width and an epilogue functor, instantiated per TU.
#pragma once

#include <algorithm>

#include "common.cuh"
#include "kernels.hpp"

namespace l1b {
namespace spmv_detail {

// Epilogue functors provide
//   skip() / start() / finish()       (device; finish does the reductions),
//   kVec, vec(v)                      the kVec n- or m-vectors the epilogue of
//                                     line i reads at index i (staged in smem),
//   line(i, value, pv)                pv[v] = vec(v)[i].

// ---------------------------------------------------------------------------
// Fallback skeleton ("row tile per warp") for operators whose 256-line tiles
// exceed the TMA stage capacity: a warp owns 32 consecutive lines, streams
// their contiguous nonzero range with coalesced loads, parks the products in
// shared memory and lane l sums line r0+l in ascending index order.
constexpr int kCapNnz = 256;
constexpr int kUnroll = 8;

__device__ __forceinline__ int pad(int off) { return off + (off >> 4); }

template <class Epi>
__device__ __forceinline__ void load_vecs(const Epi& epi, uint64_t line, double* pv) {
#pragma unroll
  for (int v = 0; v < Epi::kVec; ++v) pv[v] = epi.vec(v)[line];
}

template <typename PtrT, class Epi>
__global__ void __launch_bounds__(kThreads) spmv_warp_kernel(const PtrT* __restrict__ ptr,
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
    double pv[Epi::kVec > 0 ? Epi::kVec : 1];
    if (live) load_vecs(epi, line, pv);
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
    if (live) epi.line(line, sum, pv);
  }
  epi.finish();
}

// ---------------------------------------------------------------------------
// Main skeleton: TMA bulk-copy pipeline.  Persistent CTAs walk 256-line
// tiles; one elected thread streams each tile's row pointers, values,
// indices and epilogue vectors into a 3-stage shared-memory ring with
// cp.async.bulk (UBLKCP, evict-first for the matrix streams) completing on an
// mbarrier, two tiles ahead of the consumers.  The 256 threads then gather x
// for the tile's nonzeros (8 independent gathers each, L1/L2 hits on the
// band), park the products (padded against bank conflicts), and thread t sums
// line r0+t in ascending index order and runs the epilogue on smem-staged
// vectors.  Bytes in flight per SM ~ 2 CTAs x 2 stages x 30 KB, far above the
// ~35 KB Little's law needs at HBM bandwidth.
constexpr int kTileLines = 256;   // == kThreads
constexpr int kTileNnz = 2048;    // nonzero capacity of one tile
#ifndef L1B_SPMV_STAGES
#define L1B_SPMV_STAGES 3
#endif
#ifndef L1B_SPMV_VEC
#define L1B_SPMV_VEC 1  // stage the epilogue vectors with TMA too
#endif
#ifndef L1B_SPMV_MINB
#define L1B_SPMV_MINB 2  // CTAs per SM the register allocation targets
#endif
constexpr int kStages = L1B_SPMV_STAGES;
constexpr int kVecTma = L1B_SPMV_VEC;

// x window staged with each tile when the tile's index range fits (banded
// operators: 256 + 2 x bandwidth entries): the gathers then hit shared memory
constexpr int kTileX = 320;

template <typename PtrT, int NV>
struct TmaLayout {
  static constexpr size_t r16(size_t b) { return (b + 15) / 16 * 16; }
  static constexpr size_t vals_bytes = (kTileNnz + 2) * 8;
  static constexpr size_t idx_bytes = (kTileNnz + 8) * 4;
  static constexpr size_t ptr_bytes = r16((kTileLines + 1 + 16 / sizeof(PtrT)) * sizeof(PtrT));
  static constexpr size_t vec_bytes = kVecTma ? kTileLines * 8 : 0;
  static constexpr size_t x_bytes = kTileX * 8;
  static constexpr size_t stage_bytes = vals_bytes + idx_bytes + ptr_bytes + NV * vec_bytes + x_bytes;
  static constexpr size_t prod_off = kStages * stage_bytes;
  static constexpr size_t prod_bytes = r16((size_t)(kThreads / 32) * (256 + 256 / 16 + 2) * 8);
  static constexpr size_t bars_off = prod_off + prod_bytes;
  static constexpr size_t total = bars_off + 2 * kStages * 8;  // full + empty barriers
};

// Warp-specialised: warps 0-7 consume, warp 8 (one lane) produces.  Consumer
// warp w owns lines [32w, 32w + 32) of every tile, and their nonzeros are one
// contiguous range, so the warp computes exactly the products its own lines
// sum: a __syncwarp separates the two phases, no block barrier per tile.  A
// slot is handed back to the producer through its "empty" mbarrier (one
// arrival per consumer warp); "full" completes on the TMA bytes.
constexpr int kSpmvThreads = kThreads + 32;
constexpr int kWarpProd = 256;                              // products per warp chunk
constexpr int kWarpProdPad = kWarpProd + kWarpProd / 16 + 2;  // + the bank-conflict padding

template <typename PtrT, class Epi>
__global__ void __launch_bounds__(kSpmvThreads, L1B_SPMV_MINB) spmv_tma_kernel(const PtrT* __restrict__ ptr,
                                                               const uint32_t* __restrict__ idx,
                                                               const double* __restrict__ val,
                                                               const double* __restrict__ x,
                                                               uint64_t nlines, Epi epi,
                                                               int vec_tma, const uint32_t* __restrict__ tile_rng,
                                                               uint64_t x_len) {
  if (epi.skip()) return;
  epi.start();
  using L = TmaLayout<PtrT, Epi::kVec>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t x_lo[kStages];  // first staged x index of each slot (~0: not staged)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::bars_off);
  uint64_t* empty = full + kStages;
  double* prod = reinterpret_cast<double*>(smem + L::prod_off);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  constexpr int kConsumers = kThreads / 32;
  const uint64_t ntiles = (nlines + kTileLines - 1) / kTileLines;
  const uint64_t mine = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr int E = 16 / sizeof(PtrT);

  if (t == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumers) {
    // ---- producer: stream tile k of this CTA into slot k % kStages ---------
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      PtrT b0 = 0, b1 = 0;  // row-pointer bounds of the next tile (prefetched)
      uint32_t g0 = 1, g1 = 0;  // its index range (tile_rng)
      auto prefetch = [&](uint64_t k) {
        const uint64_t r0 = (blockIdx.x + k * gridDim.x) * (uint64_t)kTileLines;
        const uint64_t nl = min((uint64_t)kTileLines, nlines - r0);
        b0 = __ldg(ptr + r0);
        b1 = __ldg(ptr + r0 + nl);
        if (tile_rng) {
          const uint64_t tix = blockIdx.x + k * gridDim.x;
          g0 = __ldg(tile_rng + 2 * tix);
          g1 = __ldg(tile_rng + 2 * tix + 1);
        }
      };
      if (mine) prefetch(0);
      for (uint64_t k = 0; k < mine; ++k) {
        const int slot = (int)(k % kStages);
        if (k >= (uint64_t)kStages) {
          mbar_wait(&empty[slot], (uint32_t)(((k / kStages) - 1) & 1));  // tile k - kStages consumed
          fence_proxy_async();  // the consumers' generic reads before the bulk writes
        }
        const PtrT p0 = b0, p1 = b1;
        const uint32_t lo_i = g0, hi_i = g1;
        const uint64_t r0 = (blockIdx.x + k * gridDim.x) * (uint64_t)kTileLines;
        const uint64_t nl = min((uint64_t)kTileLines, nlines - r0);
        if (k + 1 < mine) prefetch(k + 1);
        unsigned char* base = smem + slot * L::stage_bytes;
        double* s_val = reinterpret_cast<double*>(base);
        uint32_t* s_idx = reinterpret_cast<uint32_t*>(base + L::vals_bytes);
        PtrT* s_ptr = reinterpret_cast<PtrT*>(base + L::vals_bytes + L::idx_bytes);
        double* s_vec = reinterpret_cast<double*>(base + L::vals_bytes + L::idx_bytes + L::ptr_bytes);
        const uint32_t ptr_b = (uint32_t)(((nl + 1 + E - 1) / E) * 16);
        const PtrT va = p0 & ~(PtrT)1, vb = (p1 + 1) & ~(PtrT)1;
        const PtrT ia = p0 & ~(PtrT)3, ib = (p1 + 3) & ~(PtrT)3;
        const uint32_t val_b = (uint32_t)(vb - va) * 8u, idx_b = (uint32_t)(ib - ia) * 4u;
        const uint32_t nv = vec_tma ? (uint32_t)(nl & ~1ull) : 0u;
        uint32_t x_b = 0;
        uint64_t xl = ~0ull;
        if (tile_rng) {  // x[lo .. hi] for this tile's gathers, when it fits and stays inside x
          const uint64_t lo = lo_i & ~1ull, hi = hi_i;
          const uint64_t cnt = (hi - lo + 2) & ~1ull;
          if (hi >= lo && cnt <= (uint64_t)kTileX && lo + cnt <= x_len) {
            xl = lo;
            x_b = (uint32_t)(cnt * 8);
          }
        }
        x_lo[slot] = xl;
        mbar_arrive_expect_tx(&full[slot], ptr_b + val_b + idx_b + Epi::kVec * nv * 8u + x_b);
        bulk_g2s(s_ptr, ptr + r0, ptr_b, &full[slot]);
        if (val_b) bulk_g2s_evict_first(s_val, val + va, val_b, &full[slot], pol);
        if (idx_b) bulk_g2s_evict_first(s_idx, idx + ia, idx_b, &full[slot], pol);
        if (nv) {
#pragma unroll
          for (int v = 0; v < Epi::kVec; ++v)
            bulk_g2s(s_vec + v * kTileLines, epi.vec(v) + r0, nv * 8u, &full[slot]);
        }
        if (x_b) bulk_g2s(s_vec + Epi::kVec * (L::vec_bytes / 8), x + xl, x_b, &full[slot]);
      }
    }
  } else {
    // ---- consumers ---------------------------------------------------------
    const int lw0 = warp * 32;
    for (uint64_t k = 0; k < mine; ++k) {
      const int slot = (int)(k % kStages);
      const uint64_t r0 = (blockIdx.x + k * gridDim.x) * (uint64_t)kTileLines;
      const int nl = (int)min((uint64_t)kTileLines, nlines - r0);
      unsigned char* base = smem + slot * L::stage_bytes;
      const double* s_val = reinterpret_cast<const double*>(base);
      const uint32_t* s_idx = reinterpret_cast<const uint32_t*>(base + L::vals_bytes);
      const PtrT* s_ptr = reinterpret_cast<const PtrT*>(base + L::vals_bytes + L::idx_bytes);
      const double* s_vec =
          reinterpret_cast<const double*>(base + L::vals_bytes + L::idx_bytes + L::ptr_bytes);
      mbar_wait(&full[slot], (uint32_t)((k / kStages) & 1));
      if (lw0 < nl) {
        const PtrT p0 = s_ptr[0];
        const PtrT va = p0 & ~(PtrT)1, ia = p0 & ~(PtrT)3;
        (void)p0;
        const uint64_t xl = x_lo[slot];
        const double* s_x = s_vec + Epi::kVec * (L::vec_bytes / 8) - (xl == ~0ull ? 0 : xl);
        const PtrT q_lo = s_ptr[lw0], q_hi = s_ptr[min(lw0 + 32, nl)];
        const int line = lw0 + lane;
        const PtrT la = line < nl ? s_ptr[line] : q_hi, le = line < nl ? s_ptr[line + 1] : q_hi;
        double* wp = prod + warp * kWarpProdPad;  // this warp's product region (no other warp touches it)
        double sum = 0.0;
        // the warp's products in chunks of kWarpProd: gathers, then every lane
        // adds its line's share in ascending index order (the same order as one
        // pass over the whole line)
        for (PtrT c0 = q_lo; c0 < q_hi; c0 += kWarpProd) {
          const PtrT c1 = min((PtrT)(c0 + kWarpProd), q_hi);
          for (PtrT q0 = c0 + lane; q0 < c1; q0 += 32 * kUnroll) {
            double vv[kUnroll];
            uint32_t ii[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const PtrT q = q0 + 32 * u;
              if (q < c1) {
                vv[u] = s_val[q - va];
                ii[u] = s_idx[q - ia];
              }
            }
            if (xl != ~0ull) {
#pragma unroll
              for (int u = 0; u < kUnroll; ++u) {
                const PtrT q = q0 + 32 * u;
                if (q < c1) wp[pad((int)(q - c0))] = vv[u] * s_x[ii[u]];
              }
            } else {
#pragma unroll
              for (int u = 0; u < kUnroll; ++u) {
                const PtrT q = q0 + 32 * u;
                if (q < c1) wp[pad((int)(q - c0))] = vv[u] * __ldg(x + ii[u]);
              }
            }
          }
          __syncwarp();
          const PtrT a = max(la, c0), e = min(le, c1);
          for (PtrT q = a; q < e; ++q) sum += wp[pad((int)(q - c0))];
          __syncwarp();  // (the next chunk reuses the region)
        }
        if (line < nl) {
          double pv[Epi::kVec > 0 ? Epi::kVec : 1];
          if (vec_tma && line < (nl & ~1)) {
#pragma unroll
            for (int v = 0; v < Epi::kVec; ++v) pv[v] = s_vec[v * kTileLines + line];
          } else {
            load_vecs(epi, r0 + line, pv);
          }
          epi.line(r0 + line, sum, pv);
        }
      }
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }
  epi.finish();
}

// ---------------------------------------------------------------------------
// dispatch over the pointer width

template <class Epi, typename PtrT>
inline void launch_p(const Csr& M, const double* x, const Epi& epi, cudaStream_t st) {
  using L = TmaLayout<PtrT, Epi::kVec>;
  if (M.tile_nnz_max <= (uint64_t)kTileNnz) {
    static int grid_cap = 0;
    if (!grid_cap) {
      L1B_CUDA(cudaFuncSetAttribute(spmv_tma_kernel<PtrT, Epi>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::total));
      int per_sm = 0;
      L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_tma_kernel<PtrT, Epi>,
                                                            kSpmvThreads, L::total));
      grid_cap = std::max(1, per_sm) * sm_count();
    }
    int vec_tma = kVecTma;
    for (int v = 0; v < Epi::kVec; ++v)
      if (reinterpret_cast<uintptr_t>(epi.vec(v)) % 16) vec_tma = 0;
    // x staging needs 16-byte aligned x (odd windows gather from global memory)
    const uint32_t* rng = reinterpret_cast<uintptr_t>(x) % 16 ? nullptr : M.tile_rng;
    const uint64_t tiles = (M.lines + kTileLines - 1) / kTileLines;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)grid_cap));
    spmv_tma_kernel<PtrT, Epi><<<grid, kSpmvThreads, L::total, st>>>(
        (const PtrT*)M.ptr, M.idx, M.val, x, M.lines, epi, vec_tma, rng, M.x_len);
    L1B_LAUNCHED();
    return;
  }
  static int grid_cap = 0;
  if (!grid_cap) {
    int per_sm = 0;
    L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_warp_kernel<PtrT, Epi>,
                                                          kThreads, 0));
    grid_cap = std::max(1, per_sm) * sm_count();
  }
  const uint64_t tiles = (M.lines + 31) / 32;
  const uint64_t blocks = (tiles + (kThreads / 32) - 1) / (kThreads / 32);
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(blocks, (uint64_t)grid_cap));
  spmv_warp_kernel<PtrT, Epi><<<grid, kThreads, 0, st>>>((const PtrT*)M.ptr, M.idx, M.val, x,
                                                         M.lines, epi);
  L1B_LAUNCHED();
}

template <class Epi>
inline void launch(const Csr& M, const double* x, const Epi& epi, cudaStream_t st) {
  if (M.ptr32)
    launch_p<Epi, uint32_t>(M, x, epi, st);
  else
    launch_p<Epi, uint64_t>(M, x, epi, st);
}

}  // namespace spmv_detail

using spmv_detail::launch;

}  // namespace l1b
