// common.cuh -- shared types, error handling and device helpers of libl1b.
//
// Layout in HBM:
//   * A rows  : CSR over the active rows [0, m_act): ptr (u32 when nnz < 2^32,
//               else u64), col u32, val f64 -- exactly OperatorSpec::row()'s
//               entries (linops.cpp:597-619), ascending, exact zeros dropped.
//   * A cols  : CSC (= CSR of A^T) over n columns, same widths, exactly
//               OperatorSpec::column() (linops.cpp:566-595).
//   * vectors : dense f64, n (x, y, ...) and m (b, residuals).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace l1b {

// ---------------------------------------------------------------------------
// errors: each maps to one l1b_status (include/l1b.h)
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct LogicError : std::logic_error {
  using std::logic_error::logic_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OutOfMemory : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Unsupported : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// NVTX range around a C-ABI entry point (header-only NVTX 3: a no-op unless a
// tool such as nsys / ncu --nvtx attaches)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define L1B_CUDA(call) ::l1b::cuda_check((call), #call, __FILE__, __LINE__)
#define L1B_LAUNCHED() ::l1b::note_launch()

extern std::atomic<uint64_t> g_launch_count;
inline void note_launch() {
  g_launch_count.fetch_add(1, std::memory_order_relaxed);
  L1B_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// operator description as kernels see it
constexpr int kMaxStages = 32;

struct StageTab {
  int count = 0;
  int offset[kMaxStages];
  double c[kMaxStages];  // cos(theta) from the host libm (linops.cpp:84-85)
  double s[kMaxStages];
  // the scaled form of the contracted arithmetic: a stage is
  // cos(theta) * [[1, -tan], [tan, 1]] on every pair, so G = (prod cos) * M
  // with M two independent fmas per pair; entries a stage leaves unpaired
  // take 1 / cos(theta) instead
  double tn[kMaxStages];  // tan(theta)
  double ic[kMaxStages];  // 1 / cos(theta)
  double cprod = 1.0;     // prod cos(theta)
  int scaled_ok = 0;      // every |cos(theta)| >= 1/4: the scaled form is well conditioned
};

struct OpView {
  uint64_t m = 0, n = 0;
  const uint32_t* p1 = nullptr;      // map, null = identity
  const uint32_t* p2 = nullptr;
  const uint32_t* p1_inv = nullptr;
  const uint32_t* p2_inv = nullptr;
  const double* sigma = nullptr;
  StageTab right, left;
};

// ---------------------------------------------------------------------------
// launch geometry
constexpr int kThreads = 256;
int sm_count();
int grid_for(uint64_t work_items, int threads = kThreads, int max_blocks_per_sm = 8);
void keep_pool(int device);  // default mem pool of `device`: freed memory stays cached

// ---------------------------------------------------------------------------
// device helpers
#ifdef __CUDACC__
// rotate_pair (linops.cpp:20-30).  The library is compiled with --fmad=false,
// so every product and sum rounds separately, as in the reference's x86-64
// build: results are bit-identical for identical inputs.
__device__ __forceinline__ void rotate_pair(double& vi, double& vj, double c, double s,
                                            bool transposed) {
  const double a = vi, b = vj;
  if (transposed) {
    vi = c * a + s * b;
    vj = -s * a + c * b;
  } else {
    vi = c * a - s * b;
    vj = s * a + c * b;
  }
}

// The contracted arithmetic mode (l1b_solver_cfg.arith = L1B_ARITH_FMA): every
// a*b + c of the hot loop as one fused multiply-add -- one rounding instead of
// two, so the results are no longer the reference's bits but at least as
// accurate (parity: <= 1e-12 relative, tests/test_gpu_rc.py, test_gpu_configs.py) --
// and every rotation in the scaled form below.  rot<false> is the exact
// (bit-identical) rotate_pair; rot<true> exists for the call sites' dead
// branches only (they take rot_scaled).
template <bool F>
__device__ __forceinline__ void rot(double& vi, double& vj, double c, double s, bool transposed) {
  rotate_pair(vi, vj, c, s, transposed);
}
// The scaled form of a rotation (contracted arithmetic):
// [[1, -tn], [tn, 1]] (transposed: tn -> -tn), two independent fmas; the
// factor cos(theta) is carried by the caller (StageTab::cprod).
__device__ __forceinline__ void rot_scaled(double& vi, double& vj, double tn, bool transposed) {
  const double a = vi, b = vj;
  if (transposed) {
    vi = __fma_rn(tn, b, a);
    vj = __fma_rn(-tn, a, b);
  } else {
    vi = __fma_rn(-tn, b, a);
    vj = __fma_rn(tn, a, b);
  }
}
// a * b - c
template <bool F>
__device__ __forceinline__ double mul_sub(double a, double b, double c) {
  return F ? __fma_rn(a, b, -c) : a * b - c;
}

// soft_threshold (solvers.cpp:153-157)
__device__ __forceinline__ double soft_threshold(double v, double t) {
  if (v > t) return v - t;
  if (v < -t) return v + t;
  return 0.0;
}

// soft_threshold on the bit patterns: |z| > t as an unsigned compare of the
// magnitude bits (t >= 0, z not NaN), then z - copysign(t, z) outside the band
// and z - z = +0 inside it -- the values of soft_threshold() bit for bit, with
// one FP64 instruction instead of two sums and the compares.  nz = (result != 0).
__device__ __forceinline__ double soft_threshold_bits(double z, double t, bool& nz) {
  // (on the 32-bit halves: a 64-bit mask of the sign would be turned back
  // into an FP64 |z|)
  const unsigned zh = (unsigned)__double2hiint(z), zl = (unsigned)__double2loint(z);
  const unsigned th = (unsigned)__double2hiint(t), tl = (unsigned)__double2loint(t);
  const unsigned ah = zh & 0x7fffffffu;
  nz = (((unsigned long long)ah << 32) | zl) > (((unsigned long long)th << 32) | tl);
  const unsigned sh = nz ? (th | (zh & 0x80000000u)) : zh, sl = nz ? tl : zl;
  return z - __hiloint2double((int)sh, (int)sl);
}
// bits of a that differ from b's, or-ed into acc (acc != 0 <=> some a != b so far)
__device__ __forceinline__ unsigned differing_bits(unsigned acc, double a, double b) {
  return acc | ((unsigned)__double2hiint(a) ^ (unsigned)__double2hiint(b)) |
         ((unsigned)__double2loint(a) ^ (unsigned)__double2loint(b));
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- TMA bulk copies + mbarriers (PTX; sm_90+ / sm_100a) -------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// orders earlier generic-proxy smem accesses before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D bulk copy global -> shared (UBLKCP), completion counted on `bar`.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, uint32_t bytes,
                                                     uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Block-wide sum of NS doubles held per thread (result valid in thread 0).
template <int NS>
__device__ __forceinline__ void block_sum(double (&v)[NS]) {
  __shared__ double red[NS][32];  // up to 1024 threads
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NS; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) red[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      v[k] = lane < (int)(blockDim.x >> 5) ? red[k][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
    }
  }
  __syncthreads();
}

// Deterministic grid reduction: every block stores its NS partial sums, the
// last block to arrive (ticket) folds all partials in a fixed order and
// returns true in all of its threads with the totals in `tot` (thread 0 of
// that block holds them; they are also broadcast through shared memory).
template <int NS>
__device__ __forceinline__ bool grid_sum(double (&v)[NS], double* partials, unsigned int* ticket,
                                         double (&tot)[NS]) {
  block_sum<NS>(v);
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) partials[(size_t)blockIdx.x * NS + k] = v[k];
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = 0.0;
  for (unsigned int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NS; ++k) acc[k] += __ldcg(&partials[(size_t)b * NS + k]);
  }
  block_sum<NS>(acc);
  __shared__ double bc[NS];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) bc[k] = acc[k];
    *ticket = 0u;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NS; ++k) tot[k] = bc[k];
  return true;
}
#endif

}  // namespace l1b
