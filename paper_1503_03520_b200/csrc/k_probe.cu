// FP64 throughput probe (measurement only): the denominator of the tile
// kernel's roofline (bench.py), measured on the GPU it runs on instead of the
// nominal 148 SMs x 64 FP64 lanes x 2 flops x clock.
#include "common.cuh"
#include "kernels.hpp"

namespace l1b {
namespace {

constexpr int kProbeChains = 8, kProbeThreads = 256;

// kProbeChains independent fma chains per thread, `rounds` fmas each
__global__ void __launch_bounds__(kProbeThreads) fp64_probe_kernel(double* out, int rounds, double b, double c) {
  double a[kProbeChains];
#pragma unroll
  for (int k = 0; k < kProbeChains; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int r = 0; r < rounds; ++r) {
#pragma unroll
    for (int k = 0; k < kProbeChains; ++k) a[k] = __fma_rn(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kProbeChains; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keeps the chains live
}

}  // namespace

double fp64_peak_tflops(int device) {
  L1B_CUDA(cudaSetDevice(device));
  double* d = nullptr;
  L1B_CUDA(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1;
  L1B_CUDA(cudaEventCreate(&e0));
  L1B_CUDA(cudaEventCreate(&e1));
  int per_sm = 0;
  L1B_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fp64_probe_kernel, kProbeThreads, 0));
  const int grid = std::max(1, per_sm) * sm_count();
  const int rounds = 1 << 14;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    L1B_CUDA(cudaEventRecord(e0));
    fp64_probe_kernel<<<grid, kProbeThreads>>>(d, rounds, 0.999999, 1e-9);
    L1B_LAUNCHED();
    L1B_CUDA(cudaEventRecord(e1));
    L1B_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    L1B_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * kProbeChains * (double)rounds * grid * kProbeThreads;
    if (rep) best = std::max(best, flops / (ms * 1e-3) / 1e12);  // (rep 0 warms up)
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return best;
}

}  // namespace l1b
