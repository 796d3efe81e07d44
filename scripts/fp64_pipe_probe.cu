// FP64 pipe probe (measurement only): dependent-issue latency and throughput of
// DFMA on one SM as a function of warps per SM and independent chains per
// thread, with and without integer instructions issued beside them.  The tile
// kernel's schedule (k_iter_rc.cu, fista_tb_kernel) is sized from these numbers.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/_build/fp64_pipe_probe scripts/fp64_pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int MIX>
__global__ void probe(double* out, long long* cyc, int rounds, double b, double c, int ib) {
  double a[ILP];
  int z[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) a[k] = threadIdx.x * 1e-3 + k, z[k] = threadIdx.x + k;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      a[k] = __fma_rn(a[k], b, c);
#pragma unroll
      for (int m = 0; m < MIX; ++m) z[k] = (z[k] ^ ib) + (z[k] >> 3);  // 2-3 integer instructions
    }
  }
  const long long t1 = clock64();
  double s = 0.0;
  int zz = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += a[k], zz += z[k];
  if (s == 12345.678 || zz == 0x7fffffff) out[0] = s + zz;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ILP, int MIX>
void run(int warps, double* d, long long* c) {
  const int rounds = 4096;
  probe<ILP, MIX><<<1, 32 * warps>>>(d, c, rounds, 0.999999, 1e-9, 5);
  probe<ILP, MIX><<<1, 32 * warps>>>(d, c, rounds, 0.999999, 1e-9, 5);
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double per_round = (double)h / rounds;
  const double warps_per_smsp = warps < 4 ? 1.0 : warps / 4.0;
  printf("ILP %d mix %d warps %2d: %7.2f cycles per round, %6.2f cycles per DFMA warp-instr per SMSP\n", ILP, MIX,
         warps, per_round, per_round / (ILP * warps_per_smsp));
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 8);
  cudaMalloc(&c, 8);
  for (int w : {1, 4, 8, 16, 32}) {
    run<1, 0>(w, d, c);
    run<2, 0>(w, d, c);
    run<4, 0>(w, d, c);
    run<8, 0>(w, d, c);
  }
  for (int w : {4, 8, 16}) {
    run<4, 1>(w, d, c);
    run<8, 1>(w, d, c);
    run<4, 2>(w, d, c);
    run<8, 2>(w, d, c);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
