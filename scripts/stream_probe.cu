// Streaming ceiling probe: 4 reads + 1 write of n doubles (the fista_rc mix), 256-bit accesses.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double (&v)[4]) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
}
template <int UNR>
__global__ void k(const double* a, const double* b, const double* c, const double* d, double* o, long n) {
  long i = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 4;
  long stride = (long)gridDim.x * blockDim.x * 4;
  for (; i < n; i += stride * UNR) {
    double va[UNR][4], vb[UNR][4], vc[UNR][4], vd[UNR][4];
#pragma unroll
    for (int u = 0; u < UNR; ++u) if (i + u * stride < n) { ld4(a + i + u * stride, va[u]); ld4(b + i + u * stride, vb[u]); ld4(c + i + u * stride, vc[u]); ld4(d + i + u * stride, vd[u]); }
#pragma unroll
    for (int u = 0; u < UNR; ++u) if (i + u * stride < n) {
      double r[4];
      for (int e = 0; e < 4; ++e) r[e] = va[u][e] + vb[u][e] * vc[u][e] - vd[u][e];
      st4(o + i + u * stride, r);
    }
  }
}
template <int UNR>
void run(int blocks_per_sm, int threads, double* a, double* b, double* c, double* d, double* o, long n) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<UNR><<<sms * blocks_per_sm, threads>>>(a, b, c, d, o, n);
  cudaEventRecord(e0);
  const int R = 20;
  for (int r = 0; r < R; ++r) k<UNR><<<sms * blocks_per_sm, threads>>>(a, b, c, d, o, n);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double t = ms / R * 1e-3;
  printf("unroll %d blocks/sm %d threads %d: %.3f ms  %.1f GB/s\n", UNR, blocks_per_sm, threads, t * 1e3, 40.0 * n / t / 1e9);
}
int main() {
  long n = 1L << 27;
  double *a, *b, *c, *d, *o;
  cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&c, n * 8); cudaMalloc(&d, n * 8); cudaMalloc(&o, n * 8);
  cudaMemset(a, 0, n * 8); cudaMemset(b, 0, n * 8); cudaMemset(c, 0, n * 8); cudaMemset(d, 0, n * 8);
  for (int bps : {2, 4, 8}) { run<1>(bps, 256, a, b, c, d, o, n); run<2>(bps, 256, a, b, c, d, o, n); run<4>(bps, 256, a, b, c, d, o, n); }
  return 0;
}
