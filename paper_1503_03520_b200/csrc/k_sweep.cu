// k_sweep.cu -- matrix-free products A = P1 Gtilde P2 Sigma G^T as Givens
// stage sweeps on device, in the reference's operation order
// (linops.cpp:422-490) and rounding (--fmad=false, host cos/sin), so the
// generator's b, e and the certificate are bit-identical to the reference.
// One thread per rotation pair; a stage is one launch (used by the generator
// and the PATH_SWEEP products; the fused multi-stage kernel is the next step,
// SURVEY.md 8(f)-1).
#include <cstring>

#include "common.cuh"
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kernels.hpp"

namespace l1b {

namespace {

__global__ void stage_kernel(double* __restrict__ v, uint64_t dim, int off, double c, double s,
                             bool transposed) {
  const uint64_t npairs = dim > (uint64_t)off ? (dim - off) / 2 : 0;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < npairs;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = off + 2 * t;
    double a = v[k], b = v[k + 1];
    rotate_pair(a, b, c, s, transposed);
    v[k] = a;
    v[k + 1] = b;
  }
}

// t[i] = j < n ? sigma[j] * v[j] : 0  with j = P2 map[i]   (linops.cpp:432-440)
__global__ void sigma_fwd(const double* __restrict__ v, double* __restrict__ t,
                          const double* __restrict__ sigma, const uint32_t* __restrict__ p2,
                          uint64_t n, uint64_t m) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = p2 ? p2[i] : i;
    t[i] = j < n ? sigma[j] * v[j] : 0.0;
  }
}

// v[j] = sigma[j] * t[i] for j = P2 map[i] < n              (linops.cpp:459-467)
__global__ void sigma_bwd(const double* __restrict__ t, double* __restrict__ v,
                          const double* __restrict__ sigma, const uint32_t* __restrict__ p2,
                          uint64_t n, uint64_t m) {
  const uint64_t lim = p2 ? m : n;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < lim;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = p2 ? p2[i] : i;
    if (j < n) v[j] = sigma[j] * t[i];
  }
}

__global__ void gather_kernel(const double* __restrict__ in, double* __restrict__ out,
                              const uint32_t* __restrict__ map, uint64_t m) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[map[i]];
}

__global__ void scatter_kernel(const double* __restrict__ in, double* __restrict__ out,
                               const uint32_t* __restrict__ map, uint64_t m) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[map[i]] = in[i];
}

__global__ void gram_scale(double* __restrict__ u, const double* __restrict__ sigma, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    u[i] /= sigma[i] * sigma[i];
}

__global__ void scatter_sparse_kernel(const uint32_t* sup, const double* val, uint64_t s,
                                      double* dense) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < s;
       k += (uint64_t)gridDim.x * blockDim.x)
    dense[sup[k]] = val[k];
}

__global__ void combine_kernel(double tau, double* __restrict__ e, double* __restrict__ b,
                               uint64_t m, double* partials, unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double ei = e[i] * tau;  // instance.cpp:70
    e[i] = ei;
    b[i] += ei;                    // instance.cpp:77
    acc[0] += ei * ei;             // instance.cpp:78
  }
  double tot[1];
  if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
}

__global__ void cert_kernel(const double* __restrict__ r, const double* __restrict__ xd,
                            double tau, uint64_t n, unsigned long long* out2) {
  double sup = 0.0, off = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double x = xd[i];
    if (x != 0.0) {
      const double sign = x > 0.0 ? 1.0 : -1.0;
      sup = fmax(sup, fabs(r[i] + tau * sign));
    } else {
      off = fmax(off, fmax(fabs(r[i]) - tau, 0.0));
    }
  }
  // non-negative doubles order like their bit patterns
  atomicMax(&out2[0], (unsigned long long)__double_as_longlong(sup));
  atomicMax(&out2[1], (unsigned long long)__double_as_longlong(off));
}

__global__ void sub_kernel(double* __restrict__ a, const double* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    a[i] -= b[i];
}

void run_stage(double* v, uint64_t dim, int off, double c, double s, bool tr, cudaStream_t st) {
  const uint64_t npairs = dim > (uint64_t)off ? (dim - off) / 2 : 0;
  if (!npairs) return;
  stage_kernel<<<grid_for(npairs), kThreads, 0, st>>>(v, dim, off, c, s, tr);
  L1B_LAUNCHED();
}

}  // namespace

void sweep_apply(const OpView& op, const double* x, double* y, cudaStream_t st) {
  double *v = nullptr, *t = nullptr;
  L1B_CUDA(cudaMallocAsync(&v, op.n * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&t, op.m * sizeof(double), st));
  L1B_CUDA(cudaMemcpyAsync(v, x, op.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  for (int s = 0; s < op.right.count; ++s)
    run_stage(v, op.n, op.right.offset[s], op.right.c[s], op.right.s[s], true, st);
  sigma_fwd<<<grid_for(op.m), kThreads, 0, st>>>(v, t, op.sigma, op.p2, op.n, op.m);
  L1B_LAUNCHED();
  for (int s = op.left.count - 1; s >= 0; --s)
    run_stage(t, op.m, op.left.offset[s], op.left.c[s], op.left.s[s], false, st);
  if (op.p1) {
    gather_kernel<<<grid_for(op.m), kThreads, 0, st>>>(t, y, op.p1, op.m);
    L1B_LAUNCHED();
  } else {
    L1B_CUDA(cudaMemcpyAsync(y, t, op.m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  L1B_CUDA(cudaFreeAsync(v, st));
  L1B_CUDA(cudaFreeAsync(t, st));
}

void sweep_apply_transpose(const OpView& op, const double* y, double* x, cudaStream_t st) {
  double *v = nullptr, *t = nullptr;
  L1B_CUDA(cudaMallocAsync(&v, op.n * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&t, op.m * sizeof(double), st));
  if (op.p1) {
    scatter_kernel<<<grid_for(op.m), kThreads, 0, st>>>(y, t, op.p1, op.m);
    L1B_LAUNCHED();
  } else {
    L1B_CUDA(cudaMemcpyAsync(t, y, op.m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  for (int s = 0; s < op.left.count; ++s)
    run_stage(t, op.m, op.left.offset[s], op.left.c[s], op.left.s[s], true, st);
  L1B_CUDA(cudaMemsetAsync(v, 0, op.n * sizeof(double), st));
  sigma_bwd<<<grid_for(op.p2 ? op.m : op.n), kThreads, 0, st>>>(t, v, op.sigma, op.p2, op.n, op.m);
  L1B_LAUNCHED();
  for (int s = op.right.count - 1; s >= 0; --s)
    run_stage(v, op.n, op.right.offset[s], op.right.c[s], op.right.s[s], false, st);
  L1B_CUDA(cudaMemcpyAsync(x, v, op.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  L1B_CUDA(cudaFreeAsync(v, st));
  L1B_CUDA(cudaFreeAsync(t, st));
}

namespace {
__global__ void abs_key_kernel(const double* __restrict__ x, uint64_t n, unsigned long long* key,
                               uint32_t* idx, unsigned long long* zeros) {
  unsigned long long z = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    // |x| ordered as its bit pattern (non-negative doubles); 0 and -0 -> 0
    const unsigned long long k = (unsigned long long)__double_as_longlong(x[i]) & 0x7fffffffffffffffull;
    key[i] = k;
    idx[i] = (uint32_t)i;
    z += k == 0;
  }
  if (z) atomicAdd(zeros, z);
}
__global__ void gather_vals(const double* __restrict__ x, const uint32_t* __restrict__ idx, uint64_t k,
                            double* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}
}  // namespace

void spectral_select(const OpView& op, const double* xhat_host, uint64_t n, uint64_t s1, uint64_t s2,
                     cudaStream_t st, std::vector<uint32_t>& sup, std::vector<double>& val) {
  double* x = nullptr;
  unsigned long long *key = nullptr, *key2 = nullptr, *zeros = nullptr;
  uint32_t *idx = nullptr, *idx2 = nullptr;
  L1B_CUDA(cudaMallocAsync(&x, n * 8, st));
  L1B_CUDA(cudaMallocAsync(&key, n * 8, st));
  L1B_CUDA(cudaMallocAsync(&key2, n * 8, st));
  L1B_CUDA(cudaMallocAsync(&idx, n * 4, st));
  L1B_CUDA(cudaMallocAsync(&idx2, n * 4, st));
  L1B_CUDA(cudaMallocAsync(&zeros, 8, st));
  L1B_CUDA(cudaMemsetAsync(zeros, 0, 8, st));
  L1B_CUDA(cudaMemcpyAsync(x, xhat_host, n * 8, cudaMemcpyHostToDevice, st));
  // op.apply_right_factor(xhat, false): stages last to first (linops.cpp:492-502)
  for (int s = op.right.count - 1; s >= 0; --s)
    run_stage(x, op.n, op.right.offset[s], op.right.c[s], op.right.s[s], false, st);
  abs_key_kernel<<<grid_for(n), kThreads, 0, st>>>(x, n, key, idx, zeros);
  L1B_LAUNCHED();
  // stable ascending |xhat| (std::stable_sort of solution.cpp:93-95): radix sort is stable
  size_t tmp_bytes = 0;
  L1B_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key2, idx, idx2, n, 0, 64, st));
  void* tmp = nullptr;
  L1B_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
  L1B_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key2, idx, idx2, n, 0, 64, st));
  L1B_LAUNCHED();
  unsigned long long z = 0;
  L1B_CUDA(cudaMemcpyAsync(&z, zeros, 8, cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  const uint64_t nz = n - z;  // the nonzeros, in sorted order: idx2[z, n)
  std::vector<std::pair<uint64_t, uint64_t>> ranges;  // [first, count) of idx2 kept
  if (nz <= s1 + s2)
    ranges.push_back({z, nz});
  else
    ranges = {{z, s1}, {n - s2, s2}};
  uint64_t kept = 0;
  for (auto& r : ranges) kept += r.second;
  uint32_t* kidx = nullptr;
  double* kval = nullptr;
  L1B_CUDA(cudaMallocAsync(&kidx, std::max<uint64_t>(kept, 1) * 4, st));
  L1B_CUDA(cudaMallocAsync(&kval, std::max<uint64_t>(kept, 1) * 8, st));
  uint64_t o = 0;
  for (auto& r : ranges) {
    if (r.second)
      L1B_CUDA(cudaMemcpyAsync(kidx + o, idx2 + r.first, r.second * 4, cudaMemcpyDeviceToDevice, st));
    o += r.second;
  }
  if (kept) {
    gather_vals<<<grid_for(kept), kThreads, 0, st>>>(x, kidx, kept, kval);
    L1B_LAUNCHED();
  }
  std::vector<uint32_t> hi(kept);
  std::vector<double> hv(kept);
  if (kept) {
    L1B_CUDA(cudaMemcpyAsync(hi.data(), kidx, kept * 4, cudaMemcpyDeviceToHost, st));
    L1B_CUDA(cudaMemcpyAsync(hv.data(), kval, kept * 8, cudaMemcpyDeviceToHost, st));
  }
  L1B_CUDA(cudaStreamSynchronize(st));
  for (void* q : {(void*)x, (void*)key, (void*)key2, (void*)idx, (void*)idx2, (void*)zeros, tmp,
                  (void*)kidx, (void*)kval})
    cudaFreeAsync(q, st);
  // ascending support (std::sort(keep), solution.cpp:104), values xhat[i]
  std::vector<uint64_t> order(kept);
  for (uint64_t k = 0; k < kept; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return hi[a] < hi[b]; });
  sup.resize(kept);
  val.resize(kept);
  for (uint64_t k = 0; k < kept; ++k) {
    sup[k] = hi[order[k]];
    val[k] = hv[order[k]];
  }
}

void sweep_gram_inverse(const OpView& op, const double* vin, double* out, cudaStream_t st) {
  if (out != vin)
    L1B_CUDA(cudaMemcpyAsync(out, vin, op.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  for (int s = 0; s < op.right.count; ++s)
    run_stage(out, op.n, op.right.offset[s], op.right.c[s], op.right.s[s], true, st);
  gram_scale<<<grid_for(op.n), kThreads, 0, st>>>(out, op.sigma, op.n);
  L1B_LAUNCHED();
  for (int s = op.right.count - 1; s >= 0; --s)
    run_stage(out, op.n, op.right.offset[s], op.right.c[s], op.right.s[s], false, st);
}

void scatter_sparse(const uint32_t* sup, const double* val, uint64_t s, double* dense, uint64_t n,
                    cudaStream_t st) {
  L1B_CUDA(cudaMemsetAsync(dense, 0, n * sizeof(double), st));
  if (!s) return;
  scatter_sparse_kernel<<<grid_for(s), kThreads, 0, st>>>(sup, val, s, dense);
  L1B_LAUNCHED();
}

void scatter_values(const uint32_t* sup, const double* val, uint64_t s, double* dense,
                    cudaStream_t st) {
  if (!s) return;
  scatter_sparse_kernel<<<grid_for(s), kThreads, 0, st>>>(sup, val, s, dense);
  L1B_LAUNCHED();
}

void generator_combine(double tau, double* e, double* b, uint64_t m, double* d_sum_sq,
                       cudaStream_t st) {
  const int grid = grid_for(m);
  double* partials = nullptr;
  unsigned int* ticket = nullptr;
  L1B_CUDA(cudaMallocAsync(&partials, grid * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&ticket, sizeof(unsigned int), st));
  L1B_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  combine_kernel<<<grid, kThreads, 0, st>>>(tau, e, b, m, partials, ticket, d_sum_sq);
  L1B_LAUNCHED();
  L1B_CUDA(cudaFreeAsync(partials, st));
  L1B_CUDA(cudaFreeAsync(ticket, st));
}

void certificate(const double* r, const double* xd, double tau, uint64_t n, double* d_out2,
                 cudaStream_t st) {
  L1B_CUDA(cudaMemsetAsync(d_out2, 0, 2 * sizeof(double), st));
  cert_kernel<<<grid_for(n), kThreads, 0, st>>>(r, xd, tau, n, (unsigned long long*)d_out2);
  L1B_LAUNCHED();
}

void vec_sub(double* a, const double* b, uint64_t n, cudaStream_t st) {
  if (!n) return;
  sub_kernel<<<grid_for(n), kThreads, 0, st>>>(a, b, n);
  L1B_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Windowed sweeps for row-block shards: v holds global entries [ws, we); a
// pair (k, k+1) of the global sweep is rotated iff both members lie in the
// window (and k + 1 < dim), so every entry whose dependency cone stays inside
// the window comes out bit-identical to the global sweep; the invalid margin
// grows by one entry per stage at window edges that are not global edges.
namespace {
__global__ void stage_window_kernel(double* __restrict__ v, uint64_t ws, uint64_t we, uint64_t dim,
                                    int off, double c, double s, bool transposed) {
  const uint64_t first = ws > (uint64_t)off ? ws + ((ws - off) & 1) : (uint64_t)off;
  const uint64_t last = min(we, dim);  // pairs need k + 1 < last
  if (last < first + 2) return;
  const uint64_t npairs = (last - first) / 2;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < npairs;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = first + 2 * t - ws;
    double a = v[k], b = v[k + 1];
    rotate_pair(a, b, c, s, transposed);
    v[k] = a;
    v[k + 1] = b;
  }
}

__global__ void window_scale(double* __restrict__ v, const double* __restrict__ sig, uint64_t len,
                             int mode, double tau) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (mode == 0) v[i] /= sig[i] * sig[i];      // (S^T S)^-1   (linops.cpp:485)
    else if (mode == 1) v[i] = sig[i] * v[i];    // Sigma        (linops.cpp:433)
    else v[i] = v[i] * tau;                      // e *= tau     (instance.cpp:70)
  }
}
}  // namespace

void window_stages(const StageTab& tab, bool forward, bool transposed, double* v, uint64_t ws,
                   uint64_t we, uint64_t dim, cudaStream_t st) {
  for (int q = 0; q < tab.count; ++q) {
    const int s = forward ? q : tab.count - 1 - q;
    stage_window_kernel<<<grid_for((we - ws) / 2 + 1), kThreads, 0, st>>>(
        v, ws, we, dim, tab.offset[s], tab.c[s], tab.s[s], transposed);
    L1B_LAUNCHED();
  }
}

namespace {
__global__ void scale_copy_kernel(const double* __restrict__ in, double a, double* __restrict__ out, uint64_t len) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i] * a;
}
}  // namespace

void scale_copy(const double* in, double a, double* out, uint64_t len, cudaStream_t st) {
  if (!len) return;
  scale_copy_kernel<<<grid_for(len), kThreads, 0, st>>>(in, a, out, len);
  L1B_LAUNCHED();
}

void window_scale_op(double* v, const double* sig, uint64_t len, int mode, double tau,
                     cudaStream_t st) {
  if (!len) return;
  window_scale<<<grid_for(len), kThreads, 0, st>>>(v, sig, len, mode, tau);
  L1B_LAUNCHED();
}

namespace {
__global__ void sum_sq_kernel(const double* __restrict__ v, uint64_t n, double* partials,
                              unsigned int* ticket, double* out) {
  double acc[1] = {0.0};
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc[0] += v[i] * v[i];
  double tot[1];
  if (grid_sum<1>(acc, partials, ticket, tot) && threadIdx.x == 0) *out = tot[0];
}

__global__ void minmax_kernel(const double* __restrict__ v, uint64_t n, unsigned long long* out) {
  // out[0] = min over bits of positive doubles, out[1] = max, out[2] = #(non-finite or <= 0)
  unsigned long long mn = ~0ull, mx = 0ull, bad = 0ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double x = v[i];
    if (!(x > 0.0) || !isfinite(x)) {
      ++bad;
      continue;
    }
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    mn = b < mn ? b : mn;
    mx = b > mx ? b : mx;
  }
  atomicMin(&out[0], mn);
  atomicMax(&out[1], mx);
  if (bad) atomicAdd(&out[2], bad);
}
}  // namespace

double device_sum_sq(const double* v, uint64_t n, cudaStream_t st) {
  const int grid = grid_for(n);
  double* scratch = nullptr;
  unsigned int* ticket = nullptr;
  L1B_CUDA(cudaMallocAsync(&scratch, (grid + 1) * sizeof(double), st));
  L1B_CUDA(cudaMallocAsync(&ticket, sizeof(unsigned int), st));
  L1B_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
  sum_sq_kernel<<<grid, kThreads, 0, st>>>(v, n, scratch + 1, ticket, scratch);
  L1B_LAUNCHED();
  double h = 0.0;
  L1B_CUDA(cudaMemcpyAsync(&h, scratch, sizeof(double), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaFreeAsync(scratch, st));
  L1B_CUDA(cudaFreeAsync(ticket, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  return h;
}

void device_min_finite(const double* v, uint64_t n, double* vmin, double* vmax, bool* finite,
                       cudaStream_t st) {
  unsigned long long* d = nullptr;
  L1B_CUDA(cudaMallocAsync(&d, 3 * sizeof(unsigned long long), st));
  const unsigned long long init[3] = {~0ull, 0ull, 0ull};
  L1B_CUDA(cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, st));
  minmax_kernel<<<grid_for(n), kThreads, 0, st>>>(v, n, d);
  L1B_LAUNCHED();
  unsigned long long h[3];
  L1B_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaFreeAsync(d, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  *finite = h[2] == 0;
  double a, b;
  std::memcpy(&a, &h[0], 8);
  std::memcpy(&b, &h[1], 8);
  *vmin = a;
  *vmax = b;
}

}  // namespace l1b
