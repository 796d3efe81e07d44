// k_solution.cu -- the generator's sequential draw loops on the device:
// uniform_sparse_solution (solution.cpp:47-75) and Permutation::realize
// (linops.cpp:224-239), both reproduced bit for bit from their draws alone.
//
// Floyd's sampling draws t_j = uniform_index(rng, j + 1) for j = n - s .. n - 1
// and inserts t_j, or j when t_j is already chosen; then the s values
// uniform_in(rng, -gamma, gamma) (rejecting 0) in ascending support order.
// The draws are one stretch of the seeded std::mt19937_64 stream (k_rng.cu's
// jump-started chunks); what is "already chosen" follows from the draws alone:
// step k (j = n - s + k) inserts j iff
//   (A) an earlier step drew the same t_j (whichever of t_i or j_i that step
//       inserted, t_j is in the set by then), or
//   (B) t_j lies in [n - s, j) -- it is the index of an earlier step -- and
//       that step inserted its own index, i.e. (A or B) held there.
// (A) is "not the first occurrence" in a stable sort of (t, k); (B) chains to
// strictly smaller steps and is resolved by a few relaxation rounds.  Result:
// the same set, sorted, and the same values as the reference's sequential loop.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <vector>

#include "kernels.hpp"

namespace l1b {
namespace {

__global__ void floyd_draws_kernel(const uint64_t* __restrict__ raw, uint64_t n, uint64_t s,
                                   uint64_t* __restrict__ t, uint32_t* __restrict__ step, int* flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < s; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t m = n - s + k + 1;  // uniform_index(rng, j + 1)
    const uint64_t lim = UINT64_MAX - UINT64_MAX % m;
    const uint64_t x = raw[k];
    if (x >= lim) atomicOr(flag, 1);  // the reference redraws: the stream shifts (host fallback)
    t[k] = x % m;
    step[k] = (uint32_t)k;
  }
}

// dup[k] = 1 unless step k is the first (in step order) to draw its value
__global__ void floyd_first_kernel(const uint64_t* __restrict__ st, const uint32_t* __restrict__ sk, uint64_t s,
                                   uint8_t* __restrict__ dup) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < s; i += (uint64_t)gridDim.x * blockDim.x)
    dup[sk[i]] = (i > 0 && st[i - 1] == st[i]) ? 1 : 0;
}

// one relaxation round of (B); sets *changed when a step turned
__global__ void floyd_chain_kernel(const uint64_t* __restrict__ t, uint64_t n, uint64_t s, uint8_t* dup,
                                   int* changed) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < s; k += (uint64_t)gridDim.x * blockDim.x) {
    if (dup[k]) continue;
    const uint64_t tk = t[k], lo = n - s, j = lo + k;
    if (tk >= lo && tk < j && *(volatile uint8_t*)&dup[tk - lo]) {
      dup[k] = 1;
      *changed = 1;
    }
  }
}

__global__ void floyd_elements_kernel(const uint64_t* __restrict__ t, const uint8_t* __restrict__ dup, uint64_t n,
                                      uint64_t s, uint64_t* __restrict__ e) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < s; k += (uint64_t)gridDim.x * blockDim.x)
    e[k] = dup[k] ? n - s + k : t[k];
}

// values uniform_in(rng, -gamma, gamma) (rng.hpp:44-47) of draws s .. 2s - 1;
// a zero (the reference redraws) shifts the stream: flagged
__global__ void floyd_values_kernel(const uint64_t* __restrict__ raw, uint64_t s, double gamma,
                                    double* __restrict__ val, int* flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < s; k += (uint64_t)gridDim.x * blockDim.x) {
    const double lo = -gamma, hi = gamma;
    const double v = lo + (hi - lo) * ((double)(raw[s + k] >> 11) * 0x1.0p-53);
    if (v == 0.0) atomicOr(flag, 2);
    val[k] = v;
  }
}

// ---- Fisher-Yates (linops.cpp:224-234): for p = m-1 .. 1: swap(map[p],
// map[j_p]), j_p = uniform_index(rng, p + 1).  Position p is final after step p
// (later steps touch smaller positions), so
//   map[p] = a[j_p] just before step p
//          = B(s) for s = the next larger step targeting j_p, else j_p itself
//            (B(p) when j_p = p)
// where B(x) = the value at position x just before step x = B(prev(x)) for
// prev(x) = the smallest step > x targeting x, else x: pointer chains to
// larger steps (pointer jumping).  map[0] = B(first step targeting 0), else 0.
__global__ void iota_kernel(uint32_t* a, uint64_t m) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < m; x += (uint64_t)gridDim.x * blockDim.x)
    a[x] = (uint32_t)x;
}
void iota_u32(uint32_t* a, uint64_t m, cudaStream_t st) {
  iota_kernel<<<grid_for(m), kThreads, 0, st>>>(a, m);
  L1B_LAUNCHED();
}

__global__ void fy_draws_kernel(const uint64_t* __restrict__ raw, uint64_t m, uint32_t* __restrict__ tgt,
                                uint32_t* __restrict__ stp, int* flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k + 1 < m; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = m - 1 - k, mod = p + 1;  // draw k belongs to step p
    const uint64_t lim = UINT64_MAX - UINT64_MAX % mod;
    const uint64_t x = raw[k];
    if (x >= lim) atomicOr(flag, 1);
    tgt[p - 1] = (uint32_t)(x % mod);  // stored in ascending step order
    stp[p - 1] = (uint32_t)p;
  }
}

// sorted by target (stable: steps ascending within a target): prev(x) and the
// successor step of each step within its target group
__global__ void fy_links_kernel(const uint32_t* __restrict__ skey, const uint32_t* __restrict__ sstp, uint64_t cnt,
                                uint32_t* __restrict__ prev, uint32_t* __restrict__ succ) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t q = skey[i], p = sstp[i];
    const bool next_same = i + 1 < cnt && skey[i + 1] == q;
    succ[p] = next_same ? sstp[i + 1] : 0xffffffffu;
    if (i == 0 || skey[i - 1] != q) {  // first step targeting q
      if (p > q) prev[q] = p;
      else if (next_same) prev[q] = sstp[i + 1];  // (p == q: step q itself; the next one is > q)
    }
  }
}

__global__ void fy_jump_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t m, int* changed) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < m; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = in[x], b = in[a];
    out[x] = b;
    if (b != a) *changed = 1;
  }
}

__global__ void fy_final_kernel(const uint32_t* __restrict__ tgt, const uint32_t* __restrict__ succ,
                                const uint32_t* __restrict__ root, const uint32_t* __restrict__ prev0, uint64_t m,
                                uint32_t* __restrict__ map) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m; p += (uint64_t)gridDim.x * blockDim.x) {
    if (p == 0) {
      const uint32_t f = *prev0;  // first step targeting 0 (0xffffffff: none)
      map[0] = f == 0xffffffffu ? 0u : root[f];
      continue;
    }
    const uint32_t q = tgt[p - 1];
    if (q == p) {
      map[p] = root[p];
    } else {
      const uint32_t s = succ[p];
      map[p] = s == 0xffffffffu ? q : root[s];
    }
  }
}

}  // namespace

bool device_permutation(uint64_t m, uint64_t seed, uint32_t* host_map, cudaStream_t st) {
  if (m == 0) return true;
  if (m > (1ull << 32)) return false;
  if (m == 1) {
    host_map[0] = 0;
    return true;
  }
  std::vector<void*> bufs;
  auto alloc = [&](auto** p, size_t bytes) {
    L1B_CUDA(cudaMallocAsync((void**)p, std::max<size_t>(bytes, 16), st));
    bufs.push_back((void*)*p);
  };
  bool ok = false;
  int* h = nullptr;
  try {
    const uint64_t cnt = m - 1;  // steps 1 .. m-1
    const uint64_t draws = (cnt + 2 * 156 - 1) / (2 * 156) * (2 * 156);
    uint64_t *win, *raw;
    uint32_t *tgt, *stp, *skey, *sstp, *prev, *succ, *ra, *rb, *map;
    int* flags;
    alloc(&win, 312 * 8);
    alloc(&raw, draws * 8);
    alloc(&tgt, cnt * 4);
    alloc(&stp, cnt * 4);
    alloc(&skey, cnt * 4);
    alloc(&sstp, cnt * 4);
    alloc(&prev, m * 4);
    alloc(&succ, m * 4);
    alloc(&flags, 16);
    L1B_CUDA(cudaMallocHost(&h, 16));
    {
      uint64_t w[312];
      mt_seed_state(seed, w);
      L1B_CUDA(cudaMemcpyAsync(win, w, sizeof(w), cudaMemcpyHostToDevice, st));
      L1B_CUDA(cudaStreamSynchronize(st));
    }
    L1B_CUDA(cudaMemsetAsync(flags, 0, 16, st));
    mt_stream_raw(win, draws, raw, st);
    fy_draws_kernel<<<grid_for(cnt), kThreads, 0, st>>>(raw, m, tgt, stp, flags);
    L1B_LAUNCHED();
    L1B_CUDA(cudaFreeAsync(raw, st));  // (the largest buffer: before the sort's scratch)
    bufs.erase(std::find(bufs.begin(), bufs.end(), (void*)raw));
    const int bits = 64 - __builtin_clzll((unsigned long long)(m - 1));
    size_t tb = 0;
    L1B_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, tgt, skey, stp, sstp, (int)cnt, 0, bits, st));
    void* tmp = nullptr;
    alloc(&tmp, tb);
    L1B_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, tgt, skey, stp, sstp, (int)cnt, 0, bits, st));
    // prev[x] = x (no earlier step wrote x) unless set; succ[] all set by the links kernel
    iota_u32(prev, m, st);
    fy_links_kernel<<<grid_for(cnt), kThreads, 0, st>>>(skey, sstp, cnt, prev, succ);
    L1B_LAUNCHED();
    // the first step targeting 0 (prev[0] != 0 when there is one)
    L1B_CUDA(cudaMemcpyAsync(flags + 2, prev, 4, cudaMemcpyDeviceToDevice, st));
    // pointer jumping: root(x) = the end of x -> prev(x) -> ... (B(x))
    ra = prev;
    alloc(&rb, m * 4);
    for (int round = 0; round < 40; ++round) {
      L1B_CUDA(cudaMemsetAsync(flags + 1, 0, 4, st));
      fy_jump_kernel<<<grid_for(m), kThreads, 0, st>>>(ra, rb, m, flags + 1);
      L1B_LAUNCHED();
      std::swap(ra, rb);
      L1B_CUDA(cudaMemcpyAsync(h, flags, 12, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
      if (!h[1]) break;
    }
    const uint32_t f0 = (uint32_t)h[2];  // prev of position 0 before the jumps
    uint32_t* d_f0 = reinterpret_cast<uint32_t*>(flags + 3);
    const uint32_t f0v = f0 == 0 ? 0xffffffffu : f0;
    L1B_CUDA(cudaMemcpyAsync(d_f0, &f0v, 4, cudaMemcpyHostToDevice, st));
    alloc(&map, m * 4);
    fy_final_kernel<<<grid_for(m), kThreads, 0, st>>>(tgt, succ, ra, d_f0, m, map);
    L1B_LAUNCHED();
    L1B_CUDA(cudaMemcpyAsync(host_map, map, m * 4, cudaMemcpyDeviceToHost, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    ok = h[0] == 0;
  } catch (...) {
    for (void* q : bufs) cudaFreeAsync(q, st);
    if (h) cudaFreeHost(h);
    throw;
  }
  for (void* q : bufs) cudaFreeAsync(q, st);
  cudaFreeHost(h);
  return ok;
}

bool device_sparse_solution(uint64_t n, uint64_t s, double gamma, uint64_t seed, std::vector<uint32_t>& sup,
                            std::vector<double>& val, cudaStream_t st) {
  sup.clear();
  val.clear();
  if (s == 0) return true;
  if (n >= (1ull << 32) + 1) return false;  // indices are stored as uint32 (the generator's limit too)
  std::vector<void*> bufs;
  auto alloc = [&](auto** p, size_t bytes) {
    L1B_CUDA(cudaMallocAsync((void**)p, std::max<size_t>(bytes, 16), st));
    bufs.push_back((void*)*p);
  };
  bool ok = false;
  try {
    uint64_t *win, *raw, *t, *st_t, *e, *e_sorted;
    uint32_t *step, *st_step;
    uint8_t* dup;
    int* flags;
    double* d_val;
    const uint64_t cnt = (2 * s + 2 * 156 - 1) / (2 * 156) * (2 * 156);  // Floyd draws, then the values
    alloc(&win, 312 * 8);
    alloc(&raw, cnt * 8);
    alloc(&t, s * 8);
    alloc(&st_t, s * 8);
    alloc(&e, s * 8);
    alloc(&e_sorted, s * 8);
    alloc(&step, s * 4);
    alloc(&st_step, s * 4);
    alloc(&dup, s);
    alloc(&flags, 16);
    alloc(&d_val, s * 8);
    {
      uint64_t w[312];
      mt_seed_state(seed, w);
      L1B_CUDA(cudaMemcpyAsync(win, w, sizeof(w), cudaMemcpyHostToDevice, st));
      L1B_CUDA(cudaStreamSynchronize(st));  // (w is a stack array)
    }
    L1B_CUDA(cudaMemsetAsync(flags, 0, 16, st));
    mt_stream_raw(win, cnt, raw, st);
    floyd_draws_kernel<<<grid_for(s), kThreads, 0, st>>>(raw, n, s, t, step, flags);
    L1B_LAUNCHED();
    const int bits = 64 - __builtin_clzll((unsigned long long)n);
    size_t tb = 0, tb2 = 0;
    L1B_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, t, st_t, step, st_step, (int)s, 0, bits, st));
    L1B_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb2, e, e_sorted, (int)s, 0, bits, st));
    void* tmp = nullptr;
    alloc(&tmp, std::max(tb, tb2));
    L1B_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, t, st_t, step, st_step, (int)s, 0, bits, st));
    floyd_first_kernel<<<grid_for(s), kThreads, 0, st>>>(st_t, st_step, s, dup);
    L1B_LAUNCHED();
    int* h = nullptr;
    L1B_CUDA(cudaMallocHost(&h, 16));
    try {
      for (uint64_t round = 0; round < s + 1; ++round) {  // (B): chains to smaller steps
        L1B_CUDA(cudaMemsetAsync(flags + 1, 0, 4, st));
        floyd_chain_kernel<<<grid_for(s), kThreads, 0, st>>>(t, n, s, dup, flags + 1);
        L1B_LAUNCHED();
        L1B_CUDA(cudaMemcpyAsync(h, flags, 8, cudaMemcpyDeviceToHost, st));
        L1B_CUDA(cudaStreamSynchronize(st));
        if (!h[1]) break;
      }
      floyd_elements_kernel<<<grid_for(s), kThreads, 0, st>>>(t, dup, n, s, e);
      L1B_LAUNCHED();
      L1B_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb2, e, e_sorted, (int)s, 0, bits, st));
      floyd_values_kernel<<<grid_for(s), kThreads, 0, st>>>(raw, s, gamma, d_val, flags);
      L1B_LAUNCHED();
      std::vector<uint64_t> e64(s);
      val.resize(s);
      L1B_CUDA(cudaMemcpyAsync(e64.data(), e_sorted, s * 8, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaMemcpyAsync(val.data(), d_val, s * 8, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaMemcpyAsync(h, flags, 4, cudaMemcpyDeviceToHost, st));
      L1B_CUDA(cudaStreamSynchronize(st));
      ok = h[0] == 0;
      sup.assign(e64.begin(), e64.end());
    } catch (...) {
      cudaFreeHost(h);
      throw;
    }
    cudaFreeHost(h);
  } catch (...) {
    for (void* q : bufs) cudaFreeAsync(q, st);
    throw;
  }
  for (void* q : bufs) cudaFreeAsync(q, st);
  if (!ok) {
    sup.clear();
    val.clear();
  }
  return ok;
}

}  // namespace l1b
