// k_build.cu -- materialise A's rows (CSR) and columns (CSC) on device, and the
// Gram diagonal, from the stage description.
//
// One thread per line runs the reference's sparse-accumulator sweep
// (linops.cpp:113-192) on a small sorted list in registers/local memory:
//   row(i)    : e_{P1 source(i)} -> left stages^T -> P2 source map with sigma
//               -> right stages (reverse)                  (linops.cpp:597-619)
//   column(j) : e_j -> right stages^T -> sigma, P2 image -> left stages
//               (reverse) -> P1 image                      (linops.cpp:566-595)
// Disjoint-pair rotations commute, so a sorted list that activates the same
// partners (value 0.0) and applies the same rotate_pair arithmetic yields the
// reference's entries bit for bit; exact zeros are dropped on emission
// (linops.cpp:186).  Two passes: count, then fill at the scanned offsets.
#include <cub/device/device_scan.cuh>

#include "kernels.hpp"
#include "common.cuh"

namespace l1b {

namespace {

constexpr int kCap = 64;  // per-line fill capacity (2^stages bound, SPEC.md "diag_AtA")

struct Line {
  uint32_t idx[kCap];
  double val[kCap];
  int cnt;
};

// One paired stage on a sorted list: in -> out (both sorted ascending).
__device__ __forceinline__ bool stage_list(const Line& in, Line& out, uint64_t dim, int off,
                                           double c, double s, bool transposed) {
  int k = 0, o = 0;
  const uint32_t uoff = (uint32_t)off;
  while (k < in.cnt) {
    const uint32_t id = in.idx[k];
    if (id < uoff) {
      if (o >= kCap) return false;
      out.idx[o] = id;
      out.val[o++] = in.val[k++];
      continue;
    }
    const uint32_t lo = id - ((id - uoff) & 1u);
    const uint32_t hi = lo + 1;
    if ((uint64_t)hi >= dim) {  // trailing unpaired coordinate (SPEC.md "Odd n/m")
      if (o >= kCap) return false;
      out.idx[o] = id;
      out.val[o++] = in.val[k++];
      continue;
    }
    double a = 0.0, b = 0.0;  // partners activate with 0.0 (linops.cpp:153-155)
    if (in.idx[k] == lo) a = in.val[k++];
    if (k < in.cnt && in.idx[k] == hi) b = in.val[k++];
    rotate_pair(a, b, c, s, transposed);
    if (o + 2 > kCap) return false;
    out.idx[o] = lo;
    out.val[o++] = a;
    out.idx[o] = hi;
    out.val[o++] = b;
  }
  out.cnt = o;
  return true;
}

__device__ __forceinline__ void sort_list(Line& l) {
  for (int i = 1; i < l.cnt; ++i) {
    const uint32_t ki = l.idx[i];
    const double kv = l.val[i];
    int j = i - 1;
    while (j >= 0 && l.idx[j] > ki) {
      l.idx[j + 1] = l.idx[j];
      l.val[j + 1] = l.val[j];
      --j;
    }
    l.idx[j + 1] = ki;
    l.val[j + 1] = kv;
  }
}

// Runs row(i) (rows) or column(i) on two ping-pong buffers; returns the one
// holding the sorted result (zeros kept), *ok = false on capacity overflow.
__device__ __forceinline__ const Line* run_line(const OpView& op, bool rows, uint64_t i, Line& l0,
                                                Line& l1, bool* ok) {
  Line* a = &l0;
  Line* b = &l1;
  if (rows) {
    a->cnt = 1;
    a->idx[0] = op.p1 ? op.p1[i] : (uint32_t)i;
    a->val[0] = 1.0;
    for (int s = 0; s < op.left.count; ++s) {
      if (!stage_list(*a, *b, op.m, op.left.offset[s], op.left.c[s], op.left.s[s], true)) { *ok = false; return a; }
      Line* t = a; a = b; b = t;
    }
    int k = 0;
    for (int e = 0; e < a->cnt; ++e) {
      const uint32_t src = a->idx[e];
      const uint32_t t = op.p2 ? op.p2[src] : src;
      if ((uint64_t)t < op.n) {
        b->idx[k] = t;
        b->val[k++] = op.sigma[t] * a->val[e];
      }
    }
    b->cnt = k;
    if (op.p2) sort_list(*b);
    { Line* t = a; a = b; b = t; }
    for (int s = op.right.count - 1; s >= 0; --s) {
      if (!stage_list(*a, *b, op.n, op.right.offset[s], op.right.c[s], op.right.s[s], false)) { *ok = false; return a; }
      Line* t = a; a = b; b = t;
    }
  } else {
    a->cnt = 1;
    a->idx[0] = (uint32_t)i;
    a->val[0] = 1.0;
    for (int s = 0; s < op.right.count; ++s) {
      if (!stage_list(*a, *b, op.n, op.right.offset[s], op.right.c[s], op.right.s[s], true)) { *ok = false; return a; }
      Line* t = a; a = b; b = t;
    }
    for (int e = 0; e < a->cnt; ++e) {
      const uint32_t src = a->idx[e];
      b->idx[e] = op.p2 ? op.p2_inv[src] : src;
      b->val[e] = op.sigma[src] * a->val[e];
    }
    b->cnt = a->cnt;
    if (op.p2) sort_list(*b);
    { Line* t = a; a = b; b = t; }
    for (int s = op.left.count - 1; s >= 0; --s) {
      if (!stage_list(*a, *b, op.m, op.left.offset[s], op.left.c[s], op.left.s[s], false)) { *ok = false; return a; }
      Line* t = a; a = b; b = t;
    }
    if (op.p1) {
      for (int e = 0; e < a->cnt; ++e) a->idx[e] = op.p1_inv[a->idx[e]];
      sort_list(*a);
    }
  }
  *ok = true;
  return a;
}

// keep_lo / keep_hi: only entries whose index (row of a column, column of a
// row) lies in [keep_lo, keep_hi) -- a general row-block shard's CSC
__global__ void count_lines(OpView op, bool rows, uint64_t first, uint64_t nlines,
                            uint32_t* counts, unsigned long long* last_nonempty,
                            unsigned int* max_len, int* overflow, uint64_t keep_lo,
                            uint64_t keep_hi) {
  Line l0, l1;
  unsigned long long last = 0;
  unsigned int mx = 0;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nlines;
       t += (uint64_t)gridDim.x * blockDim.x) {
    bool ok;
    const Line* r = run_line(op, rows, first + t, l0, l1, &ok);
    if (!ok) {
      atomicExch(overflow, 1);
      counts[t] = 0;
      continue;
    }
    unsigned int c = 0;
    for (int e = 0; e < r->cnt; ++e)
      c += r->val[e] != 0.0 && r->idx[e] >= keep_lo && r->idx[e] < keep_hi;
    counts[t] = c;
    if (c) {
      last = t + 1;
      mx = c > mx ? c : mx;
    }
  }
  if (last) atomicMax(last_nonempty, last);
  if (mx) atomicMax(max_len, mx);
}

template <typename PtrT>
__global__ void fill_lines(OpView op, bool rows, uint64_t first, uint64_t nlines,
                           const uint64_t* offs, PtrT* ptr, uint32_t* idx, double* val,
                           uint64_t idx_base, uint64_t keep_lo, uint64_t keep_hi) {
  Line l0, l1;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nlines;
       t += (uint64_t)gridDim.x * blockDim.x) {
    bool ok;
    const Line* r = run_line(op, rows, first + t, l0, l1, &ok);
    uint64_t o = offs[t];
    ptr[t] = (PtrT)o;
    if (t + 1 == nlines) ptr[nlines] = (PtrT)offs[nlines];
    if (!ok) continue;
    for (int e = 0; e < r->cnt; ++e) {
      if (r->val[e] != 0.0 && r->idx[e] >= keep_lo && r->idx[e] < keep_hi) {
        idx[o] = (uint32_t)(r->idx[e] - idx_base);
        val[o++] = r->val[e];
      }
    }
  }
}

__global__ void tile_max_kernel(const uint64_t* offs, uint64_t lines, uint64_t tile,
                                unsigned long long* out) {
  unsigned long long mx = 0;
  const uint64_t ntiles = (lines + tile - 1) / tile;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = t * tile, b = min(a + tile, lines);
    mx = max(mx, (unsigned long long)(offs[b] - offs[a]));
  }
  if (mx) atomicMax(out, mx);
}

// min / max stored index of each 256-line tile (one warp per tile)
template <typename PtrT>
__global__ void tile_range_kernel(const PtrT* __restrict__ ptr, const uint32_t* __restrict__ idx, uint64_t lines,
                                  uint32_t* __restrict__ rng, unsigned* max_idx) {
  const uint64_t ntiles = (lines + 255) / 256;
  const int lane = threadIdx.x & 31;
  for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; t < ntiles;
       t += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint64_t a = ptr[t * 256], b = ptr[min(t * 256 + 256, lines)];
    uint32_t lo = 0xffffffffu, hi = 0;
    for (uint64_t q = a + lane; q < b; q += 32) {
      const uint32_t v = idx[q];
      lo = min(lo, v);
      hi = max(hi, v);
    }
    for (int o = 16; o; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      rng[2 * t] = lo;
      rng[2 * t + 1] = hi;
      if (b > a) atomicMax(max_idx, hi);
    }
  }
}

__global__ void widen_u32(const uint32_t* in, uint64_t* out, uint64_t n) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
       t += (uint64_t)gridDim.x * blockDim.x)
    out[t] = in[t];
}

// gram_diagonal (linops.cpp:533-558): the sparse-accumulator ACTIVATION order
// is replayed (partners appended as they are first touched) so the sum of
// sigma^2 w^2 runs in the reference's order and matches it bit for bit.
__global__ void gram_diag_kernel(OpView op, uint64_t first, uint64_t ncols, double* d) {
  uint32_t idx[kCap];
  double val[kCap];
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ncols;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = first + t;
    if (op.right.count == 0) {
      d[t] = op.sigma[i] * op.sigma[i];
      continue;
    }
    int cnt = 1;
    idx[0] = (uint32_t)i;
    val[0] = 1.0;
    bool ok = true;
    for (int s = 0; s < op.right.count && ok; ++s) {
      const uint32_t off = (uint32_t)op.right.offset[s];
      const int n0 = cnt;
      for (int a = 0; a < n0; ++a) {
        const uint32_t id = idx[a];
        if (id < off) continue;
        uint32_t partner;
        if (((id - off) & 1u) == 0) {
          if ((uint64_t)id + 1 >= op.n) continue;
          partner = id + 1;
        } else {
          partner = id - 1;
        }
        bool present = false;
        for (int q = 0; q < cnt; ++q) present |= idx[q] == partner;
        if (!present) {
          if (cnt >= kCap) { ok = false; break; }
          idx[cnt] = partner;
          val[cnt++] = 0.0;
        }
      }
      for (int a = 0; a < cnt && ok; ++a) {
        const uint32_t id = idx[a];
        if (id < off || ((id - off) & 1u) || (uint64_t)id + 1 >= op.n) continue;
        int q = 0;
        while (idx[q] != id + 1) ++q;
        rotate_pair(val[a], val[q], op.right.c[s], op.right.s[s], true);
      }
    }
    double acc = 0.0;
    for (int a = 0; a < cnt; ++a) {
      const double w = val[a];
      acc += op.sigma[idx[a]] * op.sigma[idx[a]] * w * w;
    }
    d[t] = ok ? acc : __longlong_as_double(0x7ff8000000000000ULL);
  }
}

}  // namespace

// ---------------------------------------------------------------------------

void build_lines(const OpView& op, bool rows, uint64_t first, uint64_t nlines, uint64_t idx_base,
                 bool trim_tail, cudaStream_t st, LinesOut* out, uint64_t keep_lo,
                 uint64_t keep_hi) {
  if (nlines == 0) throw InvalidArgument("build_lines: empty range");
  uint32_t* counts = nullptr;
  uint64_t* offs = nullptr;
  struct Scratch {
    unsigned long long last;
    unsigned int max_len;
    int overflow;
    unsigned int max_idx;
  }* scratch = nullptr;
  L1B_CUDA(cudaMallocAsync(&counts, (nlines + 1) * sizeof(uint32_t), st));
  L1B_CUDA(cudaMallocAsync(&offs, (nlines + 1) * sizeof(uint64_t), st));
  L1B_CUDA(cudaMallocAsync(&scratch, sizeof(Scratch), st));
  L1B_CUDA(cudaMemsetAsync(scratch, 0, sizeof(Scratch), st));
  const int grid = grid_for(nlines, 128, 8);
  count_lines<<<grid, 128, 0, st>>>(op, rows, first, nlines, counts, &scratch->last,
                                    &scratch->max_len, &scratch->overflow, keep_lo, keep_hi);
  L1B_LAUNCHED();
  Scratch h;
  L1B_CUDA(cudaMemcpyAsync(&h, scratch, sizeof(Scratch), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  if (h.overflow) {
    cudaFreeAsync(counts, st);
    cudaFreeAsync(offs, st);
    cudaFreeAsync(scratch, st);
    throw Unsupported("device operator builder: per-line fill exceeds 64 entries");
  }
  const uint64_t keep = trim_tail ? (uint64_t)h.last : nlines;
  out->lines = keep;
  out->max_len = h.max_len;
  // exclusive scan of counts[0, keep) (+ a trailing zero for the total)
  uint64_t total = 0;
  if (keep > 0) {
    widen_u32<<<grid_for(keep), kThreads, 0, st>>>(counts, offs, keep);
    L1B_LAUNCHED();
    L1B_CUDA(cudaMemsetAsync(offs + keep, 0, sizeof(uint64_t), st));
    size_t tmp_bytes = 0;
    L1B_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, offs, offs, keep + 1, st));
    void* tmp = nullptr;
    L1B_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    L1B_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, offs, offs, keep + 1, st));
    L1B_LAUNCHED();
    L1B_CUDA(cudaFreeAsync(tmp, st));
    L1B_CUDA(cudaMemcpyAsync(&total, offs + keep, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    L1B_CUDA(cudaStreamSynchronize(st));
  }
  out->nnz = total;
  out->ptr32 = total < (1ull << 32);
  // +16 B slack: the TMA stages copy 16-byte aligned supersets of each range
  const size_t ptr_bytes = (keep + 1) * (out->ptr32 ? 4 : 8);
  if (cudaMalloc(&out->ptr, ptr_bytes + 16) != cudaSuccess ||
      cudaMalloc(&out->idx, (total + 4) * sizeof(uint32_t)) != cudaSuccess ||
      cudaMalloc(&out->val, (total + 2) * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    cudaFreeAsync(counts, st);
    cudaFreeAsync(offs, st);
    cudaFreeAsync(scratch, st);
    throw OutOfMemory("device operator builder: out of device memory for " +
                      std::to_string(total) + " nonzeros");
  }
  if (keep > 0) {
    if (out->ptr32)
      fill_lines<uint32_t><<<grid, 128, 0, st>>>(op, rows, first, keep, offs, (uint32_t*)out->ptr,
                                                 out->idx, out->val, idx_base, keep_lo, keep_hi);
    else
      fill_lines<uint64_t><<<grid, 128, 0, st>>>(op, rows, first, keep, offs, (uint64_t*)out->ptr,
                                                 out->idx, out->val, idx_base, keep_lo, keep_hi);
    L1B_LAUNCHED();
  } else {
    L1B_CUDA(cudaMemsetAsync(out->ptr, 0, ptr_bytes, st));
  }
  // largest nonzero count of a 256-line tile (selects the TMA SpMV kernel)
  L1B_CUDA(cudaMemsetAsync(scratch, 0, sizeof(Scratch), st));
  if (keep > 0) {
    tile_max_kernel<<<grid_for((keep + 255) / 256), kThreads, 0, st>>>(offs, keep, 256, &scratch->last);
    L1B_LAUNCHED();
  }
  if (keep > 0) {  // per-tile index ranges (x staged with the tile)
    const uint64_t ntiles = (keep + 255) / 256;
    if (cudaMalloc(&out->tile_rng, ntiles * 2 * sizeof(uint32_t)) != cudaSuccess) {
      cudaGetLastError();
      out->tile_rng = nullptr;  // the SpMV then gathers x from global memory
    } else if (out->ptr32) {
      tile_range_kernel<uint32_t><<<grid_for(ntiles * 32), kThreads, 0, st>>>((const uint32_t*)out->ptr, out->idx,
                                                                              keep, out->tile_rng, &scratch->max_idx);
      L1B_LAUNCHED();
    } else {
      tile_range_kernel<uint64_t><<<grid_for(ntiles * 32), kThreads, 0, st>>>((const uint64_t*)out->ptr, out->idx,
                                                                              keep, out->tile_rng, &scratch->max_idx);
      L1B_LAUNCHED();
    }
  }
  L1B_CUDA(cudaMemcpyAsync(&h, scratch, sizeof(Scratch), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaFreeAsync(counts, st));
  L1B_CUDA(cudaFreeAsync(offs, st));
  L1B_CUDA(cudaFreeAsync(scratch, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  out->tile_nnz_max = h.last;
  out->x_len = total ? (uint64_t)h.max_idx + 1 : 0;
}

void gram_diagonal(const OpView& op, uint64_t first, uint64_t ncols, double* d, cudaStream_t st) {
  gram_diag_kernel<<<grid_for(ncols, 128, 8), 128, 0, st>>>(op, first, ncols, d);
  L1B_LAUNCHED();
}

}  // namespace l1b
