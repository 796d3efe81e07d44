// abi.cu -- the C ABI of include/l1b.h: object lifetimes, the host half of the
// generator (sequential std::mt19937_64 streams), operator materialisation and
// the solver drivers that enqueue the device-resident loops.
//
// The host side only orchestrates: every arithmetic pass over an n- or
// m-vector runs in the kernels of k_*.cu.  The only host arithmetic is the
// RNG streams (inherently sequential: rng.hpp:14-56), cos/sin of the stage
// angles (so they come from the same libm as the reference, linops.cpp:84-85)
// and O(1) scalars.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/l1b.h"
#include "common.cuh"
#include "kernels.hpp"
#include "guard.hpp"
#include "solvers.hpp"

namespace l1b {

std::atomic<uint64_t> g_launch_count{0};

std::string& last_error_slot() {
  static thread_local std::string slot;
  return slot;
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  const std::string msg = std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                          std::to_string(line) + ")";
  if (e == cudaErrorMemoryAllocation) throw OutOfMemory(msg);
  throw CudaError(msg);
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    L1B_CUDA(cudaGetDevice(&dev));
    L1B_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return sms;
}

// the device's default stream-ordered pool keeps freed memory cached (no
// release at synchronisation points): sessions and problems allocate from it
void keep_pool(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

int grid_for(uint64_t work, int threads, int max_blocks_per_sm) {
  const uint64_t blocks = (work + threads - 1) / threads;
  const uint64_t cap = (uint64_t)max_blocks_per_sm * sm_count();
  return (int)std::max<uint64_t>(1, std::min(blocks, cap));
}

// ---------------------------------------------------------------------------
// host RNG helpers -- same streams as rng.hpp:14-56
namespace hostrng {
using Rng = std::mt19937_64;

uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline double unit(Rng& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }
inline double in(Rng& r, double lo, double hi) { return lo + (hi - lo) * unit(r); }
inline uint64_t index(Rng& r, uint64_t n) {
  const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = r();
  } while (x >= lim);
  return x % n;
}

void permutation(uint64_t n, uint64_t seed, uint32_t* map) {  // linops.cpp:224-234
  for (uint64_t i = 0; i < n; ++i) map[i] = (uint32_t)i;
  Rng r(seed);
  for (uint64_t i = n; i > 1; --i) std::swap(map[i - 1], map[index(r, i)]);
}

void spectrum_uniform(uint64_t n, double lo, double hi, double shift, uint64_t seed,
                      double* out) {  // linops.cpp:323-331
  Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) {
    double u;
    do {
      u = in(r, lo, hi);
    } while (u <= lo);
    out[i] = u + shift;
  }
}

void sparse_solution(uint64_t n, uint64_t s, double gamma, Rng& r, std::vector<uint32_t>& sup,
                     std::vector<double>& val) {  // solution.cpp:47-75
  sup.clear();
  val.clear();
  if (s == 0) return;
  std::unordered_set<uint64_t> chosen;
  chosen.reserve(s * 2);
  for (uint64_t j = n - s; j < n; ++j) {
    const uint64_t t = index(r, j + 1);
    if (!chosen.insert(t).second) chosen.insert(j);
  }
  sup.assign(chosen.begin(), chosen.end());
  std::sort(sup.begin(), sup.end());
  val.reserve(s);
  for (uint64_t k = 0; k < s; ++k) {
    double v;
    do {
      v = in(r, -gamma, gamma);
    } while (v == 0.0);
    val.push_back(v);
  }
}
}  // namespace hostrng

}  // namespace l1b

// ===========================================================================
using namespace l1b;

namespace {

// +2 entries of slack: the TMA stages copy 16-byte rounded ranges.  With a
// stream the buffer comes from the device's stream-ordered pool (kept cached,
// keep_pool): creating a problem from host data again (e2e passes, repeated
// l1b_problem_create) costs no cudaMalloc / page mapping after the first.
template <class T>
T* dev_alloc(size_t count, size_t* bytes_acc, cudaStream_t st = nullptr) {
  T* p = nullptr;
  const size_t bytes = (count + 2) * sizeof(T);
  if (st) {
    int dev = 0;
    L1B_CUDA(cudaGetDevice(&dev));
    keep_pool(dev);
    L1B_CUDA(cudaMallocAsync(&p, bytes, st));
  } else {
    L1B_CUDA(cudaMalloc(&p, bytes));
  }
  if (bytes_acc) *bytes_acc += bytes;
  return p;
}

template <class T>
T* upload(const T* host, size_t count, cudaStream_t st, size_t* bytes_acc) {
  T* p = dev_alloc<T>(count, bytes_acc, st);
  if (count) L1B_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, st));
  return p;
}

}  // namespace

struct l1b_problem {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  uint64_t m = 0, n = 0;
  double tau = 1.0;
  std::vector<int32_t> r_off, l_off;
  std::vector<double> r_theta, l_theta;
  OpView view;
  double* d_sigma = nullptr;
  uint32_t *d_p1 = nullptr, *d_p2 = nullptr, *d_p1inv = nullptr, *d_p2inv = nullptr;
  double* d_b = nullptr;
  double* d_gram = nullptr;
  double* d_sigma_c = nullptr;  // sigma * prod cos(theta): the contracted arithmetic's scaled rotations (lazily built)
  std::vector<uint32_t> xs_sup;
  std::vector<double> xs_val;
  double noise_norm = 0.0, cert_kappa = 1.0, lmax = 0.0;
  LinesOut csr, csc;
  bool sparse_built = false;
  double tail_sq = 0.0;        // sum of b_i^2 over rows >= m_active (sparse path)
  double tail_sq_band = 0.0;   // same over rows >= n (matrix-free path of banded operators)
  size_t device_bytes = 0;
  uint64_t row_begin = 0, row_end = 0;
  int world = 1, rank = 0;
  bool sharded = false;  // a row-block shard (l1b_generate with a shard descriptor)
  uint64_t halo = 0;
  uint64_t sig_begin = 0;  // shards: d_sigma holds sigma[sig_begin, sig_end)
  uint64_t sig_end = 0;    // 0: the whole problem (sigma[0, n))
  // shards: b on [b_win_lo, b_win_hi) = own rows +- the recomputing kernel's
  // halo (it rebuilds r on the rows around its own block)
  double* d_b_win = nullptr;
  uint64_t b_win_lo = 0, b_win_hi = 0;
  // general (non-banded) shard: rows [row_begin, row_end) of A, x sliced by
  // columns [col_begin, col_end) of width col_slice (the last slice padded)
  bool general = false;
  uint64_t col_begin = 0, col_end = 0, col_slice = 0;

  ~l1b_problem() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    // stream-ordered pool buffers go back to the (retained) pool: cudaFree on
    // them would hand the pages back to the driver and the next problem of the
    // same size would map them again (the e2e passes varied 0.38 - 0.6 s)
    for (void* p : {(void*)d_sigma, (void*)d_p1, (void*)d_p2, (void*)d_p1inv, (void*)d_p2inv, (void*)d_b,
                    (void*)d_b_win, (void*)d_gram, (void*)d_sigma_c})
      if (p) cudaFreeAsync(p, stream);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : {csr.ptr, (void*)csr.idx, (void*)csr.val, csc.ptr, (void*)csc.idx, (void*)csc.val,
                    (void*)csr.tile_rng, (void*)csc.tile_rng})
      if (p) cudaFree(p);  // (the CSR/CSC copy: plain allocations)
    if (stream && own_stream) cudaStreamDestroy(stream);
  }

  Csr rows() const {
    Csr c;
    c.lines = csr.lines;
    c.nnz = csr.nnz;
    c.ptr32 = csr.ptr32;
    c.ptr = csr.ptr;
    c.idx = csr.idx;
    c.val = csr.val;
    c.lanes = 32;
    c.tile_nnz_max = csr.tile_nnz_max;
    c.tile_rng = csr.tile_rng;
    c.x_len = csr.x_len;
    return c;
  }
  Csr cols() const {
    Csr c;
    c.lines = csc.lines;
    c.nnz = csc.nnz;
    c.ptr32 = csc.ptr32;
    c.ptr = csc.ptr;
    c.idx = csc.idx;
    c.val = csc.val;
    c.lanes = 32;
    c.tile_nnz_max = csc.tile_nnz_max;
    c.tile_rng = csc.tile_rng;
    c.x_len = csc.x_len;
    return c;
  }
};

namespace {

void fill_stage_tab(StageTab& tab, const std::vector<int32_t>& off, const std::vector<double>& th) {
  if (off.size() > (size_t)kMaxStages)
    throw Unsupported("at most " + std::to_string(kMaxStages) + " stages per side are supported");
  tab.count = (int)off.size();
  for (size_t k = 0; k < off.size(); ++k) {
    tab.offset[k] = off[k];
    tab.c[k] = std::cos(th[k]);
    tab.s[k] = std::sin(th[k]);
  }
  tab.cprod = 1.0;
  tab.scaled_ok = 1;
  for (size_t k = 0; k < off.size(); ++k) {
    if (std::fabs(tab.c[k]) < 0.25) tab.scaled_ok = 0;
    tab.tn[k] = tab.scaled_ok ? tab.s[k] / tab.c[k] : 0.0;
    tab.ic[k] = tab.scaled_ok ? 1.0 / tab.c[k] : 1.0;
    tab.cprod *= tab.c[k];
  }
}

std::vector<uint32_t> inverse_map(const uint32_t* map, uint64_t m) {
  std::vector<uint32_t> inv(m);
  std::vector<uint8_t> seen(m, 0);
  for (uint64_t i = 0; i < m; ++i) {
    if (map[i] >= m || seen[map[i]])
      throw InvalidArgument("Permutation: mapping is not a bijection");
    seen[map[i]] = 1;
    inv[map[i]] = (uint32_t)i;
  }
  return inv;
}

// Validation of OperatorSpec::finalize (linops.cpp:394-416) + device upload
// of the description.  sigma/p1/p2 are host arrays.
void setup_operator(l1b_problem* p, int device, uint64_t m, uint64_t n,
                    std::vector<int32_t> r_off, std::vector<double> r_th,
                    std::vector<int32_t> l_off, std::vector<double> l_th, const uint32_t* p1,
                    const uint32_t* p2, const double* sigma, double* d_sigma_ready = nullptr) {
  if (m == 0 || n == 0) throw InvalidArgument("OperatorSpec: dimensions must be positive");
  if (m < n) throw InvalidArgument("OperatorSpec: requires m >= n");
  if (m > (1ull << 32)) throw InvalidArgument("OperatorSpec: m above 2^32 exceeds uint32 indices");
  for (int32_t o : r_off)
    if (o != 0 && o != 1) throw InvalidArgument("RotationStage: offset must be 0 or 1");
  for (int32_t o : l_off)
    if (o != 0 && o != 1) throw InvalidArgument("RotationStage: offset must be 0 or 1");
  p->device = device;
  L1B_CUDA(cudaSetDevice(device));
  L1B_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  p->m = m;
  p->n = n;
  p->r_off = std::move(r_off);
  p->r_theta = std::move(r_th);
  p->l_off = std::move(l_off);
  p->l_theta = std::move(l_th);
  fill_stage_tab(p->view.right, p->r_off, p->r_theta);
  fill_stage_tab(p->view.left, p->l_off, p->l_theta);
  cudaStream_t st = p->stream;
  if (d_sigma_ready) {  // drawn on the device (k_rng.cu)
    p->d_sigma = d_sigma_ready;
    p->device_bytes += (n + 2) * sizeof(double);
  } else {
    p->d_sigma = upload(sigma, n, st, &p->device_bytes);
  }
  if (p1) {
    auto inv = inverse_map(p1, m);
    p->d_p1 = upload(p1, m, st, &p->device_bytes);
    p->d_p1inv = upload(inv.data(), m, st, &p->device_bytes);
  }
  if (p2) {
    auto inv = inverse_map(p2, m);
    p->d_p2 = upload(p2, m, st, &p->device_bytes);
    p->d_p2inv = upload(inv.data(), m, st, &p->device_bytes);
  }
  p->view.m = m;
  p->view.n = n;
  p->view.sigma = p->d_sigma;
  p->view.p1 = p->d_p1;
  p->view.p2 = p->d_p2;
  p->view.p1_inv = p->d_p1inv;
  p->view.p2_inv = p->d_p2inv;
  // Spectrum::validate (linops.cpp:359-365) and sigma_max / sigma_min, on device
  double smin = 0.0, smax = 0.0;
  bool ok = false;
  device_min_finite(p->d_sigma, n, &smin, &smax, &ok, st);
  if (!ok) throw std::runtime_error("Spectrum: all singular values must be strictly positive");
  p->lmax = smax * smax;                                     // gram_lmax (linops.cpp:560-564)
  p->cert_kappa = (smax / smin) * (smax / smin);             // solution.cpp:127-133
  L1B_CUDA(cudaStreamSynchronize(st));
}

// CSR (rows, trailing empty rows trimmed) + CSC of A, and the constant
// 1/2*||b_tail||^2 part of every objective.
void materialise(l1b_problem* p) {
  if (p->sparse_built) return;
  p->sparse_built = true;
  if (p->general) {  // general shard: CSR rows [a, b) (global columns), CSC of that block
    const uint64_t a = p->row_begin, own = p->row_end - p->row_begin;
    build_lines(p->view, true, a, own, 0, false, p->stream, &p->csr);
    p->device_bytes += (p->csr.lines + 1) * (p->csr.ptr32 ? 4 : 8) + p->csr.nnz * 12;
    build_lines(p->view, false, 0, p->n, a, false, p->stream, &p->csc, a, p->row_end);
    p->device_bytes += (p->csc.lines + 1) * (p->csc.ptr32 ? 4 : 8) + p->csc.nnz * 12;
    p->tail_sq = 0.0;  // every row belongs to some block
    return;
  }
  if (p->sharded) {  // row-block shard: rows / columns [a, b), window-local indices
    const uint64_t a = p->row_begin, own = p->row_end - p->row_begin;
    build_lines(p->view, true, a, own, a - p->halo, false, p->stream, &p->csr);
    p->device_bytes += (p->csr.lines + 1) * (p->csr.ptr32 ? 4 : 8) + p->csr.nnz * 12;
    build_lines(p->view, false, a, own, a - p->halo, false, p->stream, &p->csc);
    p->device_bytes += (p->csc.lines + 1) * (p->csc.ptr32 ? 4 : 8) + p->csc.nnz * 12;
    p->tail_sq = 0.0;  // rows >= n are structurally empty and b is exactly 0 there
    return;
  }
  build_lines(p->view, true, 0, p->m, 0, true, p->stream, &p->csr);
  p->device_bytes += (p->csr.lines + 1) * (p->csr.ptr32 ? 4 : 8) + p->csr.nnz * 12;
  build_lines(p->view, false, 0, p->n, 0, false, p->stream, &p->csc);
  p->device_bytes += (p->csc.lines + 1) * (p->csc.ptr32 ? 4 : 8) + p->csc.nnz * 12;
  p->row_begin = 0;
  p->row_end = p->csr.lines;
  p->tail_sq = 0.0;
  if (p->csr.lines < p->m) {
    std::vector<double> tail(p->m - p->csr.lines);
    L1B_CUDA(cudaMemcpyAsync(tail.data(), p->d_b + p->csr.lines, tail.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, p->stream));
    L1B_CUDA(cudaStreamSynchronize(p->stream));
    for (double v : tail) p->tail_sq += v * v;
  }
}

// sum of b_i^2 over rows >= n (empty rows of a banded operator), on device
void band_tail(l1b_problem* p) {
  p->tail_sq_band = 0.0;
  if (p->m > p->n) p->tail_sq_band = device_sum_sq(p->d_b + p->n, p->m - p->n, p->stream);
}

void check_problem(const l1b_problem* p) {
  if (!p) throw InvalidArgument("null problem");
  L1B_CUDA(cudaSetDevice(p->device));
}

void check_whole(const l1b_problem* p) {
  check_problem(p);
  if (p->sharded) throw Unsupported("operation needs the whole operator, not a row-block shard");
}

}  // namespace

// ===========================================================================
extern "C" {

int l1b_abi_version(void) { return L1B_ABI_VERSION; }
const char* l1b_last_error(void) { return last_error_slot().c_str(); }
uint64_t l1b_launch_count(void) { return g_launch_count.load(); }

uint64_t l1b_mix_seed(uint64_t seed, uint64_t salt) { return hostrng::mix_seed(seed, salt); }

int l1b_realize_permutation(uint64_t n, uint64_t seed, uint32_t* map_out) {
  return guard([&] {
    if (!map_out) throw InvalidArgument("null output");
    hostrng::permutation(n, seed, map_out);
  });
}

int l1b_realize_spectrum_uniform(uint64_t n, double lo, double hi, double shift, uint64_t seed,
                                 double* sigma_out) {
  return guard([&] { hostrng::spectrum_uniform(n, lo, hi, shift, seed, sigma_out); });
}

int l1b_mt_draws_after_jump(uint64_t seed, uint32_t log2_jump, uint64_t count, uint64_t* out) {
  return guard([&] {
    if (!out && count) throw InvalidArgument("null output");
    if (log2_jump > 63) throw InvalidArgument("jump above 2^63");
    host_draws_after_jump(seed, (int)log2_jump, count, out);
  });
}

int l1b_device_uniform_sparse_solution(int device, uint64_t n, uint64_t s, double gamma, uint64_t rng_seed,
                                       uint32_t* support_out, double* values_out, int* on_device) {
  return guard([&] {
    if (s > n) throw InvalidArgument("uniform_sparse_solution: s must not exceed n");
    if (!(gamma > 0.0)) throw InvalidArgument("uniform_sparse_solution: gamma must be positive");
    if (s && (!support_out || !values_out)) throw InvalidArgument("null output");
    L1B_CUDA(cudaSetDevice(device));
    std::vector<uint32_t> sup;
    std::vector<double> val;
    const bool dev = device_sparse_solution(n, s, gamma, rng_seed, sup, val, nullptr);
    if (!dev) {  // (a redraw: the sequential stream)
      hostrng::Rng r(rng_seed);
      hostrng::sparse_solution(n, s, gamma, r, sup, val);
    }
    if (on_device) *on_device = dev ? 1 : 0;
    std::copy(sup.begin(), sup.end(), support_out);
    std::copy(val.begin(), val.end(), values_out);
  });
}

int l1b_device_realize_permutation(int device, uint64_t n, uint64_t seed, uint32_t* map_out, int* on_device) {
  return guard([&] {
    if (!map_out && n) throw InvalidArgument("null output");
    L1B_CUDA(cudaSetDevice(device));
    const bool dev = device_permutation(n, seed, map_out, nullptr);
    if (!dev) hostrng::permutation(n, seed, map_out);
    if (on_device) *on_device = dev ? 1 : 0;
  });
}

int l1b_mt_draws_after_chunk_jump(uint64_t seed, uint64_t chunk, uint64_t count, uint64_t* out) {
  return guard([&] {
    if (!out && count) throw InvalidArgument("null output");
    host_draws_after_chunk_jump(seed, chunk, count, out);
  });
}

int l1b_device_uniform_draws(int device, uint64_t seed, uint64_t count, double lo, double hi,
                             int spectrum, double shift, uint64_t win_lo, uint64_t win_hi,
                             uint32_t min_log2_chunk, double* d_out, double* vmin, double* vmax,
                             int* exact) {
  return guard([&] {
    if (win_hi > count || win_lo > win_hi) throw InvalidArgument("draw window out of range");
    if (win_hi > win_lo && !d_out) throw InvalidArgument("null output");
    if (min_log2_chunk > 40) throw InvalidArgument("chunk above 2^40 draws");
    L1B_CUDA(cudaSetDevice(device));
    const bool ok = device_uniform_draws(seed, count, lo, hi, spectrum != 0, shift, win_lo, win_hi, d_out,
                                         vmin, vmax, 0, (int)min_log2_chunk);
    if (exact) *exact = ok ? 1 : 0;
  });
}

int l1b_device_index_stream(int device, uint64_t seed, uint64_t n, const uint64_t* piece_counts,
                            uint32_t npieces, uint32_t* d_out, uint64_t* drawn) {
  return guard([&] {
    if (n == 0 || n >= (1ull << 32)) throw InvalidArgument("index stream: n must lie in [1, 2^32)");
    if (npieces && (!piece_counts || !d_out)) throw InvalidArgument("null argument");
    L1B_CUDA(cudaSetDevice(device));
    uint64_t w[312];
    mt_seed_state(seed, w);
    uint64_t* d_w = nullptr;
    L1B_CUDA(cudaMalloc(&d_w, sizeof(w)));
    uint64_t total = 0;
    try {
      L1B_CUDA(cudaMemcpy(d_w, w, sizeof(w), cudaMemcpyHostToDevice));
      for (uint32_t k = 0; k < npieces; ++k) total += mt_stream_indices(d_w, piece_counts[k], n, d_out + total, nullptr, 0);
      L1B_CUDA(cudaStreamSynchronize(0));
    } catch (...) {
      cudaFree(d_w);
      throw;
    }
    L1B_CUDA(cudaFree(d_w));
    if (drawn) *drawn = total;
  });
}

int l1b_uniform_sparse_solution(uint64_t n, uint64_t s, double gamma, uint64_t rng_seed,
                                uint32_t* support_out, double* values_out) {
  return guard([&] {
    if (s > n) throw InvalidArgument("uniform_sparse_solution: s must not exceed n");
    if (!(gamma > 0.0)) throw InvalidArgument("uniform_sparse_solution: gamma must be positive");
    hostrng::Rng r(rng_seed);
    std::vector<uint32_t> sup;
    std::vector<double> val;
    hostrng::sparse_solution(n, s, gamma, r, sup, val);
    std::copy(sup.begin(), sup.end(), support_out);
    std::copy(val.begin(), val.end(), values_out);
  });
}

}  // extern "C"

namespace {
// The per-entry streams (sigma, the subgradient fill) are drawn on the device
// (k_rng.cu, mt19937_64 jump-ahead) for n >= 2^16; L1B_DEVICE_RNG=0 keeps the
// sequential host replay, =1 uses the device for every n.
bool device_rng_for(uint64_t n) {
  const char* e = getenv("L1B_DEVICE_RNG");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  return n >= (1ull << 16);
}

// Row-block shard of a banded instance (identity P1/P2, no left stages, so
// |col - row| <= h = #stages and rows >= n are empty).  The host replays the
// full sigma / g streams (sequential mt19937_64) but uploads only the window
// [a - 3h, b + 3h); the device runs the generator's sweeps on that window
// (k_sweep.cu window_stages), which reproduces the global b on the own rows
// bit for bit, and materialises rows [a, b) (CSR, columns local to the x
// window [a - h, b + h)) and columns [a, b) (CSC, rows local to the r window).
// The planted solution of bench.cpp:281-301 by SolutionRule::Kind.  uniform:
// uniform_sparse_solution(n, s, gamma) from Rng(mix_seed(job.seed, 4));
// two_value: the same support with gamma 1, values value_a on the first half
// and value_b on the rest; spectral: spectral_sparse_solution
// (solution.cpp:77-113) -- xhat = G gamma (Sigma^T Sigma)^{-1} 1 (right factor
// applied on the device with the reference's stage order), the s1 smallest and
// s2 = s - s1 largest |xhat| among its nonzeros (stable order), ascending.
void planted_solution(const l1b_gen_desc* g, uint64_t n, uint64_t job_seed, const double* sigma,
                      l1b_problem* p) {
  const uint64_t s = std::max<uint64_t>(1, n / g->s_divisor);
  switch (g->solution_kind) {
    case L1B_SOLUTION_UNIFORM: {
      // on the device (k_solution.cu) like the sigma / fill streams; the host
      // replay when a draw the reference redraws occurs
      if (device_rng_for(n) && device_sparse_solution(n, s, g->gamma, hostrng::mix_seed(job_seed, 4), p->xs_sup,
                                                      p->xs_val, p->stream))
        return;
      hostrng::Rng r(hostrng::mix_seed(job_seed, 4));
      hostrng::sparse_solution(n, s, g->gamma, r, p->xs_sup, p->xs_val);
      return;
    }
    case L1B_SOLUTION_TWO_VALUE: {
      if (!(device_rng_for(n) && device_sparse_solution(n, s, 1.0, hostrng::mix_seed(job_seed, 4), p->xs_sup,
                                                         p->xs_val, p->stream))) {
        hostrng::Rng r(hostrng::mix_seed(job_seed, 4));
        hostrng::sparse_solution(n, s, 1.0, r, p->xs_sup, p->xs_val);
      }
      const size_t half = p->xs_val.size() / 2;
      for (size_t k = 0; k < p->xs_val.size(); ++k) p->xs_val[k] = k < half ? g->value_a : g->value_b;
      return;
    }
    case L1B_SOLUTION_SPECTRAL: {
      const uint64_t s1 = (uint64_t)std::llround(g->s1_fraction * (double)s);
      if (s1 > s) throw InvalidArgument("spectral_sparse_solution: s1 + s2 must not exceed n");
      if (!(g->gamma > 0.0)) throw InvalidArgument("spectral_sparse_solution: gamma must be positive");
      std::vector<double> xhat(n);
      for (uint64_t i = 0; i < n; ++i) xhat[i] = g->gamma / (sigma[i] * sigma[i]);
      spectral_select(p->view, xhat.data(), n, s1, s - s1, p->stream, p->xs_sup, p->xs_val);
      return;
    }
    default:
      throw InvalidArgument("unknown solution kind");
  }
}

// L1B_GEN_TRACE=1: phase times of the shard generator on stderr
struct PhaseTrace {
  bool on;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point t0;
  PhaseTrace() : on(getenv("L1B_GEN_TRACE") != nullptr), t0(std::chrono::steady_clock::now()) {}
  void operator()(const char* what) {
    if (!on) return;
    if (st) cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[l1b gen] %-22s %8.1f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

void generate_shard(int device, const l1b_gen_desc* g, const l1b_shard_desc* sh,
                    l1b_problem** out) {
  PhaseTrace mark;
  if (g->n < 2) throw InvalidArgument("ExperimentConfig: dimensions must be at least 2");
  if (!(g->m_ratio >= 1.0)) throw InvalidArgument("ExperimentConfig: m_ratio must be >= 1");
  if (g->s_divisor == 0) throw InvalidArgument("ExperimentConfig: s_divisor must be positive");
  if (!(g->tau > 0.0)) throw InvalidArgument("generate_instance: tau must be positive");
  if (g->permute || g->left_stages)
    throw Unsupported("row-block shards need a banded operator (no permutations, no left stages)");
  if (sh->rank < 0 || sh->rank >= sh->world) throw InvalidArgument("shard: rank out of range");
  const uint64_t n = g->n;
  const uint64_t m = (uint64_t)std::llround(g->m_ratio * (double)n);
  // window overhang: #stages rounded up to even (16-byte aligned bulk copies)
  const uint64_t h = ((uint64_t)g->stages + 1) & ~1ull;
  uint64_t a = sh->row_begin, b = sh->row_end;
  if (b == 0) {  // even split, boundaries on multiples of 16 (distributed.partition)
    auto cut = [&](uint64_t g_) {
      return g_ == (uint64_t)sh->world ? n : (n * g_ / (uint64_t)sh->world) / 16 * 16;
    };
    a = cut((uint64_t)sh->rank);
    b = cut((uint64_t)sh->rank + 1);
  }
  if (!(a < b && b <= n)) throw InvalidArgument("shard: empty or out-of-range row block");
  if (a % 2) throw InvalidArgument("shard: row_begin must be even");
  const uint64_t job_seed = hostrng::mix_seed(g->seed, g->job_index);
  // b is also built on bh rows around the block for the recomputing FISTA
  // kernel (k_iter_rc.cu); sigma / x / w windows widen by the same amount
  const uint64_t bh = g->stages >= 1 && g->stages <= 4
                          ? (uint64_t)std::max(fista_rc_halo((int)g->stages), fista_rc2_halo((int)g->stages))
                          : 0;
  const uint64_t sa = a > bh + 3 * h ? (a - bh - 3 * h) & ~3ull : 0;  // 32-byte aligned view
  const uint64_t sb = std::min(n, b + bh + 3 * h);
  if (g->spectrum_kind < L1B_SPECTRUM_UNIFORM_Q || g->spectrum_kind > L1B_SPECTRUM_EXPLICIT ||
      (g->spectrum_kind == L1B_SPECTRUM_EXPLICIT && !g->sigma_explicit))
    throw InvalidArgument("unknown spectrum kind");
  auto p = std::make_unique<l1b_problem>();
  std::vector<int32_t> r_off;
  for (uint32_t i = 0; i < g->stages; ++i) r_off.push_back((int32_t)((g->stages - 1 - i) % 2));
  p->device = device;
  L1B_CUDA(cudaSetDevice(device));
  L1B_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  cudaStream_t st = p->stream;
  mark.st = st;
  mark("setup");
  // sigma: the window [sa, sb) is kept, sigma_max / sigma_min are global.  On
  // the device the whole stream is drawn (chunks jump-started) and reduced
  // without being stored; on the host (L1B_DEVICE_RNG=0, other spectra, or a
  // rejected draw) the full stream is replayed.
  const bool dev_rng = device_rng_for(n);
  double smax = 0.0, smin = 0.0;
  bool have_sigma = false;
  if (dev_rng && g->spectrum_kind == L1B_SPECTRUM_UNIFORM_Q) {
    p->d_sigma = dev_alloc<double>(sb - sa, &p->device_bytes, st);
    have_sigma = device_uniform_draws(hostrng::mix_seed(job_seed, 3), n, 0.0, std::pow(10.0, g->q), true,
                                      g->shift, sa, sb, p->d_sigma, &smin, &smax, 0);
    if (!have_sigma) {
      cudaFree(p->d_sigma);
      p->d_sigma = nullptr;
      p->device_bytes -= (sb - sa + 2) * sizeof(double);
    } else if (!(smin > 0.0) || !std::isfinite(smax)) {
      throw std::runtime_error("Spectrum: all singular values must be strictly positive");
    }
  }
  if (!have_sigma) {
    std::vector<double> sigma(n);
    if (g->spectrum_kind == L1B_SPECTRUM_UNIFORM_Q) {
      hostrng::spectrum_uniform(n, 0.0, std::pow(10.0, g->q), g->shift, hostrng::mix_seed(job_seed, 3),
                                sigma.data());
    } else if (g->spectrum_kind == L1B_SPECTRUM_ALTERNATING) {
      for (uint64_t i = 0; i < n; ++i) sigma[i] = (i % 2 == 0) ? g->odd_value : g->even_value;
    } else {
      std::copy(g->sigma_explicit, g->sigma_explicit + n, sigma.begin());
    }
    for (uint64_t i = 0; i < n; ++i)
      if (!(sigma[i] > 0.0) || !std::isfinite(sigma[i]))
        throw std::runtime_error("Spectrum: all singular values must be strictly positive");
    p->d_sigma = upload(sigma.data() + sa, sb - sa, st, &p->device_bytes);
    smax = smin = sigma[0];
    for (uint64_t i = 1; i < n; ++i) {
      smax = std::max(smax, sigma[i]);
      smin = std::min(smin, sigma[i]);
    }
    L1B_CUDA(cudaStreamSynchronize(st));
  }
  p->m = m;
  p->n = n;
  p->r_off = r_off;
  p->r_theta.assign(g->stages, g->theta);
  fill_stage_tab(p->view.right, p->r_off, p->r_theta);
  fill_stage_tab(p->view.left, p->l_off, p->l_theta);
  p->sig_begin = sa;
  p->sig_end = sb;
  p->view.m = m;
  p->view.n = n;
  p->view.sigma = p->d_sigma - sa;  // global indexing inside [sa, sb)
  p->lmax = smax * smax;
  p->cert_kappa = (smax / smin) * (smax / smin);
  p->tau = g->tau;
  p->world = sh->world;
  p->sharded = true;
  p->rank = sh->rank;
  p->row_begin = a;
  p->row_end = b;
  p->halo = h;
  if (g->solution_kind == L1B_SOLUTION_SPECTRAL)
    throw Unsupported("row-block shards: the spectral planted solution needs the whole operator");
  mark("sigma");
  planted_solution(g, n, job_seed, nullptr, p.get());
  mark("planted solution");
  const uint64_t s = p->xs_sup.size();
  // the subgradient fill on the window (instance.cpp:33-40): draws [sa, sb) of
  // Rng(mix_seed(job.seed, 5)) -- on the device only the chunks meeting the
  // window run -- then the signs of x* on the support
  double* d_g = nullptr;
  {
    std::vector<uint32_t> wsup;
    std::vector<double> wsg;
    for (uint64_t k = 0; k < s; ++k) {
      const uint64_t i = p->xs_sup[k];
      if (i >= sa && i < sb) {
        wsup.push_back((uint32_t)(i - sa));
        wsg.push_back(p->xs_val[k] > 0.0 ? 1.0 : -1.0);
      }
    }
    if (dev_rng) {
      d_g = dev_alloc<double>(sb - sa, nullptr, st);
      device_uniform_draws(hostrng::mix_seed(job_seed, 5), n, -g->fill_bound, g->fill_bound, false, 0.0, sa,
                           sb, d_g, nullptr, nullptr, st);
      uint32_t* d_ws = upload(wsup.data(), wsup.size(), st, nullptr);
      double* d_wv = upload(wsg.data(), wsg.size(), st, nullptr);
      scatter_values(d_ws, d_wv, wsup.size(), d_g, st);
      L1B_CUDA(cudaStreamSynchronize(st));
      cudaFree(d_ws);
      cudaFree(d_wv);
    } else {
      std::vector<double> gw(sb - sa);
      hostrng::Rng r(hostrng::mix_seed(job_seed, 5));
      for (uint64_t i = 0; i < sb; ++i) {
        const double v = hostrng::in(r, -g->fill_bound, g->fill_bound);
        if (i >= sa) gw[i - sa] = v;
      }
      for (size_t k = 0; k < wsup.size(); ++k) gw[wsup[k]] = wsg[k];
      d_g = upload(gw.data(), gw.size(), st, nullptr);
      L1B_CUDA(cudaStreamSynchronize(st));
    }
  }
  const uint64_t va = a > bh + h ? a - bh - h : 0, vb = std::min(n, b + bh + h), own = b - a;
  const uint64_t wa = a > bh ? a - bh : 0, wb = std::min(n, b + bh);  // b window
  // x* on the window [va, vb): zero, then its support scattered on the device
  std::vector<uint32_t> xsup;
  std::vector<double> xval;
  for (uint64_t k = 0; k < s; ++k) {
    const uint64_t i = p->xs_sup[k];
    if (i >= va && i < vb) {
      xsup.push_back((uint32_t)(i - va));
      xval.push_back(p->xs_val[k]);
    }
  }
  mark("fill + x* window");
  // w = G (S^T S)^-1 G^T g on the window (valid on [a - h, b + h))
  window_stages(p->view.right, true, true, d_g, sa, sb, n, st);
  window_scale_op(d_g, p->d_sigma, sb - sa, 0, 0.0, st);
  window_stages(p->view.right, false, false, d_g, sa, sb, n, st);
  // e_own = Sigma G^T w, b_own = Sigma G^T x* on [a, b)
  double* d_v = nullptr;
  double* d_x = dev_alloc<double>(vb - va, nullptr, st);
  {
    uint32_t* d_xs = upload(xsup.data(), xsup.size(), st, nullptr);
    double* d_xv = upload(xval.data(), xval.size(), st, nullptr);
    scatter_sparse(d_xs, d_xv, xsup.size(), d_x, vb - va, st);
    L1B_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_xs);
    cudaFree(d_xv);
  }
  L1B_CUDA(cudaMalloc(&d_v, (vb - va) * sizeof(double)));
  L1B_CUDA(cudaMemcpyAsync(d_v, d_g + (va - sa), (vb - va) * 8, cudaMemcpyDeviceToDevice, st));
  window_stages(p->view.right, true, true, d_v, va, vb, n, st);
  window_stages(p->view.right, true, true, d_x, va, vb, n, st);
  window_scale_op(d_v + (wa - va), p->d_sigma + (wa - sa), wb - wa, 1, 0.0, st);
  window_scale_op(d_x + (wa - va), p->d_sigma + (wa - sa), wb - wa, 1, 0.0, st);
  p->d_b = dev_alloc<double>(own, &p->device_bytes, st);
  L1B_CUDA(cudaMemcpyAsync(p->d_b, d_x + (a - va), own * 8, cudaMemcpyDeviceToDevice, st));
  double* d_ss = nullptr;
  L1B_CUDA(cudaMalloc(&d_ss, sizeof(double)));
  if (bh) {  // the same b = A x* + tau e, element for element, on the window
    double* d_e = nullptr;
    L1B_CUDA(cudaMalloc(&d_e, (wb - wa) * sizeof(double)));
    L1B_CUDA(cudaMemcpyAsync(d_e, d_v + (wa - va), (wb - wa) * 8, cudaMemcpyDeviceToDevice, st));
    p->d_b_win = dev_alloc<double>(wb - wa, &p->device_bytes, st);
    L1B_CUDA(cudaMemcpyAsync(p->d_b_win, d_x + (wa - va), (wb - wa) * 8, cudaMemcpyDeviceToDevice, st));
    generator_combine(p->tau, d_e, p->d_b_win, wb - wa, d_ss, st);
    p->b_win_lo = wa;
    p->b_win_hi = wb;
    L1B_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_e);
  }
  generator_combine(p->tau, d_v + (a - va), p->d_b, own, d_ss, st);  // e *= tau; b += e
  double ss = 0.0;
  L1B_CUDA(cudaMemcpyAsync(&ss, d_ss, 8, cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  p->noise_norm = std::sqrt(ss);  // this shard's part of ||e||
  for (void* q : {(void*)d_g, (void*)d_v, (void*)d_x, (void*)d_ss}) cudaFree(q);
  p->tail_sq = p->tail_sq_band = 0.0;  // rows >= n are empty and b is exactly 0 there
  mark("sweeps + b");
  // rows / columns [a, b) with indices local to the windows starting at a - h
  if (!g->lazy_sparse) materialise(p.get());
  mark("materialise");
  *out = p.release();
}

// build_instance (bench.cpp:253-316) + generate_instance (instance.cpp:53-89)
// of the whole problem on one device (the CSR/CSC copy stays lazy)
std::unique_ptr<l1b_problem> generate_whole(int device, const l1b_gen_desc* g) {
  if (g->n < 2) throw InvalidArgument("ExperimentConfig: dimensions must be at least 2");
  if (!(g->m_ratio >= 1.0)) throw InvalidArgument("ExperimentConfig: m_ratio must be >= 1");
  if (g->s_divisor == 0) throw InvalidArgument("ExperimentConfig: s_divisor must be positive");
  if (!(g->tau > 0.0)) throw InvalidArgument("generate_instance: tau must be positive");
  if (!(g->fill_bound >= 0.0 && g->fill_bound < 1.0))
    throw InvalidArgument("FillPolicy: interior bound must lie in [0, 1)");
  const uint64_t n = g->n;
  const uint64_t m = (uint64_t)std::llround(g->m_ratio * (double)n);
  const uint64_t job_seed = hostrng::mix_seed(g->seed, g->job_index);
  std::vector<int32_t> r_off, l_off;
  for (uint32_t i = 0; i < g->stages; ++i) r_off.push_back((int32_t)((g->stages - 1 - i) % 2));
  for (uint32_t i = 0; i < g->left_stages; ++i)
    l_off.push_back((int32_t)((g->left_stages - 1 - i) % 2));
  // The four seeded streams (P1, P2, sigma, the subgradient fill) are
  // independent mt19937_64 sequences: sigma and the fill are drawn on the
  // device (jump-ahead chunks), the permutations (Fisher-Yates with rejection,
  // inherently sequential) on host threads.
  std::vector<uint32_t> p1, p2;
  std::vector<double> sigma, gv;
  if (g->permute && m > (1ull << 32)) throw InvalidArgument("Permutation: m above 2^32");
  if (g->spectrum_kind == L1B_SPECTRUM_EXPLICIT && !g->sigma_explicit)
    throw InvalidArgument("explicit spectrum without values");
  if (g->spectrum_kind < L1B_SPECTRUM_UNIFORM_Q || g->spectrum_kind > L1B_SPECTRUM_EXPLICIT)
    throw InvalidArgument("unknown spectrum kind");
  const bool dev_rng = device_rng_for(n);
  L1B_CUDA(cudaSetDevice(device));
  double* d_sig = nullptr;
  if (dev_rng && g->spectrum_kind == L1B_SPECTRUM_UNIFORM_Q) {
    L1B_CUDA(cudaMalloc(&d_sig, (n + 2) * sizeof(double)));
    if (!device_uniform_draws(hostrng::mix_seed(job_seed, 3), n, 0.0, std::pow(10.0, g->q), true, g->shift,
                              0, n, d_sig, nullptr, nullptr, 0)) {
      cudaFree(d_sig);  // a rejected draw: replay the stream sequentially
      d_sig = nullptr;
    }
  }
  double* d_g = nullptr;
  if (dev_rng) {  // l1_subgradient draws (instance.cpp:33-35), Rng(mix_seed(job.seed, 5))
    L1B_CUDA(cudaMalloc(&d_g, (n + 2) * sizeof(double)));
    device_uniform_draws(hostrng::mix_seed(job_seed, 5), n, -g->fill_bound, g->fill_bound, false, 0.0, 0, n,
                         d_g, nullptr, nullptr, 0);
  }
  {
    std::vector<std::thread> pool;
    if (g->permute) {
      p1.resize(m);
      p2.resize(m);
      // Fisher-Yates on the device from its draws alone (k_solution.cu); the host
      // replay below n = 2^16 or after a redrawn index
      const bool d1 = dev_rng && device_permutation(m, hostrng::mix_seed(job_seed, 1), p1.data(), nullptr);
      const bool d2 = dev_rng && device_permutation(m, hostrng::mix_seed(job_seed, 2), p2.data(), nullptr);
      if (!d1) pool.emplace_back([&] { hostrng::permutation(m, hostrng::mix_seed(job_seed, 1), p1.data()); });
      if (!d2) pool.emplace_back([&] { hostrng::permutation(m, hostrng::mix_seed(job_seed, 2), p2.data()); });
    }
    if (!d_sig) {
      sigma.resize(n);
      pool.emplace_back([&] {
        if (g->spectrum_kind == L1B_SPECTRUM_UNIFORM_Q) {
          hostrng::spectrum_uniform(n, 0.0, std::pow(10.0, g->q), g->shift,
                                    hostrng::mix_seed(job_seed, 3), sigma.data());
        } else if (g->spectrum_kind == L1B_SPECTRUM_ALTERNATING) {
          for (uint64_t i = 0; i < n; ++i) sigma[i] = (i % 2 == 0) ? g->odd_value : g->even_value;
        } else {
          std::copy(g->sigma_explicit, g->sigma_explicit + n, sigma.begin());
        }
      });
    }
    if (!d_g) {
      gv.resize(n);
      pool.emplace_back([&] {  // l1_subgradient draws (instance.cpp:33-35), Rng(mix_seed(job.seed, 5))
        hostrng::Rng r(hostrng::mix_seed(job_seed, 5));
        for (uint64_t i = 0; i < n; ++i) gv[i] = hostrng::in(r, -g->fill_bound, g->fill_bound);
      });
    }
    for (auto& th : pool) th.join();
  }
  auto p = std::make_unique<l1b_problem>();
  setup_operator(p.get(), device, m, n, r_off, std::vector<double>(g->stages, g->theta), l_off,
                 std::vector<double>(g->left_stages, g->theta), g->permute ? p1.data() : nullptr,
                 g->permute ? p2.data() : nullptr, d_sig ? nullptr : sigma.data(), d_sig);
  p->tau = g->tau;
  if (d_sig && g->solution_kind == L1B_SOLUTION_SPECTRAL) {  // xhat needs sigma on the host
    sigma.resize(n);
    L1B_CUDA(cudaMemcpy(sigma.data(), d_sig, n * sizeof(double), cudaMemcpyDeviceToHost));
  }
  // planted solution (bench.cpp:281-301)
  planted_solution(g, n, job_seed, sigma.empty() ? nullptr : sigma.data(), p.get());
  const uint64_t s = p->xs_sup.size();
  cudaStream_t st = p->stream;
  // subgradient g: signs on the support (instance.cpp:36-40)
  if (d_g) {
    std::vector<double> sg(s);
    for (uint64_t k = 0; k < s; ++k) sg[k] = p->xs_val[k] > 0.0 ? 1.0 : -1.0;
    uint32_t* d_ssup = upload(p->xs_sup.data(), s, st, nullptr);
    double* d_sg = upload(sg.data(), s, st, nullptr);
    scatter_values(d_ssup, d_sg, s, d_g, st);
    L1B_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_ssup);
    cudaFree(d_sg);
  } else {
    for (uint64_t k = 0; k < s; ++k) gv[p->xs_sup[k]] = p->xs_val[k] > 0.0 ? 1.0 : -1.0;
    d_g = upload(gv.data(), n, st, nullptr);
  }
  // device: w = G (S^T S)^-1 G^T g; e = tau A w; b = A x* + e (instance.cpp:64-79)
  double *d_e = nullptr, *d_x = nullptr, *d_ss = nullptr;
  uint32_t* d_sup = nullptr;
  double* d_val = nullptr;
  L1B_CUDA(cudaMalloc(&d_e, m * sizeof(double)));
  L1B_CUDA(cudaMalloc(&d_x, n * sizeof(double)));
  L1B_CUDA(cudaMalloc(&d_ss, sizeof(double)));
  p->d_b = dev_alloc<double>(m, &p->device_bytes, st);
  d_sup = upload(p->xs_sup.data(), s, st, nullptr);
  d_val = upload(p->xs_val.data(), s, st, nullptr);
  sweep_gram_inverse(p->view, d_g, d_g, st);
  sweep_apply(p->view, d_g, d_e, st);
  scatter_sparse(d_sup, d_val, s, d_x, n, st);
  sweep_apply(p->view, d_x, p->d_b, st);
  generator_combine(p->tau, d_e, p->d_b, m, d_ss, st);
  double ss = 0.0;
  L1B_CUDA(cudaMemcpyAsync(&ss, d_ss, sizeof(double), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  p->noise_norm = std::sqrt(ss);
  for (void* q : {(void*)d_g, (void*)d_e, (void*)d_x, (void*)d_ss, (void*)d_sup, (void*)d_val})
    cudaFree(q);
  band_tail(p.get());
  return p;
}

// A general (permuted / left-stage) operator split over `world` devices: every
// device generates the whole instance (operator description, b, x*), then
// keeps rows [a, b) of A as CSR (global columns) and the CSC of that row block
// (local rows); x is sliced by columns for the reduce-scatter / all-gather
// FISTA of distributed.py.  Row and column cuts on multiples of 16.
void generate_general_shard(int device, const l1b_gen_desc* g, const l1b_shard_desc* sh,
                            l1b_problem** out) {
  if (sh->rank < 0 || sh->rank >= sh->world) throw InvalidArgument("shard: rank out of range");
  auto p = generate_whole(device, g);
  const uint64_t m = p->m, n = p->n, W = (uint64_t)sh->world, r = (uint64_t)sh->rank;
  uint64_t a = sh->row_begin, b = sh->row_end;
  if (b == 0) {
    auto cut = [&](uint64_t q) { return q == W ? m : (m * q / W) / 16 * 16; };
    a = cut(r);
    b = cut(r + 1);
  }
  if (!(a < b && b <= m)) throw InvalidArgument("shard: empty or out-of-range row block");
  const uint64_t cs = ((n + W - 1) / W + 15) / 16 * 16;
  p->sharded = true;
  p->general = true;
  p->world = sh->world;
  p->rank = sh->rank;
  p->row_begin = a;
  p->row_end = b;
  p->col_slice = cs;
  p->col_begin = std::min(n, r * cs);
  p->col_end = std::min(n, (r + 1) * cs);
  p->halo = 0;
  p->tail_sq = p->tail_sq_band = 0.0;
  materialise(p.get());
  *out = p.release();
}

}  // namespace

extern "C" {

// build_instance (bench.cpp:253-316) + generate_instance (instance.cpp:53-89).
int l1b_generate(int device, const l1b_gen_desc* g, const l1b_shard_desc* shard, l1b_problem** out) {
  NvtxRange nvtx("l1b_generate");
  return guard([&] {
    if (!g || !out) throw InvalidArgument("null argument");
    *out = nullptr;
    if (shard && (g->permute || g->left_stages)) {  // general row-block shard
      generate_general_shard(device, g, shard, out);
      return;
    }
    if (shard) {  // banded row-block shard (world >= 1)
      generate_shard(device, g, shard, out);
      return;
    }
    auto p = generate_whole(device, g);
    if (!g->lazy_sparse) materialise(p.get());
    *out = p.release();
  });
}

int l1b_problem_create(int device, const l1b_operator_desc* op, double tau, const double* b_host,
                       const uint32_t* xs_support, const double* xs_values, uint64_t s,
                       l1b_problem** out) {
  NvtxRange nvtx("l1b_problem_create");
  return guard([&] {
    if (!op || !out || !b_host || !op->sigma) throw InvalidArgument("null argument");
    *out = nullptr;
    if (!(tau > 0.0)) throw InvalidArgument("generate_instance: tau must be positive");
    auto p = std::make_unique<l1b_problem>();
    std::vector<int32_t> ro(op->right_offset, op->right_offset + op->n_right);
    std::vector<double> rt(op->right_theta, op->right_theta + op->n_right);
    std::vector<int32_t> lo(op->left_offset, op->left_offset + op->n_left);
    std::vector<double> lt(op->left_theta, op->left_theta + op->n_left);
    setup_operator(p.get(), device, op->m, op->n, ro, rt, lo, lt, op->p1, op->p2, op->sigma);
    p->tau = tau;
    if (s) {
      if (!xs_support || !xs_values) throw InvalidArgument("null x* arrays");
      p->xs_sup.assign(xs_support, xs_support + s);
      p->xs_val.assign(xs_values, xs_values + s);
      for (uint64_t k = 0; k < s; ++k) {
        if (p->xs_sup[k] >= op->n) throw InvalidArgument("SparseSolution: index out of range");
        if (k && p->xs_sup[k] <= p->xs_sup[k - 1])
          throw InvalidArgument("SparseSolution: support must be strictly increasing");
        if (p->xs_val[k] == 0.0) throw InvalidArgument("SparseSolution: stored values must be nonzero");
      }
    }
    p->d_b = upload(b_host, op->m, p->stream, &p->device_bytes);
    L1B_CUDA(cudaStreamSynchronize(p->stream));
    band_tail(p.get());  // the CSR/CSC copy is built on first sparse use
    *out = p.release();
  });
}

int l1b_problem_free(l1b_problem* p) {
  return guard([&] { delete p; });
}

int l1b_problem_materialize(l1b_problem* p) {
  return guard([&] {
    check_problem(p);
    materialise(p);
  });
}

int l1b_problem_info_get(const l1b_problem* p, l1b_problem_info* o) {
  return guard([&] {
    if (!p || !o) throw InvalidArgument("null argument");
    // nnz / m_active describe the CSR copy; report zeros until it exists
    o->m = p->m;
    o->n = p->n;
    o->m_active = p->sparse_built ? p->csr.lines : 0;
    o->nnz = p->sparse_built ? p->csr.nnz : 0;
    o->s = p->xs_sup.size();
    o->tau = p->tau;
    o->noise_norm = p->noise_norm;
    o->cert_kappa = p->cert_kappa;
    o->gram_lmax = p->lmax;
    double l1 = 0.0;
    for (double v : p->xs_val) l1 += std::abs(v);
    o->f_star = p->tau * l1 + 0.5 * p->noise_norm * p->noise_norm;  // instance.cpp:49-51
    o->device_bytes = p->device_bytes;
    o->row_begin = p->row_begin;
    o->row_end = p->row_end;
    o->col_begin = 0;
    o->col_end = p->n;
    o->csr_lanes = p->rows().lanes;
    o->csc_lanes = p->cols().lanes;
    o->world = p->world;
    o->rank = p->rank;
    o->halo = p->halo;
    if (p->sharded) {
      o->m_active = p->row_end - p->row_begin;
      o->col_begin = p->general ? p->col_begin : p->row_begin;
      o->col_end = p->general ? p->col_end : p->row_end;
    }
  });
}

int l1b_problem_get_b(const l1b_problem* p, double* b) {
  return guard([&] {
    check_problem(p);
    const uint64_t rows = p->sharded ? p->row_end - p->row_begin : p->m;  // shards: own rows
    const double* src = p->general ? p->d_b + p->row_begin : p->d_b;  // general: whole b kept
    L1B_CUDA(cudaMemcpyAsync(b, src, rows * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    L1B_CUDA(cudaStreamSynchronize(p->stream));
  });
}

int l1b_problem_get_b_window(const l1b_problem* p, uint64_t* lo, uint64_t* hi, double* b) {
  return guard([&] {
    check_problem(p);
    if (!lo || !hi) throw InvalidArgument("null argument");
    *lo = p->b_win_lo;
    *hi = p->b_win_hi;
    if (b && p->d_b_win && p->b_win_hi > p->b_win_lo) {
      L1B_CUDA(cudaMemcpyAsync(b, p->d_b_win, (p->b_win_hi - p->b_win_lo) * sizeof(double),
                               cudaMemcpyDeviceToHost, p->stream));
      L1B_CUDA(cudaStreamSynchronize(p->stream));
    }
  });
}

int l1b_problem_set_rhs(l1b_problem* p, const double* b_host, const double* b_win_host) {
  return guard([&] {
    check_problem(p);
    if (!b_host) throw InvalidArgument("null b");
    cudaStream_t st = p->stream;
    if (p->sharded && !p->general) {
      const uint64_t own = p->row_end - p->row_begin;
      L1B_CUDA(cudaMemcpyAsync(p->d_b, b_host, own * sizeof(double), cudaMemcpyHostToDevice, st));
      if (p->d_b_win) {
        if (!b_win_host) throw InvalidArgument("this shard keeps a b window: b_win_host needed");
        L1B_CUDA(cudaMemcpyAsync(p->d_b_win, b_win_host, (p->b_win_hi - p->b_win_lo) * sizeof(double),
                                 cudaMemcpyHostToDevice, st));
      }
      L1B_CUDA(cudaStreamSynchronize(st));  // host buffers are read during the call only
      return;
    }
    L1B_CUDA(cudaMemcpyAsync(p->d_b, b_host, p->m * sizeof(double), cudaMemcpyHostToDevice, st));
    if (p->general) {
      L1B_CUDA(cudaStreamSynchronize(st));
      return;
    }
    band_tail(p);  // (synchronises the stream)
    if (p->sparse_built)
      p->tail_sq = p->csr.lines < p->m ? device_sum_sq(p->d_b + p->csr.lines, p->m - p->csr.lines, st) : 0.0;
  });
}

int l1b_problem_get_sigma(const l1b_problem* p, double* s) {
  return guard([&] {
    check_whole(p);
    L1B_CUDA(cudaMemcpyAsync(s, p->d_sigma, p->n * sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    L1B_CUDA(cudaStreamSynchronize(p->stream));
  });
}

int l1b_problem_get_sigma_window(const l1b_problem* p, uint64_t* begin, uint64_t* end, double* s) {
  return guard([&] {
    if (!p || !begin || !end) throw InvalidArgument("null argument");
    *begin = p->sig_begin;
    *end = p->sig_end ? p->sig_end : p->n;
    if (s) {
      L1B_CUDA(cudaMemcpyAsync(s, p->d_sigma, (*end - *begin) * sizeof(double), cudaMemcpyDeviceToHost,
                               p->stream));
      L1B_CUDA(cudaStreamSynchronize(p->stream));
    }
  });
}

int l1b_problem_set_meta(l1b_problem* p, double noise_norm, double cert_kappa) {
  return guard([&] {
    if (!p) throw InvalidArgument("null problem");
    p->noise_norm = noise_norm;
    p->cert_kappa = cert_kappa;
  });
}

int l1b_problem_get_stages(const l1b_problem* p, int right, uint32_t* count, int32_t* offsets,
                           double* thetas) {
  return guard([&] {
    if (!p || !count) throw InvalidArgument("null argument");
    const auto& off = right ? p->r_off : p->l_off;
    const auto& th = right ? p->r_theta : p->l_theta;
    *count = (uint32_t)off.size();
    if (offsets) std::copy(off.begin(), off.end(), offsets);
    if (thetas) std::copy(th.begin(), th.end(), thetas);
  });
}

int l1b_problem_get_perm(const l1b_problem* p, int which, int* is_identity, uint32_t* map) {
  return guard([&] {
    if (!p || !is_identity || (which != 1 && which != 2)) throw InvalidArgument("bad argument");
    const uint32_t* d = which == 1 ? p->d_p1 : p->d_p2;
    *is_identity = d ? 0 : 1;
    if (d && map) {
      L1B_CUDA(cudaMemcpyAsync(map, d, p->m * sizeof(uint32_t), cudaMemcpyDeviceToHost, p->stream));
      L1B_CUDA(cudaStreamSynchronize(p->stream));
    }
  });
}

int l1b_problem_get_xstar(const l1b_problem* p, uint32_t* support, double* values) {
  return guard([&] {
    if (!p) throw InvalidArgument("null problem");
    std::copy(p->xs_sup.begin(), p->xs_sup.end(), support);
    std::copy(p->xs_val.begin(), p->xs_val.end(), values);
  });
}

void* l1b_problem_stream(const l1b_problem* p) { return p ? (void*)p->stream : nullptr; }

int l1b_problem_set_stream(l1b_problem* p, void* stream) {
  return guard([&] {
    check_problem(p);
    L1B_CUDA(cudaStreamSynchronize(p->stream));
    if (p->own_stream) L1B_CUDA(cudaStreamDestroy(p->stream));
    p->stream = (cudaStream_t)stream;
    p->own_stream = false;
  });
}

int l1b_apply(l1b_problem* p, int path, const double* d_x, double* d_y) {
  NvtxRange nvtx("l1b_apply");
  return guard([&] {
    check_whole(p);
    if (path == L1B_PATH_SWEEP) {
      sweep_apply(p->view, d_x, d_y, p->stream);
    } else if (path == L1B_PATH_FUSED) {
      if (!fused_supported(p->view)) throw Unsupported("fused path: banded operators only");
      fused_apply(p->view, d_x, d_y, p->stream);
      if (p->m > p->n)
        L1B_CUDA(cudaMemsetAsync(d_y + p->n, 0, (p->m - p->n) * sizeof(double), p->stream));
    } else {
      materialise(p);
      spmv(p->rows(), d_x, d_y, p->stream);
      if (p->csr.lines < p->m)
        L1B_CUDA(cudaMemsetAsync(d_y + p->csr.lines, 0, (p->m - p->csr.lines) * sizeof(double),
                                 p->stream));
    }
  });
}

int l1b_apply_transpose(l1b_problem* p, int path, const double* d_y, double* d_x) {
  return guard([&] {
    check_whole(p);
    if (path == L1B_PATH_SWEEP) {
      sweep_apply_transpose(p->view, d_y, d_x, p->stream);
    } else if (path == L1B_PATH_FUSED) {
      if (!fused_supported(p->view)) throw Unsupported("fused path: banded operators only");
      fused_apply_transpose(p->view, d_y, d_x, p->stream);
    } else {
      materialise(p);
      spmv(p->cols(), d_y, d_x, p->stream);
    }
  });
}

int l1b_gram_inverse(l1b_problem* p, const double* d_v, double* d_out) {
  return guard([&] {
    check_whole(p);
    sweep_gram_inverse(p->view, d_v, d_out, p->stream);
  });
}

namespace {
const double* gram_diag_device(l1b_problem* p) {
  if (!p->d_gram) {
    p->d_gram = dev_alloc<double>(p->n, &p->device_bytes, p->stream);
    gram_diagonal(p->view, 0, p->n, p->d_gram, p->stream);
  }
  return p->d_gram;
}
}  // namespace

int l1b_estimate_gram_lmax(l1b_problem* p, uint64_t iters, uint64_t seed, double* out) {
  return guard([&] {
    check_whole(p);
    if (!out) throw InvalidArgument("null output");
    L1B_CUDA(cudaSetDevice(p->device));
    *out = estimate_gram_lmax_device(p->view, p->m, p->n, iters, seed, p->stream);
  });
}

int l1b_gram_diagonal(l1b_problem* p, double* d_out) {
  return guard([&] {
    check_whole(p);
    const double* g = gram_diag_device(p);
    L1B_CUDA(cudaMemcpyAsync(d_out, g, p->n * sizeof(double), cudaMemcpyDeviceToDevice, p->stream));
  });
}

namespace {
void export_lines(const l1b_problem* p, const LinesOut& L, uint64_t dim, uint64_t* ptr,
                  uint32_t* idx, double* val) {
  check_problem(p);
  std::vector<uint32_t> p32;
  if (L.ptr32) {
    p32.resize(L.lines + 1);
    L1B_CUDA(cudaMemcpyAsync(p32.data(), L.ptr, p32.size() * 4, cudaMemcpyDeviceToHost, p->stream));
  } else {
    L1B_CUDA(cudaMemcpyAsync(ptr, L.ptr, (L.lines + 1) * 8, cudaMemcpyDeviceToHost, p->stream));
  }
  if (L.nnz) {
    L1B_CUDA(cudaMemcpyAsync(idx, L.idx, L.nnz * 4, cudaMemcpyDeviceToHost, p->stream));
    L1B_CUDA(cudaMemcpyAsync(val, L.val, L.nnz * 8, cudaMemcpyDeviceToHost, p->stream));
  }
  L1B_CUDA(cudaStreamSynchronize(p->stream));
  if (L.ptr32)
    for (uint64_t i = 0; i <= L.lines; ++i) ptr[i] = p32[i];
  for (uint64_t i = L.lines + 1; i <= dim; ++i) ptr[i] = L.nnz;
}
}  // namespace

int l1b_export_csr(const l1b_problem* p, uint64_t* row_ptr, uint32_t* col, double* val) {
  return guard([&] {
    materialise(const_cast<l1b_problem*>(p));
    export_lines(p, p->csr, p->m, row_ptr, col, val);
  });
}

int l1b_export_csc(const l1b_problem* p, uint64_t* col_ptr, uint32_t* row, double* val) {
  return guard([&] {
    materialise(const_cast<l1b_problem*>(p));
    export_lines(p, p->csc, p->n, col_ptr, row, val);
  });
}

int l1b_objective(l1b_problem* p, const double* d_x, double* f_out) {
  return guard([&] {
    check_whole(p);
    materialise(p);
    double* d_f = nullptr;
    L1B_CUDA(cudaMallocAsync(&d_f, sizeof(double), p->stream));
    objective(p->rows(), d_x, p->n, p->d_b, p->tau, p->tail_sq, d_f, p->stream);
    L1B_CUDA(cudaMemcpyAsync(f_out, d_f, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    L1B_CUDA(cudaFreeAsync(d_f, p->stream));
    L1B_CUDA(cudaStreamSynchronize(p->stream));
  });
}

int l1b_verify_optimality(l1b_problem* p, double tol, l1b_cert* out) {
  return guard([&] {
    check_whole(p);
    cudaStream_t st = p->stream;
    double *xd = nullptr, *res = nullptr, *r = nullptr, *mx = nullptr;
    L1B_CUDA(cudaMallocAsync(&xd, p->n * sizeof(double), st));
    L1B_CUDA(cudaMallocAsync(&res, p->m * sizeof(double), st));
    L1B_CUDA(cudaMallocAsync(&r, p->n * sizeof(double), st));
    L1B_CUDA(cudaMallocAsync(&mx, 2 * sizeof(double), st));
    uint32_t* d_sup = nullptr;
    double* d_val = nullptr;
    const uint64_t s = p->xs_sup.size();
    L1B_CUDA(cudaMallocAsync(&d_sup, std::max<uint64_t>(s, 1) * 4, st));
    L1B_CUDA(cudaMallocAsync(&d_val, std::max<uint64_t>(s, 1) * 8, st));
    if (s) {
      L1B_CUDA(cudaMemcpyAsync(d_sup, p->xs_sup.data(), s * 4, cudaMemcpyHostToDevice, st));
      L1B_CUDA(cudaMemcpyAsync(d_val, p->xs_val.data(), s * 8, cudaMemcpyHostToDevice, st));
    }
    scatter_sparse(d_sup, d_val, s, xd, p->n, st);
    sweep_apply(p->view, xd, res, st);        // instance.cpp:179
    vec_sub(res, p->d_b, p->m, st);           // :180
    sweep_apply_transpose(p->view, res, r, st);  // :182
    certificate(r, xd, p->tau, p->n, mx, st);
    double h[2];
    L1B_CUDA(cudaMemcpyAsync(h, mx, sizeof(h), cudaMemcpyDeviceToHost, st));
    for (void* q : {(void*)xd, (void*)res, (void*)r, (void*)mx, (void*)d_sup, (void*)d_val})
      L1B_CUDA(cudaFreeAsync(q, st));
    L1B_CUDA(cudaStreamSynchronize(st));
    out->max_support_violation = h[0];
    out->max_offsupport_violation = h[1];
    out->threshold = tol * p->tau;
    out->pass = h[0] <= out->threshold && h[1] <= out->threshold;
  });
}

void l1b_solver_cfg_default(l1b_solver_cfg* c) {
  std::memset(c, 0, sizeof(*c));
  c->solver = L1B_FISTA;
  c->max_iters = 100000;  // solvers.hpp:19-38
  c->max_seconds = 600.0;
  c->mu = 1e-5;
  c->eta = 0.1;
  c->pcg_max_iters = 1000;
  c->ls_max_backtracks = 50;
  c->grad_tol_rel = 1e-8;
  c->varpi = 1;
  c->block = 256;
  c->op = L1B_OP_AUTO;
  // L1B_ARITH=fma: the contracted arithmetic as the default of callers that
  // have no field for it (the reference-side drop-in maps l1bench::SolverConfig,
  // which knows no arithmetic mode, onto these defaults)
  const char* e = getenv("L1B_ARITH");
  c->arith = (e && (std::strcmp(e, "fma") == 0 || std::strcmp(e, "1") == 0)) ? L1B_ARITH_FMA : L1B_ARITH_EXACT;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// accessors used by the solver drivers (solvers.cu)
namespace l1b {
ProblemView problem_view(l1b_problem* p, bool need_sparse) {
  if (need_sparse) materialise(p);
  ProblemView v;
  v.device = p->device;
  v.stream = p->stream;
  v.m = p->m;
  v.n = p->n;
  v.tau = p->tau;
  v.lmax = p->lmax;
  v.tail_sq = p->tail_sq;
  v.tail_sq_band = p->tail_sq_band;
  v.fused_ok = fused_supported(p->view);
  v.b = p->d_b;
  v.A = p->rows();
  v.At = p->cols();
  v.op = &p->view;
  v.gram = nullptr;
  v.max_row_nnz = p->csr.max_len;
  v.max_col_nnz = p->csc.max_len;
  v.world = p->world;
  v.shard = p->sharded;
  v.rank = p->rank;
  v.row_begin = p->row_begin;
  v.row_end = p->row_end;
  v.halo = p->halo;
  v.general = p->general;
  v.col_begin = p->col_begin;
  v.col_end = p->col_end;
  v.col_slice = p->col_slice;
  if (p->d_b_win) {
    v.b_win = p->d_b_win - p->b_win_lo;
    v.b_win_lo = p->b_win_lo;
    v.b_win_hi = p->b_win_hi;
  }
  return v;
}
const double* problem_gram(l1b_problem* p) { return gram_diag_device(p); }

// sigma * prod cos(theta_s) over the right stages, indexed like view.sigma
// (global index; a shard: its window): the sigma of the contracted kernels,
// whose rotations run in the scaled form (StageTab::cprod, k_iter_rc.cu)
const double* problem_sigma_scaled(l1b_problem* p) {
  const uint64_t lo = p->sig_end ? p->sig_begin : 0, hi = p->sig_end ? p->sig_end : p->n;
  if (!p->d_sigma_c) {
    L1B_CUDA(cudaSetDevice(p->device));
    p->d_sigma_c = dev_alloc<double>(hi - lo, &p->device_bytes, p->stream);
    scale_copy(p->d_sigma, p->view.right.cprod, p->d_sigma_c, hi - lo, p->stream);
  }
  return p->d_sigma_c - lo;
}
}  // namespace l1b
