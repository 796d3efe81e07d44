// k_rng.cu -- std::mt19937_64 streams realised on the device, bit for bit.
//
// The generator's seeded streams (rng.hpp:14-56: Rng = std::mt19937_64,
// uniform_unit = (x >> 11) * 2^-53, uniform_in = lo + (hi - lo) * unit) are
// sequential by definition; the spectrum (linops.cpp:323-331) and the
// l1_subgradient fill (instance.cpp:33-35) draw one value per entry, n values
// per stream (C5: 2^32 each).  Instead of replaying them on one host core, the
// stream is cut into C chunks of J draws and every chunk starts from its own
// generator state, obtained by jumping ahead:
//
//   * Sequence form of the engine: x[0..311] from the seed, then
//       x[k+312] = x[k+156] ^ (((x[k] & UM) | (x[k+1] & LM)) >> 1) ^ (x[k+1] & 1 ? A : 0)
//     and draw k = temper(x[k+312]).  The window W_k = x[k..k+311] is the state
//     (the low 31 bits of x[k] never reach an output).
//   * W -> W_{+1} is GF(2)-linear with minimal polynomial P(t) of degree 19937
//     (times t, for those 31 don't-care bits).  P comes from Berlekamp-Massey
//     on 2 x 19937 output bits (host, once per process).
//   * W_{k+J} = sum_j p_j W_{k+j} for p(t) = t^J mod P: jumping is one
//     generation of 19937 words plus, for each of the 312 state words, an XOR
//     over the set coefficients -- the 312 words are independent; 3 x 312
//     threads each take a third of the coefficients, the whole sequence in
//     shared memory (158 KB).
//   * Chunk starts are built by a 16-ary tree of jumps (t^(16^l J) mod P by
//     repeated squaring on the host, cached): <= 3 levels x 15 sequential
//     jumps for C <= 4096 chunks.
//   * One CTA per chunk then runs the recurrence 156 words per step (the
//     largest independent batch) through a 1024-word shared-memory ring,
//     tempers, converts exactly like uniform_in and stores the draws that fall
//     in the requested window (coalesced), reducing min / max over all draws.
//
// The coordinate streams of CD / PCDM (uniform_index, mt_stream_indices) are
// cut the same way into chunks of J = 312 x 256 draws, but every chunk starts
// from the SAME base: window c = sum_j p^(c)_j W_j with p^(c) = t^(c J) mod P
// (host: one carry-less multiplication mod P per chunk, cached per process),
// so all chunk starts come from one kernel (mt_jump_many_kernel: CTAs split
// the coefficients of every jump, regenerate the base words their slice
// needs, and XOR their partial windows together).
//
// The spectrum's rejection (u <= lo, i.e. a raw draw with (x >> 11) == 0,
// probability 2^-53 per draw) would shift every later position: it is
// detected and reported, and the caller falls back to the sequential stream.
#include <immintrin.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "kernels.hpp"

namespace l1b {
namespace mt {

constexpr int NW = 312;          // state words
constexpr int MID = 156;         // recurrence offset (and the parallel batch)
constexpr int DEG = 19937;       // degree of P
constexpr int PW = 312;          // words of a polynomial of degree < 19937 (+1 spare bit)
constexpr int SEQ = DEG + NW;    // words a jump reads: x[0 .. 19936 + 311]
constexpr uint64_t MAT_A = 0xB5026F5AA96619E9ULL;
constexpr uint64_t UM = 0xFFFFFFFF80000000ULL;
constexpr uint64_t LM = 0x000000007FFFFFFFULL;
constexpr int FAN = 16;          // jump-tree fan-out
constexpr int MAX_CHUNKS = 4096;

__host__ __device__ inline uint64_t next_word(uint64_t x0, uint64_t x1, uint64_t xm) {
  const uint64_t y = (x0 & UM) | (x1 & LM);
  return xm ^ (y >> 1) ^ ((x1 & 1ull) ? MAT_A : 0ull);
}
__host__ __device__ inline uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

// std::mersenne_twister_engine::seed (initialisation multiplier 6364136223846793005)
void seed_window(uint64_t seed, uint64_t* w) {
  w[0] = seed;
  for (int i = 1; i < NW; ++i) w[i] = 6364136223846793005ULL * (w[i - 1] ^ (w[i - 1] >> 62)) + (uint64_t)i;
}

// ---------------------------------------------------------------------------
// host: characteristic polynomial and t^(2^e) mod P
using Poly = std::vector<uint64_t>;  // bit i = coefficient of t^i

// Berlekamp-Massey over GF(2) on s_k = bit 0 of draw k (any nonzero linear
// functional of the state has minimal polynomial P: P is primitive).
Poly compute_charpoly() {
  const int N = 2 * DEG + 64;
  std::vector<uint64_t> x(NW + N + 1);
  seed_window(5489u, x.data());
  for (int k = 0; k < N; ++k) x[k + NW] = next_word(x[k], x[k + 1], x[k + MID]);
  const int NWORDS = (N + 63) / 64 + 2;
  Poly rev(NWORDS + 2, 0);  // rev bit j = s_{N-1-j}
  for (int k = 0; k < N; ++k)
    if (temper(x[k + NW]) & 1ull) {
      const int j = N - 1 - k;
      rev[j >> 6] |= 1ull << (j & 63);
    }
  const int CW = NWORDS;
  Poly C(CW, 0), B(CW, 0), T;
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  for (int n = 0; n < N; ++n) {
    // d = sum_{i=0..L} c_i s_{n-i} = parity(C & rev[off ..]) with off = N-1-n
    const int off = N - 1 - n, ow = off >> 6, ob = off & 63;
    uint64_t acc = 0;
    for (int w = 0; w <= (L >> 6); ++w) {
      uint64_t r = rev[ow + w] >> ob;
      if (ob) r |= rev[ow + w + 1] << (64 - ob);
      acc ^= C[w] & r;
    }
    if (!(__builtin_popcountll(acc) & 1)) {
      ++m;
      continue;
    }
    auto add_shifted = [&](Poly& dst, const Poly& src, int sh) {  // dst ^= src << sh
      const int sw = sh >> 6, sb = sh & 63;
      for (int w = CW - 1; w >= sw; --w) {
        uint64_t v = src[w - sw] << sb;
        if (sb && w - sw - 1 >= 0) v |= src[w - sw - 1] >> (64 - sb);
        dst[w] ^= v;
      }
    };
    if (2 * L <= n) {
      T = C;
      add_shifted(C, B, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      add_shifted(C, B, m);
      ++m;
    }
  }
  if (L != DEG) throw std::runtime_error("mt19937_64 jump: characteristic polynomial has wrong degree");
  Poly P(PW + 1, 0);  // P = reverse of the connection polynomial, degree 19937
  for (int i = 0; i <= L; ++i)
    if ((C[(L - i) >> 6] >> ((L - i) & 63)) & 1ull) P[i >> 6] |= 1ull << (i & 63);
  return P;
}

struct Reducer {
  Poly P;
  std::vector<Poly> Psh;  // P << b for b = 0..63, PW + 2 words each
  Reducer() : P(compute_charpoly()) {
    Psh.assign(64, Poly(PW + 2, 0));
    for (int b = 0; b < 64; ++b)
      for (int w = 0; w <= PW; ++w) {
        Psh[b][w] ^= P[w] << b;
        if (b) Psh[b][w + 1] ^= P[w] >> (64 - b);
      }
  }
  // a^2 mod P for deg a < DEG
  Poly square(const Poly& a) const {
    Poly sq(2 * PW + 4, 0);
    for (int w = 0; w < PW; ++w) {
      uint64_t v = a[w];
      if (!v) continue;
      auto spread = [](uint64_t h) {  // 32 bits -> even bits of 64
        h &= 0xFFFFFFFFull;
        h = (h | (h << 16)) & 0x0000FFFF0000FFFFull;
        h = (h | (h << 8)) & 0x00FF00FF00FF00FFull;
        h = (h | (h << 4)) & 0x0F0F0F0F0F0F0F0Full;
        h = (h | (h << 2)) & 0x3333333333333333ull;
        h = (h | (h << 1)) & 0x5555555555555555ull;
        return h;
      };
      sq[2 * w] = spread(v);
      sq[2 * w + 1] = spread(v >> 32);
    }
    reduce(sq);
    sq.resize(PW);
    return sq;
  }
  void reduce(Poly& a) const {  // in place, a has >= 2 PW + 4 words
    for (int64_t i = 2 * (int64_t)DEG; i >= DEG; --i) {
      if (!((a[i >> 6] >> (i & 63)) & 1ull)) continue;
      const int64_t sh = i - DEG, sw = sh >> 6, sb = sh & 63;
      const Poly& q = Psh[sb];
      for (int w = 0; w < PW + 2 && sw + w < (int64_t)a.size(); ++w) a[sw + w] ^= q[w];
    }
  }
};

const Reducer& reducer() {
  static Reducer* r = new Reducer();
  return *r;
}

// t^(2^e) mod P (cached)
const Poly& pow2_poly(int e) {
  static std::mutex mu;
  static std::map<int, Poly> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(e);
  if (it != cache.end()) return it->second;
  const Reducer& R = reducer();
  // start from the largest cached exponent below e, else from t^1
  int e0 = 0;
  Poly cur(PW, 0);
  cur[0] = 2ull;  // t
  for (auto& kv : cache)
    if (kv.first <= e && kv.first > e0) {
      e0 = kv.first;
      cur = kv.second;
    }
  for (int k = e0; k < e; ++k) {
    cur = R.square(cur);
    cache.emplace(k + 1, cur);
  }
  return cache.emplace(e, cur).first->second;
}

// a * b mod P (deg a, deg b < DEG): carry-less products word by word, then the
// bit-serial reduction of Reducer
__attribute__((target("pclmul,sse2"))) void clmul_acc_hw(const uint64_t* a, const uint64_t* b, uint64_t* prod) {
  for (int i = 0; i < PW; ++i) {
    if (!a[i]) continue;
    const __m128i ai = _mm_set_epi64x(0, (long long)a[i]);
    for (int j = 0; j < PW; ++j) {
      if (!b[j]) continue;
      const __m128i r = _mm_clmulepi64_si128(ai, _mm_set_epi64x(0, (long long)b[j]), 0x00);
      prod[i + j] ^= (uint64_t)_mm_cvtsi128_si64(r);
      prod[i + j + 1] ^= (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(r, r));
    }
  }
}

void clmul_acc_sw(const uint64_t* a, const uint64_t* b, uint64_t* prod) {
  for (int i = 0; i < PW; ++i) {
    if (!a[i]) continue;
    for (int j = 0; j < PW; ++j) {
      const uint64_t y = b[j];
      if (!y) continue;
      uint64_t lo = 0, hi = 0;
      for (int k = 0; k < 64; ++k)
        if ((a[i] >> k) & 1ull) {
          lo ^= y << k;
          if (k) hi ^= y >> (64 - k);
        }
      prod[i + j] ^= lo;
      prod[i + j + 1] ^= hi;
    }
  }
}

Poly mulmod(const Poly& a, const Poly& b) {
  static const bool hw = __builtin_cpu_supports("pclmul");
  Poly prod(2 * PW + 4, 0);
  if (hw)
    clmul_acc_hw(a.data(), b.data(), prod.data());
  else
    clmul_acc_sw(a.data(), b.data(), prod.data());
  reducer().reduce(prod);
  prod.resize(PW);
  return prod;
}

// t^J mod P for any J (square-and-multiply over the cached t^(2^e))
Poly pow_t(uint64_t J) {
  Poly r(PW, 0);
  r[0] = 1;  // t^0
  for (int e = 0; J >> e; ++e)
    if ((J >> e) & 1ull) r = mulmod(r, pow2_poly(e));
  return r;
}

// t^(c J) mod P for c = 0 .. C-1, uploaded to the device (cached per device
// and J, grown on demand: one multiplication mod P per new chunk, once per
// process)
struct JumpTable {
  uint64_t J = 0;
  std::vector<Poly> host;  // host[c] = t^(c J)
  uint64_t* dev = nullptr;
  uint64_t dev_count = 0;
};

const uint64_t* jump_table(uint64_t J, uint64_t C, cudaStream_t st) {
  static std::mutex mu;
  static std::map<std::pair<int, uint64_t>, JumpTable> tabs;
  int dev = 0;
  L1B_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  JumpTable& t = tabs[{dev, J}];
  if (t.host.empty()) {
    t.J = J;
    Poly one(PW, 0);
    one[0] = 1;
    t.host.push_back(one);
  }
  if (t.dev_count >= C) return t.dev;
  const Poly step = pow_t(J);
  while (t.host.size() < C) t.host.push_back(mulmod(t.host.back(), step));
  uint64_t* d = nullptr;
  L1B_CUDA(cudaMalloc(&d, C * PW * 8));  // process-lifetime table (a few hundred KB)
  std::vector<uint64_t> flat(C * PW);
  for (uint64_t c = 0; c < C; ++c) std::memcpy(flat.data() + c * PW, t.host[c].data(), PW * 8);
  L1B_CUDA(cudaMemcpyAsync(d, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  if (t.dev) cudaFree(t.dev);
  t.dev = d;
  t.dev_count = C;
  return t.dev;
}

// ---------------------------------------------------------------------------
// device: jump tree
//
// CTA b takes window starts[b] and writes `count` windows out[b*FAN + t]
// (t < count, clipped at `total`): t = 0 is the start, t -> t+1 jumps by poly.
constexpr int JUMP_THREADS = 1024;
constexpr int JUMP_SLICES = 3;  // the coefficient words split over 3 x 312 threads
constexpr int SLICE_WORDS = (PW + JUMP_SLICES - 1) / JUMP_SLICES;

__global__ void __launch_bounds__(JUMP_THREADS) mt_jump_kernel(const uint64_t* __restrict__ starts,
                                                              const uint64_t* __restrict__ poly,
                                                              uint64_t total, uint64_t* __restrict__ out) {
  extern __shared__ uint64_t smem[];
  uint64_t* x = smem;          // SEQ words
  uint64_t* p = smem + SEQ;    // PW words
  uint64_t* part = p + PW;     // JUMP_SLICES x NW partial sums
  const int tid = threadIdx.x;
  const uint64_t first = (uint64_t)blockIdx.x * FAN;
  for (int i = tid; i < NW; i += blockDim.x) x[i] = starts[(uint64_t)blockIdx.x * NW + i];
  for (int i = tid; i < PW; i += blockDim.x) p[i] = poly[i];
  __syncthreads();
  for (int t = 0; t < FAN && first + t < total; ++t) {
    if (t > 0) {
      // x[312 ..] = the next DEG words (156 independent ones per step)
      for (int base = 0; base < DEG; base += MID) {
        const int k = base + tid;
        if (tid < MID && k < DEG) x[k + NW] = next_word(x[k], x[k + 1], x[k + MID]);
        __syncthreads();
      }
      // word k of the jumped window = XOR over set coefficients j of x[j + k]:
      // thread (slice, k) takes the coefficient words of its slice
      if (tid < JUMP_SLICES * NW) {
        const int k = tid % NW, sl = tid / NW;
        const int w1 = min(PW, (sl + 1) * SLICE_WORDS);
        uint64_t acc = 0;
        for (int w = sl * SLICE_WORDS; w < w1; ++w) {
          uint64_t bits = p[w];
          while (bits) {
            const int j = (w << 6) + __ffsll((long long)bits) - 1;
            bits &= bits - 1;
            acc ^= x[j + k];
          }
        }
        part[sl * NW + k] = acc;
      }
      __syncthreads();
      if (tid < NW) {
        uint64_t acc = 0;
        for (int sl = 0; sl < JUMP_SLICES; ++sl) acc ^= part[sl * NW + tid];
        x[tid] = acc;
      }
      __syncthreads();
    }
    for (int i = tid; i < NW; i += blockDim.x) out[(first + t) * NW + i] = x[i];
  }
}

// device: draws of chunk c = draws [c J, min((c+1) J, count)) of the stream
struct DrawArgs {
  uint64_t J, count, c0;   // chunk length, stream length, first chunk of the launch
  double lo, width, shift;
  int spectrum;            // 1: reject raw >> 11 == 0 and add shift (linops.cpp:323-331)
  uint64_t wlo, whi;       // window of draws stored to out[i - wlo]
  double* out;
  unsigned long long* minmax;  // [0] = min bits, [1] = max bits (non-negative values), or null
  int* rejected;
};

constexpr int DRAW_THREADS = 160;

__global__ void __launch_bounds__(DRAW_THREADS) mt_draw_kernel(const uint64_t* __restrict__ windows,
                                                              DrawArgs a) {
  __shared__ uint64_t ring[1024];
  __shared__ double red_min[DRAW_THREADS / 32], red_max[DRAW_THREADS / 32];
  const int tid = threadIdx.x;
  const uint64_t c = a.c0 + blockIdx.x;
  for (int i = tid; i < NW; i += blockDim.x) ring[i] = windows[c * NW + i];
  __syncthreads();
  const uint64_t d0 = c * a.J;
  const uint64_t d1 = min(a.count, d0 + a.J);
  double vmin = __longlong_as_double(0x7FF0000000000000LL), vmax = 0.0;
  bool rej = false;
  for (uint64_t base = 0; d0 + base < d1; base += MID) {
    const uint64_t k = base + (uint64_t)tid;
    if (tid < MID) {
      const uint64_t w = next_word(ring[k & 1023], ring[(k + 1) & 1023], ring[(k + MID) & 1023]);
      ring[(k + NW) & 1023] = w;
      const uint64_t d = d0 + k;
      if (d < d1) {
        const uint64_t raw = temper(w) >> 11;
        const double unit = (double)raw * 0x1.0p-53;
        double v = a.lo + a.width * unit;
        if (a.spectrum) {
          rej |= raw == 0;
          v = v + a.shift;
        }
        vmin = fmin(vmin, v);
        vmax = fmax(vmax, v);
        if (d >= a.wlo && d < a.whi) a.out[d - a.wlo] = v;
      }
    }
    __syncthreads();
  }
  if (a.minmax) {
    for (int o = 16; o; o >>= 1) {
      vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
      vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    if ((tid & 31) == 0) {
      red_min[tid >> 5] = vmin;
      red_max[tid >> 5] = vmax;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < DRAW_THREADS / 32; ++w) {
        vmin = fmin(vmin, red_min[w]);
        vmax = fmax(vmax, red_max[w]);
      }
      // non-negative doubles order like their bit patterns
      atomicMin(&a.minmax[0], (unsigned long long)__double_as_longlong(fmax(vmin, 0.0)));
      atomicMax(&a.minmax[1], (unsigned long long)__double_as_longlong(fmax(vmax, 0.0)));
      if (vmin < 0.0 || !(vmin == vmin)) atomicOr(a.rejected, 2);  // negative / NaN: not a spectrum
    }
  }
  if (rej) atomicOr(a.rejected, 1);
}


// ---------------------------------------------------------------------------
// uniform_index (rng.hpp:37-45) over a continuing stream, from the saved window
// W_k (312 words in global memory) to W_{k+count}, count a multiple of 312:
// out[q] = raw % n for draws k .. k + count - 1 (0xffffffff where raw >= lim:
// the reference redraws, the consumer skips the position).
//
// The recurrence is sequential.  Column j (0..155) of step t is
// y_j(t) = x[312 + 156 t + j] = next_word(A_j, N_j, B_j) with A_j = x[156 t + j]
// (two steps back), B_j = x[156 t + 156 + j] (one step back), N_j = A_{j+1}
// (j < 155) and N_155 = B_0.  Thread j keeps A_j, B_j in registers and
// thread 0 also runs column 155 (its N is column 0's own B), so the only
// values crossing threads are the neighbour's A and B, from two steps back:
// a thread runs TWO steps between block barriers, reading the (A, B) its
// neighbour published at the previous barrier.  The untempered words go to
// global memory; mt_temper_kernel (all SMs) tempers and reduces them after.
constexpr int IDX_THREADS = 160;
// CTA c continues from window win_in[c] for min(J, count - c J) words (a
// multiple of 2 MID) into words[c J ...]; the last CTA leaves its final window
// in win_out (one CTA = the sequential stream)
__global__ void __launch_bounds__(IDX_THREADS) mt_words_kernel(const uint64_t* __restrict__ win_in, uint64_t J,
                                                               uint64_t count, uint64_t* __restrict__ words,
                                                               uint64_t* __restrict__ win_out) {
  __shared__ uint64_t pub[2][2][MID];   // [buffer][A | B][column]
  const int tid = threadIdx.x;
  const bool rec = tid < MID - 1;       // columns 0..154 (thread 0 also 155)
  const uint64_t c = blockIdx.x, base0 = c * J;
  const uint64_t len = min(J, count - base0);
  const uint64_t* window = win_in + c * NW;
  words += base0;
  uint64_t A = 0, B = 0, A2 = 0, B2 = 0;  // A2 / B2: column 155 (thread 0)
  if (rec) {
    A = window[tid];
    B = window[MID + tid];
    pub[0][0][tid] = A;
    pub[0][1][tid] = B;
  }
  if (tid == 0) {
    A2 = window[MID - 1];
    B2 = window[2 * MID - 1];
    pub[0][0][MID - 1] = A2;
    pub[0][1][MID - 1] = B2;
  }
  __syncthreads();
  int p = 0;
  for (uint64_t base = 0; base < len; base += 2 * MID) {
    if (rec) {
      const uint64_t NA = pub[p][0][tid + 1], NB = pub[p][1][tid + 1];
      const uint64_t ya = next_word(A, NA, B);   // step t
      const uint64_t yb = next_word(B, NB, ya);  // step t + 1: A <- B, N <- neighbour's B, B <- ya
      if (tid == 0) {
        const uint64_t za = next_word(A2, B, B2);   // column 155, N = B_0(t)
        const uint64_t zb = next_word(B2, ya, za);  // N = B_0(t + 1) = y_0(t)
        A2 = za;
        B2 = zb;
        words[base + MID - 1] = za;
        words[base + 2 * MID - 1] = zb;
        pub[p ^ 1][0][MID - 1] = za;
        pub[p ^ 1][1][MID - 1] = zb;
      }
      A = ya;
      B = yb;
      words[base + tid] = ya;
      words[base + MID + tid] = yb;
      pub[p ^ 1][0][tid] = ya;
      pub[p ^ 1][1][tid] = yb;
    }
    p ^= 1;
    __syncthreads();
  }
  if (c + 1 != gridDim.x) return;
  if (rec) {
    win_out[tid] = A;
    win_out[MID + tid] = B;
  }
  if (tid == 0) {
    win_out[MID - 1] = A2;
    win_out[2 * MID - 1] = B2;
  }
}

// windows[c] ^= sum over the set coefficients j of t^(c J) mod P in slice
// blockIdx.x of x[j .. j + 312) (windows[c] zeroed before; chunk c = blockIdx.y
// + 1).  Every thread walks the same coefficient bits (uniform branches);
// thread k accumulates output word k.
constexpr int JM_SLICE = 39;  // polynomial words per CTA (8 slices)
constexpr int JM_SLICES = (PW + JM_SLICE - 1) / JM_SLICE;
constexpr int JM_THREADS = 320;
__global__ void __launch_bounds__(JM_THREADS) mt_jump_many_kernel(const uint64_t* __restrict__ window,
                                                                  const uint64_t* __restrict__ polys,
                                                                  uint64_t* __restrict__ windows) {
  __shared__ uint64_t xs[JM_SLICE * 64 + NW];
  __shared__ uint64_t ring[1024];
  __shared__ uint64_t pw[JM_SLICE];
  const uint64_t c = blockIdx.y + 1;
  const int w0 = blockIdx.x * JM_SLICE, w1 = min(PW, w0 + JM_SLICE);
  const int j0 = w0 * 64, jn = min(SEQ, w1 * 64 + NW) - j0;
  // x[j0 .. j0 + jn) of the base stream, regenerated here from the window (the
  // recurrence through a 1024-word ring, 156 words per step): no separate
  // sequential launch ahead of the jump
  for (int i = threadIdx.x; i < NW; i += blockDim.x) {
    const uint64_t v = window[i];
    ring[i] = v;
    if (i >= j0 && i < j0 + jn) xs[i - j0] = v;
  }
  for (int i = threadIdx.x; i < w1 - w0; i += blockDim.x) pw[i] = polys[c * PW + w0 + i];
  __syncthreads();
  for (int base = 0; base + NW < j0 + jn; base += MID) {
    const int k = base + threadIdx.x;  // x[k + 312] from x[k], x[k + 1], x[k + 156]
    if (threadIdx.x < MID && k + NW < j0 + jn) {
      const uint64_t v = next_word(ring[k & 1023], ring[(k + 1) & 1023], ring[(k + MID) & 1023]);
      ring[(k + NW) & 1023] = v;
      if (k + NW >= j0) xs[k + NW - j0] = v;
    }
    __syncthreads();
  }
  const int k = threadIdx.x;
  if (k >= NW) return;
  uint64_t acc = 0;
  for (int w = 0; w < w1 - w0; ++w) {
    const uint64_t bits = pw[w];  // the same for every thread: uniform predicates
    const uint64_t* xb = xs + (w << 6) + k;
#pragma unroll
    for (int b = 0; b < 64; ++b)
      if ((bits >> b) & 1ull) acc ^= xb[b];
  }
  if (acc) atomicXor((unsigned long long*)&windows[c * NW + k], (unsigned long long)acc);
}

template <bool POW2>
__global__ void mt_temper_kernel(const uint64_t* __restrict__ words, uint64_t count, uint64_t n, uint64_t lim,
                                 uint32_t* __restrict__ out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t raw = temper(words[k]);
    out[k] = raw >= lim ? 0xffffffffu : (uint32_t)(POW2 ? (raw & (n - 1)) : raw % n);
  }
}

}  // namespace mt

// Host restatement of the jump (the device kernel's arithmetic, one thread):
// the 64-bit outputs number 2^log2_jump, 2^log2_jump + 1, ... of
// std::mt19937_64(seed), reached by t^(2^log2_jump) mod P -- checks the
// polynomial machinery against a sequential stream without a GPU.
void host_draws_after_jump(uint64_t seed, int log2_jump, uint64_t count, uint64_t* out) {
  using namespace mt;
  std::vector<uint64_t> x(SEQ + 1);
  seed_window(seed, x.data());
  if (log2_jump >= 0) {
    const Poly& p = pow2_poly(log2_jump);
    for (int k = 0; k < DEG; ++k) x[k + NW] = next_word(x[k], x[k + 1], x[k + MID]);
    uint64_t w[NW] = {};
    for (int j = 0; j < DEG; ++j)
      if ((p[j >> 6] >> (j & 63)) & 1ull)
        for (int i = 0; i < NW; ++i) w[i] ^= x[j + i];
    std::copy(w, w + NW, x.begin());
  }
  std::vector<uint64_t> r(x.begin(), x.begin() + NW);
  r.resize(NW + count + 1);
  for (uint64_t k = 0; k < count; ++k) {
    r[k + NW] = next_word(r[k], r[k + 1], r[k + MID]);
    out[k] = temper(r[k + NW]);
  }
}

// ---------------------------------------------------------------------------
bool device_uniform_draws(uint64_t seed, uint64_t count, double lo, double hi, bool spectrum,
                          double shift, uint64_t wlo, uint64_t whi, double* d_out, double* vmin,
                          double* vmax, cudaStream_t st, int min_log2_chunk) {
  using namespace mt;
  if (count == 0) return true;
  whi = std::min(whi, count);
  // chunk length J = 2^e: at most MAX_CHUNKS chunks
  int e = std::max(min_log2_chunk, 1);
  while (((count + (1ull << e) - 1) >> e) > (uint64_t)MAX_CHUNKS) ++e;
  const uint64_t J = 1ull << e;
  const uint64_t C = (count + J - 1) >> e;
  int levels = 0;
  for (uint64_t span = 1; span < C; span *= FAN) ++levels;  // C <= FAN^levels
  // windows of every level, ping-pong
  uint64_t* d_poly = nullptr;
  uint64_t *d_a = nullptr, *d_b = nullptr;
  L1B_CUDA(cudaMallocAsync(&d_poly, (size_t)levels * PW * 8 + 8, st));
  L1B_CUDA(cudaMallocAsync(&d_a, (size_t)C * NW * 8, st));
  L1B_CUDA(cudaMallocAsync(&d_b, (size_t)C * NW * 8, st));
  {
    uint64_t w0[NW];
    seed_window(seed, w0);
    L1B_CUDA(cudaMemcpyAsync(d_a, w0, sizeof(w0), cudaMemcpyHostToDevice, st));
    std::vector<uint64_t> polys((size_t)levels * PW);
    for (int l = 0; l < levels; ++l) {  // level l (from the top) jumps by J * FAN^(levels-1-l)
      const Poly& q = pow2_poly(e + 4 * (levels - 1 - l));
      std::memcpy(polys.data() + (size_t)l * PW, q.data(), PW * 8);
    }
    if (levels) {
      L1B_CUDA(cudaMemcpyAsync(d_poly, polys.data(), polys.size() * 8, cudaMemcpyHostToDevice, st));
      // the host vector must outlive the copy
      L1B_CUDA(cudaStreamSynchronize(st));
    }
  }
  const int smem = (SEQ + PW + JUMP_SLICES * NW) * 8;
  L1B_CUDA(cudaFuncSetAttribute(mt_jump_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  uint64_t n_prev = 1;
  for (int l = 0; l < levels; ++l) {
    uint64_t stride = 1;  // chunks per window at this level
    for (int k = 0; k < levels - 1 - l; ++k) stride *= FAN;
    const uint64_t n_here = (C + stride - 1) / stride;
    mt_jump_kernel<<<(unsigned)n_prev, JUMP_THREADS, smem, st>>>(d_a, d_poly + (size_t)l * PW, n_here, d_b);
    L1B_LAUNCHED();
    std::swap(d_a, d_b);
    n_prev = n_here;
  }
  unsigned long long* d_mm = nullptr;
  int* d_rej = nullptr;
  L1B_CUDA(cudaMallocAsync(&d_mm, 2 * sizeof(unsigned long long) + sizeof(int) + 4, st));
  d_rej = reinterpret_cast<int*>(d_mm + 2);
  const unsigned long long init[2] = {0x7FF0000000000000ull, 0ull};
  L1B_CUDA(cudaMemcpyAsync(d_mm, init, sizeof(init), cudaMemcpyHostToDevice, st));
  L1B_CUDA(cudaMemsetAsync(d_rej, 0, sizeof(int), st));
  DrawArgs a;
  a.J = J;
  a.count = count;
  a.lo = lo;
  a.width = hi - lo;
  a.shift = shift;
  a.spectrum = spectrum ? 1 : 0;
  a.wlo = wlo;
  a.whi = whi;
  a.out = d_out;
  const bool reduce = vmin || vmax;
  a.minmax = reduce ? d_mm : nullptr;
  a.rejected = d_rej;
  // without a reduction only the chunks meeting the window run
  uint64_t c_lo = 0, c_hi = C;
  if (!reduce) {
    c_lo = wlo >> e;
    c_hi = whi > wlo ? ((whi - 1) >> e) + 1 : c_lo;
  }
  a.c0 = c_lo;
  if (c_hi > c_lo) {
    mt_draw_kernel<<<(unsigned)(c_hi - c_lo), DRAW_THREADS, 0, st>>>(d_a, a);
    L1B_LAUNCHED();
  }
  unsigned long long mm[2];
  int rej = 0;
  L1B_CUDA(cudaMemcpyAsync(mm, d_mm, sizeof(mm), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaMemcpyAsync(&rej, d_rej, sizeof(int), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  for (void* q : {(void*)d_poly, (void*)d_a, (void*)d_b, (void*)d_mm}) L1B_CUDA(cudaFreeAsync(q, st));
  if (rej & 1) return false;  // a rejected draw shifts the stream: caller replays it sequentially
  if (reduce) {
    double mn, mx;
    std::memcpy(&mn, &mm[0], 8);
    std::memcpy(&mx, &mm[1], 8);
    if (rej & 2) mn = -1.0;  // a negative or NaN value: the caller's validation rejects it
    if (vmin) *vmin = mn;
    if (vmax) *vmax = mx;
  }
  return true;
}

void mt_seed_state(uint64_t seed, uint64_t* w312) { mt::seed_window(seed, w312); }

// Chunks of kIdxChunk draws (a multiple of 312) start from windows jumped
// ahead by t^(c J) mod P, all from the same base sequence: one sequential
// generation of 19937 words, one jump kernel for every chunk, one CTA per chunk
// for the recurrence, then the tempering over all SMs.  Short streams (one
// chunk) run the recurrence directly.
constexpr uint64_t kIdxChunk = 312 * 256;

namespace {
// the untempered words of draws [0, count) of the stream continued from
// d_window (count a multiple of 312; d_window advanced past them)
void mt_stream_words(uint64_t* d_window, uint64_t count, uint64_t* words, cudaStream_t st) {
  using namespace mt;
  const uint64_t C = (count + kIdxChunk - 1) / kIdxChunk;
  if (C == 1) {
    mt_words_kernel<<<1, IDX_THREADS, 0, st>>>(d_window, count, count, words, d_window);
    L1B_LAUNCHED();
  } else {
    const uint64_t* polys = jump_table(kIdxChunk, C, st);
    uint64_t* wins = nullptr;
    L1B_CUDA(cudaMallocAsync(&wins, C * NW * 8, st));
    L1B_CUDA(cudaMemcpyAsync(wins, d_window, NW * 8, cudaMemcpyDeviceToDevice, st));
    L1B_CUDA(cudaMemsetAsync(wins + NW, 0, (C - 1) * NW * 8, st));
    mt_jump_many_kernel<<<dim3(JM_SLICES, (unsigned)(C - 1)), JM_THREADS, 0, st>>>(d_window, polys, wins);
    L1B_LAUNCHED();
    mt_words_kernel<<<(unsigned)C, IDX_THREADS, 0, st>>>(wins, kIdxChunk, count, words, d_window);
    L1B_LAUNCHED();
    L1B_CUDA(cudaFreeAsync(wins, st));
  }
}

__global__ void mt_temper_raw_kernel(uint64_t* words, uint64_t count) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < count;
       k += (uint64_t)gridDim.x * blockDim.x)
    words[k] = mt::temper(words[k]);
}
}  // namespace

uint64_t mt_stream_raw(uint64_t* d_window, uint64_t count, uint64_t* d_out, cudaStream_t st) {
  count = (count + 2 * mt::MID - 1) / (2 * mt::MID) * (2 * mt::MID);
  if (count == 0) return 0;
  mt_stream_words(d_window, count, d_out, st);
  mt_temper_raw_kernel<<<grid_for(count), kThreads, 0, st>>>(d_out, count);
  L1B_LAUNCHED();
  return count;
}

uint64_t coord_index_limit(uint64_t n) {
  uint64_t top = UINT64_MAX;
  if (const char* e = getenv("L1B_TEST_INDEX_REJECT")) {
    const int s = atoi(e);
    if (s >= 1 && s <= 63) top -= UINT64_MAX >> s;
  }
  return top - top % n;
}

uint64_t mt_stream_indices(uint64_t* d_window, uint64_t count, uint64_t n, uint32_t* d_out,
                           uint64_t* d_words, cudaStream_t st) {
  using namespace mt;
  count = (count + 2 * MID - 1) / (2 * MID) * (2 * MID);
  if (count == 0) return 0;
  const uint64_t lim = coord_index_limit(n);
  uint64_t* words = d_words;
  if (!words) L1B_CUDA(cudaMallocAsync(&words, count * 8, st));
  mt_stream_words(d_window, count, words, st);
  const int grid = grid_for(count);
  if ((n & (n - 1)) == 0) mt::mt_temper_kernel<true><<<grid, kThreads, 0, st>>>(words, count, n, lim, d_out);
  else mt::mt_temper_kernel<false><<<grid, kThreads, 0, st>>>(words, count, n, lim, d_out);
  L1B_LAUNCHED();
  if (!d_words) L1B_CUDA(cudaFreeAsync(words, st));
  return count;
}

// host restatement of the chunked jump (tests): raw outputs c J .. c J + count - 1
// of std::mt19937_64(seed) through t^(c J) mod P, J = the index-stream chunk
void host_draws_after_chunk_jump(uint64_t seed, uint64_t c, uint64_t count, uint64_t* out) {
  using namespace mt;
  std::vector<uint64_t> x(SEQ + 1);
  seed_window(seed, x.data());
  if (c) {
    const Poly p = pow_t(kIdxChunk * c);
    for (int k = 0; k < DEG; ++k) x[k + NW] = next_word(x[k], x[k + 1], x[k + MID]);
    uint64_t w[NW] = {};
    for (int j = 0; j < DEG; ++j)
      if ((p[j >> 6] >> (j & 63)) & 1ull)
        for (int i = 0; i < NW; ++i) w[i] ^= x[j + i];
    std::copy(w, w + NW, x.begin());
  }
  std::vector<uint64_t> r(x.begin(), x.begin() + NW);
  r.resize(NW + count + 1);
  for (uint64_t k = 0; k < count; ++k) {
    r[k + NW] = next_word(r[k], r[k + 1], r[k + MID]);
    out[k] = temper(r[k + NW]);
  }
}

}  // namespace l1b
