/*
 * l1oracle.c -- CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY (see l1oracle.h).  Each function cites the reference
 * lines it restates; paths are relative to /root/reference/proj.
 */
#include "l1oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* RNG -- std::mt19937_64 (C++ [rand.eng.mers] parameters) and the helpers of
 * include/l1bench/rng.hpp:14-45.                                            */

void lo_rng_seed(lo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->idx = 312;
}

static void lo_twist(lo_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  for (int i = 0; i < 312; ++i) {
    uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
  }
  r->idx = 0;
}

uint64_t lo_rng_next(lo_rng* r) {
  if (r->idx >= 312) lo_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:19-24 */
uint64_t lo_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:27-29 */
double lo_uniform_unit(lo_rng* r) { return (double)(lo_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:48-56: Box-Muller, u1 in (0, 1) */
double lo_normal(lo_rng* r) {
  double u1;
  do {
    u1 = lo_uniform_unit(r);
  } while (u1 <= 0.0);
  const double u2 = lo_uniform_unit(r);
  const double two_pi = 6.283185307179586476925286766559;
  return sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
}

/* rng.hpp:32-34 */
double lo_uniform_in(lo_rng* r, double lo, double hi) { return lo + (hi - lo) * lo_uniform_unit(r); }

/* Test hook (not in the reference): lowers the rejection limit of the CD /
 * PCDM coordinate draws by UINT64_MAX >> s, as L1B_TEST_INDEX_REJECT does in
 * the library, so the redraw paths meet the oracle.  0 = the reference's. */
static int g_index_reject = 0;
void lo_set_index_reject(int s) { g_index_reject = s; }

static uint64_t lo_coord_index(lo_rng* r, uint64_t n) {
  uint64_t top = UINT64_MAX;
  if (g_index_reject >= 1 && g_index_reject <= 63) top -= UINT64_MAX >> g_index_reject;
  const uint64_t limit = top - top % n;
  uint64_t x;
  do {
    x = lo_rng_next(r);
  } while (x >= limit);
  return x % n;
}

/* rng.hpp:37-45 */
uint64_t lo_uniform_index(lo_rng* r, uint64_t n) {
  if (n == 0) abort();
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = lo_rng_next(r);
  } while (x >= limit);
  return x % n;
}

/* ------------------------------------------------------------------------ */
/* Dense sweeps (linops.cpp:20-30, 81-108)                                   */

static inline void rot(double* vi, double* vj, double c, double s, int transposed) {
  const double a = *vi, b = *vj;
  if (transposed) {
    *vi = c * a + s * b;
    *vj = -s * a + c * b;
  } else {
    *vi = c * a - s * b;
    *vj = s * a + c * b;
  }
}

void lo_apply_stage(double* v, uint64_t dim, int offset, double theta, int transposed) {
  const double c = cos(theta), s = sin(theta);
  for (uint64_t k = (uint64_t)offset; k + 1 < dim; k += 2) rot(&v[k], &v[k + 1], c, s, transposed);
}

/* linops.cpp:422-446 */
void lo_apply(const lo_op* A, const double* x, double* y) {
  const uint64_t m = A->m, n = A->n;
  double* v = (double*)malloc(n * sizeof(double));
  double* t = (double*)malloc(m * sizeof(double));
  memcpy(v, x, n * sizeof(double));
  for (uint32_t s = 0; s < A->n_right; ++s) lo_apply_stage(v, n, A->right_offset[s], A->right_theta[s], 1);
  for (uint64_t i = 0; i < m; ++i) {
    const uint64_t j = A->p2 ? A->p2[i] : i;
    t[i] = j < n ? A->sigma[j] * v[j] : 0.0;
  }
  for (uint32_t s = A->n_left; s-- > 0;) lo_apply_stage(t, m, A->left_offset[s], A->left_theta[s], 0);
  for (uint64_t i = 0; i < m; ++i) y[i] = A->p1 ? t[A->p1[i]] : t[i];
  free(v);
  free(t);
}

/* linops.cpp:448-473 */
void lo_apply_transpose(const lo_op* A, const double* y, double* x) {
  const uint64_t m = A->m, n = A->n;
  double* t = (double*)malloc(m * sizeof(double));
  double* v = (double*)calloc(n, sizeof(double));
  if (A->p1) {
    for (uint64_t i = 0; i < m; ++i) t[A->p1[i]] = y[i];
  } else {
    memcpy(t, y, m * sizeof(double));
  }
  for (uint32_t s = 0; s < A->n_left; ++s) lo_apply_stage(t, m, A->left_offset[s], A->left_theta[s], 1);
  if (A->p2) {
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t j = A->p2[i];
      if (j < n) v[j] = A->sigma[j] * t[i];
    }
  } else {
    for (uint64_t j = 0; j < n; ++j) v[j] = A->sigma[j] * t[j];
  }
  for (uint32_t s = A->n_right; s-- > 0;) lo_apply_stage(v, n, A->right_offset[s], A->right_theta[s], 0);
  memcpy(x, v, n * sizeof(double));
  free(t);
  free(v);
}

/* linops.cpp:475-490 */
void lo_apply_gram_inverse(const lo_op* A, const double* vin, double* out) {
  const uint64_t n = A->n;
  double* u = (double*)malloc(n * sizeof(double));
  memcpy(u, vin, n * sizeof(double));
  for (uint32_t s = 0; s < A->n_right; ++s) lo_apply_stage(u, n, A->right_offset[s], A->right_theta[s], 1);
  for (uint64_t i = 0; i < n; ++i) u[i] /= A->sigma[i] * A->sigma[i];
  for (uint32_t s = A->n_right; s-- > 0;) lo_apply_stage(u, n, A->right_offset[s], A->right_theta[s], 0);
  memcpy(out, u, n * sizeof(double));
  free(u);
}

/* linops.cpp:560-564 via Spectrum::sigma_max (:349-352) */
double lo_gram_lmax(const lo_op* A) {
  double s = A->sigma[0];
  for (uint64_t i = 1; i < A->n; ++i)
    if (A->sigma[i] > s) s = A->sigma[i];
  return s * s;
}

/* linops.cpp:224-239 */
void lo_permutation_realize(uint64_t n, uint64_t seed, uint32_t* map, uint32_t* inv) {
  for (uint64_t i = 0; i < n; ++i) map[i] = (uint32_t)i;
  lo_rng r;
  lo_rng_seed(&r, seed);
  for (uint64_t i = n; i > 1; --i) {
    const uint64_t j = lo_uniform_index(&r, i);
    const uint32_t tmp = map[i - 1];
    map[i - 1] = map[j];
    map[j] = tmp;
  }
  for (uint64_t i = 0; i < n; ++i) inv[map[i]] = (uint32_t)i;
}

/* linops.cpp:320-331 */
void lo_spectrum_uniform(uint64_t n, double lo, double hi, double shift, uint64_t seed,
                         double* sigma) {
  lo_rng r;
  lo_rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) {
    double u;
    do {
      u = lo_uniform_in(&r, lo, hi);
    } while (u <= lo);
    sigma[i] = u + shift;
  }
}

void lo_uniform_stream_window(uint64_t seed, uint64_t count, double lo, double hi, int spectrum,
                              double shift, uint64_t wlo, uint64_t whi, double* out, double* vmin,
                              double* vmax) {
  lo_rng r;
  lo_rng_seed(&r, seed);
  double mn = 0.0, mx = 0.0;
  for (uint64_t i = 0; i < count; ++i) {
    double v;
    if (spectrum) {
      double u;
      do {
        u = lo_uniform_in(&r, lo, hi);
      } while (u <= lo);
      v = u + shift;
    } else {
      v = lo_uniform_in(&r, lo, hi);
    }
    if (i == 0 || v < mn) mn = v;
    if (i == 0 || v > mx) mx = v;
    if (i >= wlo && i < whi) out[i - wlo] = v;
  }
  if (vmin) *vmin = mn;
  if (vmax) *vmax = mx;
}

/* ------------------------------------------------------------------------ */
/* Sparse accumulator sweeps (linops.cpp:113-192)                            */

struct lo_ws {
  uint64_t size;
  double* acc;
  uint8_t* flag;
  uint32_t* active;
  uint64_t n_active;
  uint32_t* scratch;
  /* carry buffers for the permutation/sigma hand-offs (linops.cpp:576-593) */
  uint32_t* cidx;
  double* cval;
};

lo_ws* lo_ws_create(uint64_t size) {
  lo_ws* ws = (lo_ws*)calloc(1, sizeof(lo_ws));
  ws->size = size;
  ws->acc = (double*)calloc(size, sizeof(double));
  ws->flag = (uint8_t*)calloc(size, 1);
  ws->active = (uint32_t*)malloc(size * sizeof(uint32_t));
  ws->scratch = (uint32_t*)malloc(size * sizeof(uint32_t));
  ws->cidx = (uint32_t*)malloc(size * sizeof(uint32_t));
  ws->cval = (double*)malloc(size * sizeof(double));
  return ws;
}

void lo_ws_free(lo_ws* ws) {
  if (!ws) return;
  free(ws->acc);
  free(ws->flag);
  free(ws->active);
  free(ws->scratch);
  free(ws->cidx);
  free(ws->cval);
  free(ws);
}

/* linops.cpp:124-132 */
static inline void spa_activate(lo_ws* ws, uint32_t idx, double value) {
  if (!ws->flag[idx]) {
    ws->flag[idx] = 1;
    ws->acc[idx] = value;
    ws->active[ws->n_active++] = idx;
  } else {
    ws->acc[idx] += value;
  }
}

/* linops.cpp:134-140 */
static void spa_clear(lo_ws* ws) {
  for (uint64_t k = 0; k < ws->n_active; ++k) {
    ws->acc[ws->active[k]] = 0.0;
    ws->flag[ws->active[k]] = 0;
  }
  ws->n_active = 0;
}

/* linops.cpp:142-165 (paired stages) */
static void spa_stage(lo_ws* ws, uint64_t dim, int offset_i, double theta, int transposed) {
  const double c = cos(theta), s = sin(theta);
  const uint32_t offset = (uint32_t)offset_i;
  const uint64_t n0 = ws->n_active;
  memcpy(ws->scratch, ws->active, n0 * sizeof(uint32_t));
  for (uint64_t k = 0; k < n0; ++k) {
    const uint32_t idx = ws->scratch[k];
    if (idx < offset) continue;
    const uint32_t rel = idx - offset;
    if (rel % 2 == 0) {
      if ((uint64_t)idx + 1 < dim && !ws->flag[idx + 1]) spa_activate(ws, idx + 1, 0.0);
    } else {
      if (!ws->flag[idx - 1]) spa_activate(ws, idx - 1, 0.0);
    }
  }
  for (uint64_t k = 0; k < ws->n_active; ++k) {
    const uint32_t idx = ws->active[k];
    if (idx < offset) continue;
    const uint32_t rel = idx - offset;
    if (rel % 2 != 0 || (uint64_t)idx + 1 >= dim) continue;
    rot(&ws->acc[idx], &ws->acc[idx + 1], c, s, transposed);
  }
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* linops.cpp:179-192 */
static uint64_t spa_emit_sorted(lo_ws* ws, uint32_t* idx, double* val) {
  qsort(ws->active, ws->n_active, sizeof(uint32_t), cmp_u32);
  uint64_t k = 0;
  for (uint64_t a = 0; a < ws->n_active; ++a) {
    const double v = ws->acc[ws->active[a]];
    if (v != 0.0) {
      idx[k] = ws->active[a];
      val[k] = v;
      ++k;
    }
  }
  spa_clear(ws);
  return k;
}

/* linops.cpp:566-595 */
uint64_t lo_column(const lo_op* A, uint64_t j, lo_ws* ws, uint32_t* idx, double* val) {
  spa_activate(ws, (uint32_t)j, 1.0);
  for (uint32_t s = 0; s < A->n_right; ++s) spa_stage(ws, A->n, A->right_offset[s], A->right_theta[s], 1);
  uint64_t nc = ws->n_active;
  for (uint64_t k = 0; k < nc; ++k) {
    ws->cidx[k] = ws->active[k];
    ws->cval[k] = ws->acc[ws->active[k]];
  }
  spa_clear(ws);
  for (uint64_t k = 0; k < nc; ++k) {
    const uint32_t src = ws->cidx[k];
    const uint32_t img = A->p2 ? A->p2_inv[src] : src;
    spa_activate(ws, img, A->sigma[src] * ws->cval[k]);
  }
  for (uint32_t s = A->n_left; s-- > 0;) spa_stage(ws, A->m, A->left_offset[s], A->left_theta[s], 0);
  if (A->p1) {
    nc = ws->n_active;
    for (uint64_t k = 0; k < nc; ++k) {
      ws->cidx[k] = ws->active[k];
      ws->cval[k] = ws->acc[ws->active[k]];
    }
    spa_clear(ws);
    for (uint64_t k = 0; k < nc; ++k) spa_activate(ws, A->p1_inv[ws->cidx[k]], ws->cval[k]);
  }
  return spa_emit_sorted(ws, idx, val);
}

/* linops.cpp:597-619 */
uint64_t lo_row(const lo_op* A, uint64_t i, lo_ws* ws, uint32_t* idx, double* val) {
  spa_activate(ws, A->p1 ? A->p1[i] : (uint32_t)i, 1.0);
  for (uint32_t s = 0; s < A->n_left; ++s) spa_stage(ws, A->m, A->left_offset[s], A->left_theta[s], 1);
  const uint64_t nc = ws->n_active;
  for (uint64_t k = 0; k < nc; ++k) {
    ws->cidx[k] = ws->active[k];
    ws->cval[k] = ws->acc[ws->active[k]];
  }
  spa_clear(ws);
  for (uint64_t k = 0; k < nc; ++k) {
    const uint32_t src = ws->cidx[k];
    const uint32_t t = A->p2 ? A->p2[src] : src;
    if (t < A->n) spa_activate(ws, t, A->sigma[t] * ws->cval[k]);
  }
  for (uint32_t s = A->n_right; s-- > 0;) spa_stage(ws, A->n, A->right_offset[s], A->right_theta[s], 0);
  return spa_emit_sorted(ws, idx, val);
}

/* linops.cpp:533-558: (A^T A)_ii summed in sparse-accumulator activation order */
void lo_gram_diagonal(const lo_op* A, double* d) {
  const uint64_t n = A->n;
  if (A->n_right == 0) {
    for (uint64_t i = 0; i < n; ++i) d[i] = A->sigma[i] * A->sigma[i];
    return;
  }
  lo_ws* ws = lo_ws_create(n);
  for (uint64_t i = 0; i < n; ++i) {
    spa_activate(ws, (uint32_t)i, 1.0);
    for (uint32_t s = 0; s < A->n_right; ++s) spa_stage(ws, n, A->right_offset[s], A->right_theta[s], 1);
    double acc = 0.0;
    for (uint64_t k = 0; k < ws->n_active; ++k) {
      const uint32_t idx = ws->active[k];
      const double w = ws->acc[idx];
      acc += A->sigma[idx] * A->sigma[idx] * w * w;
    }
    d[i] = acc;
    spa_clear(ws);
  }
  lo_ws_free(ws);
}

static uint64_t build_lines(const lo_op* A, int rows, uint64_t* ptr, uint32_t* idx, double* val,
                            uint64_t cap) {
  const uint64_t dim = rows ? A->m : A->n;
  const uint64_t wsz = A->m > A->n ? A->m : A->n;
  lo_ws* ws = lo_ws_create(wsz);
  uint32_t* ti = (uint32_t*)malloc(wsz * sizeof(uint32_t));
  double* tv = (double*)malloc(wsz * sizeof(double));
  uint64_t nnz = 0;
  ptr[0] = 0;
  for (uint64_t i = 0; i < dim; ++i) {
    const uint64_t k = rows ? lo_row(A, i, ws, ti, tv) : lo_column(A, i, ws, ti, tv);
    if (nnz + k > cap) {
      nnz = UINT64_MAX;
      break;
    }
    memcpy(idx + nnz, ti, k * sizeof(uint32_t));
    memcpy(val + nnz, tv, k * sizeof(double));
    nnz += k;
    ptr[i + 1] = nnz;
  }
  free(ti);
  free(tv);
  lo_ws_free(ws);
  return nnz;
}

uint64_t lo_build_csr(const lo_op* A, uint64_t* ptr, uint32_t* idx, double* val, uint64_t cap) {
  return build_lines(A, 1, ptr, idx, val, cap);
}

uint64_t lo_build_csc(const lo_op* A, uint64_t* ptr, uint32_t* idx, double* val, uint64_t cap) {
  return build_lines(A, 0, ptr, idx, val, cap);
}

void lo_csr_matvec(uint64_t rows, const uint64_t* ptr, const uint32_t* idx, const double* val,
                   const double* x, double* y) {
  for (uint64_t i = 0; i < rows; ++i) {
    double s = 0.0;
    for (uint64_t p = ptr[i]; p < ptr[i + 1]; ++p) s += val[p] * x[idx[p]];
    y[i] = s;
  }
}

/* ------------------------------------------------------------------------ */
/* Generator                                                                 */

/* open-addressing set standing in for std::unordered_set (solution.cpp:68) */
typedef struct {
  uint64_t* keys;
  uint8_t* used;
  uint64_t mask;
} u64set;

static int u64set_insert(u64set* s, uint64_t key) {
  uint64_t h = (key * 0x9E3779B97F4A7C15ULL) & s->mask;
  while (s->used[h]) {
    if (s->keys[h] == key) return 0;
    h = (h + 1) & s->mask;
  }
  s->used[h] = 1;
  s->keys[h] = key;
  return 1;
}

/* solution.cpp:47-75 (Floyd sampling; set order is irrelevant after the sort) */
uint64_t lo_uniform_sparse_solution(uint64_t n, uint64_t s, double gamma, lo_rng* rng,
                                    uint32_t* support, double* values) {
  if (s == 0) return 0;
  uint64_t cap = 1;
  while (cap < 4 * s) cap <<= 1;
  u64set set = {(uint64_t*)malloc(cap * sizeof(uint64_t)), (uint8_t*)calloc(cap, 1), cap - 1};
  uint64_t k = 0;
  for (uint64_t j = n - s; j < n; ++j) {
    const uint64_t t = lo_uniform_index(rng, j + 1);
    if (u64set_insert(&set, t)) {
      support[k++] = (uint32_t)t;
    } else {
      u64set_insert(&set, j);
      support[k++] = (uint32_t)j;
    }
  }
  qsort(support, s, sizeof(uint32_t), cmp_u32);
  for (uint64_t q = 0; q < s; ++q) {
    double v;
    do {
      v = lo_uniform_in(rng, -gamma, gamma);
    } while (v == 0.0);
    values[q] = v;
  }
  free(set.keys);
  free(set.used);
  return s;
}

/* instance.cpp:28-42 (interior_uniform fill) */
void lo_l1_subgradient(uint64_t n, const uint32_t* support, const double* values, uint64_t s,
                       double bound, lo_rng* rng, double* g) {
  for (uint64_t i = 0; i < n; ++i) g[i] = lo_uniform_in(rng, -bound, bound);
  for (uint64_t k = 0; k < s; ++k) g[support[k]] = values[k] > 0.0 ? 1.0 : -1.0;
}

/* instance.cpp:53-89 */
double lo_generate_instance(const lo_op* A, double tau, const uint32_t* support,
                            const double* values, uint64_t s, double fill_bound, lo_rng* rng,
                            double* b) {
  const uint64_t m = A->m, n = A->n;
  double* g = (double*)malloc(n * sizeof(double));
  double* w = (double*)malloc(n * sizeof(double));
  double* e = (double*)malloc(m * sizeof(double));
  double* xd = (double*)calloc(n, sizeof(double));
  lo_l1_subgradient(n, support, values, s, fill_bound, rng, g);
  lo_apply_gram_inverse(A, g, w);
  lo_apply(A, w, e);
  for (uint64_t i = 0; i < m; ++i) e[i] *= tau;
  for (uint64_t k = 0; k < s; ++k) xd[support[k]] = values[k];
  lo_apply(A, xd, b);
  double noise_sq = 0.0;
  for (uint64_t i = 0; i < m; ++i) {
    b[i] += e[i];
    noise_sq += e[i] * e[i];
  }
  free(g);
  free(w);
  free(e);
  free(xd);
  return sqrt(noise_sq);
}

/* instance.cpp:175-202 */
lo_cert lo_verify_optimality(const lo_op* A, double tau, const double* b, const uint32_t* support,
                             const double* values, uint64_t s, double tol) {
  const uint64_t m = A->m, n = A->n;
  double* xd = (double*)calloc(n, sizeof(double));
  double* res = (double*)malloc(m * sizeof(double));
  double* r = (double*)malloc(n * sizeof(double));
  uint8_t* on = (uint8_t*)calloc(n, 1);
  for (uint64_t k = 0; k < s; ++k) xd[support[k]] = values[k];
  lo_apply(A, xd, res);
  for (uint64_t i = 0; i < m; ++i) res[i] -= b[i];
  lo_apply_transpose(A, res, r);
  lo_cert c = {0.0, 0.0, tol * tau, 0};
  for (uint64_t k = 0; k < s; ++k) {
    const uint32_t i = support[k];
    on[i] = 1;
    const double sign = values[k] > 0.0 ? 1.0 : -1.0;
    const double v = fabs(r[i] + tau * sign);
    if (v > c.max_support_violation) c.max_support_violation = v;
  }
  for (uint64_t i = 0; i < n; ++i) {
    if (on[i]) continue;
    const double v = fmax(fabs(r[i]) - tau, 0.0);
    if (v > c.max_offsupport_violation) c.max_offsupport_violation = v;
  }
  c.pass = c.max_support_violation <= c.threshold && c.max_offsupport_violation <= c.threshold;
  free(xd);
  free(res);
  free(r);
  free(on);
  return c;
}

/* ------------------------------------------------------------------------ */
/* Solver helpers (solvers.cpp:14-34, 145-157, 266-270)                      */

static double dot(const double* a, const double* b, uint64_t n) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double norm1(const double* a, uint64_t n) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += fabs(a[i]);
  return s;
}
static uint64_t count_nnz(const double* a, uint64_t n) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; ++i) c += a[i] != 0.0;
  return c;
}

double lo_soft_threshold(double v, double t) {
  if (v > t) return v - t;
  if (v < -t) return v + t;
  return 0.0;
}

double lo_cd_damping(uint64_t omega, uint64_t varpi, uint64_t n) {
  if (n <= 1 || varpi <= 1) return 1.0;
  return 1.0 + (double)(omega - 1) * (double)(varpi - 1) / (double)(n - 1);
}

double lo_objective(const lo_op* A, double tau, const double* b, const double* x) {
  double* r = (double*)malloc(A->m * sizeof(double));
  lo_apply(A, x, r);
  for (uint64_t i = 0; i < A->m; ++i) r[i] -= b[i];
  const double f = tau * norm1(x, A->n) + 0.5 * dot(r, r, A->m);
  free(r);
  return f;
}

/* Tracker (solvers.cpp:43-94) without wall-clock fields */
typedef struct {
  lo_sample* buf;
  uint64_t cap;
  lo_summary sum;
  int has_target;
  double target;
} tracker;

static void tk_init(tracker* tk, const lo_cfg* cfg, lo_sample* buf, uint64_t cap) {
  memset(tk, 0, sizeof(*tk));
  tk->buf = buf;
  tk->cap = cap;
  tk->has_target = cfg->has_target;
  tk->target = cfg->target;
  tk->sum.final_objective = NAN;
  tk->sum.matvecs_to_target = INFINITY;
}

static void tk_sample(tracker* tk, uint64_t iter, double f, uint64_t nnz, double mv, uint64_t extra) {
  if (tk->sum.n_samples < tk->cap) {
    lo_sample* s = &tk->buf[tk->sum.n_samples++];
    s->iter = iter;
    s->objective = f;
    s->nnz = nnz;
    s->matvecs = mv;
    s->extra = extra;
  }
  tk->sum.n_samples_total++;
  tk->sum.final_objective = f;
  if (!tk->sum.reached_target && tk->has_target && f <= tk->target) {
    tk->sum.reached_target = 1;
    tk->sum.matvecs_to_target = mv;
  }
}

static int tk_hit(const tracker* tk, double f) { return tk->has_target && f <= tk->target; }

static lo_summary tk_finish(tracker* tk, int status, double mv) {
  tk->sum.status = status;
  if (status == 0 && !tk->sum.reached_target) {
    tk->sum.reached_target = 1;
    if (!isfinite(tk->sum.matvecs_to_target)) tk->sum.matvecs_to_target = mv;
  }
  tk->sum.total_matvecs = mv;
  return tk->sum;
}

/* ------------------------------------------------------------------------ */
/* FISTA / ISTA with the spectrum (or fixed) L (solvers.cpp:277-382)         */

/* linops.cpp:757-778 */
double lo_estimate_gram_lmax(const lo_op* A, uint64_t iters, uint64_t seed) {
  const uint64_t n = A->n, m = A->m;
  lo_rng rng;
  lo_rng_seed(&rng, seed);
  double* v = (double*)malloc(n * sizeof(double));
  double* w = (double*)malloc(n * sizeof(double));
  double* av = (double*)malloc(m * sizeof(double));
  for (uint64_t i = 0; i < n; ++i) v[i] = lo_normal(&rng);
  double lambda = 0.0;
  for (uint64_t it = 0; it < iters; ++it) {
    double norm = 0.0;
    for (uint64_t i = 0; i < n; ++i) norm += v[i] * v[i];
    norm = sqrt(norm);
    if (norm == 0.0) break;
    for (uint64_t i = 0; i < n; ++i) v[i] /= norm;
    lo_apply(A, v, av);
    lo_apply_transpose(A, av, w);
    lambda = 0.0;
    for (uint64_t i = 0; i < n; ++i) lambda += v[i] * w[i];
    double* t = v;
    v = w;
    w = t;
  }
  free(v);
  free(w);
  free(av);
  return lambda;
}

lo_summary lo_fista(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                    lo_sample* samples, uint64_t cap, double* x_out) {
  const uint64_t n = A->n, m = A->m;
  tracker tk;
  tk_init(&tk, cfg, samples, cap);
  double mv = 0.0;
  /* LipschitzState (solvers.cpp:99-120) */
  double lval;
  int bt_on = 0;
  if (cfg->l_fixed > 0.0) {
    lval = cfg->l_fixed;
  } else if (!cfg->backtracking) {
    lval = lo_gram_lmax(A);
  } else {
    bt_on = 1;
    const double est = lo_estimate_gram_lmax(A, 30, lo_mix_seed(cfg->seed, 0x4c6d6178ULL));
    lval = est > 0.0 ? est : 1.0;
  }
  const double lcap = lval * 0x1p60;
  double* x = (double*)calloc(n, sizeof(double));
  double* y = (double*)calloc(n, sizeof(double));
  double* grad = (double*)malloc(n * sizeof(double));
  double* trial = (double*)malloc(n * sizeof(double));
  double* r_x = (double*)malloc(m * sizeof(double));
  double* r_y = (double*)malloc(m * sizeof(double));
  double* r_trial = (double*)malloc(m * sizeof(double));
  lo_apply(A, x, r_x);
  mv += 1;
  for (uint64_t i = 0; i < m; ++i) r_x[i] -= b[i];
  double f = tau * norm1(x, n) + 0.5 * dot(r_x, r_x, m);
  tk_sample(&tk, 0, f, count_nnz(x, n), mv, 0);
  memcpy(r_y, r_x, m * sizeof(double));
  double t_mom = 1.0;
  int status = 1;
  uint64_t last_sampled = 0, k = 0;
  const int acc = cfg->accelerated;
  for (;;) {
    if (tk_hit(&tk, f)) { status = 0; break; }
    if (k >= cfg->max_iters) { status = 1; break; }
    ++k;
    const double* base = acc ? y : x;
    const double* r_base = acc ? r_y : r_x;
    lo_apply_transpose(A, r_base, grad);
    mv += 1;
    const double g_base = 0.5 * dot(r_base, r_base, m);
    if (bt_on) lval = fmax(lval * 0.5, 1e-12);
    uint64_t backtracks = 0;
    for (;;) { /* solvers.cpp:325-343 */
      const double inv_l = 1.0 / lval;
      for (uint64_t i = 0; i < n; ++i) trial[i] = lo_soft_threshold(base[i] - inv_l * grad[i], tau * inv_l);
      lo_apply(A, trial, r_trial);
      mv += 1;
      for (uint64_t i = 0; i < m; ++i) r_trial[i] -= b[i];
      if (!bt_on) break;
      const double lhs = 0.5 * dot(r_trial, r_trial, m);
      double quad = g_base, step_sq = 0.0;
      for (uint64_t i = 0; i < n; ++i) {
        const double d = trial[i] - base[i];
        quad += grad[i] * d;
        step_sq += d * d;
      }
      quad += 0.5 * lval * step_sq;
      if (lhs <= quad + 1e-12 * (fabs(lhs) + fabs(quad)) || lval >= lcap) break;
      lval *= 2.0;
      ++backtracks;
    }
    int fixed_point = 1;
    for (uint64_t i = 0; i < n; ++i)
      if (trial[i] != base[i]) { fixed_point = 0; break; }
    if (acc) {
      const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t_mom * t_mom));
      const double beta = (t_mom - 1.0) / t_next;
      for (uint64_t i = 0; i < n; ++i) y[i] = trial[i] + beta * (trial[i] - x[i]);
      for (uint64_t i = 0; i < m; ++i) r_y[i] = (1.0 + beta) * r_trial[i] - beta * r_x[i];
      memcpy(x, trial, n * sizeof(double));
      memcpy(r_x, r_trial, m * sizeof(double));
      t_mom = t_next;
    } else {
      memcpy(x, trial, n * sizeof(double));
      memcpy(r_x, r_trial, m * sizeof(double));
    }
    f = tau * norm1(x, n) + 0.5 * dot(r_x, r_x, m);
    if (!isfinite(f)) { status = -1; break; }
    if (k <= 1000 || k % 10 == 0 || fixed_point) {
      tk_sample(&tk, k, f, count_nnz(x, n), mv, backtracks);
      last_sampled = k;
    }
    if (fixed_point) { status = 0; break; }
  }
  if (status >= 0 && last_sampled != k) tk_sample(&tk, k, f, count_nnz(x, n), mv, 0);
  if (x_out) memcpy(x_out, x, n * sizeof(double));
  free(x); free(y); free(grad); free(trial); free(r_x); free(r_y); free(r_trial);
  return tk_finish(&tk, status, mv);
}

/* solvers.cpp:401-410 -- omega = max row nnz, capped at n */
static uint64_t partial_separability(const lo_op* A, const uint64_t* rptr) {
  uint64_t omega = 1;
  for (uint64_t i = 0; i < A->m; ++i) {
    const uint64_t c = rptr[i + 1] - rptr[i];
    if (c > omega) omega = c;
  }
  return omega < A->n ? omega : A->n;
}

/* ------------------------------------------------------------------------ */
/* Serial randomized CD (solvers.cpp:414-482)                                */

lo_summary lo_cd(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                 const uint64_t* cptr, const uint32_t* cidx, const double* cval,
                 const uint64_t* rptr, lo_sample* samples, uint64_t cap, double* x_out) {
  const uint64_t n = A->n, m = A->m;
  tracker tk;
  tk_init(&tk, cfg, samples, cap);
  uint64_t mvc = 0; /* CountingOperator count_ */
  double mvf = 0.0;  /* CountingOperator fractional_ (linops.hpp:271-278) */
  double* lips = (double*)malloc(n * sizeof(double));
  lo_gram_diagonal(A, lips);
  uint64_t omega = 1;
  if (cfg->varpi > 1) omega = cfg->omega ? cfg->omega : partial_separability(A, rptr);
  const double beta = lo_cd_damping(omega, cfg->varpi, n);
  lo_rng rng;
  lo_rng_seed(&rng, cfg->seed);
  double* x = (double*)calloc(n, sizeof(double));
  double* r = (double*)malloc(m * sizeof(double));
  lo_apply(A, x, r);
  mvc += 1;
  for (uint64_t i = 0; i < m; ++i) r[i] -= b[i];
  double f = tau * norm1(x, n) + 0.5 * dot(r, r, m);
  tk_sample(&tk, 0, f, count_nnz(x, n), (double)mvc + mvf, 0);
  int status = 1;
  uint64_t sweep = 0;
  for (;;) {
    if (tk_hit(&tk, f)) { status = 0; break; }
    if (sweep >= cfg->max_iters) { status = 1; break; }
    ++sweep;
    uint64_t applied = 0;
    double col_ops = 0.0;
    for (uint64_t u = 0; u < n; ++u) {
      const uint64_t i = lo_coord_index(&rng, n);
      const double li = lips[i];
      if (li == 0.0) continue;
      double gi = 0.0;
      for (uint64_t p = cptr[i]; p < cptr[i + 1]; ++p) gi += cval[p] * r[cidx[p]];
      col_ops += 1.0;
      const double scale = beta * li;
      const double xi_new = lo_soft_threshold(x[i] - gi / scale, tau / scale);
      const double delta = xi_new - x[i];
      if (delta != 0.0) {
        x[i] = xi_new;
        for (uint64_t p = cptr[i]; p < cptr[i + 1]; ++p) r[cidx[p]] += delta * cval[p];
        col_ops += 1.0;
        ++applied;
      }
    }
    mvf += col_ops / (double)n;
    lo_apply(A, x, r);
    mvc += 1;
    for (uint64_t i = 0; i < m; ++i) r[i] -= b[i];
    f = tau * norm1(x, n) + 0.5 * dot(r, r, m);
    if (!isfinite(f)) { status = -1; break; }
    tk_sample(&tk, sweep, f, count_nnz(x, n), (double)mvc + mvf, applied);
  }
  if (x_out) memcpy(x_out, x, n * sizeof(double));
  free(lips); free(x); free(r);
  return tk_finish(&tk, status, (double)mvc + mvf);
}

/* ------------------------------------------------------------------------ */
/* Block PCDM (C2 mapping of SURVEY.md 8(d)).
 * Per epoch: floor(n/B) blocks.  A block is B distinct coordinates drawn
 * from the uniform_index(rng, n) stream (duplicates inside the block are
 * redrawn).  All B coordinates read the same residual (Jacobi within the
 * block, as in PCDM with tau = B processors); the CD model step
 * (solvers.cpp:457-461) with beta = cd_damping(omega, B, n).  The residual
 * update adds delta_c * A(rho, c) into r(rho) in ascending column order c
 * (the serial CD scatter of solvers.cpp:465 with the block sorted).  After
 * each epoch the residual is refreshed with A x - b (solvers.cpp:473).     */

lo_summary lo_pcdm(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                   const uint64_t* cptr, const uint32_t* cidx, const double* cval,
                   const uint64_t* rptr, const uint32_t* ridx, lo_sample* samples, uint64_t cap,
                   double* x_out) {
  (void)ridx;
  const uint64_t n = A->n, m = A->m;
  tracker tk;
  tk_init(&tk, cfg, samples, cap);
  uint64_t mvc = 0; /* CountingOperator count_ */
  double mvf = 0.0;  /* CountingOperator fractional_ (linops.hpp:271-278) */
  const uint64_t B = cfg->block < n ? cfg->block : n;
  const uint64_t per_epoch = n / B;
  double* lips = (double*)malloc(n * sizeof(double));
  lo_gram_diagonal(A, lips);
  const uint64_t omega = cfg->omega ? cfg->omega : partial_separability(A, rptr);
  const double beta = lo_cd_damping(omega, B, n);
  lo_rng rng;
  lo_rng_seed(&rng, cfg->seed);
  uint64_t* stamp = (uint64_t*)calloc(n, sizeof(uint64_t));
  uint32_t* blk = (uint32_t*)malloc(B * sizeof(uint32_t));
  double* delta = (double*)calloc(n, sizeof(double));
  double* x = (double*)calloc(n, sizeof(double));
  double* r = (double*)malloc(m * sizeof(double));
  lo_apply(A, x, r);
  mvc += 1;
  for (uint64_t i = 0; i < m; ++i) r[i] -= b[i];
  double f = tau * norm1(x, n) + 0.5 * dot(r, r, m);
  tk_sample(&tk, 0, f, count_nnz(x, n), (double)mvc + mvf, 0);
  int status = 1;
  uint64_t epoch = 0, cur = 0;
  for (;;) {
    if (tk_hit(&tk, f)) { status = 0; break; }
    if (epoch >= cfg->max_iters) { status = 1; break; }
    ++epoch;
    uint64_t applied = 0;
    double col_ops = 0.0;
    for (uint64_t q = 0; q < per_epoch; ++q) {
      ++cur;
      for (uint64_t t = 0; t < B; ++t) {
        uint64_t i;
        do {
          i = lo_coord_index(&rng, n);
        } while (stamp[i] == cur);
        stamp[i] = cur;
        blk[t] = (uint32_t)i;
      }
      for (uint64_t t = 0; t < B; ++t) {
        const uint32_t i = blk[t];
        const double li = lips[i];
        delta[i] = 0.0;
        if (li == 0.0) continue;
        double gi = 0.0;
        for (uint64_t p = cptr[i]; p < cptr[i + 1]; ++p) gi += cval[p] * r[cidx[p]];
        col_ops += 1.0;
        const double scale = beta * li;
        const double xi_new = lo_soft_threshold(x[i] - gi / scale, tau / scale);
        delta[i] = xi_new - x[i];
        if (delta[i] != 0.0) x[i] = xi_new;
      }
      qsort(blk, B, sizeof(uint32_t), cmp_u32);
      for (uint64_t t = 0; t < B; ++t) {
        const uint32_t i = blk[t];
        const double d = delta[i];
        if (d == 0.0) continue;
        for (uint64_t p = cptr[i]; p < cptr[i + 1]; ++p) r[cidx[p]] += d * cval[p];
        col_ops += 1.0;
        ++applied;
      }
    }
    mvf += col_ops / (double)n;
    lo_apply(A, x, r);
    mvc += 1;
    for (uint64_t i = 0; i < m; ++i) r[i] -= b[i];
    f = tau * norm1(x, n) + 0.5 * dot(r, r, m);
    if (!isfinite(f)) { status = -1; break; }
    tk_sample(&tk, epoch, f, count_nnz(x, n), (double)mvc + mvf, applied);
  }
  if (x_out) memcpy(x_out, x, n * sizeof(double));
  free(lips); free(stamp); free(blk); free(delta); free(x); free(r);
  return tk_finish(&tk, status, (double)mvc + mvf);
}

/* ------------------------------------------------------------------------ */
/* PCG + Newton-CG (solvers.cpp:159-264, 487-568)                            */

typedef struct {
  const lo_op* A;
  double tau;
  const double* d2psi;
  double* hess_av;
  double* mv;
} hv_ctx;

/* hessvec lambda of solvers.cpp:537-541 */
static void hessvec(hv_ctx* h, const double* v, double* out) {
  lo_apply(h->A, v, h->hess_av);
  lo_apply_transpose(h->A, h->hess_av, out);
  *h->mv += 2;
  for (uint64_t i = 0; i < h->A->n; ++i) out[i] += h->tau * h->d2psi[i] * v[i];
}

/* solvers.cpp:202-264 */
static lo_pcg_result pcg(hv_ctx* h, const double* rhs, const double* pre, double eta,
                         uint64_t max_iters, double* step) {
  const uint64_t n = h->A->n;
  lo_pcg_result res = {0, 0, 0, 0.0};
  for (uint64_t i = 0; i < n; ++i) step[i] = 0.0;
  const double rhs_norm = sqrt(dot(rhs, rhs, n));
  if (rhs_norm == 0.0) {
    res.converged = 1;
    return res;
  }
  double* r = (double*)malloc(n * sizeof(double));
  double* z = (double*)malloc(n * sizeof(double));
  double* p = (double*)malloc(n * sizeof(double));
  double* hp = (double*)malloc(n * sizeof(double));
  double* best = (double*)calloc(n, sizeof(double));
  memcpy(r, rhs, n * sizeof(double));
  for (uint64_t i = 0; i < n; ++i) z[i] = r[i] / pre[i];
  memcpy(p, z, n * sizeof(double));
  double rz = dot(r, z, n);
  double best_norm = rhs_norm;
  int done = 0;
  for (uint64_t k = 0; k < max_iters; ++k) {
    hessvec(h, p, hp);
    const double php = dot(p, hp, n);
    if (!(php > 0.0)) {
      res.negative_curvature = 1;
      break;
    }
    const double alpha = rz / php;
    for (uint64_t i = 0; i < n; ++i) {
      step[i] += alpha * p[i];
      r[i] -= alpha * hp[i];
    }
    ++res.iterations;
    const double rn = sqrt(dot(r, r, n));
    if (rn < best_norm) {
      best_norm = rn;
      memcpy(best, step, n * sizeof(double));
    }
    if (rn <= eta * rhs_norm) {
      res.converged = 1;
      res.rel_residual = rn / rhs_norm;
      done = 1;
      break;
    }
    for (uint64_t i = 0; i < n; ++i) z[i] = r[i] / pre[i];
    const double rz_next = dot(r, z, n);
    const double beta = rz_next / rz;
    rz = rz_next;
    for (uint64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  if (!done) {
    memcpy(step, best, n * sizeof(double));
    res.rel_residual = best_norm / rhs_norm;
  }
  free(r); free(z); free(p); free(hp); free(best);
  return res;
}

lo_pcg_result lo_pcg_at(const lo_op* A, double tau, double mu, const double* x,
                        const double* rhs, const double* precond, double eta, uint64_t max_iters,
                        double* step) {
  const uint64_t n = A->n;
  double* d2psi = (double*)malloc(n * sizeof(double));
  double* hav = (double*)malloc(A->m * sizeof(double));
  for (uint64_t i = 0; i < n; ++i) {
    const double q = mu * mu + x[i] * x[i];
    d2psi[i] = mu * mu / (q * sqrt(q));
  }
  double mv = 0.0;
  hv_ctx h = {A, tau, d2psi, hav, &mv};
  lo_pcg_result r = pcg(&h, rhs, precond, eta, max_iters, step);
  free(d2psi);
  free(hav);
  return r;
}

static double pseudo_huber(const double* x, uint64_t n, double mu) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += sqrt(mu * mu + x[i] * x[i]) - mu;
  return s;
}

/* solvers.cpp:487-568 */
lo_summary lo_newton_cg(const lo_op* A, double tau, const double* b, const lo_cfg* cfg,
                        lo_sample* samples, uint64_t cap, double* x_out) {
  const uint64_t n = A->n, m = A->m;
  const double mu = cfg->mu;
  tracker tk;
  tk_init(&tk, cfg, samples, cap);
  double mv = 0.0;
  double* gram = (double*)malloc(n * sizeof(double));
  lo_gram_diagonal(A, gram);
  double* atb = (double*)malloc(n * sizeof(double));
  lo_apply_transpose(A, b, atb);
  mv += 1;
  const double nb = sqrt(dot(atb, atb, n));
  const double grad_tol = cfg->grad_tol_rel * (nb > 1.0 ? nb : 1.0);
  double* x = (double*)calloc(n, sizeof(double));
  double* r = (double*)malloc(m * sizeof(double));
  lo_apply(A, x, r);
  mv += 1;
  for (uint64_t i = 0; i < m; ++i) r[i] -= b[i];
  double* grad = (double*)malloc(n * sizeof(double));
  double* d2psi = (double*)malloc(n * sizeof(double));
  double* pre = (double*)malloc(n * sizeof(double));
  double* ad = (double*)malloc(m * sizeof(double));
  double* xt = (double*)malloc(n * sizeof(double));
  double* rt = (double*)malloc(m * sizeof(double));
  double* hav = (double*)malloc(m * sizeof(double));
  double* rhs = (double*)malloc(n * sizeof(double));
  double* step_v = (double*)malloc(n * sizeof(double));
  int status = 1;
  uint64_t step = 0, last_pcg = 0;
  for (;;) {
    const double f_true = tau * norm1(x, n) + 0.5 * dot(r, r, m);
    if (!isfinite(f_true)) { status = -1; break; }
    tk_sample(&tk, step, f_true, count_nnz(x, n), mv, last_pcg);
    if (tk_hit(&tk, f_true)) { status = 0; break; }
    const double f_smooth = tau * pseudo_huber(x, n, mu) + 0.5 * dot(r, r, m);
    lo_apply_transpose(A, r, grad);
    mv += 1;
    for (uint64_t i = 0; i < n; ++i) {
      const double q = mu * mu + x[i] * x[i];
      const double root = sqrt(q);
      grad[i] += tau * x[i] / root;
      d2psi[i] = mu * mu / (q * root);
      pre[i] = tau * d2psi[i] + gram[i];
    }
    if (sqrt(dot(grad, grad, n)) <= grad_tol) { status = 0; break; }
    if (step >= cfg->max_iters) { status = 1; break; }
    ++step;
    for (uint64_t i = 0; i < n; ++i) rhs[i] = -grad[i];
    hv_ctx h = {A, tau, d2psi, hav, &mv};
    const lo_pcg_result pr = pcg(&h, rhs, pre, cfg->eta, cfg->pcg_max_iters, step_v);
    last_pcg = pr.iterations;
    tk.sum.total_pcg_iterations += pr.iterations;
    lo_apply(A, step_v, ad);
    mv += 1;
    const double slope = dot(grad, step_v, n);
    double alpha = 1.0;
    uint64_t bt = 0;
    for (;;) {
      for (uint64_t i = 0; i < n; ++i) xt[i] = x[i] + alpha * step_v[i];
      for (uint64_t i = 0; i < m; ++i) rt[i] = r[i] + alpha * ad[i];
      const double f_trial = tau * pseudo_huber(xt, n, mu) + 0.5 * dot(rt, rt, m);
      if (f_trial <= f_smooth + 1e-4 * alpha * slope || bt >= cfg->ls_max_backtracks) break;
      alpha *= 0.5;
      ++bt;
    }
    double* tmp = x; x = xt; xt = tmp;
    tmp = r; r = rt; rt = tmp;
    tk.sum.newton_steps++;
  }
  if (x_out) memcpy(x_out, x, n * sizeof(double));
  free(gram); free(atb); free(x); free(r); free(grad); free(d2psi); free(pre); free(ad);
  free(xt); free(rt); free(hav); free(rhs); free(step_v);
  return tk_finish(&tk, status, mv);
}
