// solvers.cu -- host drivers of the device-resident solver loops.
//
// FISTA/ISTA (solvers.cpp:277-382): two fused kernels per iteration (k_spmv.cu)
// and no host round trip: the stop decision (fixed point, target, iteration
// budget, divergence) is taken on device and turns later launches into
// no-ops, so the host enqueues chunks and only polls a pinned copy of the stop
// flag between chunks (time budget = the reference's loop-head check at chunk
// granularity).  Trace samples are stamped with %globaltimer on device.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "guard.hpp"
#include "nccl_rt.hpp"
#include "solvers.hpp"

using namespace l1b;

namespace l1b {
void validate_cfg(const l1b_solver_cfg* c, uint64_t n);
void run_pcdm(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
              l1b_summary* summary, double* x_host, double* d_x);
void run_newton_cg(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
                  l1b_summary* summary, double* x_host, double* d_x);
void run_fista_backtracking(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
                            l1b_summary* summary, double* x_host, double* d_x);
}  // namespace l1b

// Small page-locked blocks (the stop flags and the state read back at the end
// of a solve), cached for the process: cudaMallocHost / cudaFreeHost are
// heavyweight driver calls (page locking, device-wide synchronisation) that a
// solve should not pay on every call.
constexpr size_t kPinnedBlock = 4096;
struct PinnedCache {
  std::mutex m;
  std::vector<void*> free_;
  void* get() {
    {
      std::lock_guard<std::mutex> g(m);
      if (!free_.empty()) {
        void* p = free_.back();
        free_.pop_back();
        return p;
      }
    }
    void* p = nullptr;
    L1B_CUDA(cudaMallocHost(&p, kPinnedBlock));
    return p;
  }
  void put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(m);
    free_.push_back(p);
  }
};
PinnedCache& pinned_cache() {
  static PinnedCache* c = new PinnedCache();  // (never destroyed: no driver calls at exit)
  return *c;
}
void pinned_release(void* p) { pinned_cache().put(p); }

// (see l1b_session::tile_plan) kmax = the session's iterations per tile launch, 0: no tiles
static std::vector<int> plan_tile_launches(int kmax_, uint64_t iters) {
  std::vector<int> ks;
  if (kmax_ <= 0) return ks;
  const uint64_t kmax = (uint64_t)kmax_, kmin = std::min<uint64_t>(6, kmax);  // (K = 2: tests)
  uint64_t l = iters / kmax + (iters % kmax >= kmin ? 1 : 0), r = iters;
  for (; l > 0 && r >= kmin; --l) {
    uint64_t k = std::min((r + l - 1) / l, kmax);
    const uint64_t down = (k + 2) % 4;  // to the next value = 2 mod 4 below
    k = k > down ? k - down : kmin;
    k = std::max(k, kmin);
    if (k > r) break;
    ks.push_back((int)k);
    r -= k;
  }
  return ks;
}

struct l1b_session {
  l1b_problem* prob = nullptr;
  ProblemView v;
  l1b_solver_cfg cfg;
  bool accel = true;
  bool shard = false;
  bool fused = false;   // matrix-free fused kernels (k_fused.cu) instead of CSR/CSC
  bool single = false;  // ... as one kernel per iteration (one device): x / r rotate
  bool recompute = false;  // ... with r_k, r_{k-1} rebuilt from x (k_iter_rc.cu): no R buffers
  bool pairs = false;      // ... shard k1 = two iterations (fista_rc_iter2), halos of two x buffers
  bool general = false;    // general row-block shard: reduce-scatter g, all-gather x (distributed.py)
  double *g_full = nullptr, *x_full = nullptr;  // n_pad = world * col_slice entries each
  uint64_t n_pad = 0, col_off = 0;              // own slice: [col_off, col_off + nx)
  double* X[4] = {nullptr, nullptr, nullptr, nullptr};
  int nbuf = 3;  // x rotation period: 4 for the recomputing kernels (two-iteration launches)
  double* R[3] = {nullptr, nullptr, nullptr};
  uint64_t xh = 0, rh = 0;  // single-kernel windows: x / r halo widths (shards: H / 2H)
  uint64_t nx = 0, nr = 0, halo = 0;  // own columns / own rows / window overhang
  double *x_win = nullptr, *r_y_win = nullptr;  // shard windows (x, r_y point inside)
  double *x = nullptr, *y = nullptr, *r_x = nullptr, *r_y = nullptr, *partials = nullptr;
  FistaDev* st = nullptr;
  FistaSample* trace = nullptr;
  FistaDev* h_st = nullptr;  // pinned
  uint64_t cap = 0;
  uint64_t launched = 0;
  std::chrono::steady_clock::time_point t0;
  bool time_out = false;

  // launch j computes iteration j+1 from x_j (X[j%P]) and x_{j-1} (X[(j+P-1)%P]), P = nbuf
  IterBufs iter_bufs(uint64_t j) const {
    // global-index views: window entry xh + (g - lo) holds global entry g
    const int64_t lo = shard ? (int64_t)v.row_begin : 0;
    auto gx = [&](double* p) { return p + (int64_t)xh - lo; };
    auto gr = [&](double* p) { return p + (int64_t)rh - lo; };
    IterBufs ib;
    const uint64_t P = (uint64_t)nbuf;
    ib.x_k = gx(X[j % P]);
    ib.x_km1 = gx(X[(j + P - 1) % P]);
    ib.r_k = recompute ? nullptr : gr(R[j % 3]);
    ib.r_km1 = recompute ? nullptr : gr(R[(j + 2) % 3]);
    ib.x_next = gx(X[(j + 1) % P]);
    ib.r_next = recompute ? nullptr : gr(R[(j + 1) % 3]);
    ib.b = recompute && shard ? v.b_win : v.b - lo;
    ib.st = st;
    ib.trace = trace;
    ib.partials = partials;
    return ib;
  }

  // launch j of the single-kernel loop (iteration j + 1)
  // launches j and j+1 as one two-iteration kernel (recomputing path, one device)
  // neighbours' x buffers (global-index views) when the halo travels by the
  // kernels' own peer stores (l1b_session_attach_peers)
  bool peers_on = false;
  double* peer_left[4] = {nullptr, nullptr, nullptr, nullptr};
  double* peer_right[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<void*> ipc_opened;
  std::vector<double*> x_raw;  // cudaMalloc'd x buffers (shards: exportable over IPC)

  // native shard driver (l1b_session_attach_nccl): the library's own NCCL
  // communicator; graph[q] = two launches starting at launched % 4 == 2q,
  // captured once and replayed
  ncclComm_t comm = nullptr;
  int comm_rank = 0, comm_world = 1;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  uint64_t graph_kernels[2] = {0, 0};

  PeerViews peers(uint64_t j) const {  // x_{j+1}, x_{j+2} of the neighbours
    PeerViews pv;
    if (!peers_on) return pv;
    pv.on = 1;
    pv.halo = (int64_t)xh;
    for (int w = 0; w < 2; ++w) {
      pv.left[w] = peer_left[(j + 1 + w) % 4];
      pv.right[w] = peer_right[(j + 1 + w) % 4];
    }
    return pv;
  }

  // contracted arithmetic: honoured where every rotation stage has
  // |cos(theta)| >= 1/4 (the scaled form of the two-iteration and tile
  // kernels, StageTab::scaled_ok); steeper stages keep the exact arithmetic.
  // opf = the operator with sigma * prod cos(theta) as its sigma (the contracted kernels' view)
  bool fma() const { return cfg.arith == L1B_ARITH_FMA && v.op->right.scaled_ok != 0; }
  OpView opf;
  const OpView& op2() const { return fma() ? opf : *v.op; }

  // tile kernel (K iterations per launch, one device): tbk = K (0: off),
  // tb = its per-CTA sums, tb_starts = (j, K) of every launch (a stop inside one is
  // replayed from its inputs, which no later launch overwrites)
  int tbk = 0;
  double* tb = nullptr;
  std::vector<std::pair<uint64_t, int>> tb_starts;

  void iteratek(uint64_t j, cudaStream_t stream, int K = 0) {
    if (K == 0) K = tbk;
    fista_rc_iterk(op2(), iter_bufs(j), X[(j + K - 1) % 4], X[(j + K) % 4], K, false, tb, stream, fma());
    tb_starts.emplace_back(j, K);
  }
  // The tile launches `iters` iterations take (each K = 2 mod 4, 6 <= K <=
  // tbk: the rotation of the x buffers; what is left, < 6 iterations, goes to
  // two-iteration / single launches).  A remainder of 6 or more gets its own
  // launch and the iterations are spread evenly (20 = 10 + 10, not 14 + 6: a
  // launch costs a tile start, and a short one keeps less of its tiles).
  std::vector<int> tile_plan(uint64_t iters) const { return plan_tile_launches(tbk, iters); }

  void iterate2(uint64_t j, cudaStream_t stream) const {
    const int64_t lo = shard ? (int64_t)v.row_begin : 0;
    fista_rc_iter2(op2(), iter_bufs(j), X[(j + 2) % 4] + (int64_t)xh - lo, (uint64_t)lo,
                   shard ? v.row_end : v.n, stream, peers(j), fma());
  }

  void iterate(uint64_t j, cudaStream_t stream, bool flush = false) const {
    const uint64_t lo = shard ? v.row_begin : 0, hi = shard ? v.row_end : v.n;
    if (recompute)
      fista_rc_iter(op2(), iter_bufs(j), lo, hi, stream, flush, flush ? PeerViews() : peers(j), fma());
    else
      fista_fused_iter(*v.op, iter_bufs(j), lo, hi, stream);
  }

  FistaBufs bufs() const {
    FistaBufs b;
    b.x = x;
    b.y = y;
    b.r_x = r_x;
    b.r_y = r_y;
    b.b = general ? v.b + v.row_begin : v.b;
    b.x_gather = general ? x_full : shard ? x_win : x;
    b.r_y_gather = shard ? r_y_win : r_y;
    b.lo = shard ? v.row_begin : 0;
    b.hi = shard ? v.row_end : v.n;
    b.gather_base = shard ? (int64_t)v.row_begin - (int64_t)v.halo : 0;
    b.st = st;
    b.trace = trace;
    b.partials = partials;
    return b;
  }

  ~l1b_session() {
    cudaSetDevice(v.device);
    if (v.stream) cudaStreamSynchronize(v.stream);
    for (auto& g : graph)
      if (g) cudaGraphExecDestroy(g);
    if (comm) nccl().CommDestroy(comm);
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
    for (double* q : x_raw) cudaFree(q);
    for (void* q : allocs) cudaFreeAsync(q, v.stream);  // back to the stream-ordered pool
    if (v.stream) cudaStreamSynchronize(v.stream);
    if (h_st) pinned_release(h_st);
  }
  std::vector<void*> allocs;
  // stream-ordered allocations from the device pool (kept cached between
  // sessions, see keep_pool): a session costs no cudaMalloc after the first
  void* valloc(size_t bytes) {
    void* q = nullptr;
    L1B_CUDA(cudaMallocAsync(&q, std::max<size_t>(bytes, 16), v.stream));
    allocs.push_back(q);
    return q;
  }
  double* dalloc(uint64_t count) { return (double*)valloc((count + 2) * sizeof(double)); }
};

namespace {

bool rc2_enabled();  // L1B_RC2 switch (below)

uint64_t sample_capacity(uint64_t max_iters) {
  uint64_t c = std::min<uint64_t>(max_iters, 1000) + 2;
  if (max_iters > 1000) c += (max_iters - 1000) / 10 + 1;
  return std::min<uint64_t>(c, 1ull << 22);
}

// Keep freed pool memory cached on the device (release threshold = max), so
// repeated solves on resident instances do not go back to the driver.

void session_reset(l1b_session* s);

void session_begin(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_session* s) {
  keep_pool(problem_view(p, false).device);
  s->prob = p;
  {
    const ProblemView probe = problem_view(p, false);
    if (cfg->op == L1B_OP_MATRIX_FREE && !probe.fused_ok)
      throw Unsupported("matrix-free FISTA needs a banded operator (no P1/P2, no left stages, one device)");
    s->fused = probe.fused_ok && (cfg->op == L1B_OP_MATRIX_FREE || cfg->op == L1B_OP_AUTO);
  }
  s->v = problem_view(p, !s->fused);
  s->cfg = *cfg;
  s->accel = cfg->solver == L1B_FISTA;
  const ProblemView& v = s->v;
  cudaStream_t st = v.stream;
  s->shard = v.shard;
  s->single = s->fused && fused_iter_supported(*v.op);
  {
    // recomputing kernel: one device, 32-byte aligned sigma / b (256-bit loads);
    // L1B_ITER_RC=0 selects the stored-residual kernel (comparison runs)
    // (shards: b on the rows around the block, blocks on multiples of 4 and at
    // least one halo wide -- the exchange only reaches the next rank)
    const char* e = getenv("L1B_ITER_RC");
    bool ok = s->single && !(e && e[0] == '0') && (uintptr_t)v.op->sigma % 32 == 0;
    if (ok && s->shard) {
      const uint64_t H3 = (uint64_t)std::max(fista_rc_halo(v.op->right.count),
                                             fista_rc2_halo(v.op->right.count));
      ok = v.b_win && (uintptr_t)v.b_win % 32 == 0 && v.row_begin % 4 == 0 &&
           v.row_end - v.row_begin >= H3 && v.b_win_lo <= (v.row_begin > H3 ? v.row_begin - H3 : 0) &&
           v.b_win_hi >= std::min(v.n, v.row_end + H3);
    } else if (ok) {
      ok = (uintptr_t)v.b % 32 == 0;
    }
    s->recompute = ok;
  }
  if (s->single) {
    // x_k, x_{k-1}, x_{k+1} and r_k, r_{k-1}, r_{k+1} over the n active rows
    // (a shard: its own rows plus halos of H for x and 2H for r);
    // X[2] / R[2] stand for the iterate "before" the first one (x_{-1} = x_0)
    const uint64_t H = ((uint64_t)v.op->right.count + 1) & ~1ull;
    s->nx = s->nr = s->shard ? v.row_end - v.row_begin : v.n;
    s->pairs = s->shard && s->recompute && rc2_enabled();
    s->xh = s->shard ? (s->recompute ? (uint64_t)std::max(fista_rc_halo(v.op->right.count),
                                                          fista_rc2_halo(v.op->right.count))
                                     : H)
                     : 0;
    s->rh = s->shard && !s->recompute ? 2 * H : 0;
    s->halo = s->xh;
    s->nbuf = s->recompute ? 4 : 3;
    for (int q = 0; q < s->nbuf; ++q) {
      if (s->shard && s->recompute) {  // plain allocations: exportable to peer processes (IPC)
        double* p = nullptr;
        L1B_CUDA(cudaMalloc(&p, (s->nx + 2 * s->xh + 2) * sizeof(double)));
        s->x_raw.push_back(p);
        s->X[q] = p;
      } else {
        s->X[q] = s->dalloc(s->nx + 2 * s->xh);
      }
      L1B_CUDA(cudaMemsetAsync(s->X[q], 0, (s->nx + 2 * s->xh) * 8, st));
      if (s->recompute) continue;
      s->R[q] = s->dalloc(s->nr + 2 * s->rh);
      L1B_CUDA(cudaMemsetAsync(s->R[q], 0, (s->nr + 2 * s->rh) * 8, st));
    }
    s->x = s->X[0] + s->xh;
    s->y = s->x;
    s->r_x = s->recompute ? nullptr : s->R[0] + s->rh;  // null: init only sums ||b||^2
    s->r_y = s->recompute ? nullptr : s->R[2] + s->rh;
  } else if (v.general) {
    // general shard: K1a writes the partial A^T r_y over all columns into
    // g_full; the caller reduce-scatters it (rank r's slice = entries
    // [r*cs, (r+1)*cs)); the prox updates the own slice of x_full, which the
    // caller all-gathers before K2 (CSR rows with global columns)
    s->general = true;
    const uint64_t cs = v.col_slice;
    s->n_pad = (uint64_t)v.world * cs;
    s->col_off = (uint64_t)v.rank * cs;
    s->nx = v.col_end - v.col_begin;
    s->nr = v.row_end - v.row_begin;
    s->g_full = s->dalloc(s->n_pad);
    s->x_full = s->dalloc(s->n_pad);
    L1B_CUDA(cudaMemsetAsync(s->g_full, 0, s->n_pad * 8, st));
    L1B_CUDA(cudaMemsetAsync(s->x_full, 0, s->n_pad * 8, st));
    s->x = s->x_full + s->col_off;
    s->r_y = s->dalloc(s->nr);
    if (s->accel) {
      s->y = s->dalloc(cs);
      s->r_x = s->dalloc(s->nr);
    } else {
      s->y = s->x;  // ISTA: base = x (solvers.cpp:317-318)
      s->r_x = s->r_y;
    }
  } else if (s->shard) {
    // windows: [halo | own | halo]; K1 writes own x, K2 gathers the x window,
    // K2 writes own r_y, K1 gathers the r_y window
    s->halo = v.halo;
    s->nx = s->nr = v.row_end - v.row_begin;
    s->x_win = s->dalloc(s->nx + 2 * s->halo);
    s->r_y_win = s->dalloc(s->nr + 2 * s->halo);
    L1B_CUDA(cudaMemsetAsync(s->x_win, 0, (s->nx + 2 * s->halo) * 8, st));
    L1B_CUDA(cudaMemsetAsync(s->r_y_win, 0, (s->nr + 2 * s->halo) * 8, st));
    s->x = s->x_win + s->halo;
    s->r_y = s->r_y_win + s->halo;
    if (s->accel) {
      s->y = s->dalloc(s->nx);
      s->r_x = s->dalloc(s->nr);
    } else {
      s->y = s->x;  // ISTA: base = x (solvers.cpp:317-318)
      s->r_x = s->r_y;
    }
  } else {
    s->nx = v.n;
    s->nr = v.m;
    s->x = s->dalloc(v.n);
    s->r_x = s->dalloc(v.m);
    if (s->accel) {
      s->y = s->dalloc(v.n);
      s->r_y = s->dalloc(v.m);
    } else {
      s->y = s->x;  // ISTA: base = x (solvers.cpp:317-318)
      s->r_y = s->r_x;
    }
  }
  s->partials = s->dalloc((uint64_t)spmv_grid_max() * 4);
  s->cap = sample_capacity(cfg->max_iters);
  s->trace = (FistaSample*)s->valloc(s->cap * sizeof(FistaSample));
  s->st = (FistaDev*)s->valloc(sizeof(FistaDev));
  static_assert(sizeof(FistaDev) <= kPinnedBlock, "FistaDev outgrew the pinned block");
  s->h_st = (FistaDev*)pinned_cache().get();
  if (s->recompute && !s->shard && rc2_enabled() && tb_enabled(v.n, (int)v.op->right.count)) {
    s->tbk = tb_iters();
    s->tb = s->dalloc(fista_tb_scratch());
  }
  if (s->recompute && s->fma()) {  // sigma * prod cos(theta), built once per problem
    s->opf = *v.op;
    s->opf.sigma = problem_sigma_scaled(p);
  }
  if (s->recompute) fista_rc_prepare(*v.op, s->fma());  // module load + grid sizing before t0
  session_reset(s);
}

// x_0 = 0 and the loop state of iteration 0 (begin, and l1b_session_restart)
void session_reset(l1b_session* s) {
  const ProblemView& v = s->v;
  const l1b_solver_cfg* cfg = &s->cfg;
  cudaStream_t st = v.stream;
  s->tb_starts.clear();
  if (s->single)  // every rotating buffer, halos included (the first launch reads X[3] as x_{-1})
    for (int q = 0; q < s->nbuf; ++q) L1B_CUDA(cudaMemsetAsync(s->X[q], 0, (s->nx + 2 * s->xh) * 8, st));
  L1B_CUDA(cudaMemsetAsync(s->x, 0, s->nx * sizeof(double), st));
  if (s->accel && !s->single) L1B_CUDA(cudaMemsetAsync(s->y, 0, s->nx * sizeof(double), st));
  FistaDev h;
  std::memset(&h, 0, sizeof(h));
  h.t = 1.0;  // solvers.cpp:304
  h.lval = cfg->l_fixed > 0.0 ? cfg->l_fixed : v.lmax;  // LipschitzState (:103-115)
  h.tau = v.tau;
  h.target = cfg->target;
  h.has_target = cfg->has_target ? 1 : 0;
  h.tail_sq = s->fused ? v.tail_sq_band : v.tail_sq;
  h.max_iters = cfg->max_iters;
  h.cap = s->cap;
  h.accel = s->accel ? 1 : 0;
  h.defer = s->shard ? 1 : 0;
  h.init_tail = s->single ? v.tail_sq_band : 0.0;  // the init kernel covers rows [0, nr)
  h.lagged = s->recompute ? 1 : 0;
  *s->h_st = h;
  L1B_CUDA(cudaMemcpyAsync(s->st, s->h_st, sizeof(FistaDev), cudaMemcpyHostToDevice, st));
  s->launched = 0;
  s->time_out = false;
  s->t0 = std::chrono::steady_clock::now();
  // residuals over all (own) rows: rows >= m_active keep r = -b for the whole run
  fista_init(s->bufs(), s->nr, st);  // (single: writes r_0 into R[0] and R[2])
}

// Small single-device instances run a whole chunk of iterations in one
// cooperative launch (k_iter_rc.cu fista_rc_loop); L1B_PERSIST=0 disables.
constexpr uint64_t kPersistMaxN = 1ull << 20;

bool persist_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("L1B_PERSIST");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

// Large single-device instances run two iterations per launch (24n instead
// of 40n bytes per iteration); L1B_RC2=0 keeps one per launch.

bool rc2_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("L1B_RC2");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

// `iters` single-device recomputing iterations as two-iteration launches (+ one
// single launch for an odd count); returns false when the session is not one
bool step_pairs(l1b_session* s, uint64_t iters, cudaStream_t st) {
  if (!(s->recompute && !s->shard && rc2_enabled())) return false;
  uint64_t i = 0;
  for (const int k : s->tile_plan(iters)) {
    s->iteratek(s->launched + i, st, k);
    i += (uint64_t)k;
  }
  for (; i + 2 <= iters; i += 2) s->iterate2(s->launched + i, st);
  if (i < iters) s->iterate(s->launched + i, st);
  return true;
}

// small single-device recomputing sessions step through fista_rc_loop (one
// launch per chunk; also for single iterations, so that every iteration of a
// session reduces its sums in the same order)
bool uses_loop(const l1b_session* s) {
  return s->recompute && !s->shard && !s->tbk && s->v.n <= kPersistMaxN && persist_enabled();
}

void session_step(l1b_session* s, uint64_t iters) {
  const FistaBufs b = s->bufs();
  if (uses_loop(s)) {
    fista_rc_loop(*s->v.op, s->iter_bufs(s->launched), s->X, s->launched, iters, 0, s->v.n,
                  s->v.stream);
    s->launched += iters;
    return;
  }
  if (step_pairs(s, iters, s->v.stream)) {
    s->launched += iters;
    return;
  }
  for (uint64_t i = 0; i < iters; ++i) {
    if (s->single) {
      s->iterate(s->launched + i, s->v.stream);
    } else if (s->fused) {
      fista_fused_k1(*s->v.op, b, s->v.stream);
      fista_fused_k2(*s->v.op, b, s->v.stream);
    } else {
      fista_k1(s->v.At, b, s->v.stream);
      fista_k2(s->v.A, b, s->v.stream);
    }
  }
  s->launched += iters;
}

void session_finish(l1b_session* s, l1b_sample* samples, uint64_t cap, l1b_summary* sum,
                    double* x_host, double* d_x) {
  cudaStream_t st = s->v.stream;
  // the recomputing kernel records each iterate one kernel late: record the last one
  // (shards: l1b_session_flush).  Loop sessions record it with one more
  // iteration of the loop kernel (its x is discarded), so that every record
  // of a small instance reduces its sums the same way.
  if (s->recompute && !s->shard) {
    if (uses_loop(s))
      fista_rc_loop(*s->v.op, s->iter_bufs(s->launched), s->X, s->launched, 1, 0, s->v.n, st);
    else
      s->iterate(s->launched, st, true);
  }
  L1B_CUDA(cudaMemcpyAsync(s->h_st, s->st, sizeof(FistaDev), cudaMemcpyDeviceToHost, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  const FistaDev h = *s->h_st;
  const char* name = s->accel ? "fista" : "ista";
  if (h.status < 0)
    throw std::runtime_error(std::string(name) + ": objective diverged to a non-finite value");
  int status = h.stop ? h.status : (s->time_out ? L1B_TIME_BUDGET : L1B_ITER_BUDGET);
  const uint64_t kept = std::min<uint64_t>(h.n_samples, s->cap);
  std::vector<FistaSample> tr(kept);
  if (kept)
    L1B_CUDA(cudaMemcpyAsync(tr.data(), s->trace, kept * sizeof(FistaSample),
                             cudaMemcpyDeviceToHost, st));
  const double* xf = s->single ? s->X[h.k % (uint64_t)s->nbuf] + s->xh : s->x;  // x after the last executed iteration
  // a tile launch stores only its last two iterates: a stop before those is
  // replayed from the launch's inputs (same operations: the same x)
  for (auto it = s->tb_starts.rbegin(); it != s->tb_starts.rend(); ++it) {
    const uint64_t j = it->first;
    if (h.k <= j) continue;
    if (h.k + 1 < j + (uint64_t)it->second) {
      double* dst = s->X[(j + 1) % 4];
      fista_rc_iterk(s->op2(), s->iter_bufs(j), nullptr, dst, (int)(h.k - j), true, s->tb, st, s->fma());
      xf = dst;
    }
    break;
  }
  if (x_host) L1B_CUDA(cudaMemcpyAsync(x_host, xf, s->nx * 8, cudaMemcpyDeviceToHost, st));
  if (d_x) L1B_CUDA(cudaMemcpyAsync(d_x, xf, s->nx * 8, cudaMemcpyDeviceToDevice, st));
  L1B_CUDA(cudaStreamSynchronize(st));
  // final sample when the last iteration was not sampled (solvers.cpp:379)
  if (h.last_sampled != h.k) tr.push_back(FistaSample{h.k, h.f, h.nnz, h.last_ts});
  std::memset(sum, 0, sizeof(*sum));
  if (uses_loop(s))
    sum->path = L1B_RAN_FISTA_LOOP | L1B_RAN_FISTA_RECOMPUTE;
  else if (s->recompute)
    sum->path = (rc2_enabled() ? L1B_RAN_FISTA_TWO_ITER : 0u) | L1B_RAN_FISTA_RECOMPUTE |
                (s->tb_starts.empty() ? 0u : L1B_RAN_FISTA_TILE) | (s->fma() ? L1B_RAN_FMA : 0u);
  else
    sum->path = s->single ? L1B_RAN_FISTA_STORED : s->fused ? L1B_RAN_FISTA_MF_PAIR : L1B_RAN_FISTA_SPARSE;
  sum->status = status;
  sum->time_to_target = INFINITY;
  sum->matvecs_to_target = INFINITY;
  sum->final_objective = NAN;
  const uint64_t total = h.n_samples + (h.last_sampled != h.k ? 1 : 0);
  for (size_t i = 0; i < tr.size(); ++i) {
    l1b_sample o;
    o.iter = tr[i].iter;
    o.elapsed_s = (double)(tr[i].ts_ns - h.t0_ns) * 1e-9;
    o.objective = tr[i].f;
    o.nnz = (uint64_t)tr[i].nnz;
    o.matvecs = 1.0 + 2.0 * (double)tr[i].iter;  // CountingOperator: 1 + 2 per iteration
    o.extra = 0;
    if (samples && i < cap) samples[i] = o;
    sum->final_objective = o.objective;
    if (!sum->reached_target && s->cfg.has_target && o.objective <= s->cfg.target) {
      sum->reached_target = 1;  // Tracker::sample (solvers.cpp:61-69)
      sum->time_to_target = o.elapsed_s;
      sum->matvecs_to_target = o.matvecs;
    }
  }
  sum->n_samples = total;
  sum->iterations = h.k;
  sum->elapsed_s = (double)(h.last_ts - h.t0_ns) * 1e-9;
  sum->total_matvecs = 1.0 + 2.0 * (double)h.k;
  if (status == L1B_TARGET_REACHED && !sum->reached_target) {  // Tracker::finish (:79-93)
    sum->reached_target = 1;
    sum->time_to_target = sum->elapsed_s;
    sum->matvecs_to_target = sum->total_matvecs;
  }
}


}  // namespace

namespace l1b {

void validate_cfg(const l1b_solver_cfg* c, uint64_t n) {  // SolverConfig::validate (solvers.cpp:133-143)
  if (!c) throw InvalidArgument("null solver config");
  if (c->solver < L1B_ISTA || c->solver > L1B_PCDM)
    throw InvalidArgument("SolverConfig: unknown solver id");
  if (!(c->mu > 0.0)) throw InvalidArgument("SolverConfig: mu must be positive");
  if (!(c->eta > 0.0 && c->eta < 1.0)) throw InvalidArgument("SolverConfig: eta must lie in (0, 1)");
  if (c->varpi < 1) throw InvalidArgument("SolverConfig: varpi must be at least 1");
  if (c->omega && (c->omega < 1 || c->omega > n))
    throw InvalidArgument("SolverConfig: omega must lie in [1, n]");
  if (c->l_fixed < 0.0 || std::isnan(c->l_fixed))
    throw InvalidArgument("SolverConfig: fixed L must be positive");
  if (c->l_policy != L1B_L_SPECTRUM && c->l_policy != L1B_L_BACKTRACKING)
    throw InvalidArgument("SolverConfig: unknown Lipschitz policy");
  if (c->arith != L1B_ARITH_EXACT && c->arith != L1B_ARITH_FMA)
    throw InvalidArgument("SolverConfig: unknown arithmetic mode");
  if (!(c->max_seconds > 0.0)) throw InvalidArgument("SolverConfig: max_seconds must be positive");
}

}  // namespace l1b

extern "C" {

int l1b_session_begin(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_session** out) {
  return guard([&] {
    if (!p || !out) throw InvalidArgument("null argument");
    *out = nullptr;
    ProblemView v = problem_view(p, false);
    validate_cfg(cfg, v.n);
    if (cfg->solver != L1B_FISTA && cfg->solver != L1B_ISTA)
      throw InvalidArgument("sessions drive FISTA / ISTA only");
    if (cfg->l_policy == L1B_L_BACKTRACKING && !(cfg->l_fixed > 0.0))
      throw Unsupported("sessions run a constant L (spectrum or l_fixed); LPolicy::backtracking runs in l1b_solve");
    L1B_CUDA(cudaSetDevice(v.device));
    auto* s = new l1b_session();
    try {
      session_begin(p, cfg, s);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int l1b_session_buffers(l1b_session* s, l1b_shard_buffers* out) {
  return guard([&] {
    if (!s || !out) throw InvalidArgument("null argument");
    out->x_win = s->shard ? s->x_win : s->x;
    out->r_y_win = s->shard ? s->r_y_win : s->r_y;
    out->scal = &s->st->scal[0];
    out->own = s->nx;
    out->halo = s->halo;
    out->single = s->single ? 1 : 0;
    for (int q = 0; q < 4; ++q) out->x_bufs[q] = s->X[q];
    for (int q = 0; q < 3; ++q) out->r_bufs[q] = s->R[q];
    out->x_nbufs = s->nbuf;
    out->x_halo = s->xh;
    out->r_halo = s->rh;
    out->lagged = s->recompute ? 1 : 0;
    out->pairs = s->pairs ? 1 : 0;
    out->scal8 = &s->st->scal8[0];
    out->general = s->general ? 1 : 0;
    out->g_full = s->g_full;
    out->x_full = s->x_full;
    out->n_pad = s->n_pad;
    out->col_begin = s->col_off;
    out->col_count = s->general ? s->nx : 0;
  });
}

int l1b_fp64_peak(int device, double* tflops) {
  return guard([&] {
    if (!tflops) throw InvalidArgument("null argument");
    *tflops = fp64_peak_tflops(device);
  });
}

int l1b_session_tile_geometry(l1b_session* s, int* iters, int64_t* span, int64_t* valid) {
  return guard([&] {
    if (!s || !iters || !span || !valid) throw InvalidArgument("null argument");
    *iters = s->tbk;
    *span = *valid = 0;
    if (s->tbk) fista_tb_geometry((int)s->v.op->right.count, s->tbk, span, valid);
  });
}

int l1b_session_tile_plan(l1b_session* s, uint64_t iters, int* ks, int cap, int* count) {
  return guard([&] {
    if (!s || !count || (cap > 0 && !ks)) throw InvalidArgument("null argument");
    const std::vector<int> plan = s->tile_plan(iters);
    *count = (int)plan.size();
    for (int i = 0; i < cap && i < (int)plan.size(); ++i) ks[i] = plan[(size_t)i];
  });
}

int l1b_tile_plan(int kmax, uint64_t iters, int* ks, int cap, int* count) {
  return guard([&] {
    if (!count || (cap > 0 && !ks)) throw InvalidArgument("null argument");
    if (kmax < 0 || (kmax > 0 && kmax % 4 != 2)) throw InvalidArgument("tile plan: K must be 2 mod 4");
    const std::vector<int> plan = plan_tile_launches(kmax, iters);
    *count = (int)plan.size();
    for (int i = 0; i < cap && i < (int)plan.size(); ++i) ks[i] = plan[(size_t)i];
  });
}

int l1b_session_kernel_mode(l1b_session* s, int* mode) {
  return guard([&] {
    if (!s || !mode) throw InvalidArgument("null argument");
    *mode = s->general ? L1B_KMODE_GENERAL_SHARD
            : !s->single ? (s->fused ? L1B_KMODE_MATRIX_FREE_PAIR : L1B_KMODE_SPARSE)
            : !s->recompute ? L1B_KMODE_STORED_RESIDUAL
            : s->tbk ? L1B_KMODE_RECOMPUTE_TILE
            : (!s->shard && rc2_enabled()) ? L1B_KMODE_RECOMPUTE_TWO
                                           : L1B_KMODE_RECOMPUTE;
  });
}

namespace {
void attach_side(l1b_session* s, double* const* bufs, uint64_t peer_lo, double** out) {
  for (int q = 0; q < 4; ++q) out[q] = bufs ? bufs[q] + (int64_t)s->xh - (int64_t)peer_lo : nullptr;
}
void check_peer_session(const l1b_session* s) {
  if (!s) throw InvalidArgument("null session");
  if (!(s->shard && s->recompute && s->nbuf == 4))
    throw LogicError("peer halos need a row-block shard session on the recomputing kernels");
}
}  // namespace

int l1b_session_attach_peers(l1b_session* s, double* const* left_bufs, uint64_t left_row_begin,
                             double* const* right_bufs, uint64_t right_row_begin) {
  return guard([&] {
    check_peer_session(s);
    attach_side(s, left_bufs, left_row_begin, s->peer_left);
    attach_side(s, right_bufs, right_row_begin, s->peer_right);
    s->peers_on = left_bufs || right_bufs;
  });
}

int l1b_session_export_x_ipc(l1b_session* s, void* handles) {
  return guard([&] {
    check_peer_session(s);
    if (!handles) throw InvalidArgument("null output");
    L1B_CUDA(cudaSetDevice(s->v.device));
    for (int q = 0; q < 4; ++q)
      L1B_CUDA(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handles) + q, s->X[q]));
  });
}

int l1b_session_attach_peers_ipc(l1b_session* s, const void* left_handles, uint64_t left_row_begin,
                                 const void* right_handles, uint64_t right_row_begin) {
  return guard([&] {
    check_peer_session(s);
    L1B_CUDA(cudaSetDevice(s->v.device));
    double* lb[4] = {nullptr, nullptr, nullptr, nullptr};
    double* rb[4] = {nullptr, nullptr, nullptr, nullptr};
    auto open = [&](const void* h, double** out) {
      for (int q = 0; q < 4; ++q) {
        void* p = nullptr;
        L1B_CUDA(cudaIpcOpenMemHandle(&p, reinterpret_cast<const cudaIpcMemHandle_t*>(h)[q],
                                      cudaIpcMemLazyEnablePeerAccess));
        s->ipc_opened.push_back(p);
        out[q] = static_cast<double*>(p);
      }
    };
    if (left_handles) open(left_handles, lb);
    if (right_handles) open(right_handles, rb);
    attach_side(s, left_handles ? lb : nullptr, left_row_begin, s->peer_left);
    attach_side(s, right_handles ? rb : nullptr, right_row_begin, s->peer_right);
    s->peers_on = left_handles || right_handles;
  });
}

int l1b_session_prox(l1b_session* s) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    if (!s->general) throw LogicError("prox is the middle step of general-shard sessions");
    L1B_CUDA(cudaSetDevice(s->v.device));
    fista_prox(s->g_full + s->col_off, s->x, s->y, s->nx, s->st, s->partials, s->v.stream);
  });
}

int l1b_session_flush(l1b_session* s) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    if (!s->recompute || !s->shard) return;  // single device: inside l1b_session_end
    L1B_CUDA(cudaSetDevice(s->v.device));
    s->iterate(s->launched, s->v.stream, true);
  });
}

int l1b_session_k1(l1b_session* s) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    L1B_CUDA(cudaSetDevice(s->v.device));
    if (s->single && s->pairs) {  // two iterations (the extra one past a stop is discarded)
      s->iterate2(s->launched, s->v.stream);
      s->launched += 2;
    } else if (s->single) {  // the whole iteration; k2 is then a no-op
      s->iterate(s->launched, s->v.stream);
      s->launched += 1;
    } else if (s->general) {  // partial A^T r_y of the own rows, all n columns
      spmv(s->v.At, s->r_y, s->g_full, s->v.stream);
    } else if (s->fused) {
      fista_fused_k1(*s->v.op, s->bufs(), s->v.stream);
    } else {
      fista_k1(s->v.At, s->bufs(), s->v.stream);
    }
  });
}

int l1b_session_k2(l1b_session* s) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    L1B_CUDA(cudaSetDevice(s->v.device));
    if (s->single) return;
    if (s->fused)
      fista_fused_k2(*s->v.op, s->bufs(), s->v.stream);
    else
      fista_k2(s->v.A, s->bufs(), s->v.stream);
    s->launched += 1;
  });
}

int l1b_session_finalize(l1b_session* s) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    if (!s->shard) throw LogicError("finalize is for row-block shards (single-device sessions finalise in K2)");
    L1B_CUDA(cudaSetDevice(s->v.device));
    fista_finalize_launch(s->bufs(), s->v.stream);
  });
}

int l1b_session_step(l1b_session* s, uint64_t iters) {
  NvtxRange nvtx("l1b_session_step");
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    if (s->shard) throw LogicError("shard sessions are stepped by the caller (k1 / k2 / finalize)");
    L1B_CUDA(cudaSetDevice(s->v.device));
    session_step(s, iters);
  });
}

int l1b_session_profile(l1b_session* s, uint64_t iters, double* ms_out, int n_ms) {
  return guard([&] {
    if (!s || !ms_out || n_ms < 2) throw InvalidArgument("bad arguments");
    if (s->shard) throw LogicError("profile drives single-device sessions");
    L1B_CUDA(cudaSetDevice(s->v.device));
    cudaStream_t st = s->v.stream;
    std::vector<cudaEvent_t> ev(3 * iters);
    for (auto& e : ev) L1B_CUDA(cudaEventCreate(&e));
    const FistaBufs b = s->bufs();
    if (uses_loop(s)) {  // one-iteration launches of the loop kernel, timed each
      for (uint64_t i = 0; i < iters; ++i) {
        L1B_CUDA(cudaEventRecord(ev[3 * i], st));
        fista_rc_loop(*s->v.op, s->iter_bufs(s->launched + i), s->X, s->launched + i, 1, 0, s->v.n, st);
        L1B_CUDA(cudaEventRecord(ev[3 * i + 1], st));
        L1B_CUDA(cudaEventRecord(ev[3 * i + 2], st));
      }
      s->launched += iters;
      L1B_CUDA(cudaStreamSynchronize(st));
      double k1 = 0.0, k2 = 0.0;
      for (uint64_t i = 0; i < iters; ++i) {
        float a = 0.f, c = 0.f;
        L1B_CUDA(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
        L1B_CUDA(cudaEventElapsedTime(&c, ev[3 * i + 1], ev[3 * i + 2]));
        k1 += a;
        k2 += c;
      }
      for (auto& e : ev) cudaEventDestroy(e);
      ms_out[0] = k1;
      ms_out[1] = k2;
      return;
    }
    // tile / two-iteration launches, timed each -- where session_step uses them too
    if (s->recompute && !s->shard && rc2_enabled()) {
      // ms_out[0] = the tile launches (tile sessions; else the two-iteration
      // launches), ms_out[1] = what is left after them (two-iteration / single
      // launches; empty for sessions without tiles and an even count)
      const std::vector<int> plan = s->tile_plan(iters);
      uint64_t i = 0;
      size_t e = 0;
      auto rec = [&] { L1B_CUDA(cudaEventRecord(ev[e++], st)); };
      std::vector<std::pair<size_t, int>> spans;  // (first event, slot)
      for (const int k : plan) {
        spans.emplace_back(e, 0);
        rec();
        s->iteratek(s->launched + i, st, k);
        rec();
        i += (uint64_t)k;
      }
      const int rest_slot = s->tbk ? 1 : 0;
      for (; i + 2 <= iters; i += 2) {
        spans.emplace_back(e, rest_slot);
        rec();
        s->iterate2(s->launched + i, st);
        rec();
      }
      if (i < iters) {
        spans.emplace_back(e, 1);
        rec();
        s->iterate(s->launched + i, st);
        rec();
      }
      s->launched += iters;
      L1B_CUDA(cudaStreamSynchronize(st));
      double k1 = 0.0, k2 = 0.0;
      for (const auto& sp : spans) {
        float a = 0.f;
        L1B_CUDA(cudaEventElapsedTime(&a, ev[sp.first], ev[sp.first + 1]));
        (sp.second ? k2 : k1) += a;
      }
      for (auto& e : ev) cudaEventDestroy(e);
      ms_out[0] = k1;
      ms_out[1] = k2;
      return;
    }
    for (uint64_t i = 0; i < iters; ++i) {
      L1B_CUDA(cudaEventRecord(ev[3 * i], st));
      if (s->single)
        s->iterate(s->launched + i, st);
      else if (s->fused)
        fista_fused_k1(*s->v.op, b, st);
      else
        fista_k1(s->v.At, b, st);
      L1B_CUDA(cudaEventRecord(ev[3 * i + 1], st));
      if (s->single) {
      } else if (s->fused) {
        fista_fused_k2(*s->v.op, b, st);
      } else {
        fista_k2(s->v.A, b, st);
      }
      L1B_CUDA(cudaEventRecord(ev[3 * i + 2], st));
    }
    s->launched += iters;
    L1B_CUDA(cudaStreamSynchronize(st));
    double k1 = 0.0, k2 = 0.0;
    for (uint64_t i = 0; i < iters; ++i) {
      float a = 0.f, c = 0.f;
      L1B_CUDA(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
      L1B_CUDA(cudaEventElapsedTime(&c, ev[3 * i + 1], ev[3 * i + 2]));
      k1 += a;
      k2 += c;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    ms_out[0] = k1;
    ms_out[1] = k2;
  });
}

int l1b_session_sync(l1b_session* s, int* stopped, uint64_t* iterations) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    L1B_CUDA(cudaSetDevice(s->v.device));
    L1B_CUDA(cudaMemcpyAsync(s->h_st, s->st, sizeof(FistaDev), cudaMemcpyDeviceToHost, s->v.stream));
    L1B_CUDA(cudaStreamSynchronize(s->v.stream));
    if (stopped) *stopped = s->h_st->stop;
    if (iterations) *iterations = s->h_st->k;
  });
}

int l1b_session_restart(l1b_session* s) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    if (s->general) throw Unsupported("restart: general shards keep no restartable state");
    L1B_CUDA(cudaSetDevice(s->v.device));
    session_reset(s);
  });
}

int l1b_session_read(l1b_session* s, l1b_sample* samples, uint64_t cap, l1b_summary* summary,
                     double* x_host) {
  return guard([&] {
    if (!s) throw InvalidArgument("null session");
    if (!s->shard) throw LogicError("read: single-device sessions report through l1b_session_end");
    L1B_CUDA(cudaSetDevice(s->v.device));
    l1b_summary tmp;
    session_finish(s, samples, cap, summary ? summary : &tmp, x_host, nullptr);
  });
}

int l1b_session_end(l1b_session* s, l1b_sample* samples, uint64_t cap, l1b_summary* summary,
                    double* x_host) {
  const int rc = guard([&] {
    if (!s) throw InvalidArgument("null session");
    L1B_CUDA(cudaSetDevice(s->v.device));
    l1b_summary tmp;
    session_finish(s, samples, cap, summary ? summary : &tmp, x_host, nullptr);
  });
  delete s;
  return rc;
}

int l1b_solve(l1b_problem* p, const l1b_solver_cfg* cfg, l1b_sample* samples, uint64_t cap,
              l1b_summary* summary, double* x_host, double* d_x) {
  NvtxRange nvtx("l1b_solve");
  return guard([&] {
    if (!p || !summary) throw InvalidArgument("null argument");
    ProblemView v = problem_view(p, false);
    validate_cfg(cfg, v.n);
    if (v.shard)
      throw Unsupported("a row-block shard is solved by the distributed driver (l1b_session_k1/k2/finalize)");
    L1B_CUDA(cudaSetDevice(v.device));
    if (cfg->solver == L1B_PCDM || cfg->solver == L1B_CD) {
      run_pcdm(p, cfg, samples, cap, summary, x_host, d_x);
      return;
    }
    if (cfg->solver == L1B_NEWTON_CG) {
      run_newton_cg(p, cfg, samples, cap, summary, x_host, d_x);
      return;
    }
    if (cfg->l_policy == L1B_L_BACKTRACKING && !(cfg->l_fixed > 0.0)) {  // LipschitzState (:103-119)
      run_fista_backtracking(p, cfg, samples, cap, summary, x_host, d_x);
      return;
    }
    // host-side setup before session_begin: the device clock of the trace
    // starts in its init kernel
    // L1B_SOLVE_TRACE=1: host-side phase times on stderr
    const bool tracing = getenv("L1B_SOLVE_TRACE") != nullptr;
    auto tp = std::chrono::steady_clock::now();
    auto ptrace = [&](const char* what) {
      if (!tracing) return;
      const auto now = std::chrono::steady_clock::now();
      fprintf(stderr, "[l1b_solve] %-16s %9.1f us\n", what, std::chrono::duration<double, std::micro>(now - tp).count());
      tp = now;
    };
    int* h_flags = nullptr;
    h_flags = (int*)pinned_cache().get();
    l1b_session s;
    try {
      session_begin(p, cfg, &s);
    } catch (...) {
      pinned_cache().put(h_flags);
      throw;
    }
    ptrace("session begun");
    cudaStream_t st = v.stream;
    cudaEvent_t ev[2];
    L1B_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    L1B_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    bool pending[2] = {false, false};
    int slot = 0;
    // small instances run whole chunks in one launch (fista_rc_loop): start at
    // the full chunk, each launch costs a reload of the instance
    // (tile sessions: chunks of whole K-iteration launches)
    const uint64_t tk = (uint64_t)s.tbk;
    uint64_t chunk = uses_loop(&s) ? 64 : tk ? tk : 4;
    try {
      while (s.launched < cfg->max_iters) {
        // loop-head time check (solvers.cpp:314), at chunk granularity
        const double el =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - s.t0).count();
        if (el > cfg->max_seconds) {
          s.time_out = true;
          break;
        }
        const uint64_t k = std::min<uint64_t>(chunk, cfg->max_iters - s.launched);
        session_step(&s, k);
        L1B_CUDA(cudaMemcpyAsync(&h_flags[slot], &s.st->stop, sizeof(int), cudaMemcpyDeviceToHost, st));
        L1B_CUDA(cudaEventRecord(ev[slot], st));
        pending[slot] = true;
        slot ^= 1;
        if (pending[slot]) {  // the previous chunk: one chunk of look-ahead stays queued
          L1B_CUDA(cudaEventSynchronize(ev[slot]));
          pending[slot] = false;
          if (h_flags[slot]) break;
        }
        chunk = std::min<uint64_t>(chunk * 2, tk ? 4 * tk : 64);
      }
      L1B_CUDA(cudaStreamSynchronize(st));
      ptrace("iterations done");
    } catch (...) {
      cudaEventDestroy(ev[0]);
      cudaEventDestroy(ev[1]);
      pinned_cache().put(h_flags);
      throw;
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    pinned_cache().put(h_flags);
    session_finish(&s, samples, cap, summary, x_host, d_x);
    ptrace("finished");
  });
}


}  // extern "C"

// ---------------------------------------------------------------------------
// Native shard driver: the loop distributed.py drives from Python
// (k1 -> halos -> all-reduce -> finalize per launch), issued here on the
// session's stream with the library's own NCCL communicator and, for the
// steady state, replayed from a CUDA graph of two launches (x rotates with
// period 4, a launch advances it by 2), so no host work sits between the
// kernels of consecutive launches.  Lagged two-iteration shards (the default
// for banded 1..4-stage operators) only.

namespace {

void check_native(const l1b_session* s) {
  if (!s) throw InvalidArgument("null session");
  if (!(s->shard && s->single && s->recompute && s->pairs))
    throw Unsupported("native shard driver: lagged two-iteration shards only (distributed.py drives the others)");
}

void check_comm(const l1b_session* s) {
  check_native(s);
  if (!s->comm) throw LogicError("no NCCL communicator: call l1b_session_attach_nccl first");
}

// launch j (iteration j+1, j+2): k1, then the x halos of both new iterates
// (unless the kernel stored them into the neighbours), all-reduce of the 8
// sums, finalize (records two iterations, lagged)
void native_exchange(l1b_session* s, uint64_t j) {
  const NcclApi& N = nccl();
  cudaStream_t st = s->v.stream;
  if (!s->peers_on && s->comm_world > 1) {
    const size_t h = s->xh, own = s->nx;
    L1B_NCCL(N.GroupStart());
    for (int w = 1; w <= 2; ++w) {
      double* win = s->X[(j + w) % 4];
      if (s->comm_rank > 0) {
        L1B_NCCL(N.Send(win + h, h, ncclDouble, s->comm_rank - 1, s->comm, st));
        L1B_NCCL(N.Recv(win, h, ncclDouble, s->comm_rank - 1, s->comm, st));
      }
      if (s->comm_rank < s->comm_world - 1) {
        L1B_NCCL(N.Send(win + own, h, ncclDouble, s->comm_rank + 1, s->comm, st));
        L1B_NCCL(N.Recv(win + own + h, h, ncclDouble, s->comm_rank + 1, s->comm, st));
      }
    }
    L1B_NCCL(N.GroupEnd());
  }
  L1B_NCCL(N.AllReduce(s->st->scal8, s->st->scal8, 8, ncclDouble, ncclSum, s->comm, st));
  fista_finalize_launch(s->bufs(), st);
}

void native_launch(l1b_session* s, cudaEvent_t k1_begin = nullptr, cudaEvent_t k1_end = nullptr) {
  const uint64_t j = s->launched;
  if (k1_begin) L1B_CUDA(cudaEventRecord(k1_begin, s->v.stream));
  s->iterate2(j, s->v.stream);
  if (k1_end) L1B_CUDA(cudaEventRecord(k1_end, s->v.stream));
  s->launched += 2;
  native_exchange(s, j);
}

void native_reduce_finalize(l1b_session* s) {
  L1B_NCCL(nccl().AllReduce(s->st->scal, s->st->scal, 4, ncclDouble, ncclSum, s->comm, s->v.stream));
  fista_finalize_launch(s->bufs(), s->v.stream);
}

}  // namespace

extern "C" {

int l1b_nccl_get_unique_id(void* id_out) {
  return guard([&] {
    if (!id_out) throw InvalidArgument("null output");
    ncclUniqueId id;
    L1B_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int l1b_nccl_version(int* version) {
  return guard([&] {
    if (!version) throw InvalidArgument("null output");
    *version = nccl().version;
  });
}

int l1b_session_attach_nccl(l1b_session* s, const void* unique_id, int rank, int world) {
  return guard([&] {
    check_native(s);
    if (!unique_id) throw InvalidArgument("null unique id");
    if (world != s->v.world || rank != s->v.rank)
      throw InvalidArgument("communicator rank / size differ from the shard's");
    if (s->comm) throw LogicError("session already has a communicator");
    if (!s->v.stream) throw InvalidArgument("the native driver needs a non-default stream (graph capture)");
    L1B_CUDA(cudaSetDevice(s->v.device));
    const NcclApi& N = nccl();
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    L1B_NCCL(N.CommInitRank(&s->comm, world, id, rank));
    s->comm_rank = rank;
    s->comm_world = world;
    // connect every channel this session uses (all-reduce, neighbour send /
    // recv) outside of any capture: NCCL sets connections up on first use
    double* tmp = s->dalloc(2 * s->xh + 8);
    L1B_CUDA(cudaMemsetAsync(tmp, 0, (2 * s->xh + 8) * 8, s->v.stream));
    L1B_NCCL(N.AllReduce(tmp, tmp, 8, ncclDouble, ncclSum, s->comm, s->v.stream));
    if (world > 1) {
      L1B_NCCL(N.GroupStart());
      if (rank > 0) {
        L1B_NCCL(N.Send(tmp + 8, s->xh, ncclDouble, rank - 1, s->comm, s->v.stream));
        L1B_NCCL(N.Recv(tmp + 8 + s->xh, s->xh, ncclDouble, rank - 1, s->comm, s->v.stream));
      }
      if (rank < world - 1) {
        L1B_NCCL(N.Send(tmp + 8, s->xh, ncclDouble, rank + 1, s->comm, s->v.stream));
        L1B_NCCL(N.Recv(tmp + 8 + s->xh, s->xh, ncclDouble, rank + 1, s->comm, s->v.stream));
      }
      L1B_NCCL(N.GroupEnd());
    }
    L1B_CUDA(cudaStreamSynchronize(s->v.stream));
  });
}

int l1b_session_nccl_start(l1b_session* s) {
  return guard([&] {
    check_comm(s);
    L1B_CUDA(cudaSetDevice(s->v.device));
    native_reduce_finalize(s);  // f_0 from the summed ||b_own||^2
  });
}

int l1b_session_nccl_steps(l1b_session* s, uint64_t launches, int use_graph, double* k1_ms) {
  NvtxRange nvtx("l1b_session_nccl_steps");
  return guard([&] {
    check_comm(s);
    L1B_CUDA(cudaSetDevice(s->v.device));
    cudaStream_t st = s->v.stream;
    if (k1_ms) {  // events around every k1 (no graph): the per-rank kernel time
      std::vector<cudaEvent_t> ev(2 * launches);
      for (auto& e : ev) L1B_CUDA(cudaEventCreate(&e));
      for (uint64_t i = 0; i < launches; ++i) native_launch(s, ev[2 * i], ev[2 * i + 1]);
      L1B_CUDA(cudaStreamSynchronize(st));
      double tot = 0.0;
      for (uint64_t i = 0; i < launches; ++i) {
        float a = 0.f;
        L1B_CUDA(cudaEventElapsedTime(&a, ev[2 * i], ev[2 * i + 1]));
        tot += a;
      }
      for (auto& e : ev) cudaEventDestroy(e);
      *k1_ms = tot;
      return;
    }
    uint64_t i = 0;
    if (use_graph) {
      for (; i + 2 <= launches; i += 2) {
        const int q = (int)((s->launched % 4) / 2);
        if (!s->graph[q]) {  // capture launches j, j+1 (host bookkeeping rewound afterwards)
          const uint64_t j0 = s->launched, k0 = g_launch_count.load();
          cudaGraph_t g = nullptr;
          L1B_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          try {
            native_launch(s);
            native_launch(s);
          } catch (...) {
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            s->launched = j0;
            throw;
          }
          L1B_CUDA(cudaStreamEndCapture(st, &g));
          s->graph_kernels[q] = g_launch_count.load() - k0;
          g_launch_count.fetch_sub(s->graph_kernels[q]);  // counted when replayed
          const cudaError_t e = cudaGraphInstantiate(&s->graph[q], g, 0);
          cudaGraphDestroy(g);
          L1B_CUDA(e);
          s->launched = j0;
        }
        L1B_CUDA(cudaGraphLaunch(s->graph[q], st));
        g_launch_count.fetch_add(s->graph_kernels[q]);
        s->launched += 4;
      }
    }
    for (; i < launches; ++i) native_launch(s);
    nccl_check_async(s->comm);  // a peer's failure surfaces here, not as a hang later
  });
}

int l1b_session_nccl_finish(l1b_session* s) {
  return guard([&] {
    check_comm(s);
    L1B_CUDA(cudaSetDevice(s->v.device));
    s->iterate(s->launched, s->v.stream, true);  // flush: ||r||^2 of the last iterate
    native_reduce_finalize(s);
    nccl_check_async(s->comm);
  });
}

}  // extern "C"
