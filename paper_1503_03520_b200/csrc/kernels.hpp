// kernels.hpp -- host-side launchers of the device kernels (one per .cu file).
#pragma once

#include <vector>

#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace l1b {

// ---- k_build.cu ----------------------------------------------------------
struct LinesOut {
  uint64_t lines = 0;    // lines kept (trailing empty lines trimmed when asked)
  uint64_t nnz = 0;
  uint32_t max_len = 0;
  uint64_t tile_nnz_max = 0;  // max nonzeros over 256-line tiles
  bool ptr32 = true;
  void* ptr = nullptr;   // (lines + 1) x u32 or u64 (+16 B of slack for the bulk copies)
  uint32_t* idx = nullptr;
  double* val = nullptr;
  uint32_t* tile_rng = nullptr;  // per 256-line tile: min, max index (the SpMV stages x[min..max])
  uint64_t x_len = 0;            // largest index + 1: entries of x the products read
};
// Lines [first, first + nlines) of A (rows) or A^T (columns = CSC of A).
// Indices are stored minus idx_base (wrapping), i.e. local to a window; only
// entries with index in [keep_lo, keep_hi) are kept (a general shard's CSC).
void build_lines(const OpView& op, bool rows, uint64_t first, uint64_t nlines, uint64_t idx_base,
                 bool trim_tail, cudaStream_t st, LinesOut* out, uint64_t keep_lo = 0,
                 uint64_t keep_hi = ~0ull);
void gram_diagonal(const OpView& op, uint64_t first, uint64_t ncols, double* d, cudaStream_t st);

// ---- k_rng.cu (std::mt19937_64 streams on the device, bit-exact) ----------
// Draws [0, count) of Rng(seed) as uniform_in(lo, hi) (rng.hpp:44-47); with
// `spectrum` the draws follow Spectrum::uniform (linops.cpp:323-331): + shift,
// rejection of u <= lo.  Draws [wlo, whi) are stored to d_out[i - wlo]; when
// vmin / vmax are given, the min / max over all draws (non-negative values).
// Returns false when a draw would be rejected (the stream shifts; the caller
// replays it sequentially).  Chunks hold >= 2^min_log2_chunk draws.  Syncs.
bool device_uniform_draws(uint64_t seed, uint64_t count, double lo, double hi, bool spectrum,
                          double shift, uint64_t wlo, uint64_t whi, double* d_out, double* vmin,
                          double* vmax, cudaStream_t st, int min_log2_chunk = 12);
// uniform_index(rng, n) draws (rng.hpp:37-45) continuing a device-resident
// stream: d_window = the 312-word state (mt_seed_state, updated in place);
// d_out[q] = index of draw q, 0xffffffff where the reference would redraw.
// Draws count rounded up to a multiple of 312 (returned; d_out must hold them).
// d_words: scratch of as many 64-bit words (null: allocated on the stream).
// Streams longer than one chunk (312 x 256 draws) run in parallel chunks
// started by jump-ahead (k_rng.cu).
void mt_seed_state(uint64_t seed, uint64_t* w312);
// The rejection limit of the CD / PCDM coordinate draws: UINT64_MAX -
// UINT64_MAX % n (rng.hpp:37-45).  Test hook: L1B_TEST_INDEX_REJECT=s lowers
// it by UINT64_MAX >> s (a draw is redrawn with probability ~2^-s), so the
// redraw paths, hit once per ~2^64/n draws otherwise, run under parity tests
// (oracle: lo_set_index_reject).  Read per call.
uint64_t coord_index_limit(uint64_t n);
uint64_t mt_stream_indices(uint64_t* d_window, uint64_t count, uint64_t n, uint32_t* d_out,
                           uint64_t* d_words, cudaStream_t st);
// the raw 64-bit outputs of the same continued stream (count rounded up to 312)
uint64_t mt_stream_raw(uint64_t* d_window, uint64_t count, uint64_t* d_out, cudaStream_t st);
// ---- k_solution.cu ------------------------------------------------------------
// uniform_sparse_solution (solution.cpp:47-75) from Rng(seed) on the device:
// the support ascending and the values; false when a draw the reference
// would redraw occurs (the caller replays the stream on the host).  Syncs.
bool device_sparse_solution(uint64_t n, uint64_t s, double gamma, uint64_t seed, std::vector<uint32_t>& sup,
                            std::vector<double>& val, cudaStream_t st);
// Permutation::realize (linops.cpp:224-239) from Rng(seed) on the device into
// host_map (m entries); false on a draw the reference redraws.  Syncs.
bool device_permutation(uint64_t m, uint64_t seed, uint32_t* host_map, cudaStream_t st);
// host: raw 64-bit outputs 2^log2_jump .. 2^log2_jump + count - 1 of
// std::mt19937_64(seed) through the jump polynomial (log2_jump < 0: no jump)
void host_draws_after_jump(uint64_t seed, int log2_jump, uint64_t count, uint64_t* out);
// host: raw outputs c J .. c J + count - 1 through t^(c J) mod P, J = the
// coordinate-stream chunk (the start of chunk c in mt_stream_indices)
void host_draws_after_chunk_jump(uint64_t seed, uint64_t c, uint64_t count, uint64_t* out);
constexpr uint64_t kIdxChunkDraws = 312 * 256;

// ---- k_bt.cu ----------------------------------------------------------------
// estimate_gram_lmax (linops.cpp:757-778) with the matrix-free products (syncs)
double estimate_gram_lmax_device(const OpView& op, uint64_t m, uint64_t n, uint64_t iters, uint64_t seed,
                                 cudaStream_t st);

// ---- k_sweep.cu (matrix-free, bit-exact vs linops.cpp) ---------------------
void sweep_apply(const OpView& op, const double* x, double* y, cudaStream_t st);
void sweep_apply_transpose(const OpView& op, const double* y, double* x, cudaStream_t st);
// spectral_sparse_solution's selection (solution.cpp:77-113) given xhat =
// gamma / sigma^2 on the host: right factor applied on the device, the s1
// smallest and s2 largest |xhat| nonzeros (stable), ascending support
void spectral_select(const OpView& op, const double* xhat_host, uint64_t n, uint64_t s1, uint64_t s2,
                     cudaStream_t st, std::vector<uint32_t>& sup, std::vector<double>& val);
void sweep_gram_inverse(const OpView& op, const double* v, double* out, cudaStream_t st);
void scatter_sparse(const uint32_t* sup, const double* val, uint64_t s, double* dense, uint64_t n,
                    cudaStream_t st);
// dense[sup[k]] = val[k] (no zero fill)
void scatter_values(const uint32_t* sup, const double* val, uint64_t s, double* dense,
                    cudaStream_t st);
// b += tau * e-part: e *= tau; b += e; returns sum(e^2) through *sum_sq (device)
void generator_combine(double tau, double* e, double* b, uint64_t m, double* d_sum_sq,
                       cudaStream_t st);
void vec_sub(double* a, const double* b, uint64_t n, cudaStream_t st);  // a -= b
double device_sum_sq(const double* v, uint64_t n, cudaStream_t st);      // sum v_i^2 (syncs)
// min over i of sigma_i and a flag for any non-finite entry (syncs)
void device_min_finite(const double* v, uint64_t n, double* vmin, double* vmax, bool* finite,
                       cudaStream_t st);
// max_S |r_i + tau sign(x_i)|, max_{S^c} (|r_i| - tau)_+  (instance.cpp:187-198)
void certificate(const double* r, const double* xd, double tau, uint64_t n, double* d_out2,
                 cudaStream_t st);

// windowed sweeps of a row-block shard (global entries [ws, we) of a dim-vector)
void window_stages(const StageTab& tab, bool forward, bool transposed, double* v, uint64_t ws,
                   uint64_t we, uint64_t dim, cudaStream_t st);
// mode 0: v /= sig^2, 1: v = sig * v, 2: v *= tau
// out[i] = in[i] * a
void scale_copy(const double* in, double a, double* out, uint64_t len, cudaStream_t st);
void window_scale_op(double* v, const double* sig, uint64_t len, int mode, double tau,
                     cudaStream_t st);

// ---- k_spmv.cu -------------------------------------------------------------
struct Csr {  // CSR of A (rows) or of A^T (= CSC of A)
  uint64_t lines = 0;
  uint64_t nnz = 0;
  bool ptr32 = true;
  const void* ptr = nullptr;
  const uint32_t* idx = nullptr;
  const double* val = nullptr;
  int lanes = 32;  // lines per warp tile (fallback kernel)
  uint64_t tile_nnz_max = ~0ull;  // max nonzeros of a 256-line tile (TMA kernel when <= 2048)
  const uint32_t* tile_rng = nullptr;  // per 256-line tile: min, max index (null: not staged)
  uint64_t x_len = 0;                  // x entries the products may read (staging never reads past)
};

// y[0, lines) = M x
void spmv(const Csr& M, const double* x, double* y, cudaStream_t st);
// out = tau*||x||_1 + 0.5*(sum_{i<lines} (Mx - b)_i^2 + tail_sq) into *d_f
void objective(const Csr& A, const double* x, uint64_t n, const double* b, double tau,
               double tail_sq, double* d_f, cudaStream_t st);

// FISTA / ISTA device loop state (solvers.cpp:277-382)
struct FistaSample {
  uint64_t iter;
  double f;
  double nnz;
  uint64_t ts_ns;
};
struct FistaDev {
  double t, lval, tau, f, nnz, target, tail_sq;
  double init_tail;  // sum b_i^2 of the rows the init kernel does not cover
  double beta_y;     // momentum that forms y / r_y from the last two iterates (single-kernel path)
  uint64_t k, max_iters, n_samples, cap, last_sampled, t0_ns, last_ts;
  int stop, status, accel, has_target;
  int defer;        // shards: K2 / init leave scal for the caller's all-reduce
  int initialized;  // sample 0 written
  unsigned int ticket[4];
  double scal[4];  // l1, nnz, mismatches, ||r||^2 of the last iteration
  // lagged objective (recomputing kernel): kernel j sums ||r_j||^2 while it
  // produces x_{j+1}; x_{j+1}'s l1 / nnz / mismatches wait here for kernel j+1
  double pend[3];
  uint64_t pend_ts;
  int pend_valid;
  int lagged;    // the recomputing kernel: fista_finalize_lagged
  int flushing;  // set by its flush launch (deferred finalize records, then stops stashing)
  // two-iteration kernel: ||r_k||^2, (l1, nnz, mism) of x_{k+1}, ||r_{k+1}||^2,
  // (l1, nnz, mism) of x_{k+2}
  double scal8[8];
  int pair_pending;  // shards: the last kernel ran two iterations (finalize: lagged2)
  // tile kernel (K iterations per launch): t and beta_y as the last launch
  // found them -- a stop inside a launch replays it from there (fista_rc_iterk)
  double snap_t, snap_beta;
};

struct FistaBufs {
  double *x, *y;          // n (own columns)
  double *r_x, *r_y;      // rows (own rows)
  const double* x_gather;    // vector K2 gathers (x, or the shard's x window)
  const double* r_y_gather;  // vector K1 gathers (r_y, or the shard's r_y window)
  // own range [lo, hi) of rows == columns in global indices; gather windows
  // start at global index gather_base (0 on one device, a - halo on a shard)
  uint64_t lo = 0, hi = 0;
  int64_t gather_base = 0;
  const double* b;
  FistaDev* st;
  FistaSample* trace;
  double* partials;       // grid_max * 4
};

int spmv_grid_max();
void fista_init(const FistaBufs& fb, uint64_t m_rows, cudaStream_t st);
// K1: x, y <- prox/momentum of A^T r_y      (CSC over n columns)
void fista_k1(const Csr& At, const FistaBufs& fb, cudaStream_t st);
// K2: r_x, r_y <- A x - b, residual momentum (CSR over active rows) + finalize
void fista_k2(const Csr& A, const FistaBufs& fb, cudaStream_t st);
// matrix-free products / FISTA kernels for banded operators (k_fused.cu);
// vectors need 2 entries of slack past their end (16-byte bulk copies)
bool fused_supported(const OpView& op);
void fused_apply(const OpView& op, const double* x, double* y, cudaStream_t st);
void fused_apply_transpose(const OpView& op, const double* r, double* g, cudaStream_t st);
void fista_fused_k1(const OpView& op, const FistaBufs& fb, cudaStream_t st);
void fista_fused_k2(const OpView& op, const FistaBufs& fb, cudaStream_t st);
// one kernel per FISTA iteration (k_fused.cu): x / r rotate through 3 buffers,
// y and r_y are formed on the fly from the last two iterates
struct IterBufs {
  const double* x_k;    // x after iteration k (window reads)
  const double* x_km1;  // x after iteration k-1
  const double* r_k;    // r = A x - b after iteration k (rows [0, n))
  const double* r_km1;
  double* x_next;       // x after iteration k+1 (own writes)
  double* r_next;
  const double* b;
  FistaDev* st;
  FistaSample* trace;
  double* partials;
};
bool fused_iter_supported(const OpView& op);  // banded, 1..4 stages
// lines [lo, hi) (a shard's own block, [0, n) on one device); every IterBufs
// pointer is indexed by GLOBAL entry
void fista_fused_iter(const OpView& op, const IterBufs& ib, uint64_t lo, uint64_t hi,
                      cudaStream_t st);
// the same iteration with r_k, r_{k-1} recomputed from x_k, x_{k-1} (k_iter_rc.cu):
// reads x_k, x_km1, sigma, b, writes x_next (32-byte aligned, lo % 4 == 0);
// r_* of ib unused.  A shard's x windows need fista_rc_halo(stages) entries.
// Neighbour shards' x windows as global-index views (x_{k+1}, x_{k+2}), for
// kernels that store the halo entries themselves (peer memory over NVLink).
struct PeerViews {
  int on = 0;
  int64_t halo = 0;
  double* left[2] = {nullptr, nullptr};
  double* right[2] = {nullptr, nullptr};
};
// The objective lags one kernel (fista_finalize_lagged); flush = true records
// the last iterate's (x_k of ib) after the loop.
// fma: the contracted arithmetic (L1B_ARITH_FMA, common.cuh rot<true>)
void fista_rc_iter(const OpView& op, const IterBufs& ib, uint64_t lo, uint64_t hi, cudaStream_t st,
                   bool flush = false, const PeerViews& peers = PeerViews(), bool fma = false);
int fista_rc_halo(int stages);
// x-window halo of the two-iteration kernel (default 8-entries-per-lane variant)
int fista_rc2_halo(int stages);
// `iters` iterations j0, j0+1, ... of the same kernel in ONE cooperative launch
// (grid barriers between iterations; x rotates through X[j % 3]) -- small
// instances, where a launch per iteration costs more than the iteration.
void fista_rc_loop(const OpView& op, const IterBufs& ib, double* const X[4], uint64_t j0,
                   uint64_t iters, uint64_t lo, uint64_t hi, cudaStream_t st);
// two iterations (x_{k+1} into ib.x_next, x_{k+2} into x_next2) in one kernel:
// 24n bytes per iteration (k_iter_rc.cu fista_rc2_kernel); one device
void fista_rc_iter2(const OpView& op, const IterBufs& ib, double* x_next2, uint64_t lo, uint64_t hi,
                    cudaStream_t st, const PeerViews& peers = PeerViews(), bool fma = false);
// K iterations in one launch (k_iter_rc.cu fista_tb_kernel: tiles of 16 warps
// advance K iterations with their x halos exchanged in shared memory):
// x_{k+K-1} into out1, x_{k+K} into out2; K in [2, kTbKMax].  tb = device
// scratch of fista_tb_scratch(K) doubles.  replay: the same iterations from
// the launch's snapshot of t / beta_y without any bookkeeping, only out2
// written (a stop inside the launch: x of the stopping iteration).  One device.
constexpr int kTbKMax = 14;
void fista_rc_iterk(const OpView& op, const IterBufs& ib, double* out1, double* out2, int K, bool replay,
                    double* tb, cudaStream_t st, bool fma);
uint64_t fista_tb_scratch();
void fista_tb_geometry(int stages, int K, int64_t* span, int64_t* valid);
// k_probe.cu: dense FP64 fma throughput of this GPU (TFLOP/s, best of 3 timed runs)
double fp64_peak_tflops(int device);
// n from which the tile kernel runs (L1B_TB=0: never; L1B_TB_K: iterations per launch)
bool tb_enabled(uint64_t n, int stages);
int tb_iters();
// loads the recomputing kernels and sizes their grids (outside the timed loop)
void fista_rc_prepare(const OpView& op, bool fma = false);
// general shards: prox / momentum on the own column slice from the reduced g
void fista_prox(const double* g, double* x, double* y, uint64_t cols, FistaDev* st,
                double* partials, cudaStream_t stream);
// deferred finalisation (shards): after the caller summed st->scal across ranks
void fista_finalize_launch(const FistaBufs& fb, cudaStream_t st);

}  // namespace l1b
