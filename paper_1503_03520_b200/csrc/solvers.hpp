// solvers.hpp -- what the solver drivers see of a problem.
#pragma once

#include <cuda_runtime.h>

#include "../../include/l1b.h"
#include "common.cuh"
#include "kernels.hpp"

namespace l1b {

struct ProblemView {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t m = 0, n = 0;
  double tau = 1.0, lmax = 0.0, tail_sq = 0.0, tail_sq_band = 0.0;
  bool fused_ok = false;  // banded operator: the matrix-free fused kernels apply
  const double* b = nullptr;  // m
  Csr A;                      // CSR over active rows
  Csr At;                     // CSC over n columns
  const OpView* op = nullptr;
  const double* gram = nullptr;
  uint64_t max_row_nnz = 0;  // omega of solvers.cpp:401-410 (max nnz over rows)
  uint64_t max_col_nnz = 0;
  // row-block shard (world > 1): own rows == own columns [row_begin, row_end);
  // A / At index x / r windows that start `halo` entries before row_begin
  int world = 1, rank = 0;
  bool shard = false;
  uint64_t row_begin = 0, row_end = 0, halo = 0;
  // shards: b by global row index, valid on [b_win_lo, b_win_hi) (null if absent)
  const double* b_win = nullptr;
  uint64_t b_win_lo = 0, b_win_hi = 0;
  // general (non-banded) shard: A's rows [row_begin, row_end) as CSR with global
  // columns + the CSC of that block (local rows); x sliced by columns
  bool general = false;
  uint64_t col_begin = 0, col_end = 0, col_slice = 0;
};

ProblemView problem_view(l1b_problem* p, bool need_sparse = true);
const double* problem_gram(l1b_problem* p);  // lazily built diag(A^T A)
const double* problem_sigma_scaled(l1b_problem* p);  // lazily built sigma * prod cos(theta) (contracted arithmetic)

}  // namespace l1b
