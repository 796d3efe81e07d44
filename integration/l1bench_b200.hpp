// l1bench_b200.hpp -- drop-in device solvers for the reference's C++ API.
//
// A program that links the reference (`l1bench`, proj/include/l1bench) swaps
//     l1bench::run_solver(inst, cfg, &x)
// for
//     l1bench::b200::run_solver(inst, cfg, &x)
// (same types, same argument meaning, same exceptions); the instance is
// uploaded through the C ABI (include/l1b.h) and the whole solver loop runs on
// the GPU.  See INTEGRATION.md.
#pragma once

#include <vector>

#include "l1bench/instance.hpp"
#include "l1bench/solvers.hpp"

namespace l1bench::b200 {

// solvers.hpp:106-117 equivalents (ids: ista, fista, cd, newton_cg; + pcdm)
SolverTrace run_solver(const ProblemInstance& inst, const SolverConfig& cfg,
                       std::vector<double>* x_out = nullptr);
SolverTrace fista_run(const ProblemInstance& inst, const SolverConfig& cfg,
                      std::vector<double>* x_out = nullptr);
SolverTrace ista_run(const ProblemInstance& inst, const SolverConfig& cfg,
                     std::vector<double>* x_out = nullptr);
SolverTrace coordinate_descent_run(const ProblemInstance& inst, const SolverConfig& cfg,
                                   std::vector<double>* x_out = nullptr);
SolverTrace newton_cg_run(const ProblemInstance& inst, const SolverConfig& cfg,
                          std::vector<double>* x_out = nullptr);

}  // namespace l1bench::b200
