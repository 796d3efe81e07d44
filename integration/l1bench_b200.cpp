// l1bench_b200.cpp -- the reference-side binding of libl1b:
// converts the reference's ProblemInstance / SolverConfig into the C ABI's
// plain structs, calls l1b_problem_create + l1b_solve, and converts the trace
// back, rethrowing the reference's exception types with the ABI's message.
#include "l1bench_b200.hpp"

#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>

#include "l1b.h"
#include "l1bench/bench.hpp"

namespace l1bench::b200 {

namespace {

[[noreturn]] void rethrow(int rc) {
  const std::string msg = l1b_last_error();
  switch (rc) {
    case L1B_EINVAL: throw std::invalid_argument(msg);
    case L1B_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

void check(int rc) {
  if (rc != L1B_OK) rethrow(rc);
}

struct Problem {
  l1b_problem* p = nullptr;
  ~Problem() {
    if (p) l1b_problem_free(p);
  }
};

// OperatorSpec (linops.hpp:159-206) -> l1b_operator_desc; paired stages only
void upload(const ProblemInstance& inst, Problem* out) {
  if (inst.is_wide()) throw std::invalid_argument("b200: wide (m < n) instances are not supported");
  const OperatorSpec& spec = *inst.factored;
  std::vector<int32_t> ro, lo;
  std::vector<double> rt, lt;
  for (const auto& st : spec.right_stages) {
    if (st.kind != RotationStage::Kind::paired) throw std::invalid_argument("b200: explicit-list stages are not supported");
    ro.push_back(st.offset);
    rt.push_back(st.theta);
  }
  for (const auto& st : spec.left_stages) {
    if (st.kind != RotationStage::Kind::paired) throw std::invalid_argument("b200: explicit-list stages are not supported");
    lo.push_back(st.offset);
    lt.push_back(st.theta);
  }
  l1b_operator_desc d{};
  d.m = spec.m;
  d.n = spec.n;
  d.n_right = (uint32_t)ro.size();
  d.right_offset = ro.data();
  d.right_theta = rt.data();
  d.n_left = (uint32_t)lo.size();
  d.left_offset = lo.data();
  d.left_theta = lt.data();
  d.p1 = spec.p1.kind == Permutation::Kind::identity ? nullptr : spec.p1.map().data();
  d.p2 = spec.p2.kind == Permutation::Kind::identity ? nullptr : spec.p2.map().data();
  d.sigma = spec.spectrum.values().data();
  check(l1b_problem_create(0, &d, inst.tau, inst.b.data(), inst.x_star.support.data(),
                           inst.x_star.values.data(), inst.x_star.nnz(), &out->p));
}

}  // namespace

SolverTrace run_solver(const ProblemInstance& inst, const SolverConfig& cfg,
                       std::vector<double>* x_out) {
  cfg.validate(inst.cols());  // the reference's own validation first (solvers.cpp:133-143)
  l1b_solver_cfg c;
  l1b_solver_cfg_default(&c);
  if (cfg.id == "ista") c.solver = L1B_ISTA;
  else if (cfg.id == "fista") c.solver = L1B_FISTA;
  else if (cfg.id == "cd") c.solver = L1B_CD;
  else if (cfg.id == "newton_cg") c.solver = L1B_NEWTON_CG;
  else throw std::invalid_argument("run_solver: unknown solver id '" + cfg.id + "'");
  c.l_policy = cfg.l_policy == LPolicy::backtracking ? L1B_L_BACKTRACKING : L1B_L_SPECTRUM;
  c.max_iters = cfg.max_iters;
  c.max_seconds = cfg.max_seconds;
  c.has_target = cfg.target_objective.has_value();
  c.target = cfg.target_objective.value_or(0.0);
  c.mu = cfg.mu;
  c.eta = cfg.eta;
  c.pcg_max_iters = cfg.pcg_max_iters;
  c.ls_max_backtracks = cfg.ls_max_backtracks;
  c.grad_tol_rel = cfg.grad_tol_rel;
  c.l_fixed = cfg.l_fixed.value_or(0.0);
  c.varpi = cfg.varpi;
  c.omega = cfg.omega.value_or(0);
  c.seed = cfg.seed;
  Problem prob;
  upload(inst, &prob);
  const uint64_t cap = std::min<uint64_t>(cfg.max_iters + 4, 1u << 22);
  std::vector<l1b_sample> samples(cap);
  l1b_summary s{};
  std::vector<double> x(inst.cols());
  check(l1b_solve(prob.p, &c, samples.data(), cap, &s, x.data(), nullptr));
  SolverTrace tr;
  tr.solver = cfg.id;
  for (uint64_t i = 0; i < std::min<uint64_t>(s.n_samples, cap); ++i) {
    const auto& q = samples[i];
    tr.samples.push_back({q.iter, q.elapsed_s, q.objective, q.nnz, q.matvecs, q.extra});
  }
  tr.status = static_cast<StopReason>(s.status);
  tr.reached_target = s.reached_target != 0;
  tr.final_objective = s.final_objective;
  tr.elapsed_s = s.elapsed_s;
  tr.total_matvecs = s.total_matvecs;
  tr.total_pcg_iterations = s.total_pcg_iterations;
  tr.newton_steps = s.newton_steps;
  tr.time_to_target = s.time_to_target;
  tr.matvecs_to_target = s.matvecs_to_target;
  if (x_out) *x_out = std::move(x);
  return tr;
}

namespace {
SolverTrace with_id(const ProblemInstance& inst, SolverConfig cfg, const char* id,
                    std::vector<double>* x_out) {
  cfg.id = id;
  return b200::run_solver(inst, cfg, x_out);
}
}  // namespace

SolverTrace fista_run(const ProblemInstance& i, const SolverConfig& c, std::vector<double>* x) {
  return with_id(i, c, "fista", x);
}
SolverTrace ista_run(const ProblemInstance& i, const SolverConfig& c, std::vector<double>* x) {
  return with_id(i, c, "ista", x);
}
SolverTrace coordinate_descent_run(const ProblemInstance& i, const SolverConfig& c,
                                   std::vector<double>* x) {
  return with_id(i, c, "cd", x);
}
SolverTrace newton_cg_run(const ProblemInstance& i, const SolverConfig& c, std::vector<double>* x) {
  return with_id(i, c, "newton_cg", x);
}

}  // namespace l1bench::b200

// ---------------------------------------------------------------------------
// Self-test entry for tests/test_gpu_dropin.py: builds an instance with the
// reference's own build_instance, solves it with the reference and with the
// drop-in, and reports the largest relative iterate / objective difference.
extern "C" int b200_dropin_compare(const char* solver, uint64_t n, uint32_t stages, int q,
                                   uint64_t seed, uint64_t iters, double* out) {
  using namespace l1bench;
  try {
    ExperimentConfig cfg;
    cfg.n_list = {n};
    cfg.stage_counts = {stages};
    cfg.spectrum.q_list = {q};
    cfg.s_divisor = 100;
    cfg.seed = seed;
    SolverConfig sc;
    std::string id = solver;  // "<solver>_bt": the backtracking Lipschitz policy
    const bool bt = id.size() > 3 && id.compare(id.size() - 3, 3, "_bt") == 0;
    if (bt) id.resize(id.size() - 3);
    sc.id = id;
    if (bt) sc.l_policy = LPolicy::backtracking;
    sc.max_iters = iters;
    sc.varpi = 4;
    sc.seed = 5;
    cfg.solvers = {sc};
    cfg.reference = id;
    const ProblemInstance inst = build_instance(cfg, enumerate_jobs(cfg).at(0));
    std::vector<double> xr, xb;
    const SolverTrace tr = l1bench::run_solver(inst, sc, &xr);
    const SolverTrace tb = l1bench::b200::run_solver(inst, sc, &xb);
    double dx = 0.0, mx = 0.0, df = 0.0;
    for (size_t i = 0; i < xr.size(); ++i) {
      dx = std::max(dx, std::abs(xr[i] - xb[i]));
      mx = std::max(mx, std::abs(xr[i]));
    }
    const size_t k = std::min(tr.samples.size(), tb.samples.size());
    for (size_t i = 0; i < k; ++i)
      df = std::max(df, std::abs(tr.samples[i].objective - tb.samples[i].objective) /
                            std::max(1e-300, std::abs(tr.samples[i].objective)));
    out[0] = mx > 0 ? dx / mx : dx;
    out[1] = df;
    out[2] = (double)tr.samples.size();
    out[3] = (double)tb.samples.size();
    out[4] = (double)static_cast<int>(tr.status);
    out[5] = (double)static_cast<int>(tb.status);
    return 0;
  } catch (const std::exception& e) {
    return 1;
  }
}
