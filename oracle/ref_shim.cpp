// ref_shim.cpp -- extern "C" handle over the UNMODIFIED reference library
// (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libl1ref.so).  TEST/BASELINE INFRASTRUCTURE ONLY: used by
// tests/ to pin the oracle restatement, by tests/golden/make_golden.py to
// write the golden vectors, and by bench.py --impl reference / cpu_baseline.
// Every call goes through the reference's public API (include/l1bench/*.hpp).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "l1bench/bench.hpp"
#include "l1bench/serialize.hpp"
#include "l1bench/instance.hpp"
#include "l1bench/linops.hpp"
#include "l1bench/solvers.hpp"

using namespace l1bench;

namespace {
thread_local std::string g_err;

struct RefInst {
  ProblemInstance inst;
  ColumnWorkspace ws;
  SparseColumn col;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

typedef struct {
  uint64_t iter;
  double elapsed_s;
  double objective;
  uint64_t nnz;
  double matvecs;
  uint64_t extra;
} ref_sample;

typedef struct {
  int status;
  int reached_target;
  double final_objective;
  double elapsed_s;
  double total_matvecs;
  uint64_t total_pcg_iterations;
  uint64_t newton_steps;
  double time_to_target;
  double matvecs_to_target;
  uint64_t n_samples_total;
} ref_summary;

typedef struct {
  const char* id;
  uint64_t max_iters;
  double max_seconds;
  int has_target;
  double target;
  double mu, eta, grad_tol_rel;
  uint64_t pcg_max_iters, ls_max_backtracks;
  double l_fixed;  // <= 0: unset
  uint64_t varpi;
  uint64_t omega;  // 0: unset
  uint64_t seed;
  int backtracking;  // LPolicy::backtracking
} ref_cfg;

const char* ref_last_error() { return g_err.c_str(); }

// ExperimentConfig / enumerate_jobs / build_instance (bench.hpp:37-102).  With
// sigma_explicit != nullptr the same assembly is done through the operator
// API with Spectrum::from_values (SURVEY.md 8(d) C1 mapping).
void* ref_build_instance2(uint64_t n, double m_ratio, uint64_t stages, uint64_t left_stages,
                          int permute, int q, double shift, uint64_t s_divisor, double gamma,
                          double tau, double theta, uint64_t seed, const double* sigma_explicit,
                          int solution_kind, double s1_fraction, double value_a, double value_b);

void* ref_build_instance(uint64_t n, double m_ratio, uint64_t stages, uint64_t left_stages,
                         int permute, int q, double shift, uint64_t s_divisor, double gamma,
                         double tau, double theta, uint64_t seed, const double* sigma_explicit) {
  return ref_build_instance2(n, m_ratio, stages, left_stages, permute, q, shift, s_divisor, gamma,
                             tau, theta, seed, sigma_explicit, 0, 0.5, -1e4, 1e-1);
}

// SpectrumRule::Kind::alternating (bench.hpp:16-23, bench.cpp:278) for the next
// ref_build_instance2 call: the odd / even values (on = 0: uniform_q again)
static thread_local int g_alt_on = 0;
static thread_local double g_alt_odd = 0.1, g_alt_even = 100.0;
void ref_next_spectrum_alternating(int on, double odd_value, double even_value) {
  g_alt_on = on;
  g_alt_odd = odd_value;
  g_alt_even = even_value;
}

// + SolutionRule (bench.hpp:25-32): kind 0 uniform, 1 spectral, 2 two_value
void* ref_build_instance2(uint64_t n, double m_ratio, uint64_t stages, uint64_t left_stages,
                          int permute, int q, double shift, uint64_t s_divisor, double gamma,
                          double tau, double theta, uint64_t seed, const double* sigma_explicit,
                          int solution_kind, double s1_fraction, double value_a, double value_b) {
  RefInst* out = nullptr;
  int rc = guarded([&] {
    ExperimentConfig cfg;
    cfg.solution.kind = solution_kind == 1   ? SolutionRule::Kind::spectral
                        : solution_kind == 2 ? SolutionRule::Kind::two_value
                                             : SolutionRule::Kind::uniform;
    cfg.solution.s1_fraction = s1_fraction;
    cfg.solution.value_a = value_a;
    cfg.solution.value_b = value_b;
    cfg.name = "ref";
    cfg.n_list = {static_cast<std::size_t>(n)};
    cfg.m_ratio = m_ratio;
    cfg.spectrum.q_list = {q};
    cfg.spectrum.shift = shift;
    if (g_alt_on) {
      cfg.spectrum.kind = SpectrumRule::Kind::alternating;
      cfg.spectrum.odd_value = g_alt_odd;
      cfg.spectrum.even_value = g_alt_even;
      g_alt_on = 0;
    }
    cfg.theta_list = {theta};
    cfg.stage_counts = {static_cast<std::size_t>(stages)};
    cfg.left_stage_count = static_cast<std::size_t>(left_stages);
    cfg.permute = permute != 0;
    cfg.solution.gamma = gamma;
    cfg.s_divisor = static_cast<std::size_t>(s_divisor);
    cfg.tau_list = {tau};
    SolverConfig sc;
    sc.id = "fista";
    cfg.solvers = {sc};
    cfg.reference = "fista";
    cfg.seed = seed;
    const auto jobs = enumerate_jobs(cfg);
    auto* ri = new RefInst();
    if (!sigma_explicit) {
      ri->inst = build_instance(cfg, jobs.at(0));
    } else {
      const InstanceJob& job = jobs.at(0);
      const std::size_t m = static_cast<std::size_t>(std::llround(m_ratio * static_cast<double>(n)));
      auto spec = std::make_shared<OperatorSpec>();
      spec->m = m;
      spec->n = n;
      for (std::size_t i = 0; i < stages; ++i) {
        spec->right_stages.push_back(
            RotationStage::paired(n, static_cast<int>((stages - 1 - i) % 2), theta));
      }
      for (std::size_t i = 0; i < left_stages; ++i) {
        spec->left_stages.push_back(
            RotationStage::paired(m, static_cast<int>((left_stages - 1 - i) % 2), theta));
      }
      if (permute) {
        spec->p1 = Permutation::random(m, mix_seed(job.seed, 1));
        spec->p2 = Permutation::random(m, mix_seed(job.seed, 2));
      }
      spec->spectrum = Spectrum::from_values(std::vector<double>(sigma_explicit, sigma_explicit + n));
      spec->finalize();
      const std::size_t s = std::max<std::size_t>(1, n / s_divisor);
      Rng rng = make_rng(mix_seed(job.seed, 4));
      SparseSolution x = uniform_sparse_solution(n, s, gamma, rng);
      Rng gen = make_rng(mix_seed(job.seed, 5));
      ri->inst = generate_instance(tau, spec, std::move(x), FillPolicy::interior(), gen);
    }
    out = ri;
  });
  return rc == 0 ? out : nullptr;
}

void ref_free(void* h) { delete static_cast<RefInst*>(h); }

// serialize.cpp's own save_instance / load_instance (instance files)
int ref_save_instance(void* h, const char* path) {
  return guarded([&] { save_instance(static_cast<RefInst*>(h)->inst, path); });
}
void* ref_load_instance(const char* path) {
  RefInst* out = nullptr;
  const int rc = guarded([&] {
    auto* ri = new RefInst();
    ri->inst = load_instance(path);
    out = ri;
  });
  return rc == 0 ? out : nullptr;
}

void ref_dims(void* h, uint64_t* m, uint64_t* n) {
  auto* ri = static_cast<RefInst*>(h);
  *m = ri->inst.rows();
  *n = ri->inst.cols();
}

double ref_tau(void* h) { return static_cast<RefInst*>(h)->inst.tau; }
double ref_noise_norm(void* h) { return static_cast<RefInst*>(h)->inst.noise_norm; }
double ref_cert_kappa(void* h) { return static_cast<RefInst*>(h)->inst.cert_kappa; }
double ref_f_star(void* h) { return static_cast<RefInst*>(h)->inst.objective_at_planted(); }
double ref_gram_lmax(void* h) { return *static_cast<RefInst*>(h)->inst.factored->gram_lmax(); }

void ref_get_b(void* h, double* b) {
  const auto& v = static_cast<RefInst*>(h)->inst.b;
  std::memcpy(b, v.data(), v.size() * sizeof(double));
}

void ref_get_sigma(void* h, double* s) {
  const auto& v = static_cast<RefInst*>(h)->inst.factored->spectrum.values();
  std::memcpy(s, v.data(), v.size() * sizeof(double));
}

uint64_t ref_xstar_nnz(void* h) { return static_cast<RefInst*>(h)->inst.x_star.nnz(); }

void ref_get_xstar(void* h, uint32_t* support, double* values) {
  const auto& x = static_cast<RefInst*>(h)->inst.x_star;
  std::memcpy(support, x.support.data(), x.support.size() * sizeof(uint32_t));
  std::memcpy(values, x.values.data(), x.values.size() * sizeof(double));
}

// Returns 1 and fills map when the permutation is non-identity.
int ref_get_perm(void* h, int which, uint32_t* map) {
  const auto& spec = *static_cast<RefInst*>(h)->inst.factored;
  const Permutation& p = which == 1 ? spec.p1 : spec.p2;
  if (p.kind == Permutation::Kind::identity) return 0;
  std::memcpy(map, p.map().data(), p.map().size() * sizeof(uint32_t));
  return 1;
}

uint32_t ref_n_stages(void* h, int right) {
  const auto& spec = *static_cast<RefInst*>(h)->inst.factored;
  return static_cast<uint32_t>(right ? spec.right_stages.size() : spec.left_stages.size());
}

void ref_stage(void* h, int right, uint32_t k, int32_t* offset, double* theta) {
  const auto& spec = *static_cast<RefInst*>(h)->inst.factored;
  const RotationStage& st = right ? spec.right_stages.at(k) : spec.left_stages.at(k);
  *offset = st.offset;
  *theta = st.theta;
}

uint64_t ref_row(void* h, uint64_t i, uint32_t* idx, double* val) {
  auto* ri = static_cast<RefInst*>(h);
  ri->inst.op().row(i, ri->ws, ri->col);
  std::memcpy(idx, ri->col.idx.data(), ri->col.nnz() * sizeof(uint32_t));
  std::memcpy(val, ri->col.val.data(), ri->col.nnz() * sizeof(double));
  return ri->col.nnz();
}

uint64_t ref_column(void* h, uint64_t j, uint32_t* idx, double* val) {
  auto* ri = static_cast<RefInst*>(h);
  ri->inst.op().column(j, ri->ws, ri->col);
  std::memcpy(idx, ri->col.idx.data(), ri->col.nnz() * sizeof(uint32_t));
  std::memcpy(val, ri->col.val.data(), ri->col.nnz() * sizeof(double));
  return ri->col.nnz();
}

void ref_apply(void* h, const double* x, double* y) {
  const auto& op = static_cast<RefInst*>(h)->inst.op();
  op.apply(std::span<const double>(x, op.cols()), std::span<double>(y, op.rows()));
}

void ref_apply_transpose(void* h, const double* y, double* x) {
  const auto& op = static_cast<RefInst*>(h)->inst.op();
  op.apply_transpose(std::span<const double>(y, op.rows()), std::span<double>(x, op.cols()));
}

void ref_gram_diagonal(void* h, double* d) {
  const auto v = static_cast<RefInst*>(h)->inst.op().gram_diagonal();
  std::memcpy(d, v.data(), v.size() * sizeof(double));
}

void ref_gram_inverse(void* h, const double* v, double* out) {
  const auto& spec = *static_cast<RefInst*>(h)->inst.factored;
  spec.apply_gram_inverse(std::span<const double>(v, spec.n), std::span<double>(out, spec.n));
}

double ref_objective(void* h, const double* x) {
  const auto& inst = static_cast<RefInst*>(h)->inst;
  return objective(inst, std::span<const double>(x, inst.cols()));
}

int ref_verify(void* h, double tol, double* out3) {
  const auto rep = verify_optimality(static_cast<RefInst*>(h)->inst, tol);
  out3[0] = rep.max_support_violation;
  out3[1] = rep.max_offsupport_violation;
  out3[2] = rep.threshold;
  return rep.pass ? 1 : 0;
}

void ref_smoothed_hessvec(void* h, const double* x, double mu, const double* v, double* out) {
  const auto& inst = static_cast<RefInst*>(h)->inst;
  const std::size_t n = inst.cols();
  const auto r = smoothed_hessvec(inst, std::span<const double>(x, n), mu, std::span<const double>(v, n));
  std::memcpy(out, r.data(), n * sizeof(double));
}

void ref_smoothed_gradient(void* h, const double* x, double mu, double* out) {
  const auto& inst = static_cast<RefInst*>(h)->inst;
  const std::size_t n = inst.cols();
  const auto r = smoothed_gradient(inst, std::span<const double>(x, n), mu);
  std::memcpy(out, r.data(), n * sizeof(double));
}

double ref_smoothed_objective(void* h, const double* x, double mu) {
  const auto& inst = static_cast<RefInst*>(h)->inst;
  return smoothed_objective(inst, std::span<const double>(x, inst.cols()), mu);
}

// pcg_solve (solvers.hpp:82-84) with the smoothed Hessian at x.
int ref_pcg(void* h, const double* x, double mu, const double* rhs, const double* precond,
            double eta, uint64_t max_iters, double* step, uint64_t* iters, int* converged) {
  return guarded([&] {
    const auto& inst = static_cast<RefInst*>(h)->inst;
    const std::size_t n = inst.cols();
    std::vector<double> xv(x, x + n);
    auto hv = [&](std::span<const double> v, std::span<double> out) {
      const auto r = smoothed_hessvec(inst, xv, mu, v);
      std::copy(r.begin(), r.end(), out.begin());
    };
    PcgResult res = pcg_solve(hv, std::span<const double>(rhs, n), std::span<const double>(precond, n),
                              eta, max_iters);
    std::memcpy(step, res.step.data(), n * sizeof(double));
    *iters = res.iterations;
    *converged = res.converged ? 1 : 0;
  });
}

int ref_solve(void* h, const ref_cfg* c, ref_sample* samples, uint64_t cap, uint64_t* n_samples,
              ref_summary* summary, double* x_out) {
  return guarded([&] {
    const auto& inst = static_cast<RefInst*>(h)->inst;
    SolverConfig cfg;
    cfg.id = c->id;
    cfg.max_iters = c->max_iters;
    cfg.max_seconds = c->max_seconds;
    if (c->has_target) cfg.target_objective = c->target;
    cfg.mu = c->mu;
    cfg.eta = c->eta;
    cfg.grad_tol_rel = c->grad_tol_rel;
    cfg.pcg_max_iters = c->pcg_max_iters;
    cfg.ls_max_backtracks = c->ls_max_backtracks;
    if (c->l_fixed > 0.0) cfg.l_fixed = c->l_fixed;
    cfg.varpi = c->varpi;
    if (c->omega) cfg.omega = c->omega;
    cfg.seed = c->seed;
    if (c->backtracking) cfg.l_policy = LPolicy::backtracking;
    std::vector<double> x;
    SolverTrace tr = run_solver(inst, cfg, &x);
    const std::size_t k = std::min<std::size_t>(cap, tr.samples.size());
    for (std::size_t i = 0; i < k; ++i) {
      const auto& s = tr.samples[i];
      samples[i] = {s.iter, s.elapsed_s, s.objective, s.nnz, s.matvecs, s.extra};
    }
    *n_samples = k;
    summary->status = static_cast<int>(tr.status);
    summary->reached_target = tr.reached_target ? 1 : 0;
    summary->final_objective = tr.final_objective;
    summary->elapsed_s = tr.elapsed_s;
    summary->total_matvecs = tr.total_matvecs;
    summary->total_pcg_iterations = tr.total_pcg_iterations;
    summary->newton_steps = tr.newton_steps;
    summary->time_to_target = tr.time_to_target;
    summary->matvecs_to_target = tr.matvecs_to_target;
    summary->n_samples_total = tr.samples.size();
    if (x_out) std::memcpy(x_out, x.data(), x.size() * sizeof(double));
  });
}

}  // extern "C"
