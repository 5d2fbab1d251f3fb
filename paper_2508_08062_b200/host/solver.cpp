// solver.cpp — the drop-in C++ solver API over the sm_100a C-ABI.
//
// solve()/select_step_sizes()/kkt_metrics()/pdhg_step()/matvec*() keep the
// reference signatures (proj/include/aapdhg/solver.hpp:81-99,
// pdhg_core.hpp:33, sparse_linalg.hpp:34-47) and throw the reference's
// exception types; all arithmetic runs in libaapdhg_cuda.so.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <thread>
#include <cstring>
#include <string>
#include <vector>

#include "aapdhg/aapdhg.hpp"
#include "aapdhg_cuda.h"

namespace aapdhg {
namespace {

[[noreturn]] void raise(int rc, const char* msg) {
  const std::string m = msg && *msg ? msg : ("aapdhg_cuda error " + std::to_string(rc));
  switch (rc) {
    case AAPDHG_ERR_INPUT: throw InputError(m);
    case AAPDHG_ERR_DIMENSION: throw DimensionError(m);
    case AAPDHG_ERR_UNSUPPORTED: throw UnsupportedError(m);
    case AAPDHG_ERR_SINGULAR: throw SingularError(m);
    default: throw Error(m);
  }
}

void check(int rc, const char* err) {
  if (rc != AAPDHG_OK) raise(rc, err);
}

aapdhg_problem_view view_of(const ProblemData& p) {
  if (int(p.l.size()) != p.n() || int(p.u.size()) != p.n() || p.k.ncols != p.n() ||
      int(p.q.size()) != p.k.nrows || p.m1() + p.m2() != p.k.nrows)
    throw DimensionError("ProblemData: inconsistent sizes");
  aapdhg_problem_view v{};
  v.k.nrows = p.k.nrows;
  v.k.ncols = p.k.ncols;
  v.k.nnz = int64_t(p.k.vals.size());
  v.k.row_ptr = p.k.row_ptr.data();
  v.k.col_idx = p.k.col_idx.data();
  v.k.vals = p.k.vals.data();
  v.m1 = p.m1();
  v.c = p.c.data();
  v.q = p.q.data();
  v.l = p.l.data();
  v.u = p.u.data();
  return v;
}

aapdhg_solve_params params_of(const SolverConfig& cfg) {
  aapdhg_solve_params prm{};
  prm.method = cfg.method == Method::kAaPdhg    ? AAPDHG_METHOD_AA
               : cfg.method == Method::kFaaPdhg ? AAPDHG_METHOD_FAA
                                                : AAPDHG_METHOD_PDHG;
  prm.reduction = cfg.reduction == Reduction::kSerial ? AAPDHG_REDUCE_SERIAL
                  : cfg.reduction == Reduction::kTree ? AAPDHG_REDUCE_TREE
                                                      : AAPDHG_REDUCE_AUTO;
  prm.m = cfg.m;
  prm.safeguard_d = cfg.safeguard_d;
  prm.safeguard_eps = cfg.safeguard_eps;
  prm.beta = cfg.aa.beta;
  prm.d_hat = cfg.aa.d_hat.empty() ? nullptr : cfg.aa.d_hat.data();
  prm.eta = cfg.aa.eta;
  prm.c_s = cfg.filter.c_s;
  prm.kappa_bar = cfg.filter.kappa_bar;
  prm.toll = cfg.toll;
  prm.kkt_eps = cfg.kkt_eps;
  prm.kkt_terminate = cfg.kkt_terminate ? 1 : 0;
  prm.max_iters = cfg.max_iters;
  prm.max_wall_seconds = cfg.max_wall_seconds;
  prm.tau = cfg.tau;
  prm.sigma = cfg.sigma;
  return prm;
}

void record_sink(const aapdhg_record* recs, uint64_t count, void* ctx) {
  auto* out = static_cast<std::vector<TrajectoryRecord>*>(ctx);
  for (uint64_t t = 0; t < count; ++t) {
    TrajectoryRecord r;
    r.k = recs[t].k;
    r.g_norm = recs[t].g_norm;
    r.aa_step = recs[t].aa_step != 0;
    r.i = recs[t].i;
    r.j = recs[t].j;
    r.kkt.r_gap = recs[t].r_gap;
    r.kkt.r_primal = recs[t].r_primal;
    r.kkt.r_dual = recs[t].r_dual;
    r.objective = recs[t].objective;
    r.elapsed_s = recs[t].elapsed_s;
    out->push_back(r);
  }
}

// Owns a device handle for the duration of one call.
struct Handle {
  aapdhg_handle* h = nullptr;
  Handle(const ProblemData& p, int device) {
    char err[512] = {0};
    const aapdhg_problem_view v = view_of(p);
    check(aapdhg_cuda_problem_create(&v, device, &h, err, sizeof err), err);
  }
  ~Handle() { aapdhg_cuda_problem_destroy(h); }
};

ProblemData matrix_only(const SparseMatrix& m) {
  ProblemData p;
  p.k = m;
  p.a.nrows = m.nrows;  // all rows "equality": m1 = 0
  p.c.assign(std::size_t(m.ncols), 0.0);
  p.l.assign(std::size_t(m.ncols), 0.0);
  p.u.assign(std::size_t(m.ncols), kInf);
  p.q.assign(std::size_t(m.nrows), 0.0);
  p.b = p.q;
  return p;
}

SolveOutput run_solve(aapdhg_handle* h, const ProblemData& p, const SolverConfig& cfg,
                      const Iterate* u0) {
  const std::size_t n = std::size_t(p.n()), m = p.q.size();
  if (u0 && (u0->x.size() != n || u0->y.size() != m))
    throw DimensionError("solve: start iterate dims mismatch");
  if (!cfg.aa.d_hat.empty() && cfg.aa.d_hat.size() != n + m)
    throw DimensionError("aa: d_hat size mismatch");
  const aapdhg_solve_params prm = params_of(cfg);
  SolveOutput out;
  SolveResult& r = out.result;
  r.u.x.assign(n, 0.0);
  r.u.y.assign(m, 0.0);
  r.lambda.assign(n, 0.0);
  aapdhg_solve_result res{};
  char err[512] = {0};
  check(aapdhg_cuda_solve(h, &prm, u0 ? u0->x.data() : nullptr, u0 ? u0->y.data() : nullptr,
                          &res, r.u.x.data(), r.u.y.data(), r.lambda.data(), record_sink,
                          &out.trajectory, err, sizeof err),
        err);
  r.status = SolveStatus(res.status);
  r.iterations = res.iterations;
  r.i = res.i;
  r.j = res.j;
  r.aa_failures = res.aa_failures;
  r.g_norm = res.g_norm;
  r.kkt.r_gap = res.r_gap;
  r.kkt.r_primal = res.r_primal;
  r.kkt.r_dual = res.r_dual;
  r.objective = res.objective;
  r.steps.tau = res.tau;
  r.steps.sigma = res.sigma;
  r.wall_seconds = res.wall_seconds;
  return out;
}

}  // namespace

// ---- vec.hpp helpers (host; the reference's serial order) ------------------
double dot(const Vec& a, const Vec& b) {
  if (a.size() != b.size()) throw DimensionError("dot: size mismatch");
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double nrm2sq(const Vec& a) {
  double s = 0.0;
  for (double v : a) s += v * v;
  return s;
}
void axpy(double alpha, const Vec& x, Vec& y) {
  if (x.size() != y.size()) throw DimensionError("axpy: size mismatch");
  for (std::size_t i = 0; i < x.size(); ++i) y[i] += alpha * x[i];
}
Vec sub(const Vec& a, const Vec& b) {
  if (a.size() != b.size()) throw DimensionError("sub: size mismatch");
  Vec o(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) o[i] = a[i] - b[i];
  return o;
}
Vec add(const Vec& a, const Vec& b) {
  if (a.size() != b.size()) throw DimensionError("add: size mismatch");
  Vec o(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) o[i] = a[i] + b[i];
  return o;
}
Vec scaled(const Vec& a, double alpha) {
  Vec o(a.size());
  for (std::size_t i = 0; i < a.size(); ++i) o[i] = alpha * a[i];
  return o;
}

// ---- device products ---------------------------------------------------------
void matvec(const SparseMatrix& m, const Vec& v, Vec& out) {
  if (int(v.size()) != m.ncols) throw DimensionError("matvec: dim mismatch");
  const ProblemData p = matrix_only(m);
  Handle h(p, 0);
  out.assign(std::size_t(m.nrows), 0.0);
  char err[512] = {0};
  check(aapdhg_cuda_matvec(h.h, v.data(), out.data(), err, sizeof err), err);
}
Vec matvec(const SparseMatrix& m, const Vec& v) {
  Vec o;
  matvec(m, v, o);
  return o;
}
void matvec_transpose(const SparseMatrix& m, const Vec& v, Vec& out) {
  if (int(v.size()) != m.nrows) throw DimensionError("matvec_transpose: dim mismatch");
  const ProblemData p = matrix_only(m);
  Handle h(p, 0);
  out.assign(std::size_t(m.ncols), 0.0);
  char err[512] = {0};
  check(aapdhg_cuda_matvec_transpose(h.h, v.data(), out.data(), err, sizeof err), err);
}
Vec matvec_transpose(const SparseMatrix& m, const Vec& v) {
  Vec o;
  matvec_transpose(m, v, o);
  return o;
}
double power_iteration_norm(const SparseMatrix& m, int max_iters, double rel_tol,
                            std::uint64_t seed) {
  const ProblemData p = matrix_only(m);
  Handle h(p, 0);
  double out = 0.0;
  int32_t rounds = 0;
  char err[512] = {0};
  check(aapdhg_cuda_power_norm(h.h, max_iters, rel_tol, seed, AAPDHG_REDUCE_AUTO, &out,
                               &rounds, err, sizeof err),
        err);
  return out;
}

// ---- pdhg_core ---------------------------------------------------------------
Iterate pdhg_step(const Iterate& u, const ProblemData& p, const StepSizes& s) {
  if (int(u.x.size()) != p.n() || u.y.size() != p.q.size())
    throw DimensionError("pdhg_step: iterate dims mismatch");
  Handle h(p, 0);
  Iterate out{Vec(u.x.size()), Vec(u.y.size())};
  char err[512] = {0};
  check(aapdhg_cuda_pdhg_step(h.h, s.tau, s.sigma, u.x.data(), u.y.data(), out.x.data(),
                              out.y.data(), err, sizeof err),
        err);
  return out;
}

std::pair<Vec, double> fixed_point_residual(const Iterate& u, const Iterate& tu) {
  if (u.x.size() != tu.x.size() || u.y.size() != tu.y.size())
    throw DimensionError("fixed_point_residual: dims mismatch");
  Vec g = sub(concat_iterate(tu), concat_iterate(u));
  const double nrm = nrm2(g);
  return {std::move(g), nrm};
}

Vec concat_iterate(const Iterate& u) {
  Vec out = u.x;
  out.insert(out.end(), u.y.begin(), u.y.end());
  return out;
}

Iterate split_iterate(const Vec& v, int n) {
  if (int(v.size()) < n) throw DimensionError("split_iterate: vector too short");
  return {Vec(v.begin(), v.begin() + n), Vec(v.begin() + n, v.end())};
}

// ---- solver ------------------------------------------------------------------
double KktMetrics::max() const {
  return std::fmax(std::fmax(r_gap, r_primal), r_dual);
}

bool safeguard_pass(double g_norm, double g0_norm, std::size_t i, double d, double eps) {
  return g_norm <= d * g0_norm * std::pow(double(i) + 1.0, -(1.0 + eps));
}

std::pair<KktMetrics, Vec> kkt_metrics(const Iterate& u, const ProblemData& p,
                                       const LambdaSpec& spec) {
  if (spec.size() != std::size_t(p.n())) throw DimensionError("project_lambda: size mismatch");
  if (int(u.x.size()) != p.n() || u.y.size() != p.q.size())
    throw DimensionError("kkt_metrics: iterate dims mismatch");
  // the device derives Lambda from (l, u) exactly as build_lambda_set does
  Handle h(p, 0);
  double kkt[4];
  Vec lam(std::size_t(p.n()));
  char err[512] = {0};
  check(aapdhg_cuda_kkt_metrics(h.h, AAPDHG_REDUCE_AUTO, u.x.data(), u.y.data(), kkt,
                                lam.data(), err, sizeof err),
        err);
  KktMetrics m;
  m.r_gap = kkt[0];
  m.r_primal = kkt[1];
  m.r_dual = kkt[2];
  return {m, std::move(lam)};
}

StepSizes select_step_sizes(const ProblemData& p, const SolverConfig& cfg) {
  Handle h(p, cfg.device);
  const aapdhg_solve_params prm = params_of(cfg);
  StepSizes s;
  char err[512] = {0};
  check(aapdhg_cuda_select_step_sizes(h.h, &prm, &s.tau, &s.sigma, err, sizeof err), err);
  return s;
}

SolveOutput solve(const ProblemData& p, const SolverConfig& cfg, const Iterate& u0) {
  Handle h(p, cfg.device);
  return run_solve(h.h, p, cfg, &u0);
}

SolveOutput solve(const ProblemData& p, const SolverConfig& cfg) {
  Handle h(p, cfg.device);
  return run_solve(h.h, p, cfg, nullptr);
}

DeviceProblem::DeviceProblem(const ProblemData& p, int device) : p_(&p) {
  char err[512] = {0};
  const aapdhg_problem_view v = view_of(p);
  aapdhg_handle* h = nullptr;
  check(aapdhg_cuda_problem_create(&v, device, &h, err, sizeof err), err);
  h_ = h;
}

DeviceProblem::~DeviceProblem() { aapdhg_cuda_problem_destroy(static_cast<aapdhg_handle*>(h_)); }

SolveOutput DeviceProblem::solve(const SolverConfig& cfg, const Iterate& u0) const {
  return run_solve(static_cast<aapdhg_handle*>(h_), *p_, cfg, &u0);
}

SolveOutput DeviceProblem::solve(const SolverConfig& cfg) const {
  return run_solve(static_cast<aapdhg_handle*>(h_), *p_, cfg, nullptr);
}

double m_inner_product(const Vec& u, const Vec& v, const ProblemData& p, const StepSizes& s) {
  if (s.tau != s.sigma) throw UnsupportedError("m_inner_product requires tau == sigma");
  const std::size_t n = std::size_t(p.n()), m = std::size_t(p.m1() + p.m2());
  if (u.size() != n + m || v.size() != n + m)
    throw DimensionError("m_inner_product: size mismatch");
  const Vec ux(u.begin(), u.begin() + long(n)), uy(u.begin() + long(n), u.end());
  const Vec vx(v.begin(), v.begin() + long(n)), vy(v.begin() + long(n), v.end());
  double out = dot(ux, vx) + dot(uy, vy);
  out += s.tau * dot(matvec_transpose(p.k, uy), vx);
  out += s.tau * dot(matvec(p.k, ux), vy);
  return out;
}

// ---- host projections (pdhg_core.cpp:10-43 semantics: std::min/std::max, same
// error types and messages) -----------------------------------------------------
Vec project_box(const Vec& x, const Vec& l, const Vec& u) {
  if (x.size() != l.size() || x.size() != u.size())
    throw DimensionError("project_box: size mismatch");
  Vec out(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) out[i] = std::min(std::max(x[i], l[i]), u[i]);
  return out;
}

Vec project_dual(const Vec& y, int m1) {
  if (m1 < 0 || std::size_t(m1) > y.size()) throw DimensionError("project_dual: bad m1");
  Vec out = y;
  for (std::size_t i = 0; i < std::size_t(m1); ++i) out[i] = std::max(out[i], 0.0);
  return out;
}

Vec project_lambda(const Vec& v, const LambdaSpec& spec) {
  if (v.size() != spec.size()) throw DimensionError("project_lambda: size mismatch");
  Vec out(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) {
    const LambdaTag t = spec[i];
    out[i] = t == LambdaTag::kZero     ? 0.0
             : t == LambdaTag::kNonpos ? std::min(v[i], 0.0)
             : t == LambdaTag::kNonneg ? std::max(v[i], 0.0)
                                       : v[i];
  }
  return out;
}

Iterate project_feasible(const Iterate& u, const ProblemData& p) {
  return {project_box(u.x, p.l, p.u), project_dual(u.y, p.m1())};
}

DenseMatrix DenseMatrix::identity(int n) {
  DenseMatrix m(n, n);
  for (int i = 0; i < n; ++i) m.at(i, i) = 1.0;
  return m;
}

// ---- sweep mode (proj/src/cli.cpp:142-214) ----------------------------------
namespace {
std::string short_num(double v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%g", v);
  return buf;
}
}  // namespace

std::vector<SweepCase> sweep_cases(const SolverConfig& base, const std::vector<double>& d,
                                   const std::vector<double>& eps,
                                   const std::vector<std::size_t>& m,
                                   const std::vector<double>& kappa_bar) {
  std::vector<SweepCase> cases;
  for (std::size_t id = 0; id < std::max<std::size_t>(1, d.size()); ++id)
    for (std::size_t ie = 0; ie < std::max<std::size_t>(1, eps.size()); ++ie)
      for (std::size_t im = 0; im < std::max<std::size_t>(1, m.size()); ++im)
        for (std::size_t ik = 0; ik < std::max<std::size_t>(1, kappa_bar.size()); ++ik) {
          SweepCase sc{base, ""};
          std::string name;
          if (!d.empty()) {
            sc.cfg.safeguard_d = d[id];
            name += "D" + short_num(d[id]);
          }
          if (!eps.empty()) {
            sc.cfg.safeguard_eps = eps[ie];
            name += std::string(name.empty() ? "" : "_") + "eps" + short_num(eps[ie]);
          }
          if (!m.empty()) {
            sc.cfg.m = m[im];
            name += std::string(name.empty() ? "" : "_") + "m" + std::to_string(m[im]);
          }
          if (!kappa_bar.empty()) {
            sc.cfg.filter.kappa_bar = kappa_bar[ik];
            name += std::string(name.empty() ? "" : "_") + "kappa" + short_num(kappa_bar[ik]);
          }
          sc.name = name;
          cases.push_back(std::move(sc));
        }
  return cases;
}

std::vector<SweepOutcome> solve_sweep(const ProblemData& p, const std::vector<SweepCase>& cases,
                                      std::size_t workers, const std::vector<int>& devices) {
  if (devices.empty()) throw InputError("solve_sweep: no devices");
  if (workers == 0) {
    workers = 1;
    if (const char* env = std::getenv("AAPDHG_SWEEP_WORKERS")) {
      const long parsed = std::strtol(env, nullptr, 10);
      if (parsed > 0) workers = std::size_t(parsed);
    }
  }
  workers = std::max<std::size_t>(1, std::min(workers, cases.size()));
  std::vector<SweepOutcome> out(cases.size());
  std::atomic<std::size_t> next{0};
  auto work = [&](std::size_t w) {
    std::unique_ptr<DeviceProblem> dp;
    std::string setup_error;
    try {
      dp.reset(new DeviceProblem(p, devices[w % devices.size()]));
    } catch (const std::exception& e) {
      setup_error = e.what();
    }
    for (std::size_t idx = next.fetch_add(1); idx < cases.size(); idx = next.fetch_add(1)) {
      if (!dp) {
        out[idx].error = setup_error;
        continue;
      }
      try {
        out[idx].output = dp->solve(cases[idx].cfg);
        out[idx].ok = true;
      } catch (const std::exception& e) {
        out[idx].error = e.what();
      }
    }
  };
  if (workers == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (std::size_t w = 0; w < workers; ++w) pool.emplace_back(work, w);
    for (std::thread& t : pool) t.join();
  }
  return out;
}

}  // namespace aapdhg
