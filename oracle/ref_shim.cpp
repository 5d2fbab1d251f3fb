// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle side, never product).
//
// A C-ABI shim over the UNMODIFIED reference sources compiled from
// /root/reference/proj/src (see oracle/Makefile). It lets the Python tests,
// the golden-fixture script and bench.py's reference arm call the
// reference's own solve(), pdhg_step(), kkt_metrics(), aa_apply(),
// build_filtered_memory()/filtered_aa_apply(), power_iteration_norm() and the
// test-support instance generators with the same POD structs as the CUDA
// C-ABI (include/aapdhg_cuda.h). Nothing here re-implements the algorithm.
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <vector>

#include "aapdhg/anderson.hpp"
#include "aapdhg/errors.hpp"
#include "aapdhg/filtering.hpp"
#include "aapdhg/lp_model.hpp"
#include "aapdhg/pdhg_core.hpp"
#include "aapdhg/solver.hpp"
#include "aapdhg/sparse_linalg.hpp"
#include "aapdhg_cuda.h"
#include "support/test_support.hpp"

namespace R = aapdhg;

namespace {

void put_err(char* err, size_t errlen, const std::string& msg) {
  if (!err || errlen == 0) return;
  std::strncpy(err, msg.c_str(), errlen - 1);
  err[errlen - 1] = '\0';
}

template <class F>
int guard(char* err, size_t errlen, F&& f) {
  try {
    f();
    return AAPDHG_OK;
  } catch (const R::SingularError& e) {
    put_err(err, errlen, e.what());
    return AAPDHG_ERR_SINGULAR;
  } catch (const R::InputError& e) {
    put_err(err, errlen, e.what());
    return AAPDHG_ERR_INPUT;
  } catch (const R::DimensionError& e) {
    put_err(err, errlen, e.what());
    return AAPDHG_ERR_DIMENSION;
  } catch (const R::UnsupportedError& e) {
    put_err(err, errlen, e.what());
    return AAPDHG_ERR_UNSUPPORTED;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return AAPDHG_ERR_INTERNAL;
  }
}

R::SparseMatrix rows_of(const aapdhg_csr_view& k, int r0, int r1) {
  R::SparseMatrix s;
  s.nrows = r1 - r0;
  s.ncols = k.ncols;
  const int base = k.row_ptr[r0];
  s.row_ptr.resize(std::size_t(s.nrows) + 1);
  for (int r = r0; r <= r1; ++r) s.row_ptr[std::size_t(r - r0)] = k.row_ptr[r] - base;
  s.col_idx.assign(k.col_idx + base, k.col_idx + k.row_ptr[r1]);
  s.vals.assign(k.vals + base, k.vals + k.row_ptr[r1]);
  return s;
}

R::ProblemData problem_of(const aapdhg_problem_view* v) {
  const int n = v->k.ncols, m = v->k.nrows, m1 = v->m1;
  R::ProblemData p;
  p.g = rows_of(v->k, 0, m1);
  p.a = rows_of(v->k, m1, m);
  p.k = R::vstack(p.g, p.a);
  p.c.assign(v->c, v->c + n);
  p.l.assign(v->l, v->l + n);
  p.u.assign(v->u, v->u + n);
  p.q.assign(v->q, v->q + m);
  p.h.assign(v->q, v->q + m1);
  p.b.assign(v->q + m1, v->q + m);
  p.name = "shim";
  return p;
}

R::SolverConfig config_of(const aapdhg_solve_params* prm, std::size_t N) {
  R::SolverConfig cfg;
  cfg.method = prm->method == AAPDHG_METHOD_AA    ? R::Method::kAaPdhg
               : prm->method == AAPDHG_METHOD_FAA ? R::Method::kFaaPdhg
                                                  : R::Method::kPdhg;
  cfg.m = prm->m;
  cfg.safeguard_d = prm->safeguard_d;
  cfg.safeguard_eps = prm->safeguard_eps;
  cfg.aa.beta = prm->beta;
  if (prm->d_hat) cfg.aa.d_hat.assign(prm->d_hat, prm->d_hat + N);
  cfg.aa.eta = prm->eta;
  cfg.filter.c_s = prm->c_s;
  cfg.filter.kappa_bar = prm->kappa_bar;
  cfg.toll = prm->toll;
  cfg.kkt_eps = prm->kkt_eps;
  cfg.kkt_terminate = prm->kkt_terminate != 0;
  cfg.max_iters = prm->max_iters;
  cfg.max_wall_seconds = prm->max_wall_seconds;
  cfg.tau = prm->tau;
  cfg.sigma = prm->sigma;
  return cfg;
}

std::vector<R::Vec> columns(const double* cols, int p, std::size_t N) {
  std::vector<R::Vec> out;
  for (int j = 0; j < p; ++j) out.emplace_back(cols + std::size_t(j) * N, cols + std::size_t(j + 1) * N);
  return out;
}

struct GenProblem {
  R::ProblemData p;
};

}  // namespace

extern "C" {

int aapdhg_ref_solve(const aapdhg_problem_view* prob, const aapdhg_solve_params* prm,
                     const double* x0, const double* y0, aapdhg_solve_result* res,
                     double* x_out, double* y_out, double* lambda_out,
                     aapdhg_record_sink sink, void* ctx, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    const R::ProblemData p = problem_of(prob);
    const std::size_t n = std::size_t(p.n()), m = p.q.size();
    const R::SolverConfig cfg = config_of(prm, n + m);
    R::Iterate u0;
    u0.x = x0 ? R::Vec(x0, x0 + n) : R::Vec(n, 0.0);
    u0.y = y0 ? R::Vec(y0, y0 + m) : R::Vec(m, 0.0);
    const R::SolveOutput out = R::solve(p, cfg, u0);
    const R::SolveResult& r = out.result;
    res->status = int32_t(r.status);
    res->iterations = r.iterations;
    res->i = r.i;
    res->j = r.j;
    res->aa_failures = r.aa_failures;
    res->g_norm = r.g_norm;
    res->r_gap = r.kkt.r_gap;
    res->r_primal = r.kkt.r_primal;
    res->r_dual = r.kkt.r_dual;
    res->objective = r.objective;
    res->tau = r.steps.tau;
    res->sigma = r.steps.sigma;
    res->wall_seconds = r.wall_seconds;
    if (x_out) std::memcpy(x_out, r.u.x.data(), n * sizeof(double));
    if (y_out) std::memcpy(y_out, r.u.y.data(), m * sizeof(double));
    if (lambda_out) std::memcpy(lambda_out, r.lambda.data(), n * sizeof(double));
    if (sink) {
      std::vector<aapdhg_record> recs(out.trajectory.size());
      for (std::size_t t = 0; t < recs.size(); ++t) {
        const R::TrajectoryRecord& s = out.trajectory[t];
        aapdhg_record& d = recs[t];
        std::memset(&d, 0, sizeof d);
        d.k = s.k;
        d.g_norm = s.g_norm;
        d.aa_step = s.aa_step ? 1 : 0;
        d.i = s.i;
        d.j = s.j;
        d.r_gap = s.kkt.r_gap;
        d.r_primal = s.kkt.r_primal;
        d.r_dual = s.kkt.r_dual;
        d.objective = s.objective;
        d.elapsed_s = s.elapsed_s;
      }
      sink(recs.data(), recs.size(), ctx);
    }
  });
}

int aapdhg_ref_select_step_sizes(const aapdhg_problem_view* prob,
                                 const aapdhg_solve_params* prm, double* tau,
                                 double* sigma, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    const R::ProblemData p = problem_of(prob);
    const R::StepSizes s = R::select_step_sizes(p, config_of(prm, p.c.size() + p.q.size()));
    *tau = s.tau;
    *sigma = s.sigma;
  });
}

int aapdhg_ref_power_norm(const aapdhg_problem_view* prob, int32_t max_iters,
                          double rel_tol, uint64_t seed, double* out, char* err,
                          size_t errlen) {
  return guard(err, errlen, [&] {
    const R::ProblemData p = problem_of(prob);
    *out = R::power_iteration_norm(p.k, max_iters, rel_tol, seed);
  });
}

int aapdhg_ref_matvec(const aapdhg_problem_view* prob, const double* x, double* out,
                      char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    const R::ProblemData p = problem_of(prob);
    const R::Vec r = R::matvec(p.k, R::Vec(x, x + p.n()));
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int aapdhg_ref_matvec_transpose(const aapdhg_problem_view* prob, const double* y,
                                double* out, char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    const R::ProblemData p = problem_of(prob);
    const R::Vec r = R::matvec_transpose(p.k, R::Vec(y, y + p.q.size()));
    std::memcpy(out, r.data(), r.size() * sizeof(double));
  });
}

int aapdhg_ref_pdhg_step(const aapdhg_problem_view* prob, double tau, double sigma,
                         const double* x, const double* y, double* xn, double* yn,
                         char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    const R::ProblemData p = problem_of(prob);
    R::Iterate u{R::Vec(x, x + p.n()), R::Vec(y, y + p.q.size())};
    const R::Iterate t = R::pdhg_step(u, p, R::StepSizes{tau, sigma});
    std::memcpy(xn, t.x.data(), t.x.size() * sizeof(double));
    std::memcpy(yn, t.y.data(), t.y.size() * sizeof(double));
  });
}

int aapdhg_ref_kkt_metrics(const aapdhg_problem_view* prob, const double* x,
                           const double* y, double* kkt, double* lambda, char* err,
                           size_t errlen) {
  return guard(err, errlen, [&] {
    const R::ProblemData p = problem_of(prob);
    R::Iterate u{R::Vec(x, x + p.n()), R::Vec(y, y + p.q.size())};
    const auto [m, lam] = R::kkt_metrics(u, p, R::build_lambda_set(p.l, p.u));
    kkt[0] = m.r_gap;
    kkt[1] = m.r_primal;
    kkt[2] = m.r_dual;
    kkt[3] = R::dot(p.c, u.x);
    if (lambda) std::memcpy(lambda, lam.data(), lam.size() * sizeof(double));
  });
}

int aapdhg_ref_aa_apply(int32_t p, int64_t N, const double* du_cols,
                        const double* dg_cols, double beta, const double* d_hat,
                        double eta, const double* u, const double* g, double* out,
                        char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    R::AAMemory mem;
    mem.capacity = std::size_t(p > 0 ? p : 1);
    mem.du_cols = columns(du_cols, p, std::size_t(N));
    mem.dg_cols = columns(dg_cols, p, std::size_t(N));
    R::AAParams prm;
    prm.beta = beta;
    prm.eta = eta;
    if (d_hat) prm.d_hat.assign(d_hat, d_hat + N);
    const R::Vec r = R::aa_apply(mem, prm, R::Vec(u, u + N), R::Vec(g, g + N));
    std::memcpy(out, r.data(), std::size_t(N) * sizeof(double));
  });
}

int aapdhg_ref_filtered_aa_apply(int32_t p, int64_t N, const double* e_cols,
                                 const double* f_cols, double c_s, double kappa_bar,
                                 double beta, const double* d_hat, const double* u,
                                 const double* g, double* out, int32_t* kept,
                                 char* err, size_t errlen) {
  return guard(err, errlen, [&] {
    const auto e = columns(e_cols, p, std::size_t(N));
    const auto f = columns(f_cols, p, std::size_t(N));
    R::FilterParams fp;
    fp.c_s = c_s;
    fp.kappa_bar = kappa_bar;
    const R::FilteredMemory fm = R::build_filtered_memory(e, f, fp);
    // identify surviving columns (kept lists preserve order)
    std::size_t t = 0;
    for (int j = 0; j < p; ++j) {
      const bool hit = t < fm.f.size() && fm.f[t] == f[std::size_t(j)] && fm.e[t] == e[std::size_t(j)];
      if (kept) kept[j] = hit ? 1 : 0;
      if (hit) ++t;
    }
    R::AAParams prm;
    prm.beta = beta;
    if (d_hat) prm.d_hat.assign(d_hat, d_hat + N);
    const R::Vec r = R::filtered_aa_apply(fm, prm, R::Vec(u, u + N), R::Vec(g, g + N));
    std::memcpy(out, r.data(), std::size_t(N) * sizeof(double));
  });
}

int aapdhg_ref_safeguard_pass(double g_norm, double g0_norm, uint64_t i, double d,
                              double eps) {
  return R::safeguard_pass(g_norm, g0_norm, std::size_t(i), d, eps) ? 1 : 0;
}

// ---- test-support generators (proj/tests/support/test_support.cpp) ------

// kind: 0 toy, 1 random_box_lp (index-th draw from mt19937_64(seed)),
//       2 transport_lp(a, b, seed, slack), 3 setcover_lp(a, b, c, seed)
void* aapdhg_ref_gen(int32_t kind, int32_t a, int32_t b, int32_t c, uint64_t seed,
                     double slack, int32_t index) {
  try {
    auto* g = new GenProblem;
    switch (kind) {
      case 0: g->p = testsup::toy_problem(); break;
      case 1: {
        std::mt19937_64 rng(seed);
        for (int t = 0; t <= index; ++t) g->p = testsup::random_box_lp(rng);
        break;
      }
      case 2: g->p = testsup::transport_lp(a, b, unsigned(seed), slack); break;
      case 3: g->p = testsup::setcover_lp(a, b, c, unsigned(seed)); break;
      default: delete g; return nullptr;
    }
    return g;
  } catch (...) {
    return nullptr;
  }
}

void aapdhg_ref_gen_dims(void* h, int32_t* n, int32_t* m1, int32_t* m2, int64_t* nnz) {
  const auto& p = static_cast<GenProblem*>(h)->p;
  *n = p.n();
  *m1 = p.m1();
  *m2 = p.m2();
  *nnz = int64_t(p.k.nnz());
}

void aapdhg_ref_gen_copy(void* h, int32_t* row_ptr, int32_t* col_idx, double* vals,
                         double* c, double* q, double* l, double* u) {
  const auto& p = static_cast<GenProblem*>(h)->p;
  std::memcpy(row_ptr, p.k.row_ptr.data(), p.k.row_ptr.size() * sizeof(int32_t));
  std::memcpy(col_idx, p.k.col_idx.data(), p.k.col_idx.size() * sizeof(int32_t));
  std::memcpy(vals, p.k.vals.data(), p.k.vals.size() * sizeof(double));
  std::memcpy(c, p.c.data(), p.c.size() * sizeof(double));
  std::memcpy(q, p.q.data(), p.q.size() * sizeof(double));
  std::memcpy(l, p.l.data(), p.l.size() * sizeof(double));
  std::memcpy(u, p.u.data(), p.u.size() * sizeof(double));
}

void aapdhg_ref_gen_free(void* h) { delete static_cast<GenProblem*>(h); }

}  // extern "C"
