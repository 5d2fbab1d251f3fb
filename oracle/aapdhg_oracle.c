/*
 * aapdhg_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference CPU algorithm for the AA-PDHG /
 * FAA-PDHG solve path. Every function cites the reference lines it restates
 * (paths relative to the reference checkout). Arithmetic is written in the
 * reference's exact expression order and compiled with -ffp-contract=off so
 * that results are bit-identical to the reference built -O3 on x86-64
 * (pinned in tests/test_oracle_pin.py against oracle/_ref and the golden
 * fixtures in tests/golden/).
 */
#define _POSIX_C_SOURCE 200809L
#include "aapdhg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* std::min / std::max semantics (libstdc++: max(a,b) = a<b ? b : a,
 * min(a,b) = b<a ? b : a) — matters for signed zeros.                       */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

static void set_err(char* err, size_t errlen, const char* msg) {
  if (!err || errlen == 0) return;
  strncpy(err, msg, errlen - 1);
  err[errlen - 1] = '\0';
}

static void* xmalloc(size_t bytes) {
  void* p = calloc(bytes ? bytes : 1, 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory (%zu bytes)\n", bytes);
    abort();
  }
  return p;
}

/* vec.hpp:16-29 — serial dot / nrm2sq in index order. */
static double dotv(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double nrm2sq(const double* a, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * a[i];
  return s;
}

/* ---- sparse_linalg.cpp -------------------------------------------------- */

/* matvec, proj/src/sparse_linalg.cpp:60-69: row-serial sum in CSR order. */
static void matvec(const aapdhg_csr_view* k, const double* v, double* out) {
  for (int32_t r = 0; r < k->nrows; ++r) {
    double s = 0.0;
    for (int32_t e = k->row_ptr[r]; e < k->row_ptr[r + 1]; ++e)
      s += k->vals[e] * v[k->col_idx[e]];
    out[r] = s;
  }
}

/* matvec_transpose, proj/src/sparse_linalg.cpp:77-87: zero-initialised
 * row-ascending scatter, rows with v[row]==0 skipped. */
static void matvec_t(const aapdhg_csr_view* k, const double* v, double* out) {
  for (int32_t c = 0; c < k->ncols; ++c) out[c] = 0.0;
  for (int32_t r = 0; r < k->nrows; ++r) {
    const double vr = v[r];
    if (vr == 0.0) continue;
    for (int32_t e = k->row_ptr[r]; e < k->row_ptr[r + 1]; ++e)
      out[k->col_idx[e]] += k->vals[e] * vr;
  }
}

/* std::mt19937_64 (published MT19937-64 algorithm, as in <random>). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;
static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}
/* libstdc++ generate_canonical<double,53> for a 64-bit engine (one draw,
 * divided by 2^64, clamped below 1), then uniform_real_distribution(a,b):
 * canonical * (b - a) + a. */
static double mt64_uniform(mt64* g, double a, double b) {
  double c = (double)mt64_next(g) / 18446744073709551616.0;
  if (c >= 1.0) c = nextafter(1.0, 0.0);
  return c * (b - a) + a;
}

void aapdhg_oracle_power_start(uint64_t seed, int64_t n, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = mt64_uniform(&g, -1.0, 1.0);
}

/* power_iteration_norm, proj/src/sparse_linalg.cpp:95-123. */
int aapdhg_oracle_power_norm(const aapdhg_problem_view* prob, int32_t max_iters,
                             double rel_tol, uint64_t seed, double* out,
                             int32_t* rounds) {
  const aapdhg_csr_view* k = &prob->k;
  int all_zero = 1;
  for (int64_t e = 0; e < k->nnz; ++e)
    if (k->vals[e] != 0.0) { all_zero = 0; break; }
  if (rounds) *rounds = 0;
  if (all_zero) { *out = 0.0; return AAPDHG_OK; }
  const int64_t n = k->ncols;
  double* x = xmalloc(sizeof(double) * (size_t)n);
  double* mx = xmalloc(sizeof(double) * (size_t)k->nrows);
  double* mtmx = xmalloc(sizeof(double) * (size_t)n);
  aapdhg_oracle_power_start(seed, n, x);
  double xn = sqrt(nrm2sq(x, n));
  if (xn == 0.0) { x[0] = 1.0; xn = 1.0; }
  for (int64_t i = 0; i < n; ++i) x[i] /= xn;
  double est = 0.0;
  int done = 0;
  for (int it = 0; it < max_iters; ++it) {
    matvec(k, x, mx);
    matvec_t(k, mx, mtmx);
    const double lam = sqrt(nrm2sq(mtmx, n));
    const double next = sqrt(lam);
    if (rounds) *rounds = it + 1;
    if (lam == 0.0) { est = 0.0; done = 1; break; }
    for (int64_t i = 0; i < n; ++i) x[i] = mtmx[i] / lam;
    if (it > 0 && fabs(next - est) < rel_tol * next) { est = next; done = 1; break; }
    est = next;
  }
  (void)done;
  *out = est;
  free(x); free(mx); free(mtmx);
  return AAPDHG_OK;
}

/* ---- pdhg_core.cpp ------------------------------------------------------ */

/* project_box / project_dual, proj/src/pdhg_core.cpp:10-25. */
static void project_feasible(const aapdhg_problem_view* p, double* x, double* y) {
  const int32_t n = p->k.ncols;
  for (int32_t i = 0; i < n; ++i) x[i] = smin(smax(x[i], p->l[i]), p->u[i]);
  for (int32_t i = 0; i < p->m1; ++i) y[i] = smax(y[i], 0.0);
}

/* pdhg_step, proj/src/pdhg_core.cpp:45-63. `kty`, `kxn`, `kx` are scratch. */
static void pdhg_step(const aapdhg_problem_view* p, double tau, double sigma,
                      const double* x, const double* y, double* xn, double* yn,
                      double* kty, double* kxn, double* kx) {
  const int32_t n = p->k.ncols, m = p->k.nrows;
  matvec_t(&p->k, y, kty);
  for (int32_t i = 0; i < n; ++i) xn[i] = x[i] - tau * (p->c[i] - kty[i]);
  for (int32_t i = 0; i < n; ++i) xn[i] = smin(smax(xn[i], p->l[i]), p->u[i]);
  matvec(&p->k, xn, kxn);
  matvec(&p->k, x, kx);
  for (int32_t i = 0; i < m; ++i) yn[i] = y[i] + sigma * (p->q[i] - (2.0 * kxn[i] - kx[i]));
  for (int32_t i = 0; i < p->m1; ++i) yn[i] = smax(yn[i], 0.0);
}

int aapdhg_oracle_pdhg_step(const aapdhg_problem_view* p, double tau, double sigma,
                            const double* x, const double* y, double* xn, double* yn) {
  const int32_t n = p->k.ncols, m = p->k.nrows;
  double* kty = xmalloc(sizeof(double) * (size_t)n);
  double* kxn = xmalloc(sizeof(double) * (size_t)m);
  double* kx = xmalloc(sizeof(double) * (size_t)m);
  pdhg_step(p, tau, sigma, x, y, xn, yn, kty, kxn, kx);
  free(kty); free(kxn); free(kx);
  return AAPDHG_OK;
}

int aapdhg_oracle_matvec(const aapdhg_problem_view* p, const double* x, double* out) {
  matvec(&p->k, x, out);
  return AAPDHG_OK;
}
int aapdhg_oracle_matvec_transpose(const aapdhg_problem_view* p, const double* y, double* out) {
  matvec_t(&p->k, y, out);
  return AAPDHG_OK;
}

/* ---- solver.cpp: KKT ---------------------------------------------------- */

/* build_lambda_set (proj/src/lp_model.cpp:293-306) + project_lambda
 * (proj/src/pdhg_core.cpp:27-39) fused: lambda_i = P_Lambda_i(v_i). */
static double project_lambda1(double v, double l, double u) {
  const int lo = isfinite(l), hi = isfinite(u);
  if (!lo && !hi) return 0.0;    /* kZero   */
  if (!lo) return smin(v, 0.0);  /* kNonpos */
  if (!hi) return smax(v, 0.0);  /* kNonneg */
  return v;                      /* kFree   */
}

typedef struct {
  double r_gap, r_primal, r_dual, primal_obj;
} kkt_t;

/* kkt_metrics, proj/src/solver.cpp:64-110. Scratch: kty[n], kx[m]. */
static kkt_t kkt_metrics(const aapdhg_problem_view* p, const double* x, const double* y,
                         double* lambda_out, double* kty, double* kx) {
  const int32_t n = p->k.ncols, m = p->k.nrows, m1 = p->m1;
  matvec_t(&p->k, y, kty);
  /* reduced = c - kty kept implicitly; lambda = P_Lambda(reduced) */
  double bound_terms = 0.0;
  for (int32_t i = 0; i < n; ++i) {
    const double red = p->c[i] - kty[i];
    const double lam = project_lambda1(red, p->l[i], p->u[i]);
    if (lambda_out) lambda_out[i] = lam;
    if (isfinite(p->l[i]) && lam > 0.0) bound_terms += p->l[i] * lam;
    if (isfinite(p->u[i]) && lam < 0.0) bound_terms += p->u[i] * lam;
  }
  const double dual_core = dotv(p->q, y, m) + bound_terms;
  const double primal_obj = dotv(p->c, x, n);
  kkt_t r;
  r.r_gap = fabs(dual_core - primal_obj) / (1.0 + fabs(dual_core) + fabs(primal_obj));
  matvec(&p->k, x, kx);
  double infeas_sq = 0.0;
  for (int32_t i = 0; i < m1; ++i) {
    const double v = smax(p->q[i] - kx[i], 0.0);
    infeas_sq += v * v;
  }
  for (int32_t i = m1; i < m; ++i) {
    const double v = p->q[i] - kx[i];
    infeas_sq += v * v;
  }
  r.r_primal = sqrt(infeas_sq) / (1.0 + sqrt(nrm2sq(p->q, m)));
  double dual_sq = 0.0;
  for (int32_t i = 0; i < n; ++i) {
    const double red = p->c[i] - kty[i];
    const double v = red - project_lambda1(red, p->l[i], p->u[i]);
    dual_sq += v * v;
  }
  r.r_dual = sqrt(dual_sq) / (1.0 + sqrt(nrm2sq(p->c, n)));
  r.primal_obj = primal_obj;
  return r;
}

int aapdhg_oracle_kkt_metrics(const aapdhg_problem_view* p, const double* x,
                              const double* y, double* kkt, double* lambda) {
  double* kty = xmalloc(sizeof(double) * (size_t)p->k.ncols);
  double* kx = xmalloc(sizeof(double) * (size_t)p->k.nrows);
  const kkt_t r = kkt_metrics(p, x, y, lambda, kty, kx);
  kkt[0] = r.r_gap;
  kkt[1] = r.r_primal;
  kkt[2] = r.r_dual;
  kkt[3] = r.primal_obj;
  free(kty); free(kx);
  return AAPDHG_OK;
}

/* safeguard_pass, proj/src/solver.cpp:59-62 (equality passes). */
int aapdhg_oracle_safeguard_pass(double g_norm, double g0_norm, uint64_t i, double d,
                                 double eps) {
  return g_norm <= d * g0_norm * pow((double)i + 1.0, -(1.0 + eps));
}

/* ---- anderson.cpp ------------------------------------------------------- */

/* damp, proj/src/anderson.cpp:10-20: beta*v, or (beta*d_hat_i)*v_i. */
static inline double damp1(double beta, const double* d_hat, int64_t i, double v) {
  return d_hat ? beta * d_hat[i] * v : beta * v;
}

/* cholesky_solve, proj/src/anderson.cpp:26-51; a is p x p column-major and
 * overwritten; returns AAPDHG_ERR_SINGULAR on a pivot <= 0. */
static int cholesky_solve(int p, double* a, double* rhs) {
#define A(i, j) a[(size_t)(j) * (size_t)p + (size_t)(i)]
  for (int j = 0; j < p; ++j) {
    double d = A(j, j);
    for (int k = 0; k < j; ++k) d -= A(j, k) * A(j, k);
    if (d <= 0.0) return AAPDHG_ERR_SINGULAR;
    d = sqrt(d);
    A(j, j) = d;
    for (int i = j + 1; i < p; ++i) {
      double s = A(i, j);
      for (int k = 0; k < j; ++k) s -= A(i, k) * A(j, k);
      A(i, j) = s / d;
    }
  }
  for (int i = 0; i < p; ++i) {
    double s = rhs[i];
    for (int k = 0; k < i; ++k) s -= A(i, k) * rhs[k];
    rhs[i] = s / A(i, i);
  }
  for (int i = p - 1; i >= 0; --i) {
    double s = rhs[i];
    for (int k = i + 1; k < p; ++k) s -= A(k, i) * rhs[k];
    rhs[i] = s / A(i, i);
  }
#undef A
  return AAPDHG_OK;
}

/* aa_apply, proj/src/anderson.cpp:106-135. du[j], dg[j] oldest first. */
static int aa_apply(int p, int64_t N, const double* const* du, const double* const* dg,
                    double beta, const double* d_hat, double eta, const double* u,
                    const double* g, double* out) {
  for (int64_t i = 0; i < N; ++i) out[i] = u[i] + damp1(beta, d_hat, i, g[i]);
  if (p == 0) return AAPDHG_OK;
  double* gram = xmalloc(sizeof(double) * (size_t)p * (size_t)p);
  double* w = xmalloc(sizeof(double) * (size_t)p);
  double frob_sq = 0.0;
  for (int i = 0; i < p; ++i) {
    for (int j = i; j < p; ++j) {
      const double v = dotv(dg[i], dg[j], N);
      gram[(size_t)j * p + i] = v;
      gram[(size_t)i * p + j] = v;
    }
    frob_sq += gram[(size_t)i * p + i];
  }
  const double eta_eff = eta * frob_sq;
  for (int i = 0; i < p; ++i) gram[(size_t)i * p + i] += eta_eff;
  for (int i = 0; i < p; ++i) w[i] = dotv(dg[i], g, N);
  const int rc = cholesky_solve(p, gram, w);
  if (rc == AAPDHG_OK) {
    for (int j = 0; j < p; ++j) {
      const double a = -w[j];
      for (int64_t i = 0; i < N; ++i) out[i] += a * du[j][i];
      for (int64_t i = 0; i < N; ++i) out[i] += a * damp1(beta, d_hat, i, dg[j][i]);
    }
  }
  free(gram); free(w);
  return rc;
}

int aapdhg_oracle_aa_apply(int32_t p, int64_t N, const double* du_cols,
                           const double* dg_cols, double beta, const double* d_hat,
                           double eta, const double* u, const double* g, double* out) {
  const double** du = xmalloc(sizeof(double*) * (size_t)(p ? p : 1));
  const double** dg = xmalloc(sizeof(double*) * (size_t)(p ? p : 1));
  for (int j = 0; j < p; ++j) {
    du[j] = du_cols + (size_t)j * (size_t)N;
    dg[j] = dg_cols + (size_t)j * (size_t)N;
  }
  const int rc = aa_apply(p, N, du, dg, beta, d_hat, eta, u, g, out);
  free(du); free(dg);
  return rc;
}

/* ---- filtering.cpp ------------------------------------------------------ */

/* qr_diagonal, proj/src/filtering.cpp:25-50: |diag R| of Householder QR of
 * the N x p column list (w overwritten, column-major N x p). */
static void qr_diagonal(int64_t N, int p, double* w, double* diag, double* v) {
#define W(i, j) w[(size_t)(j) * (size_t)N + (size_t)(i)]
  const int steps = (int64_t)p < N ? p : (int)N;
  for (int j = 0; j < steps; ++j) {
    double nrm_sq = 0.0;
    for (int64_t i = j; i < N; ++i) nrm_sq += W(i, j) * W(i, j);
    const double nrm = sqrt(nrm_sq);
    diag[j] = nrm;
    if (nrm == 0.0) continue;
    const double alpha = W(j, j) >= 0.0 ? -nrm : nrm;
    v[j] = W(j, j) - alpha;
    for (int64_t i = j + 1; i < N; ++i) v[i] = W(i, j);
    double vv = 0.0;
    for (int64_t i = j; i < N; ++i) vv += v[i] * v[i];
    if (vv == 0.0) continue;
    for (int col = j + 1; col < p; ++col) {
      double vw = 0.0;
      for (int64_t i = j; i < N; ++i) vw += v[i] * W(i, col);
      const double coef = 2.0 * vw / vv;
      for (int64_t i = j; i < N; ++i) W(i, col) -= coef * v[i];
    }
  }
#undef W
}

/* length_bounds, proj/src/filtering.cpp:92-114. */
void aapdhg_oracle_length_bounds(int32_t m, const double* fn_sq, double c_s, double* b) {
  if (m == 0) return;
  const double cs2 = c_s * c_s;
  const double ct = sqrt(smax(0.0, 1.0 - cs2));
  const double ct2 = ct * ct;
  b[0] = 1.0 / fn_sq[0];
  for (int jj = 1; jj < m; ++jj) {
    const int j = jj + 1;
    double acc = ct2 * pow((ct + c_s) / c_s, 2.0 * (j - 2)) / fn_sq[0];
    for (int i = 2; i <= j - 1; ++i)
      acc += ct2 * pow(ct + c_s, 2.0 * (j - i - 1)) /
             (fn_sq[i - 1] * pow(c_s, 2.0 * (j - i)));
    acc += 1.0 / fn_sq[jj];
    b[jj] = acc / cs2;
  }
}

/* economy_qr (proj/src/sparse_linalg.cpp:131-192) followed by the
 * back_substitute of filtered_aa_apply (proj/src/filtering.cpp:170-176,
 * proj/src/sparse_linalg.cpp:200-218): computes w = R^{-1} Q' g.
 * f: N x p column-major copy (overwritten). Returns SINGULAR per the floor. */
static int qr_solve(int64_t N, int p, double* f, const double* g, double* w) {
  if (p < 1 || p > N) return AAPDHG_ERR_DIMENSION;
#define W(i, j) f[(size_t)(j) * (size_t)N + (size_t)(i)]
  double** refl = xmalloc(sizeof(double*) * (size_t)p);
  for (int j = 0; j < p; ++j) {
    const int64_t len = N - j;
    double* v = xmalloc(sizeof(double) * (size_t)len);
    double norm = 0.0;
    for (int64_t i = j; i < N; ++i) norm += W(i, j) * W(i, j);
    norm = sqrt(norm);
    const double alpha = W(j, j) >= 0.0 ? -norm : norm;
    if (norm > 0.0) {
      for (int64_t i = j; i < N; ++i) v[i - j] = W(i, j);
      v[0] -= alpha;
      const double vn = sqrt(nrm2sq(v, len));
      if (vn > 0.0) {
        for (int64_t i = 0; i < len; ++i) v[i] /= vn;
        for (int c = j; c < p; ++c) {
          double s = 0.0;
          for (int64_t i = j; i < N; ++i) s += v[i - j] * W(i, c);
          s *= 2.0;
          for (int64_t i = j; i < N; ++i) W(i, c) -= s * v[i - j];
        }
      } else {
        for (int64_t i = 0; i < len; ++i) v[i] = 0.0;
      }
    }
    refl[j] = v;
  }
  double* r = xmalloc(sizeof(double) * (size_t)p * (size_t)p); /* column-major */
#define RR(i, j) r[(size_t)(j) * (size_t)p + (size_t)(i)]
  for (int j = 0; j < p; ++j)
    for (int i = 0; i <= j; ++i) RR(i, j) = W(i, j);
  /* Q' g column by column: q_c = H_0 ... H_{p-1} e_c, then (q_c . g) */
  double* col = xmalloc(sizeof(double) * (size_t)N);
  double* qtg = xmalloc(sizeof(double) * (size_t)p);
  for (int c = 0; c < p; ++c) {
    for (int64_t i = 0; i < N; ++i) col[i] = 0.0;
    col[c] = 1.0;
    for (int j = p - 1; j >= 0; --j) {
      const double* v = refl[j];
      double s = 0.0;
      for (int64_t i = j; i < N; ++i) s += v[i - j] * col[i];
      s *= 2.0;
      for (int64_t i = j; i < N; ++i) col[i] -= s * v[i - j];
    }
    /* nonnegative-diagonal sign convention (sparse_linalg.cpp:185-190) */
    if (RR(c, c) < 0.0)
      for (int64_t i = 0; i < N; ++i) col[i] = -col[i];
    double s = 0.0;
    for (int64_t i = 0; i < N; ++i) s += col[i] * g[i];
    qtg[c] = s;
  }
  for (int j = 0; j < p; ++j)
    if (RR(j, j) < 0.0)
      for (int c = j; c < p; ++c) RR(j, c) = -RR(j, c);
  /* back_substitute, proj/src/sparse_linalg.cpp:200-218 */
  double fro = 0.0;
  for (size_t t = 0; t < (size_t)p * (size_t)p; ++t) fro += r[t] * r[t];
  const double floor_v = 1e-14 * sqrt(fro);
  int rc = AAPDHG_OK;
  for (int i = 0; i < p; ++i)
    if (fabs(RR(i, i)) <= floor_v) rc = AAPDHG_ERR_SINGULAR;
  if (rc == AAPDHG_OK) {
    for (int i = 0; i < p; ++i) w[i] = qtg[i];
    for (int i = p - 1; i >= 0; --i) {
      double s = w[i];
      for (int j = i + 1; j < p; ++j) s -= RR(i, j) * w[j];
      w[i] = s / RR(i, i);
    }
  }
#undef RR
#undef W
  for (int j = 0; j < p; ++j) free(refl[j]);
  free(refl); free(r); free(col); free(qtg);
  return rc;
}

/* build_filtered_memory (proj/src/filtering.cpp:140-157) over column lists
 * e[], f[] (oldest first, count p): writes keep[p] (1 = survives).
 * reverse_columns (:61-67) -> angle_filter (:69-90) -> length_filter
 * (:116-138) -> reverse back. Returns SINGULAR on a zero leading column. */
static int filter_memory(int p, int64_t N, const double* const* e, const double* const* f,
                         double c_s, double kappa_bar, int* keep) {
  for (int j = 0; j < p; ++j) keep[j] = 0;
  if (p == 0) return AAPDHG_OK;
  /* reversed order: r-th column is original index p-1-r */
  double* wmat = xmalloc(sizeof(double) * (size_t)N * (size_t)p);
  for (int r = 0; r < p; ++r)
    memcpy(wmat + (size_t)r * (size_t)N, f[p - 1 - r], sizeof(double) * (size_t)N);
  const int steps = (int64_t)p < N ? p : (int)N;
  double* diag = xmalloc(sizeof(double) * (size_t)(steps ? steps : 1));
  double* v = xmalloc(sizeof(double) * (size_t)N);
  qr_diagonal(N, p, wmat, diag, v);
  int* akeep = xmalloc(sizeof(int) * (size_t)p);
  int rc = AAPDHG_OK;
  for (int r = 0; r < p; ++r) {
    akeep[r] = 1;
    const double fn = sqrt(nrm2sq(f[p - 1 - r], N));
    const double sine = ((int64_t)r < N && fn > 0.0) ? diag[r] / fn : 0.0;
    if (r == 0) {
      if (fn == 0.0) rc = AAPDHG_ERR_SINGULAR;
      continue;
    }
    if (sine < c_s) akeep[r] = 0;
  }
  if (rc == AAPDHG_OK) {
    /* surviving columns in reversed order */
    int m = 0;
    int* idx = xmalloc(sizeof(int) * (size_t)p);
    for (int r = 0; r < p; ++r)
      if (akeep[r]) idx[m++] = p - 1 - r;
    double* fn_sq = xmalloc(sizeof(double) * (size_t)m);
    double* b = xmalloc(sizeof(double) * (size_t)m);
    for (int t = 0; t < m; ++t) fn_sq[t] = nrm2sq(f[idx[t]], N);
    aapdhg_oracle_length_bounds(m, fn_sq, c_s, b);
    double* ep = xmalloc(sizeof(double) * (size_t)(m + 1));
    double* bp = xmalloc(sizeof(double) * (size_t)(m + 1));
    ep[0] = 0.0;
    bp[0] = 0.0;
    for (int t = 0; t < m; ++t) {
      ep[t + 1] = ep[t] + nrm2sq(e[idx[t]], N);
      bp[t + 1] = bp[t] + b[t];
    }
    const double cap = kappa_bar * kappa_bar;
    int kk = 0;
    for (int t = m; t >= 1; --t)
      if (ep[t] * bp[t] <= cap) { kk = t; break; }
    for (int t = 0; t < kk; ++t) keep[idx[t]] = 1;
    free(idx); free(fn_sq); free(b); free(ep); free(bp);
  }
  free(wmat); free(diag); free(v); free(akeep);
  return rc;
}

/* filtered_aa_apply, proj/src/filtering.cpp:159-181, on the kept columns
 * (oldest first). */
static int filtered_apply(int p, int64_t N, const double* const* e, const double* const* f,
                          double beta, const double* d_hat, const double* u, const double* g,
                          double* out) {
  for (int64_t i = 0; i < N; ++i) out[i] = u[i] + damp1(beta, d_hat, i, g[i]);
  if (p == 0) return AAPDHG_OK;
  double* fm = xmalloc(sizeof(double) * (size_t)N * (size_t)p);
  for (int j = 0; j < p; ++j) memcpy(fm + (size_t)j * (size_t)N, f[j], sizeof(double) * (size_t)N);
  double* w = xmalloc(sizeof(double) * (size_t)p);
  const int rc = qr_solve(N, p, fm, g, w);
  if (rc == AAPDHG_OK) {
    for (int j = 0; j < p; ++j) {
      const double a = -w[j];
      for (int64_t i = 0; i < N; ++i) out[i] += a * e[j][i];
      for (int64_t i = 0; i < N; ++i) out[i] += a * damp1(beta, d_hat, i, f[j][i]);
    }
  }
  free(fm); free(w);
  return rc;
}

int aapdhg_oracle_filtered_aa_apply(int32_t p, int64_t N, const double* e_cols,
                                    const double* f_cols, double c_s, double kappa_bar,
                                    double beta, const double* d_hat, const double* u,
                                    const double* g, double* out, int32_t* kept) {
  const double** e = xmalloc(sizeof(double*) * (size_t)(p ? p : 1));
  const double** f = xmalloc(sizeof(double*) * (size_t)(p ? p : 1));
  int* keep = xmalloc(sizeof(int) * (size_t)(p ? p : 1));
  for (int j = 0; j < p; ++j) {
    e[j] = e_cols + (size_t)j * (size_t)N;
    f[j] = f_cols + (size_t)j * (size_t)N;
  }
  int rc = filter_memory(p, N, e, f, c_s, kappa_bar, keep);
  if (rc == AAPDHG_OK) {
    int t = 0;
    for (int j = 0; j < p; ++j) {
      if (kept) kept[j] = keep[j];
      if (keep[j]) { e[t] = e[j]; f[t] = f[j]; ++t; }
    }
    rc = filtered_apply(t, N, e, f, beta, d_hat, u, g, out);
  }
  free(e); free(f); free(keep);
  return rc;
}

/* ---- solver.cpp --------------------------------------------------------- */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* validate, proj/src/solver.cpp:25-38. */
static int validate(const aapdhg_solve_params* c, char* err, size_t errlen) {
  const char* msg = NULL;
  if (c->m < 1) msg = "solver: m must be >= 1";
  else if (c->safeguard_d <= 0.0) msg = "solver: D must be > 0";
  else if (c->safeguard_eps <= 0.0) msg = "solver: eps must be > 0";
  else if (c->toll <= 0.0) msg = "solver: toll must be > 0";
  else if (c->kkt_eps <= 0.0) msg = "solver: kkt_eps must be > 0";
  else if (c->beta <= 0.0 || c->beta > 1.0) msg = "solver: beta must be in (0, 1]";
  else if (c->eta < 0.0) msg = "solver: eta must be >= 0";
  else if (c->c_s <= 0.0 || c->c_s > 1.0) msg = "solver: c_s must be in (0, 1]";
  else if (c->kappa_bar <= 0.0) msg = "solver: kappa_bar must be > 0";
  if (msg) { set_err(err, errlen, msg); return AAPDHG_ERR_INPUT; }
  return AAPDHG_OK;
}

/* select_step_sizes, proj/src/solver.cpp:112-123. */
int aapdhg_oracle_select_step_sizes(const aapdhg_problem_view* prob,
                                    const aapdhg_solve_params* prm, double* tau,
                                    double* sigma, char* err, size_t errlen) {
  if (prm->tau > 0.0 || prm->sigma > 0.0) {
    if (!(prm->tau > 0.0 && prm->sigma > 0.0)) {
      set_err(err, errlen, "step sizes: override requires both tau and sigma");
      return AAPDHG_ERR_INPUT;
    }
    *tau = prm->tau;
    *sigma = prm->sigma;
    return AAPDHG_OK;
  }
  double k_norm = 0.0;
  aapdhg_oracle_power_norm(prob, 5000, 1e-4, 12345u, &k_norm, NULL);
  if (k_norm == 0.0) { *tau = 1.0; *sigma = 1.0; return AAPDHG_OK; }
  const double s = 0.9 / k_norm;
  *tau = s;
  *sigma = s;
  return AAPDHG_OK;
}

/* difference memory: FIFO of (du, dg) column pointers, oldest first. */
typedef struct {
  double** du;
  double** dg;
  int size, cap;
} memory_t;

static void memory_push(memory_t* mem, double* du, double* dg, size_t cap) {
  mem->du[mem->size] = du;
  mem->dg[mem->size] = dg;
  mem->size++;
  while ((size_t)mem->size > cap) {
    free(mem->du[0]);
    free(mem->dg[0]);
    memmove(mem->du, mem->du + 1, sizeof(double*) * (size_t)(mem->size - 1));
    memmove(mem->dg, mem->dg + 1, sizeof(double*) * (size_t)(mem->size - 1));
    mem->size--;
  }
}

typedef struct {
  aapdhg_record* recs;
  uint64_t count, cap;
} recbuf_t;

static void rec_push(recbuf_t* rb, const aapdhg_record* r) {
  if (rb->count == rb->cap) {
    rb->cap = rb->cap ? 2 * rb->cap : 1024;
    aapdhg_record* nr = realloc(rb->recs, sizeof(aapdhg_record) * rb->cap);
    if (!nr) abort();
    rb->recs = nr;
  }
  rb->recs[rb->count++] = *r;
}

/* solve, proj/src/solver.cpp:125-253 (+ default start :255-260). */
int aapdhg_oracle_solve(const aapdhg_problem_view* prob, const aapdhg_solve_params* prm,
                        const double* x0, const double* y0, aapdhg_solve_result* res,
                        double* x_out, double* y_out, double* lambda_out,
                        aapdhg_record_sink sink, void* ctx, char* err, size_t errlen) {
  const double t0 = now_s();
  int rc = validate(prm, err, errlen);
  if (rc) return rc;
  const aapdhg_problem_view* p = prob;
  const int32_t n = p->k.ncols, m = p->k.nrows;
  const int64_t N = (int64_t)n + m;
  if (prm->d_hat)
    for (int64_t i = 0; i < N; ++i)
      if (prm->d_hat[i] <= 0.0) { set_err(err, errlen, "aa: d_hat entries must be > 0"); return AAPDHG_ERR_INPUT; }
  for (int32_t i = 0; i < n; ++i)
    if (p->l[i] > p->u[i]) { set_err(err, errlen, "build_lambda_set: l > u"); return AAPDHG_ERR_INPUT; }
  double tau, sigma;
  rc = aapdhg_oracle_select_step_sizes(p, prm, &tau, &sigma, err, errlen);
  if (rc) return rc;

  const double beta = prm->beta;
  const double* d_hat = prm->d_hat;
  uint64_t i_cnt = 0, j_cnt = 0, aa_failures = 0;
  recbuf_t rb = {NULL, 0, 0};

  /* iterates stored stacked (x; y) */
  double* u_prev = xmalloc(sizeof(double) * (size_t)N);
  double* u = xmalloc(sizeof(double) * (size_t)N);
  double* uh = xmalloc(sizeof(double) * (size_t)N);
  double* u_next = xmalloc(sizeof(double) * (size_t)N);
  double* g_prev = xmalloc(sizeof(double) * (size_t)N);
  double* gk = xmalloc(sizeof(double) * (size_t)N);
  double* cand = xmalloc(sizeof(double) * (size_t)N);
  double* kty = xmalloc(sizeof(double) * (size_t)n);
  double* kxa = xmalloc(sizeof(double) * (size_t)m);
  double* kxb = xmalloc(sizeof(double) * (size_t)m);
  const size_t cap = (size_t)prm->m;
  memory_t mem = {xmalloc(sizeof(double*) * (cap + 1)), xmalloc(sizeof(double*) * (cap + 1)), 0, (int)cap};

#define STEP(src, dst) pdhg_step(p, tau, sigma, (src), (src) + n, (dst), (dst) + n, kty, kxa, kxb)
#define RESID(a, b, g, out_norm)                               \
  do {                                                         \
    for (int64_t t_ = 0; t_ < N; ++t_) (g)[t_] = (b)[t_] - (a)[t_]; \
    (out_norm) = sqrt(nrm2sq((g), N));                         \
  } while (0)

  int status = -1;
  double g_final = 0.0;
  const double* u_final = NULL;

  /* record, solver.cpp:138-151: KKT evaluated at the produced iterate. */
#define RECORD(K, GN, AA, IK, JK, PRODUCED, KKT_OUT)                               \
  do {                                                                            \
    aapdhg_record r_;                                                             \
    memset(&r_, 0, sizeof r_);                                                    \
    r_.k = (K);                                                                   \
    r_.g_norm = (GN);                                                             \
    r_.aa_step = (AA);                                                            \
    r_.i = (IK);                                                                  \
    r_.j = (JK);                                                                  \
    const kkt_t kk_ = kkt_metrics(p, (PRODUCED), (PRODUCED) + n, NULL, kty, kxa); \
    r_.r_gap = kk_.r_gap;                                                         \
    r_.r_primal = kk_.r_primal;                                                   \
    r_.r_dual = kk_.r_dual;                                                       \
    r_.objective = dotv(p->c, (PRODUCED), n);                                     \
    r_.elapsed_s = now_s() - t0;                                                  \
    rec_push(&rb, &r_);                                                           \
    (KKT_OUT) = smax(smax(kk_.r_gap, kk_.r_primal), kk_.r_dual);                  \
  } while (0)

  for (int32_t t = 0; t < n; ++t) u_prev[t] = x0 ? x0[t] : 0.0;
  for (int32_t t = 0; t < m; ++t) u_prev[n + t] = y0 ? y0[t] : 0.0;
  project_feasible(p, u_prev, u_prev + n);
  STEP(u_prev, uh);
  double g0n;
  RESID(u_prev, uh, g_prev, g0n);
  double kmax;
  RECORD(0, g0n, 0, 0, 0, uh, kmax);
  if (g0n == 0.0) {
    status = AAPDHG_SOLVE_FIXED_POINT_START;
    u_final = u_prev;
    g_final = 0.0;
  } else if (prm->kkt_terminate && kmax <= prm->kkt_eps) {
    STEP(uh, u_next);
    double gn;
    RESID(uh, u_next, gk, gn);
    status = AAPDHG_SOLVE_KKT_TOL;
    u_final = uh;
    g_final = gn;
  } else {
    memcpy(u, uh, sizeof(double) * (size_t)N);
    /* FAA carried memory uses the same FIFO container (solver.cpp:42-53) */
    for (uint64_t k = 1;; ++k) {
      STEP(u, uh);
      double gkn;
      RESID(u, uh, gk, gkn);
      if (gkn < prm->toll) { status = AAPDHG_SOLVE_RESIDUAL_TOL; u_final = u; g_final = gkn; break; }
      if (i_cnt + j_cnt >= prm->max_iters) { status = AAPDHG_SOLVE_MAX_ITERS; u_final = u; g_final = gkn; break; }
      if (now_s() - t0 >= prm->max_wall_seconds) { status = AAPDHG_SOLVE_TIMEOUT; u_final = u; g_final = gkn; break; }

      if (prm->method != AAPDHG_METHOD_PDHG) {
        double* du = xmalloc(sizeof(double) * (size_t)N);
        double* dg = xmalloc(sizeof(double) * (size_t)N);
        for (int64_t t = 0; t < N; ++t) du[t] = u[t] - u_prev[t];
        for (int64_t t = 0; t < N; ++t) dg[t] = gk[t] - g_prev[t];
        memory_push(&mem, du, dg, cap);
      }
      const uint64_t i_pre = i_cnt, j_pre = j_cnt;
      int aa_step = 0;
      if (prm->method != AAPDHG_METHOD_PDHG &&
          aapdhg_oracle_safeguard_pass(gkn, g0n, i_cnt, prm->safeguard_d, prm->safeguard_eps)) {
        int arc;
        if (prm->method == AAPDHG_METHOD_AA) {
          arc = aa_apply(mem.size, N, (const double* const*)mem.du, (const double* const*)mem.dg,
                         beta, d_hat, prm->eta, u, gk, cand);
        } else {
          int* keep = xmalloc(sizeof(int) * (size_t)(mem.size ? mem.size : 1));
          arc = filter_memory(mem.size, N, (const double* const*)mem.du,
                              (const double* const*)mem.dg, prm->c_s, prm->kappa_bar, keep);
          if (arc == AAPDHG_OK) {
            const double** ke = xmalloc(sizeof(double*) * (size_t)(mem.size ? mem.size : 1));
            const double** kf = xmalloc(sizeof(double*) * (size_t)(mem.size ? mem.size : 1));
            int kp = 0;
            for (int t = 0; t < mem.size; ++t)
              if (keep[t]) { ke[kp] = mem.du[t]; kf[kp] = mem.dg[t]; ++kp; }
            arc = filtered_apply(kp, N, ke, kf, beta, d_hat, u, gk, cand);
            if (arc == AAPDHG_OK) {
              /* carried memory replaced only on success (solver.cpp:221-224) */
              int t2 = 0;
              for (int t = 0; t < mem.size; ++t) {
                if (keep[t]) { mem.du[t2] = mem.du[t]; mem.dg[t2] = mem.dg[t]; ++t2; }
                else { free(mem.du[t]); free(mem.dg[t]); }
              }
              mem.size = t2;
            }
            free(ke); free(kf);
          }
          free(keep);
        }
        if (arc == AAPDHG_OK) {
          memcpy(u_next, cand, sizeof(double) * (size_t)N);
          project_feasible(p, u_next, u_next + n);
          aa_step = 1;
          ++i_cnt;
        } else if (arc == AAPDHG_ERR_SINGULAR) {
          memcpy(u_next, uh, sizeof(double) * (size_t)N);
          ++j_cnt;
          ++aa_failures;
        } else {
          set_err(err, errlen, "economy_qr: need 1 <= p <= n");
          rc = arc;
          break;
        }
      } else {
        memcpy(u_next, uh, sizeof(double) * (size_t)N);
        ++j_cnt;
      }
      RECORD(k, gkn, aa_step, i_pre, j_pre, u_next, kmax);
      if (prm->kkt_terminate && kmax <= prm->kkt_eps) {
        double gn;
        STEP(u_next, uh);
        RESID(u_next, uh, gk, gn);
        status = AAPDHG_SOLVE_KKT_TOL;
        u_final = u_next;
        g_final = gn;
        break;
      }
      /* u_prev = u; g_prev = gk; u = u_next (solver.cpp:249-251) */
      double* tmp = u_prev;
      u_prev = u;
      u = u_next;
      u_next = tmp;
      tmp = g_prev;
      g_prev = gk;
      gk = tmp;
    }
  }

  if (rc == AAPDHG_OK) {
    /* finish, solver.cpp:153-166 */
    double* lam = xmalloc(sizeof(double) * (size_t)n);
    const kkt_t fk = kkt_metrics(p, u_final, u_final + n, lam, kty, kxa);
    res->status = status;
    res->iterations = i_cnt + j_cnt;
    res->i = i_cnt;
    res->j = j_cnt;
    res->aa_failures = aa_failures;
    res->g_norm = g_final;
    res->r_gap = fk.r_gap;
    res->r_primal = fk.r_primal;
    res->r_dual = fk.r_dual;
    res->objective = dotv(p->c, u_final, n);
    res->tau = tau;
    res->sigma = sigma;
    res->wall_seconds = now_s() - t0;
    if (x_out) memcpy(x_out, u_final, sizeof(double) * (size_t)n);
    if (y_out) memcpy(y_out, u_final + n, sizeof(double) * (size_t)m);
    if (lambda_out) memcpy(lambda_out, lam, sizeof(double) * (size_t)n);
    free(lam);
    if (sink && rb.count) sink(rb.recs, rb.count, ctx);
  }
#undef STEP
#undef RESID
#undef RECORD
  for (int t = 0; t < mem.size; ++t) { free(mem.du[t]); free(mem.dg[t]); }
  free(mem.du); free(mem.dg);
  free(u_prev); free(u); free(uh); free(u_next); free(g_prev); free(gk); free(cand);
  free(kty); free(kxa); free(kxb); free(rb.recs);
  return rc;
}
