// modules.cpp — the drop-in's anderson.hpp / filtering.hpp / QR building
// blocks (proj/include/aapdhg/anderson.hpp:12-48, filtering.hpp:14-59,
// sparse_linalg.hpp:60-72), so that code written against the reference's
// module API — its own test_anderson / test_filtering / test_sparse_linalg
// suites and acceptance_test — builds and runs on the B200 library.
//
// The column-level numerics run on the device through the per-op C-ABI
// entries on a workspace handle sized to the columns
// (aapdhg_cuda_workspace_create): aa_apply -> aapdhg_cuda_aa_apply (the
// solve loop's Gram / Cholesky / mix kernels), the FAA kept sets and
// candidates -> aapdhg_cuda_faa_op (its filters and double-double least
// squares), economy_qr -> aapdhg_cuda_economy_qr. What stays on the host is
// container bookkeeping (memory_push, reverse_columns), argument checks with
// the reference's exception types, p x p triangular solves
// (back_substitute), the closed-form length bounds, and the Alg-1
// standard_aa_* test oracles (small dense solves on residual lists).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "aapdhg/aapdhg.hpp"
#include "aapdhg_cuda.h"

namespace aapdhg {
namespace {

[[noreturn]] void raise_rc(int rc, const char* msg) {
  const std::string m = msg && *msg ? msg : ("aapdhg_cuda error " + std::to_string(rc));
  switch (rc) {
    case AAPDHG_ERR_INPUT: throw InputError(m);
    case AAPDHG_ERR_DIMENSION: throw DimensionError(m);
    case AAPDHG_ERR_UNSUPPORTED: throw UnsupportedError(m);
    case AAPDHG_ERR_SINGULAR: throw SingularError(m);
    default: throw Error(m);
  }
}

void check_rc(int rc, const char* err) {
  if (rc != AAPDHG_OK) raise_rc(rc, err);
}

int device_of_env() {
  const char* d = std::getenv("AAPDHG_DEVICE");
  return d && *d ? std::atoi(d) : 0;
}

// One workspace handle per (thread, column length): the per-op entries are
// not re-entrant on a handle, threads get their own. (Kept for the thread's
// life; the device memory returns to the library's block cache at exit.)
aapdhg_handle* workspace(std::size_t n) {
  thread_local std::map<std::size_t, aapdhg_handle*>* ws = new std::map<std::size_t, aapdhg_handle*>();
  auto it = ws->find(n);
  if (it != ws->end()) return it->second;
  aapdhg_handle* h = nullptr;
  char err[512] = {0};
  check_rc(aapdhg_cuda_workspace_create(device_of_env(), int64_t(n), &h, err, sizeof err), err);
  (*ws)[n] = h;
  return h;
}

// columns -> one p x n block (column j at j * n)
std::vector<double> pack(const ColumnList& cols, std::size_t n) {
  std::vector<double> out(cols.size() * n);
  for (std::size_t j = 0; j < cols.size(); ++j)
    std::copy(cols[j].begin(), cols[j].end(), out.begin() + std::ptrdiff_t(j * n));
  return out;
}

std::size_t common_length(const ColumnList& e, const ColumnList& f, const char* what) {
  if (e.size() != f.size()) throw DimensionError(std::string(what) + ": column count mismatch");
  const std::size_t n = f.empty() ? 0 : f[0].size();
  for (const Vec& c : f)
    if (c.size() != n) throw DimensionError(std::string(what) + ": column length mismatch");
  for (const Vec& c : e)
    if (c.size() != n) throw DimensionError(std::string(what) + ": column length mismatch");
  return n;
}

// FAA steps on the device: kept flags of the columns in memory order
std::vector<int32_t> faa_kept(const ColumnList& e, const ColumnList& f, std::size_t n,
                              double c_s, double kappa_bar, int skip) {
  const int p = int(f.size());
  std::vector<int32_t> kept(std::size_t(std::max(p, 1)), 0);
  if (p == 0 || n == 0) return kept;
  const std::vector<double> ec = pack(e, n), fc = pack(f, n);
  char err[512] = {0};
  check_rc(aapdhg_cuda_faa_op(workspace(n), AAPDHG_REDUCE_AUTO, p, ec.data(), fc.data(), c_s,
                              kappa_bar, 1.0, nullptr, skip, nullptr, nullptr, nullptr,
                              kept.data(), err, sizeof err),
           err);
  return kept;
}

// the p x p symmetric eigen-decomposition (cyclic Jacobi): a = V diag(w) V'
void sym_eigen(std::vector<double> a, int n, std::vector<double>& w, std::vector<double>& v) {
  v.assign(std::size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) v[std::size_t(i) * n + i] = 1.0;
  auto A = [&](int i, int j) -> double& { return a[std::size_t(i) * n + j]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? tot : off) += A(i, j) * A(i, j);
    if (off <= 1e-32 * (tot + off) || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (A(p, q) == 0.0) continue;
        const double theta = (A(q, q) - A(p, p)) / (2.0 * A(p, q));
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- J' A J
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = v[std::size_t(k) * n + p], vkq = v[std::size_t(k) * n + q];
          v[std::size_t(k) * n + p] = c * vkp - s * vkq;
          v[std::size_t(k) * n + q] = s * vkp + c * vkq;
        }
      }
  }
  w.resize(std::size_t(n));
  for (int i = 0; i < n; ++i) w[std::size_t(i)] = A(i, i);
}

}  // namespace

// ---- anderson.hpp -------------------------------------------------------------
void memory_push(AAMemory& mem, Vec du, Vec dg) {
  if (du.size() != dg.size()) throw DimensionError("memory_push: du and dg lengths differ");
  if (!mem.empty() && du.size() != mem.du_cols.front().size())
    throw DimensionError("memory_push: column length differs from the memory's");
  mem.du_cols.push_back(std::move(du));
  mem.dg_cols.push_back(std::move(dg));
  while (mem.du_cols.size() > mem.capacity) {
    mem.du_cols.erase(mem.du_cols.begin());
    mem.dg_cols.erase(mem.dg_cols.begin());
  }
}

Vec damp(const AAParams& params, const Vec& v) {
  Vec out(v.size());
  if (params.d_hat.empty()) {
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = params.beta * v[i];
    return out;
  }
  if (params.d_hat.size() != v.size()) throw DimensionError("damp: d_hat length mismatch");
  for (double d : params.d_hat)
    if (!(d > 0.0)) throw InputError("damp: d_hat entries must be > 0");
  // (beta d_i) v_i: the association of the device's damping (common.cuh damp1)
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = params.beta * params.d_hat[i] * v[i];
  return out;
}

Vec aa_apply(const AAMemory& mem, const AAParams& params, const Vec& u, const Vec& g) {
  const std::size_t n = u.size();
  if (g.size() != n) throw DimensionError("aa_apply: u and g lengths differ");
  if (mem.du_cols.size() != mem.dg_cols.size())
    throw DimensionError("aa_apply: du / dg column counts differ");
  for (std::size_t j = 0; j < mem.size(); ++j)
    if (mem.du_cols[j].size() != n || mem.dg_cols[j].size() != n)
      throw DimensionError("aa_apply: memory column length differs from u");
  if (!params.d_hat.empty() && params.d_hat.size() != n)
    throw DimensionError("aa_apply: d_hat length mismatch");
  if (n == 0) return {};
  const std::vector<double> du = pack(mem.du_cols, n), dg = pack(mem.dg_cols, n);
  Vec out(n);
  char err[512] = {0};
  check_rc(aapdhg_cuda_aa_apply(workspace(n), AAPDHG_REDUCE_AUTO, int32_t(mem.size()), du.data(),
                                dg.data(), params.beta,
                                params.d_hat.empty() ? nullptr : params.d_hat.data(), params.eta,
                                u.data(), g.data(), out.data(), err, sizeof err),
           err);
  return out;
}

Vec standard_aa_weights(const std::vector<Vec>& residuals) {
  const int q = int(residuals.size());
  if (q == 0) throw InputError("standard_aa_weights: no residuals");
  const std::size_t n = residuals[0].size();
  for (const Vec& r : residuals)
    if (r.size() != n) throw DimensionError("standard_aa_weights: residual lengths differ");
  if (q == 1) return Vec{1.0};
  // min a'Ga s.t. 1'a = 1: the bordered system [G 1; 1' 0][a; l] = [0; 1],
  // solved with its pseudo-inverse (the minimum-norm solution when G is
  // singular, e.g. duplicate residuals)
  const int b = q + 1;
  std::vector<double> m(std::size_t(b) * b, 0.0);
  for (int i = 0; i < q; ++i) {
    for (int j = 0; j < q; ++j) m[std::size_t(i) * b + j] = dot(residuals[std::size_t(i)], residuals[std::size_t(j)]);
    m[std::size_t(i) * b + q] = m[std::size_t(q) * b + i] = 1.0;
  }
  std::vector<double> w, v;
  sym_eigen(m, b, w, v);
  double wmax = 0.0;
  for (double x : w) wmax = std::max(wmax, std::fabs(x));
  const double tol = wmax * double(b) * 1e-13;
  Vec sol(std::size_t(b), 0.0);
  for (int k = 0; k < b; ++k) {
    if (std::fabs(w[std::size_t(k)]) <= tol) continue;
    // coefficient of eigenvector k: (v_k . rhs) / w_k with rhs = e_q
    const double c = v[std::size_t(q) * b + k] / w[std::size_t(k)];
    for (int i = 0; i < b; ++i) sol[std::size_t(i)] += c * v[std::size_t(i) * b + k];
  }
  return Vec(sol.begin(), sol.begin() + q);
}

Vec standard_aa_step(const std::vector<Vec>& points, const std::vector<Vec>& images,
                     const Vec& weights, double beta) {
  if (points.size() != images.size() || weights.size() != points.size() || points.empty())
    throw DimensionError("standard_aa_step: points / images / weights counts differ");
  const std::size_t n = points[0].size();
  for (std::size_t i = 0; i < points.size(); ++i)
    if (points[i].size() != n || images[i].size() != n)
      throw DimensionError("standard_aa_step: vector lengths differ");
  Vec out(n);
  for (std::size_t t = 0; t < n; ++t) {
    double a = 0.0, b = 0.0;
    for (std::size_t i = 0; i < points.size(); ++i) {
      a += weights[i] * points[i][t];
      b += weights[i] * images[i][t];
    }
    out[t] = (1.0 - beta) * a + beta * b;
  }
  return out;
}

// ---- sparse_linalg.hpp: QR --------------------------------------------------------
QRFactors economy_qr(const DenseMatrix& f) {
  const int n = f.nrows, p = f.ncols;
  if (p > n) throw DimensionError("economy_qr: more columns than rows");
  QRFactors qr;
  qr.q = DenseMatrix(n, p);
  qr.r = DenseMatrix(p, p);
  if (p == 0) return qr;
  char err[512] = {0};
  check_rc(aapdhg_cuda_economy_qr(workspace(std::size_t(n)), AAPDHG_REDUCE_AUTO, p,
                                  f.data.data(), qr.q.data.data(), qr.r.data.data(), err,
                                  sizeof err),
           err);
  return qr;
}

DenseMatrix back_substitute(const DenseMatrix& r, const DenseMatrix& b) {
  const int k = r.nrows;
  if (r.ncols != k || b.nrows != k) throw DimensionError("back_substitute: dimension mismatch");
  double fro = 0.0;
  for (double x : r.data) fro += x * x;
  const double floor_v = 1e-14 * std::sqrt(fro);
  for (int i = 0; i < k; ++i)
    if (std::fabs(r.at(i, i)) <= floor_v) throw SingularError("back_substitute: singular triangle");
  DenseMatrix x(k, b.ncols);
  for (int c = 0; c < b.ncols; ++c)
    for (int i = k - 1; i >= 0; --i) {
      double s = b.at(i, c);
      for (int j = i + 1; j < k; ++j) s -= r.at(i, j) * x.at(j, c);
      x.at(i, c) = s / r.at(i, i);
    }
  return x;
}

Vec back_substitute(const DenseMatrix& r, const Vec& b) {
  DenseMatrix bm(int(b.size()), 1);
  std::copy(b.begin(), b.end(), bm.data.begin());
  const DenseMatrix x = back_substitute(r, bm);
  return x.data;
}

// ---- filtering.hpp -----------------------------------------------------------------
std::pair<ColumnList, ColumnList> reverse_columns(ColumnList e, ColumnList f) {
  if (e.size() != f.size()) throw DimensionError("reverse_columns: column count mismatch");
  std::reverse(e.begin(), e.end());
  std::reverse(f.begin(), f.end());
  return {std::move(e), std::move(f)};
}

// The device step reads the memory oldest first and filters newest first;
// a list given in filter order is passed reversed.
std::pair<ColumnList, ColumnList> angle_filter(ColumnList e, ColumnList f, double c_s) {
  const std::size_t n = common_length(e, f, "angle_filter");
  const std::size_t p = f.size();
  if (p == 0) return {std::move(e), std::move(f)};
  auto [er, fr] = reverse_columns(e, f);
  const std::vector<int32_t> kept = faa_kept(er, fr, n, c_s, 1e300, 2 /* skip length */);
  ColumnList eo, fo;
  for (std::size_t i = 0; i < p; ++i)
    if (kept[p - 1 - i]) {
      eo.push_back(std::move(e[i]));
      fo.push_back(std::move(f[i]));
    }
  return {std::move(eo), std::move(fo)};
}

Vec length_bounds(const ColumnList& f, double c_s) {
  const std::size_t m = f.size();
  Vec b(m);
  if (m == 0) return b;
  std::vector<double> fn2(m);
  for (std::size_t j = 0; j < m; ++j) fn2[j] = nrm2sq(f[j]);
  // b_1 = 1/||f_1||^2;  b_j = ( ct^2 ((ct+cs)/cs)^{2(j-2)} / ||f_1||^2
  //   + sum_{i=2}^{j-1} ct^2 (ct+cs)^{2(j-i-1)} / (||f_i||^2 cs^{2(j-i)})
  //   + 1/||f_j||^2 ) / cs^2,  ct = sqrt(1 - cs^2)   (paper Alg. 6)
  const double cs2 = c_s * c_s;
  const double ct = std::sqrt(std::max(0.0, 1.0 - cs2));
  const double ct2 = ct * ct;
  b[0] = 1.0 / fn2[0];
  for (std::size_t jj = 1; jj < m; ++jj) {
    const int j = int(jj) + 1;
    double acc = ct2 * std::pow((ct + c_s) / c_s, 2.0 * (j - 2)) / fn2[0];
    for (int i = 2; i <= j - 1; ++i)
      acc += ct2 * std::pow(ct + c_s, 2.0 * (j - i - 1)) /
             (fn2[std::size_t(i) - 1] * std::pow(c_s, 2.0 * (j - i)));
    acc += 1.0 / fn2[jj];
    b[jj] = acc / cs2;
  }
  return b;
}

std::pair<ColumnList, ColumnList> length_filter(ColumnList e, ColumnList f, double c_s,
                                                double kappa_bar) {
  const std::size_t n = common_length(e, f, "length_filter");
  const std::size_t p = f.size();
  if (p == 0) return {std::move(e), std::move(f)};
  auto [er, fr] = reverse_columns(e, f);
  const std::vector<int32_t> kept = faa_kept(er, fr, n, c_s, kappa_bar, 1 /* skip angle */);
  ColumnList eo, fo;  // a prefix of the given (newest-first) order
  for (std::size_t i = 0; i < p; ++i)
    if (kept[p - 1 - i]) {
      eo.push_back(std::move(e[i]));
      fo.push_back(std::move(f[i]));
    }
  return {std::move(eo), std::move(fo)};
}

FilteredMemory build_filtered_memory(ColumnList e, ColumnList f, const FilterParams& params) {
  const std::size_t n = common_length(e, f, "build_filtered_memory");
  FilteredMemory fm;
  const std::size_t p = f.size();
  if (p == 0) return fm;
  const std::vector<int32_t> kept = faa_kept(e, f, n, params.c_s, params.kappa_bar, 0);
  for (std::size_t j = 0; j < p; ++j)
    if (kept[j]) {
      fm.e.push_back(std::move(e[j]));
      fm.f.push_back(std::move(f[j]));
    }
  DenseMatrix fd(int(n), int(fm.f.size()));
  for (std::size_t j = 0; j < fm.f.size(); ++j)
    std::copy(fm.f[j].begin(), fm.f[j].end(), fd.data.begin() + std::ptrdiff_t(j * n));
  fm.qr = fm.f.empty() ? QRFactors{DenseMatrix(int(n), 0), DenseMatrix(0, 0)} : economy_qr(fd);
  return fm;
}

Vec filtered_aa_apply(const FilteredMemory& fm, const AAParams& params, const Vec& u,
                      const Vec& g) {
  const std::size_t n = u.size();
  if (g.size() != n) throw DimensionError("filtered_aa_apply: u and g lengths differ");
  const std::size_t p = fm.f.size();
  if (fm.e.size() != p) throw DimensionError("filtered_aa_apply: e / f column counts differ");
  for (std::size_t j = 0; j < p; ++j)
    if (fm.e[j].size() != n || fm.f[j].size() != n)
      throw DimensionError("filtered_aa_apply: column length differs from u");
  if (!params.d_hat.empty() && params.d_hat.size() != n)
    throw DimensionError("filtered_aa_apply: d_hat length mismatch");
  if (p > 0) {
    // the triangle's singularity test of back_substitute (sparse_linalg.hpp:70-72)
    const DenseMatrix& r = fm.qr.r;
    if (r.nrows != int(p) || r.ncols != int(p))
      throw DimensionError("filtered_aa_apply: R does not match the memory");
    double fro = 0.0;
    for (double x : r.data) fro += x * x;
    for (int i = 0; i < int(p); ++i)
      if (std::fabs(r.at(i, i)) <= 1e-14 * std::sqrt(fro))
        throw SingularError("back_substitute: singular triangle");
  }
  if (n == 0) return {};
  const std::vector<double> ec = pack(fm.e, n), fc = pack(fm.f, n);
  Vec out(n);
  std::vector<int32_t> kept(std::max<std::size_t>(p, 1));
  char err[512] = {0};
  check_rc(aapdhg_cuda_faa_op(workspace(n), AAPDHG_REDUCE_AUTO, int32_t(p), ec.data(), fc.data(),
                              0.2, 1e300, params.beta,
                              params.d_hat.empty() ? nullptr : params.d_hat.data(),
                              1 | 2 /* the memory is already filtered */, u.data(), g.data(),
                              out.data(), kept.data(), err, sizeof err),
           err);
  return out;
}

}  // namespace aapdhg
