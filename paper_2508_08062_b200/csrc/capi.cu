// capi.cu — extern "C" entry points of include/aapdhg_cuda.h.
// Exceptions never cross the boundary: they map onto aapdhg_status codes
// (InputError / DimensionError / UnsupportedError / SingularError /
// CUDA runtime errors) with the message copied into the caller's buffer.
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "aapdhg_cuda.h"
#include "engine.h"
#include "shard.h"

using aapdhg_b200::CudaError;
using aapdhg_b200::Problem;
using aapdhg_b200::ShardGroup;
using aapdhg_b200::StatusError;

struct aapdhg_handle {
  Problem* prob;      // whole-LP handle
  ShardGroup* group;  // sharded handle (prob == nullptr)
};

namespace {

void put_err(char* err, size_t errlen, const char* msg) {
  if (!err || errlen == 0) return;
  std::strncpy(err, msg, errlen - 1);
  err[errlen - 1] = '\0';
}

template <class F>
int guard(char* err, size_t errlen, F&& f) {
  try {
    return f();
  } catch (const StatusError& e) {
    put_err(err, errlen, e.what());
    return e.code;
  } catch (const CudaError& e) {
    put_err(err, errlen, e.what());
    return AAPDHG_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    put_err(err, errlen, "host allocation failed");
    return AAPDHG_ERR_INTERNAL;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return AAPDHG_ERR_INTERNAL;
  }
}

int need(const void* p, const char* what, char* err, size_t errlen) {
  if (p) return AAPDHG_OK;
  put_err(err, errlen, what);
  return AAPDHG_ERR_INPUT;
}

// single-op entry points work on whole-LP handles only
int whole(const aapdhg_handle* h, const char* what, char* err, size_t errlen) {
  if (!h || !h->group) return AAPDHG_OK;
  put_err(err, errlen, (std::string(what) + ": not available on a sharded handle").c_str());
  return AAPDHG_ERR_UNSUPPORTED;
}

}  // namespace

extern "C" {

int aapdhg_cuda_abi_version(void) { return AAPDHG_ABI_VERSION; }

int aapdhg_cuda_device_info(char* out, size_t outlen) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return AAPDHG_ERR_CUDA;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return AAPDHG_ERR_CUDA;
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s, sm_%d%d, %d SMs", p.name, p.major, p.minor,
                p.multiProcessorCount);
  put_err(out, outlen, buf);
  return AAPDHG_OK;
}

int aapdhg_cuda_problem_create(const aapdhg_problem_view* prob, int device,
                               aapdhg_handle** out, char* err, size_t errlen) {
  if (int rc = need(out, "problem_create: null out", err, errlen)) return rc;
  *out = nullptr;
  return guard(err, errlen, [&] {
    auto* h = new aapdhg_handle{new Problem(prob, device), nullptr};
    *out = h;
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_problem_create_dist(const aapdhg_problem_view* prob, int device,
                                    const aapdhg_dist_view* dist, aapdhg_handle** out,
                                    char* err, size_t errlen) {
  if (int rc = need(out, "problem_create_dist: null out", err, errlen)) return rc;
  *out = nullptr;
  return guard(err, errlen, [&] {
    auto* h = new aapdhg_handle{nullptr, new ShardGroup(prob, device, dist)};
    *out = h;
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_nccl_id(uint8_t* out, size_t len, char* err, size_t errlen) {
  if (int rc = need(out, "nccl_id: null out", err, errlen)) return rc;
  return guard(err, errlen, [&] {
    aapdhg_b200::nccl_unique_id(out, len);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_balance_partition(int32_t workers, int32_t nslices, const int32_t* cur_starts,
                                  const double* phase_ns, const int32_t* sm,
                                  const int32_t* slice_work, int32_t* new_starts) {
  if (workers <= 0 || nslices < 0 || !cur_starts || !phase_ns || !sm || !slice_work ||
      !new_starts)
    return AAPDHG_ERR_INPUT;
  try {
    std::vector<int32_t> cur(cur_starts, cur_starts + workers + 1);
    std::vector<double> t(phase_ns, phase_ns + workers);
    std::vector<int> s(sm, sm + workers);
    std::vector<int32_t> wt(slice_work, slice_work + nslices);
    const std::vector<int32_t> out = aapdhg_b200::rebalance_partition(cur, t, s, wt);
    for (int32_t w = 0; w <= workers; ++w) new_starts[w] = out[size_t(w)];
    return AAPDHG_OK;
  } catch (...) {
    return AAPDHG_ERR_INPUT;
  }
}

int aapdhg_cuda_partition(const aapdhg_csr_view* k, int32_t world, int32_t* row_bounds,
                          int32_t* col_bounds) {
  if (!k || !row_bounds || !col_bounds || world < 1) return AAPDHG_ERR_INPUT;
  if (world > k->nrows || world > k->ncols) return AAPDHG_ERR_UNSUPPORTED;
  return guard(nullptr, 0, [&] {
    const aapdhg_b200::Partition p = aapdhg_b200::plan_partition(*k, world);
    for (int r = 0; r <= world; ++r) {
      row_bounds[r] = p.rows[r];
      col_bounds[r] = p.cols[r];
    }
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_problem_destroy(aapdhg_handle* h) {
  if (!h) return AAPDHG_OK;
  delete h->prob;
  delete h->group;
  delete h;
  return AAPDHG_OK;
}

int aapdhg_cuda_problem_dims(const aapdhg_handle* h, int32_t* n, int32_t* m1, int32_t* m2,
                             int64_t* nnz) {
  if (!h) return AAPDHG_ERR_INPUT;
  if (h->group) {
    if (n) *n = h->group->n();
    if (m1) *m1 = h->group->m1();
    if (m2) *m2 = h->group->m() - h->group->m1();
    if (nnz) *nnz = h->group->nnz();
    return AAPDHG_OK;
  }
  if (n) *n = h->prob->n();
  if (m1) *m1 = h->prob->m1();
  if (m2) *m2 = h->prob->m() - h->prob->m1();
  if (nnz) *nnz = h->prob->nnz();
  return AAPDHG_OK;
}

int aapdhg_cuda_solve(aapdhg_handle* h, const aapdhg_solve_params* prm, const double* x0,
                      const double* y0, aapdhg_solve_result* res, double* x_out,
                      double* y_out, double* lambda_out, aapdhg_record_sink sink, void* ctx,
                      char* err, size_t errlen) {
  if (int rc = need(h, "solve: null handle", err, errlen)) return rc;
  if (int rc = need(prm, "solve: null params", err, errlen)) return rc;
  if (int rc = need(res, "solve: null result", err, errlen)) return rc;
  return guard(err, errlen, [&] {
    if (h->group) h->group->solve(prm, x0, y0, res, x_out, y_out, lambda_out, sink, ctx);
    else h->prob->solve(prm, x0, y0, res, x_out, y_out, lambda_out, sink, ctx);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_select_step_sizes(aapdhg_handle* h, const aapdhg_solve_params* prm,
                                  double* tau, double* sigma, char* err, size_t errlen) {
  if (int rc = need(h && prm && tau && sigma ? h : nullptr, "select_step_sizes: null argument",
                    err, errlen))
    return rc;
  return guard(err, errlen, [&] {
    if (h->group) h->group->select_step_sizes(prm, tau, sigma);
    else h->prob->select_step_sizes(prm, tau, sigma);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_power_norm(aapdhg_handle* h, int32_t max_iters, double rel_tol, uint64_t seed,
                           int32_t reduction, double* out, int32_t* rounds, char* err,
                           size_t errlen) {
  if (int rc = whole(h, "power_norm", err, errlen)) return rc;
  if (int rc = need(h && out ? h : nullptr, "power_norm: null argument", err, errlen)) return rc;
  return guard(err, errlen, [&] {
    int r = 0;
    const bool serial = reduction == AAPDHG_REDUCE_SERIAL ||
                        (reduction == AAPDHG_REDUCE_AUTO &&
                         int64_t(h->prob->n()) + h->prob->m() <= 65536);
    *out = h->prob->power_norm(max_iters, rel_tol, seed, serial, &r);
    if (rounds) *rounds = r;
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_matvec(aapdhg_handle* h, const double* x, double* out, char* err,
                       size_t errlen) {
  if (int rc = whole(h, "matvec", err, errlen)) return rc;
  if (int rc = need(h && (out || h->prob->m() == 0) && (x || h->prob->n() == 0) ? h : nullptr,
                    "matvec: null argument",
                    err, errlen))
    return rc;
  return guard(err, errlen, [&] {
    h->prob->matvec(x, out);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_matvec_transpose(aapdhg_handle* h, const double* y, double* out, char* err,
                                 size_t errlen) {
  if (int rc = whole(h, "matvec_transpose", err, errlen)) return rc;
  if (int rc = need(h && (out || h->prob->n() == 0) && (y || h->prob->m() == 0) ? h : nullptr,
                    "matvec_transpose: null argument", err, errlen))
    return rc;
  return guard(err, errlen, [&] {
    h->prob->matvec_transpose(y, out);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_pdhg_step(aapdhg_handle* h, double tau, double sigma, const double* x,
                          const double* y, double* xn, double* yn, char* err, size_t errlen) {
  if (int rc = whole(h, "pdhg_step", err, errlen)) return rc;
  if (int rc = need(h && (xn || h->prob->n() == 0) && (yn || h->prob->m() == 0) ? h : nullptr,
                    "pdhg_step: null argument", err, errlen))
    return rc;
  return guard(err, errlen, [&] {
    h->prob->pdhg_step(tau, sigma, x, y, xn, yn);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_kkt_metrics(aapdhg_handle* h, int32_t reduction, const double* x,
                            const double* y, double* kkt, double* lambda, char* err,
                            size_t errlen) {
  if (int rc = whole(h, "kkt_metrics", err, errlen)) return rc;
  if (int rc = need(h && kkt ? h : nullptr, "kkt_metrics: null argument", err, errlen)) return rc;
  return guard(err, errlen, [&] {
    h->prob->kkt_metrics(reduction, x, y, kkt, lambda);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_aa_apply(aapdhg_handle* h, int32_t reduction, int32_t p, const double* du_cols,
                         const double* dg_cols, double beta, const double* d_hat, double eta,
                         const double* u, const double* g, double* out, char* err,
                         size_t errlen) {
  if (int rc = whole(h, "aa_apply", err, errlen)) return rc;
  if (int rc = need(h && u && g && out ? h : nullptr, "aa_apply: null argument", err, errlen))
    return rc;
  return guard(err, errlen, [&] {
    const int rc = h->prob->aa_apply(reduction, false, p, du_cols, dg_cols, beta, d_hat, eta,
                                     0.2, 1e9, u, g, out, nullptr);
    if (rc == AAPDHG_ERR_SINGULAR) put_err(err, errlen, "aa: normal equations not positive definite");
    return rc;
  });
}

int aapdhg_cuda_filtered_aa_apply(aapdhg_handle* h, int32_t reduction, int32_t p,
                                  const double* e_cols, const double* f_cols, double c_s,
                                  double kappa_bar, double beta, const double* d_hat,
                                  const double* u, const double* g, double* out,
                                  int32_t* kept, char* err, size_t errlen) {
  if (int rc = whole(h, "filtered_aa_apply", err, errlen)) return rc;
  if (int rc = need(h && u && g && out ? h : nullptr, "filtered_aa_apply: null argument", err,
                    errlen))
    return rc;
  return guard(err, errlen, [&] {
    const int rc = h->prob->aa_apply(reduction, true, p, e_cols, f_cols, beta, d_hat, 0.0, c_s,
                                     kappa_bar, u, g, out, kept);
    if (rc == AAPDHG_ERR_SINGULAR) put_err(err, errlen, "filtered memory: singular");
    return rc;
  });
}

int aapdhg_cuda_workspace_create(int32_t device, int64_t n, aapdhg_handle** out, char* err,
                                 size_t errlen) {
  if (int rc = need(out, "workspace_create: null out", err, errlen)) return rc;
  *out = nullptr;
  if (n < 1 || n > (int64_t(1) << 31)) {
    put_err(err, errlen, "workspace_create: vector length out of range");
    return AAPDHG_ERR_DIMENSION;
  }
  return guard(err, errlen, [&] {
    // a 1 x (n-1) LP with one unit entry: the per-op entries only use its
    // n-vectors and history buffers
    const int nc = int(n - 1);
    int32_t rp[2] = {0, nc > 0 ? 1 : 0};
    int32_t ci[1] = {0};
    double v[1] = {1.0};
    std::vector<double> zc(size_t(std::max(nc, 1)), 0.0), inf(size_t(std::max(nc, 1)), 1.0 / 0.0);
    double q[1] = {1.0};
    aapdhg_problem_view view{};
    view.k = aapdhg_csr_view{1, nc, int64_t(rp[1]), rp, ci, v};
    view.m1 = 0;
    view.c = zc.data();
    view.q = q;
    view.l = zc.data();
    view.u = inf.data();
    auto* h = new aapdhg_handle{new Problem(&view, device), nullptr};
    *out = h;
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_faa_op(aapdhg_handle* h, int32_t reduction, int32_t p, const double* e_cols,
                       const double* f_cols, double c_s, double kappa_bar, double beta,
                       const double* d_hat, int32_t skip, const double* u, const double* g,
                       double* out, int32_t* kept, char* err, size_t errlen) {
  if (int rc = whole(h, "faa_op", err, errlen)) return rc;
  if (int rc = need(h && (f_cols || p == 0) && (!out || (u && g)) ? h : nullptr,
                    "faa_op: null argument", err, errlen))
    return rc;
  return guard(err, errlen, [&] {
    const int rc = h->prob->aa_op(reduction, true, p, e_cols, f_cols, beta, d_hat, 0.0, c_s,
                                  kappa_bar, skip, u, g, out, kept, nullptr, nullptr);
    if (rc == AAPDHG_ERR_SINGULAR) put_err(err, errlen, "filtered memory: singular");
    return rc;
  });
}

int aapdhg_cuda_economy_qr(aapdhg_handle* h, int32_t reduction, int32_t p, const double* f_cols,
                           double* q_out, double* r_out, char* err, size_t errlen) {
  if (int rc = whole(h, "economy_qr", err, errlen)) return rc;
  if (int rc = need(h && f_cols && q_out && r_out ? h : nullptr, "economy_qr: null argument", err,
                    errlen))
    return rc;
  return guard(err, errlen, [&] {
    const int rc = h->prob->aa_op(reduction, true, p, nullptr, f_cols, 1.0, nullptr, 0.0, 0.2,
                                  1e300, aapdhg_b200::kFaaSkipAngle | aapdhg_b200::kFaaSkipLength,
                                  nullptr, nullptr, nullptr, nullptr, r_out, q_out);
    if (rc == AAPDHG_ERR_SINGULAR) put_err(err, errlen, "economy_qr: rank-deficient columns");
    return rc;
  });
}

int aapdhg_cuda_csr_from_triplets(int32_t device, int32_t nrows_in, int32_t nrows_out,
                                  int32_t ncols, int64_t count, const aapdhg_triplet* triplets,
                                  const int32_t* row_map, const uint8_t* row_neg,
                                  int32_t* row_ptr, int32_t* col_idx, double* vals, int64_t* nnz,
                                  char* err, size_t errlen) {
  if (int rc = need(row_ptr && nnz && (count == 0 || (triplets && col_idx && vals)) ? row_ptr
                                                                                    : nullptr,
                    "csr_from_triplets: null argument", err, errlen))
    return rc;
  return guard(err, errlen, [&] {
    *nnz = aapdhg_b200::csr_from_triplets(device, nrows_in, nrows_out, ncols, count, triplets,
                                          row_map, row_neg, row_ptr, col_idx, vals);
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_set_stream(aapdhg_handle* h, void* stream) {
  if (!h) return AAPDHG_ERR_INPUT;
  return guard(nullptr, 0, [&] {
    if (h->group) h->group->set_stream(static_cast<cudaStream_t>(stream));
    else h->prob->set_stream(static_cast<cudaStream_t>(stream));
    return AAPDHG_OK;
  });
}

int aapdhg_cuda_set_profiling(aapdhg_handle* h, int32_t enable) {
  if (!h) return AAPDHG_ERR_INPUT;
  if (h->group) return enable ? AAPDHG_ERR_UNSUPPORTED : AAPDHG_OK;
  h->prob->set_profiling(enable != 0);
  return AAPDHG_OK;
}

int aapdhg_cuda_kernel_times(aapdhg_handle* h, char* names, size_t names_len, double* ms,
                             uint64_t* launches, int32_t cap, int32_t* count) {
  if (!h) return AAPDHG_ERR_INPUT;
  if (h->group) {
    if (count) *count = 0;
    if (names && names_len) names[0] = '\0';
    return AAPDHG_OK;
  }
  const auto& st = h->prob->kernel_stats();
  std::string all;
  int k = 0;
  for (const auto& kv : st) {
    if (k < cap) {
      // eager launches run every kernel of an iteration, predicated off on
      // the device when it has nothing to do (no AA attempt, past the end):
      // launches under 30% of the kernel's longest are such no-ops
      float mx = 0.f;
      for (float v : kv.second.each) mx = v > mx ? v : mx;
      double tot = 0.0;
      uint64_t n = 0;
      for (float v : kv.second.each)
        if (v >= 0.3f * mx) {
          tot += v;
          ++n;
        }
      if (ms) ms[k] = tot;
      if (launches) launches[k] = n;
      all += kv.first;
      all += '\n';
    }
    ++k;
  }
  if (names && names_len) put_err(names, names_len, all.c_str());
  if (count) *count = k;
  return AAPDHG_OK;
}

int aapdhg_cuda_last_plain_loop(aapdhg_handle* h, uint64_t* iterations, double* seconds,
                                uint64_t* launches) {
  if (!h || h->group) return AAPDHG_ERR_INPUT;
  uint64_t it = 0, la = 0;
  double sec = 0.0;
  h->prob->last_plain_stats(&it, &sec, &la);
  if (iterations) *iterations = it;
  if (seconds) *seconds = sec;
  if (launches) *launches = la;
  return AAPDHG_OK;
}

int aapdhg_cuda_last_launch_count(aapdhg_handle* h, uint64_t* launches,
                                  uint64_t* loop_iterations) {
  if (!h) return AAPDHG_ERR_INPUT;
  if (launches) *launches = h->group ? h->group->last_launches() : h->prob->last_launches();
  if (loop_iterations)
    *loop_iterations = h->group ? h->group->last_loop_iters() : h->prob->last_loop_iters();
  return AAPDHG_OK;
}

}  // extern "C"
