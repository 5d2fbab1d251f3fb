// engine.cu — host orchestration of the sm_100a AA-PDHG / FAA-PDHG solver.
//
// The reference solve() (proj/src/solver.cpp:125-253) runs entirely on the
// device: one iteration = the kernel sequence in launch_iteration(), whose
// branches (termination, safeguard, AA success / SingularError fallback)
// are predicates in device memory, so iterations are replayed from a CUDA
// graph without any host round trip. The host only polls the small
// DevState mirror (pinned) between graph batches to stream trajectory
// records out and to stop.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <random>
#include <thread>

#include "engine.h"
#include "aa.cuh"
#include "pipeline.cuh"
#include "shard.cuh"

namespace aapdhg_b200 {

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

constexpr uint64_t kMaxBatch = 4096;  // iterations per graph launch (max)
constexpr uint64_t kRecCap = 1 << 16;  // device record ring
constexpr uint64_t kPowTabMax = 1 << 22;
constexpr int kPowerBatch = 8;

// tuning overrides (experiments, INTEGRATION.md "Environment switches")
int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

int num_items_host(int p, int method) {
  return p * (p + 1) / 2 + p + (method == AAPDHG_METHOD_FAA ? p : 0);
}

// host <-> device copies (memory.cu): pinned host buffers are DMA'd
// directly, pageable ones staged through pinned chunks; d2h returns with the
// data on the host
void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  host_to_device(dst, src, bytes, s);
}
void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  device_to_host(dst, src, bytes, s);
}

int grid_for(int64_t n, int per_block = kThreads, int cap = 148 * 8) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace

// The streams of the handle this thread is working for (Problem::enter):
// a growing buffer waits for them only, never for the whole device — a
// device-wide synchronize would break another thread's graph capture
// (concurrent handles: solve_sweep).
thread_local cudaStream_t g_tls_sync[2] = {nullptr, nullptr};

// Device buffers come from the per-device block cache (memory.cu); a block
// returns to it when its owner is done with it (owners synchronise first).
DevBuf::~DevBuf() {
  if (p) cache_free(p, bytes);
}

void DevBuf::reserve(size_t b) {
  if (b == 0) b = 16;
  if (p && b <= bytes) return;
  if (p) {  // growth: work in flight may still read the old block
    if (g_tls_sync[0] || g_tls_sync[1]) {
      for (cudaStream_t st : g_tls_sync)
        if (st) AAPDHG_CUDA(cudaStreamSynchronize(st));
    } else {
      AAPDHG_CUDA(cudaDeviceSynchronize());
    }
    cache_free(p, bytes);
  }
  p = nullptr;
  bytes = 0;
  p = cache_alloc(b);
  bytes = b;
}

struct SolveSetup {
  IterBufs B;
  DotBufs D;
  SolveScratch W;
  const DevParams* P;
  DevState* S;
  bool serial, push;
  bool ring = false;     // AA-PDHG's ring history (DevParams::ring)
  int method, cap, nblk1, nblk2, ndot_blk, items_max;
  bool persist = false;  // plain iterations in k_plain_loop (graph replay only)
  int pgrid = 0;         // workers + the control CTA
  CsrDev pk1, pk2;       // the K' / K layouts on <= pgrid - 1 worker CTAs
  GridBar* gb = nullptr;
  int np1 = 0, np2 = 0;  // partial rows: CTAs, or slices (calibrated partition)
  bool split = false;    // L2-blocked TREE: all blocks as passes, then k_dual_epi / k_primal_epi
  int epi = 0;           // their grid (grid-stride rows)
  bool epi_pipe = false; // k_dual_epi per K column block, K's passes beside it (side_)
  unsigned long long* bal = nullptr;  // per-CTA phase times (calibrating)
};

// ---- k_plain_loop partition calibration ------------------------------------
// The worker CTAs of the persistent grid sit on the same SMs launch after
// launch, and some SMs gather measurably slower than others (up to ~20% on
// configs[1]: profiles/exp_sm_balance.py). Each barrier waits for the slowest
// SM, so the slices are shared out per SM in proportion to the rate each SM
// achieved in earlier launches (slices per microsecond of its slowest CTA),
// evenly over the SM's CTAs (<= kWarps each). The partials are per slice
// (CsrDev::sl_start), so every partition gives the same bits. The partition
// is kept per device and layout shape, so a new handle of the same LP starts
// calibrated; it is refined after each of the first AAPDHG_BALANCE_ROUNDS
// (default 3) solves that ran at least kBalMinIters plain iterations.
namespace {
constexpr uint64_t kBalMinIters = 16;
struct BalEntry {
  std::vector<int32_t> s1, s2;  // slice starts per worker CTA (workers + 1)
  std::vector<int32_t> w1, w2;  // slice work (per-lane lengths) of K' / K
  int rounds = 0;
};
std::mutex g_bal_mu;
std::map<std::string, BalEntry> g_bal;

std::string bal_key(int device, const CsrDev& a, const CsrDev& b, int workers) {
  char k[160];
  std::snprintf(k, sizeof k, "%d/%d/%d/%d/%d/%d/%d/%lld/%lld", device, workers, a.nslices, a.sf,
                b.nslices, b.sf, a.nrows, (long long)a.nnz, (long long)b.nnz);
  return k;
}

std::vector<int32_t> proportional_starts(int ns, int workers) {
  std::vector<int32_t> st(static_cast<size_t>(workers) + 1);
  for (int w = 0; w <= workers; ++w) st[size_t(w)] = int32_t(int64_t(w) * ns / workers);
  return st;
}

// new starts from one phase's measurements: t[w] mean phase time of worker w,
// sm[w] its SM, cur the current starts, wt[s] the work of slice s (its
// per-lane length). Each SM gets work in proportion to the rate it showed
// (work per microsecond of its slowest CTA), split evenly over its CTAs; the
// slices go to the CTAs in order, <= kWarps each.
}  // namespace

std::vector<int32_t> rebalance_partition(const std::vector<int32_t>& cur, const std::vector<double>& t,
                               const std::vector<int>& sm, const std::vector<int32_t>& wt) {
  const int W = int(cur.size()) - 1;
  const int ns = int(wt.size());
  int nsm = 0;
  for (int w = 0; w < W; ++w) nsm = std::max(nsm, sm[size_t(w)] + 1);
  std::vector<double> work(static_cast<size_t>(nsm), 0.0), tmax(static_cast<size_t>(nsm), 0.0);
  std::vector<int> nct(static_cast<size_t>(nsm), 0);
  for (int w = 0; w < W; ++w) {
    const int q = sm[size_t(w)];
    for (int32_t x = cur[size_t(w)]; x < cur[size_t(w) + 1]; ++x) work[size_t(q)] += wt[size_t(x)];
    tmax[size_t(q)] = std::max(tmax[size_t(q)], t[size_t(w)]);
    ++nct[size_t(q)];
  }
  std::vector<double> rate(static_cast<size_t>(nsm), 0.0);
  double rmean = 0.0;
  int nr = 0;
  for (int q = 0; q < nsm; ++q)
    if (work[size_t(q)] > 0 && tmax[size_t(q)] > 0) {
      rate[size_t(q)] = work[size_t(q)] / tmax[size_t(q)];
      rmean += rate[size_t(q)];
      ++nr;
    }
  if (nr == 0) return cur;
  rmean /= nr;
  double rsum = 0.0, wtot = 0.0;
  for (int q = 0; q < nsm; ++q) {
    if (nct[size_t(q)] == 0) rate[size_t(q)] = 0.0;
    else if (rate[size_t(q)] == 0.0) rate[size_t(q)] = rmean;  // (idle last time)
    rsum += rate[size_t(q)];
  }
  for (int x = 0; x < ns; ++x) wtot += wt[size_t(x)];
  // cumulative work targets in CTA order; a slice goes to the CTA whose
  // target range holds its midpoint
  std::vector<int32_t> st(static_cast<size_t>(W) + 1, 0);
  double target = 0.0, cum = 0.0;
  int x = 0;
  for (int w = 0; w < W; ++w) {
    const int q = sm[size_t(w)];
    target += wtot * rate[size_t(q)] / rsum / nct[size_t(q)];
    int took = 0;
    while (x < ns && took < kWarps && (w == W - 1 || cum + 0.5 * wt[size_t(x)] <= target)) {
      cum += wt[size_t(x)];
      ++x;
      ++took;
    }
    st[size_t(w) + 1] = x;
  }
  // slices the caps left over: move the boundaries down from the end (each
  // CTA still <= kWarps slices)
  st[size_t(W)] = ns;
  for (int w = W - 1; w >= 0; --w)
    st[size_t(w)] = std::min(st[size_t(w) + 1], std::max(st[size_t(w)], st[size_t(w) + 1] - kWarps));
  if (st[0] != 0) return cur;  // (infeasible: keep the partition)
  return st;
}


// Before a persistent launch: the partition (cached for this device and
// layout shape, else proportional) into bal_start1_ / bal_start2_; *measure:
// whether this solve records phase times (bal_stats_).
void Problem::bal_setup(const CsrDev& a, const CsrDev& b, int workers, bool* measure) {
  const std::string key = bal_key(device_, a, b, workers);
  BalEntry e;
  {
    std::lock_guard<std::mutex> g(g_bal_mu);
    auto it = g_bal.find(key);
    if (it != g_bal.end()) e = it->second;
  }
  if (e.s1.empty()) {
    e.s1 = proportional_starts(a.nslices, workers);
    e.s2 = proportional_starts(b.nslices, workers);
    e.w1.resize(size_t(a.nslices));
    e.w2.resize(size_t(b.nslices));
    d2h(e.w1.data(), a.sl_len, sizeof(int32_t) * e.w1.size(), stream_);
    d2h(e.w2.data(), b.sl_len, sizeof(int32_t) * e.w2.size(), stream_);
    sync();
    std::lock_guard<std::mutex> g(g_bal_mu);
    g_bal[key] = e;
  }
  bal_start1_.reserve(sizeof(int32_t) * (size_t(workers) + 1));
  bal_start2_.reserve(sizeof(int32_t) * (size_t(workers) + 1));
  h2d(bal_start1_.p, e.s1.data(), sizeof(int32_t) * e.s1.size(), stream_);
  h2d(bal_start2_.p, e.s2.data(), sizeof(int32_t) * e.s2.size(), stream_);
  *measure = e.rounds < env_int("AAPDHG_BALANCE_ROUNDS", 3);
  if (*measure) {
    bal_stats_.reserve(sizeof(unsigned long long) * 4 * size_t(workers));
    AAPDHG_CUDA(cudaMemsetAsync(bal_stats_.p, 0, bal_stats_.bytes, stream_));
  }
}

// After a measured solve: the per-CTA phase times -> a new partition for the
// next launch on this device and layout shape.
void Problem::bal_collect(const CsrDev& a, const CsrDev& b, int workers) {
  std::vector<unsigned long long> st(4 * static_cast<size_t>(workers));
  d2h(st.data(), bal_stats_.p, sizeof(unsigned long long) * st.size(), stream_);
  sync();
  std::vector<double> t1(static_cast<size_t>(workers)), t2(static_cast<size_t>(workers));
  std::vector<int> sm(static_cast<size_t>(workers));
  for (int w = 0; w < workers; ++w) {
    const unsigned long long c = st[4 * size_t(w) + 2];
    if (c < kBalMinIters) return;  // too few iterations: keep the partition
    t1[size_t(w)] = double(st[4 * size_t(w)]) / double(c);
    t2[size_t(w)] = double(st[4 * size_t(w) + 1]) / double(c);
    sm[size_t(w)] = int(st[4 * size_t(w) + 3]);
  }
  const std::string key = bal_key(device_, a, b, workers);
  std::lock_guard<std::mutex> g(g_bal_mu);
  auto it = g_bal.find(key);
  if (it == g_bal.end()) return;
  BalEntry& e = it->second;
  const auto n1 = rebalance_partition(e.s1, t1, sm, e.w1),
             n2 = rebalance_partition(e.s2, t2, sm, e.w2);
  if (env_int("AAPDHG_VERBOSE", 0)) {
    auto moved = [](const std::vector<int32_t>& a, const std::vector<int32_t>& b) {
      int c = 0;
      for (size_t i = 0; i < a.size(); ++i) c += a[i] != b[i];
      return c;
    };
    double m1 = 0, m2 = 0, a1 = 0, a2 = 0;
    for (int w = 0; w < workers; ++w) {
      m1 = std::max(m1, t1[size_t(w)]);
      m2 = std::max(m2, t2[size_t(w)]);
      a1 += t1[size_t(w)] / workers;
      a2 += t2[size_t(w)] / workers;
    }
    std::fprintf(stderr, "aapdhg: balance round %d: K1 mean %.2f max %.2f us, K2 mean %.2f max "
                 "%.2f us; boundaries moved %d / %d\n", e.rounds, a1 / 1e3, m1 / 1e3, a2 / 1e3,
                 m2 / 1e3, moved(n1, e.s1), moved(n2, e.s2));
  }
  e.s1 = n1;
  e.s2 = n2;
  ++e.rounds;
}

// k_plain_loop spins on grid barriers, so it must never share the GPU with a
// second persistent grid (two partially resident grids would wait on each
// other): one persistent solve per device at a time, the others take the
// per-kernel graph.
static std::atomic<int> g_persist_busy[64];
struct PersistLock {
  int dev = -1;
  bool try_lock(int d) {
    if (d < 0 || d >= 64) return false;
    int z = 0;
    if (!g_persist_busy[d].compare_exchange_strong(z, 1)) return false;
    dev = d;
    return true;
  }
  ~PersistLock() {
    if (dev >= 0) g_persist_busy[dev].store(0);
  }
};

// SELL-32 slices of the short rows with split factor sf (see CsrDev):
// slice = 32 / sf rows; element k of the slice's row rho sits at
// sl_ptr + 32 (k / sf) + rho sf + (k % sf).
// Uploads one CSR with its two sliced layouts: `ser` (sf = 1, CSR-ordered
// row sums for the SERIAL mode) and `tree` (sf chosen so the slices fill
// ~48 warps on every SM; aliases `ser` when sf = 1).
// (rp / ci / v may be host or device memory; nnz < 0: rp[nrows], host rp)
void Problem::upload_csr(const int32_t* rp, const int32_t* ci, const double* v, int nrows,
                         int ncols, CsrStore& st, CsrDev& ser, CsrDev& tree, int64_t nnz_in) {
  const int64_t nnz = nnz_in >= 0 ? nnz_in : rp[nrows];
  st.rp.reserve(sizeof(int32_t) * (size_t(nrows) + 1));
  st.ci.reserve(sizeof(int32_t) * size_t(std::max<int64_t>(nnz, 1)));
  st.v.reserve(sizeof(double) * size_t(std::max<int64_t>(nnz, 1)));
  h2d(st.rp.p, rp, sizeof(int32_t) * (size_t(nrows) + 1), stream_);
  h2d(st.ci.p, ci, sizeof(int32_t) * size_t(nnz), stream_);
  h2d(st.v.p, v, sizeof(double) * size_t(nnz), stream_);
  device_validate(st, nrows, ncols, nnz);
  finish_csr(nrows, ncols, nnz, st, ser, tree);  // layouts built on the device (ingest.cu)
}

// L2 column blocking (TREE mode only). A matrix whose gathered vector is
// larger than the L2 budget (AAPDHG_L2_BLOCK_KB, default 80 MB per block:
// configs[4]'s x in 4 passes, y in 2 — fewer passes beat the extra gather
// misses of a block above L2's clean ~48 MB, profiles/r02/cfg4_l2_persist.txt;
// blocking starts above AAPDHG_L2_BLOCK_MIN_KB, default 64 MB) is split into column blocks; each block's
// rows are the same rows restricted to its columns (CSR order kept), so a
// pass gathers only from an L2-resident slice of the vector instead of one
// DRAM sector per nonzero. Row sums become (((b0 + b1) + b2) + ...) — fixed
// order, deterministic, not the CPU's association.
void Problem::build_blocks(const CsrStore& src, int nrows, int ncols, Blocked& out,
                           const char* kb_env) {
  const int64_t kb = env_int(kb_env, env_int("AAPDHG_L2_BLOCK_KB", 80 << 10));  // per block
  const int64_t min_kb = env_int("AAPDHG_L2_BLOCK_MIN_KB", 64 << 10);  // start above
  const int64_t vec_bytes = int64_t(ncols) * 8;
  if (kb <= 0 || nrows == 0 || vec_bytes <= (min_kb << 10)) return;
  const int64_t per = std::max<int64_t>((kb << 10) / 8, 1);
  const int nb = int((int64_t(ncols) + per - 1) / per);
  if (nb < 2) return;
  const int64_t W = (int64_t(ncols) + nb - 1) / nb;
  out.width = W;
  building_blocks_ = true;
  for (int b = 0; b < nb; ++b) {
    out.store.emplace_back(new CsrStore());
    int64_t nnz_b = 0;
    device_block(src, nrows, b * W, std::min<int64_t>(int64_t(ncols), (b + 1) * W),
                 *out.store.back(), &nnz_b);
    CsrDev ser, tree;
    finish_csr(nrows, ncols, nnz_b, *out.store.back(), ser, tree);
    out.blk.push_back(tree);
  }
  building_blocks_ = false;
  out.partial.reserve(sizeof(double) * size_t(nrows));
}

int Problem::launch_blocked_passes(cudaStream_t s, const Blocked& bk, const VecRef& x,
                                   const DevState* S, int pred_aa, const int32_t* stop,
                                   bool all) {
  int nodes = 0;
  for (int b = 0; b + (all ? 0 : 1) < bk.nb(); ++b) {
    prof_begin(s, "k_spmv_pass");
    k_spmv_pass<<<bk.blk[b].grid(), kThreads, 0, s>>>(bk.blk[b], x, bk.partial.as<double>(),
                                                     b == 0 ? 1 : pass_prefetch_, S, pred_aa, stop);
    prof_end(s);
    AAPDHG_CUDA(cudaGetLastError());
    ++nodes;
  }
  return nodes;
}

// out = A x (CSR-ordered row sums).
int Problem::spmv(cudaStream_t s, const CsrDev& A, const VecRef& x, const RowsumArgs& o,
                  bool serial, const DevState* S, int pred, const int32_t* stop) {
  if (A.grid() == 0) return 0;
  RowsumArgs r = o;
  r.pred_aa_ok = pred;
  r.stop = stop;
  prof_begin(s, "k_spmv");
  if (serial) k_spmv<true><<<A.grid(), kThreads, 0, s>>>(A, x, r, S);
  else k_spmv<false><<<A.grid(), kThreads, 0, s>>>(A, x, r, S);
  prof_end(s);
  AAPDHG_CUDA(cudaGetLastError());
  return 1;
}

// out = K x (transpose: K'y), through the L2 column blocks when the TREE
// layout has them (the passes, then the last block on their partial sums)
int Problem::spmv_any(cudaStream_t s, bool transpose, const VecRef& x, RowsumArgs r, bool serial,
                      const DevState* S, const int32_t* stop) {
  const Blocked& bk = transpose ? ktb_ : kb_;
  if (!serial && bk.nb() > 1) {
    const int nodes = launch_blocked_passes(s, bk, x, S, 0, stop);
    r.rinit = bk.partial.as<double>();
    return nodes + spmv(s, bk.blk.back(), x, r, false, S, 0, stop);
  }
  return spmv(s, transpose ? KTm(serial) : Km(serial), x, r, serial, S, 0, stop);
}

static VecRef vref(const double* p) { return VecRef{p, nullptr, 0, 0, 0}; }
static RowsumArgs rout(double* out) {
  RowsumArgs r{};
  r.out = out;
  return r;
}

// k_aa_solve's dynamic shared memory: Gram, work (R) and R's low parts (FAA)
size_t Problem::aa_smem(int cap) { return sizeof(double) * 3 * size_t(cap) * size_t(cap); }


// ---------------------------------------------------------------------------
// O(1) checks on the host; the O(nnz) ones run on the device after the
// upload (Problem::device_validate) or, for the sharded path that slices
// the LP on the host, in validate_problem_deep.
void validate_problem_header(const aapdhg_problem_view* v) {
  if (!v) throw StatusError(AAPDHG_ERR_INPUT, "problem_create: null problem");
  const aapdhg_csr_view& k = v->k;
  if (k.nrows < 0 || k.ncols < 0 || k.nnz < 0)
    throw StatusError(AAPDHG_ERR_DIMENSION, "problem_create: negative dimension");
  if (v->m1 < 0 || v->m1 > k.nrows)
    throw StatusError(AAPDHG_ERR_DIMENSION, "problem_create: bad m1");
  if (!k.row_ptr || (k.nnz > 0 && (!k.col_idx || !k.vals)))
    throw StatusError(AAPDHG_ERR_INPUT, "problem_create: null CSR array");
  if (k.row_ptr[0] != 0 || int64_t(k.row_ptr[k.nrows]) != k.nnz)
    throw StatusError(AAPDHG_ERR_DIMENSION, "problem_create: row_ptr does not span nnz");
  if (k.ncols > 0 && (!v->c || !v->l || !v->u))
    throw StatusError(AAPDHG_ERR_INPUT, "problem_create: null c/l/u");
  if (k.nrows > 0 && !v->q) throw StatusError(AAPDHG_ERR_INPUT, "problem_create: null q");
}

const char* csr_flag_message(int flags) {
  if (flags & kCsrBadRowPtr) return "problem_create: row_ptr not monotone";
  if (flags & kCsrBadColumn) return "problem_create: column index out of range";
  if (flags & kCsrUnsorted) return "problem_create: column indices not strictly increasing in a row";
  return nullptr;
}

void validate_problem_deep(const aapdhg_problem_view* v) {
  const aapdhg_csr_view& k = v->k;
  int flags = 0;
  for (int r = 0; r < k.nrows; ++r)
    if (k.row_ptr[r + 1] < k.row_ptr[r]) flags |= kCsrBadRowPtr;
  for (int64_t e = 0; e < k.nnz; ++e)
    if (k.col_idx[e] < 0 || k.col_idx[e] >= k.ncols) flags |= kCsrBadColumn;
  if (!(flags & kCsrBadRowPtr))
    for (int r = 0; r < k.nrows; ++r)
      for (int32_t e = k.row_ptr[r] + 1; e < k.row_ptr[r + 1]; ++e)
        if (k.col_idx[e] <= k.col_idx[e - 1]) flags |= kCsrUnsorted;
  if (const char* msg = csr_flag_message(flags)) throw StatusError(AAPDHG_ERR_DIMENSION, msg);
}

void validate_problem_view(const aapdhg_problem_view* v) {
  validate_problem_header(v);
  validate_problem_deep(v);
}

// K' as CSR with the entries of each row in ascending original row of K
// (stable counting sort), the order matvec_transpose accumulates in
// (sparse_linalg.cpp:77-87).
void transpose_csr(const aapdhg_csr_view& k, std::vector<int32_t>& trp, std::vector<int32_t>& tci,
                   std::vector<double>& tv) {
  const int n = k.ncols, m = k.nrows;
  trp.assign(static_cast<size_t>(n) + 1, 0);
  tci.resize(static_cast<size_t>(k.nnz));
  tv.resize(static_cast<size_t>(k.nnz));
  for (int64_t e = 0; e < k.nnz; ++e) trp[size_t(k.col_idx[e]) + 1]++;
  for (int j = 0; j < n; ++j) trp[j + 1] += trp[j];
  std::vector<int32_t> next(trp.begin(), trp.end() - 1);
  for (int r = 0; r < m; ++r)
    for (int32_t e = k.row_ptr[r]; e < k.row_ptr[r + 1]; ++e) {
      const int32_t pos = next[size_t(k.col_idx[e])]++;
      tci[size_t(pos)] = r;
      tv[size_t(pos)] = k.vals[e];
    }
}

// Per-device one-time setup (the kernels' attributes are process state):
// done once per device, not per handle.
static std::mutex g_dev_mu;
static bool g_dev_ready[64];
static int g_dev_sms[64];

void Problem::init_device(int device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw CudaError("no CUDA device available (the sm_100a path has no CPU fallback)");
  if (device < 0 || device >= ndev) throw CudaError("device ordinal out of range");
  AAPDHG_CUDA(cudaSetDevice(device));
  {
    std::lock_guard<std::mutex> g(g_dev_mu);
    if (device >= 64 || !g_dev_ready[device]) {
      int major = 0;
      AAPDHG_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
      if (major < 10) {
        cudaDeviceProp prop;
        AAPDHG_CUDA(cudaGetDeviceProperties(&prop, device));
        throw CudaError(std::string("device ") + prop.name + " is not sm_100 class");
      }
      int sms = 0;
      AAPDHG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      // the gather kernels want L1, not shared memory (a few KB per CTA): 10%
      // of the shared-memory maximum keeps 6 CTAs/SM and leaves more L1 than
      // the driver's default 64 KB carveout (configs[1]: 47.3 -> 46.5 us per
      // plain iteration, profiles/exp_carveout.py); -1 = driver default
      const int carve = env_int("AAPDHG_CARVEOUT", 10);
      if (carve >= 0) {
        auto set = [&](const void* f) {
          AAPDHG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
        };
        set((const void*)k_plain_loop<true>);
        set((const void*)k_plain_loop<false>);
        set((const void*)k_dual_side<false, true>);
        set((const void*)k_dual_side<false, false>);
        set((const void*)k_primal_side<false, true>);
        set((const void*)k_primal_side<false, false>);
      }
      AAPDHG_CUDA(cudaFuncSetAttribute(k_aa_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(aa_smem(kMaxMemory))));
      AAPDHG_CUDA(cudaFuncSetAttribute(k_serial_control, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSerSmem)));
      AAPDHG_CUDA(cudaFuncSetAttribute(k_serial_xchains, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(kSerSmem)));
      if (device < 64) {
        g_dev_sms[device] = sms;
        g_dev_ready[device] = true;
      }
      num_sms_ = sms;
    } else {
      num_sms_ = g_dev_sms[device];
    }
  }
  AAPDHG_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
  stream_ = own_stream_;
  AAPDHG_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  g_tls_sync[0] = stream_;
  g_tls_sync[1] = side_;
  AAPDHG_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  AAPDHG_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  AAPDHG_CUDA(cudaEventCreateWithFlags(&ev_out_, cudaEventDisableTiming));
  AAPDHG_CUDA(cudaEventCreateWithFlags(&ev_out_done_, cudaEventDisableTiming));
  for (auto& e : ev_blk_) AAPDHG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  pdl_ = env_int("AAPDHG_PDL", 1) != 0;
  // later column passes fetch their row partial with the metadata: 3 = into a
  // register (default), 2 = an L2 prefetch, 0 = after the gather chain
  pass_prefetch_ = env_int("AAPDHG_PASS_PREFETCH", 3);
  if (pass_prefetch_ != 2 && pass_prefetch_ != 3) pass_prefetch_ = 0;
}

// c, q, l, u on the device plus the scratch of power iteration / per-op /
// KKT evaluation.
// c, q, l, u to the device. Page-locked sources go on side_ (copy engine)
// while the device builds the layouts on stream_ (the caller joins with
// join_vectors); pageable ones are staged on stream_ (host memcpy).
void Problem::upload_vectors(const double* c, const double* q, const double* l, const double* u) {
  c_.reserve(sizeof(double) * n_);
  q_.reserve(sizeof(double) * m_);
  l_.reserve(sizeof(double) * n_);
  u_.reserve(sizeof(double) * n_);
  vec_async_ = host_is_pinned(c) && host_is_pinned(q) && host_is_pinned(l) && host_is_pinned(u);
  cudaStream_t s = vec_async_ ? side_ : stream_;
  if (vec_async_) {  // (the reservations above may have used stream_-ordered memsets)
    AAPDHG_CUDA(cudaEventRecord(ev_fork_, stream_));
    AAPDHG_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
  }
  h2d(c_.p, c, sizeof(double) * n_, s);
  h2d(q_.p, q, sizeof(double) * m_, s);
  h2d(l_.p, l, sizeof(double) * n_, s);
  h2d(u_.p, u, sizeof(double) * n_, s);
  if (vec_async_) AAPDHG_CUDA(cudaEventRecord(ev_join_, side_));
}

void Problem::init_vectors() {
  if (vec_async_) AAPDHG_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
  pw_x_.reserve(sizeof(double) * std::max<int64_t>(n_, 1));
  pw_mx_.reserve(sizeof(double) * std::max<int64_t>(m_, 1));
  pw_mtmx_.reserve(sizeof(double) * std::max<int64_t>(n_, 1));
  pw_state_.reserve(sizeof(PowerState));
  lam_.reserve(sizeof(double) * std::max<int64_t>(n_, 1));
  scal_.reserve(sizeof(double) * 64);
  const int64_t nbig = std::max<int64_t>(std::max<int64_t>(n_, m_), 1);
  part_small_.reserve(sizeof(double) * 5 * (nbig / kThreads + 2));
  static_assert(sizeof(DevState) <= 4096, "state mirror exceeds a pinned pool block");
  h_state_ = static_cast<DevState*>(pinned_small_alloc(sizeof(DevState)));
  h_batch_ = static_cast<int32_t*>(pinned_small_alloc(sizeof(int32_t)));
}

namespace {
// AAPDHG_TIMING=1: problem_create phase times on stderr
struct PhaseTimer {
  bool on = env_int("AAPDHG_TIMING", 0) != 0;
  Clock::time_point t = Clock::now();
  void operator()(const char* what) {
    if (!on) return;
    std::fprintf(stderr, "[aapdhg] %-26s %10.1f us\n", what, 1e6 * secs(t));
    t = Clock::now();
  }
};
}  // namespace

Problem::Problem(const aapdhg_problem_view* v, int device) : device_(device) {
  PhaseTimer ph;
  validate_problem_header(v);
  const aapdhg_csr_view& k = v->k;
  ph("validate");
  init_device(device);
  ph("init_device");
  n_ = k.ncols;
  m_ = k.nrows;
  m1_ = v->m1;
  nnz_ = k.nnz;
  N_ = int64_t(n_) + m_;
  nglob_ = N_;

  // K uploaded and checked on the device, then K's layouts, the transpose
  // K' and its layouts (a second host thread building K' on side_ was
  // measured: no gain inside the bench's process, more variance). Page-
  // locked values go over PCIe on side_ while stream_ sorts the transpose's
  // keys (it needs the structure only); then c, q, l, u the same way beside
  // the layout builds.
  const bool vpin = nnz_ > 0 && host_is_pinned(k.vals) && env_int("AAPDHG_INGEST_OVERLAP", 1);
  if (vpin) {
    k_store_.rp.reserve(sizeof(int32_t) * (size_t(m_) + 1));
    k_store_.ci.reserve(sizeof(int32_t) * size_t(nnz_));
    k_store_.v.reserve(sizeof(double) * size_t(nnz_));
    h2d(k_store_.rp.p, k.row_ptr, sizeof(int32_t) * (size_t(m_) + 1), stream_);
    h2d(k_store_.ci.p, k.col_idx, sizeof(int32_t) * size_t(nnz_), stream_);
    AAPDHG_CUDA(cudaEventRecord(ev_fork_, stream_));
    AAPDHG_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
    h2d(k_store_.v.p, k.vals, sizeof(double) * size_t(nnz_), side_);
    AAPDHG_CUDA(cudaEventRecord(ev_blk_[0], side_));
    upload_vectors(v->c, v->q, v->l, v->u);  // (side_, behind the values)
    device_validate(k_store_, m_, n_, nnz_, false);
    ph("upload K structure");
    // the structure of every layout while the values are in flight (the
    // SELL fills and the blocks' value copies queued: defer_fills_)
    TransposeScratch ts;
    device_transpose_sort(k_store_, m_, n_, nnz_, t_store_, ts);
    device_transpose_permute(k_store_, nnz_, t_store_, ts, nullptr, 1);
    ph("transpose structure");
    defer_fills_ = true;
    finish_csr(m_, n_, nnz_, k_store_, Ks_, Kt_);
    finish_csr(n_, m_, nnz_, t_store_, KTs_, KTt_);
    ph("K, K' SELL structure");
    build_blocks(k_store_, m_, n_, kb_, "AAPDHG_L2_BLOCK_KB_K");
    build_blocks(t_store_, n_, m_, ktb_, "AAPDHG_L2_BLOCK_KB_KT");
    defer_fills_ = false;
    ph("L2 blocks structure");
    AAPDHG_CUDA(cudaStreamWaitEvent(stream_, ev_blk_[0], 0));  // the values are on the device
    device_validate_values(k_store_, nnz_);
    ph("K values");
    device_transpose_permute(k_store_, nnz_, t_store_, ts, nullptr, 2);
    flush_fills();
    ph("value fills");
  } else {
    upload_csr(k.row_ptr, k.col_idx, k.vals, m_, n_, k_store_, Ks_, Kt_);
    ph("upload K + SELL");
    upload_vectors(v->c, v->q, v->l, v->u);  // (page-locked: beside the layout builds)
    ph("vectors (issued)");
    device_transpose(k_store_, m_, n_, nnz_, t_store_);
    ph("transpose");
    finish_csr(n_, m_, nnz_, t_store_, KTs_, KTt_);
    ph("K' SELL");
    build_blocks(k_store_, m_, n_, kb_, "AAPDHG_L2_BLOCK_KB_K");    // K x: blocks of x
    build_blocks(t_store_, n_, m_, ktb_, "AAPDHG_L2_BLOCK_KB_KT");  // K'y: blocks of y
    ph("L2 blocks");
  }

  init_vectors();
  device_flags_vectors();
  ph("vectors");
  // ||q|| and ||c|| (constants of kkt_metrics): TREE order on the device;
  // the SERIAL (index-ordered, vec.hpp:16-29) ones on first use (serial_norms)
  nrm_q_[1] = std::sqrt(device_dot(q_.as<double>(), nullptr, m_, false));
  nrm_c_[1] = std::sqrt(device_dot(c_.as<double>(), nullptr, n_, false));
  ph("norms");
}

void Problem::enter() {
  AAPDHG_CUDA(cudaSetDevice(device_));
  g_tls_sync[0] = stream_;
  g_tls_sync[1] = side_;
}

Problem::~Problem() {
  PhaseTimer ph;
  // the device buffers go back to the block cache: nothing may still use them
  // (this handle's streams; not the device: another thread may be capturing)
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  if (side_) cudaStreamSynchronize(side_);
  if (g_tls_sync[0] == stream_ || g_tls_sync[1] == side_) g_tls_sync[0] = g_tls_sync[1] = nullptr;
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  ph("destroy: graph");
  for (auto& e : event_pool_) cudaEventDestroy(e);
  for (auto& p : pending_) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  pinned_small_free(h_state_);
  pinned_small_free(h_batch_);
  ph("destroy: pinned");
  delete sh_su_;
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (ev_out_) cudaEventDestroy(ev_out_);
  if (ev_out_done_) cudaEventDestroy(ev_out_done_);
  for (auto& e : ev_blk_)
    if (e) cudaEventDestroy(e);
  if (side_) cudaStreamDestroy(side_);
  if (own_stream_) cudaStreamDestroy(own_stream_);
  ph("destroy: streams");
}

void Problem::set_stream(cudaStream_t s) {
  enter();
  AAPDHG_CUDA(cudaStreamSynchronize(stream_));
  stream_ = s ? s : own_stream_;
  if (graph_exec_) {  // a graph is replayed on whatever stream; keep it
  }
}

void Problem::sync() { AAPDHG_CUDA(cudaStreamSynchronize(stream_)); }

bool Problem::resolve_serial(int reduction) const {
  if (reduction == AAPDHG_REDUCE_SERIAL) return true;
  if (m_ == 0 || n_ == 0) return true;  // TREE control rides on the K xhat kernel
  if (reduction == AAPDHG_REDUCE_TREE) return false;
  return N_ <= 65536;
}

// a.b (b == nullptr: a.a) on the device in the requested order; synchronous.
double Problem::device_dot(const double* a, const double* b, int64_t n, bool serial) {
  double* part = part_small_.as<double>();
  const int nb = grid_for(n);
  if (!serial && n > 0) k_sumsq_partials<<<nb, kThreads, 0, stream_>>>(a, b, n, part, nullptr);
  k_dot_final<<<1, kCtrlThreads, 0, stream_>>>(a, b, n, part, n > 0 ? nb : 0, serial ? 1 : 0,
                                                scal_.as<double>() + 40);
  AAPDHG_CUDA(cudaGetLastError());
  double out = 0.0;
  d2h(&out, scal_.as<double>() + 40, sizeof(double), stream_);
  sync();
  return out;
}

// (i+1)^-(1+eps) for i < need (at most kPowTabMax; device pow() beyond),
// host std::pow as the reference's safeguard_pass (solver.cpp:59-62). The
// table is kept across solves and grown lazily, so a solve uploads only the
// entries its launches can reach.
void Problem::ensure_pow_table(double eps, uint64_t need) {
  need = std::min<uint64_t>(std::max<uint64_t>(need, 1), kPowTabMax);
  if (!(eps == pow_eps_)) {
    pow_host_.clear();
    pow_len_ = 0;
    pow_eps_ = eps;
  }
  if (need <= pow_len_) return;
  const uint64_t from = pow_len_;
  const uint64_t len = std::min<uint64_t>(std::max<uint64_t>(need, 2 * from), kPowTabMax);
  pow_host_.resize(len);
  for (uint64_t i = from; i < len; ++i) pow_host_[i] = std::pow(double(i) + 1.0, -(1.0 + eps));
  if (sizeof(double) * len > pow_tab_.bytes) {  // new block: upload everything
    pow_tab_.reserve(sizeof(double) * len);
    h2d(pow_tab_.p, pow_host_.data(), sizeof(double) * len, stream_);
  } else {
    h2d(pow_tab_.as<double>() + from, pow_host_.data() + from, sizeof(double) * (len - from),
        stream_);
  }
  pow_len_ = len;
}

// the SERIAL-order ||q||, ||c|| (index-ordered chains, bitwise the
// reference's dot, vec.hpp:16-29), computed on first SERIAL use
void Problem::ensure_serial_norms() {
  if (serial_norms_) return;
  nrm_q_[0] = std::sqrt(device_dot(q_.as<double>(), nullptr, m_, true));
  nrm_c_[0] = std::sqrt(device_dot(c_.as<double>(), nullptr, n_, true));
  serial_norms_ = true;
}

void Problem::ensure_iter_buffers(int method, int cap, bool ring) {
  int nblk1 = std::max(KTs_.grid(), KTt_.grid()), nblk2 = std::max(Ks_.grid(), Kt_.grid());
  for (const CsrDev& b : ktb_.blk) nblk1 = std::max(nblk1, b.grid());
  for (const CsrDev& b : kb_.blk) nblk2 = std::max(nblk2, b.grid());
  upool_.reserve(sizeof(double) * 4 * std::max<int64_t>(N_, 1));
  kxpool_.reserve(sizeof(double) * 3 * std::max<int64_t>(m_, 1));
  T_.reserve(sizeof(double) * std::max<int64_t>(n_, 1));
  T2_.reserve(sizeof(double) * std::max<int64_t>(n_, 1));
  nblk1 = std::max(nblk1, num_sms_ * kSpmvBlocksPerSM * std::max(kb_.nb(), 1));  // (k_dual_epi per K block)
  nblk2 = std::max(nblk2, num_sms_ * kSpmvBlocksPerSM);
  part1_.reserve(sizeof(double) * P1_COUNT * std::max(nblk1, 1));
  part2_.reserve(sizeof(double) * P2_COUNT * std::max(nblk2, 1));

  gram_.reserve(sizeof(double) * kMaxMemory * kMaxMemory);
  work_.reserve(sizeof(double) * kMaxMemory * kMaxMemory);
  vec_.reserve(sizeof(double) * 8 * kMaxMemory);
  rec_.reserve(sizeof(aapdhg_record) * kRecCap);
  rec_cap_ = kRecCap;
  dparams_.reserve(sizeof(DevParams));
  dstate_.reserve(sizeof(DevState));
  if (!ticket_.p) {  // k_spmv_commit's last-CTA ticket (returns to 0 after each launch)
    ticket_.reserve(sizeof(unsigned int) * 4);
    AAPDHG_CUDA(cudaMemsetAsync(ticket_.p, 0, ticket_.bytes, stream_));
  }
  ndot_tile_ = int((N_ + kDotChunk - 1) / kDotChunk);
  if (method != AAPDHG_METHOD_PDHG) {
    if (ring) {
      // the ring history: cap + 2 slots of g and of the stored du (ring_push,
      // pipeline.cuh); no dg columns
      gpool_.reserve(sizeof(double) * size_t(cap + 2) * std::max<int64_t>(N_, 1));
      du_.reserve(sizeof(double) * size_t(cap + 2) * std::max<int64_t>(N_, 1));
    } else {
      gpool_.reserve(sizeof(double) * 2 * std::max<int64_t>(N_, 1));
      // cap + 1 slots: the next push never lands in a slot the memory holds
      // (advance, pipeline.cuh)
      du_.reserve(sizeof(double) * size_t(cap + 1) * std::max<int64_t>(N_, 1));
      dg_.reserve(sizeof(double) * size_t(cap + 1) * std::max<int64_t>(N_, 1));
    }
    // hi parts, then (FAA) the low parts of the double-double partials
    const int items = num_items_host(cap, AAPDHG_METHOD_FAA);
    partdot_.reserve(2 * sizeof(double) * size_t(items) *
                     std::max(std::max(ndot_tile_, num_sms_), 1));
  }
}

// FAA's double-double partials: the second half of partdot_
double* Problem::faa_part_lo(int method, int cap) const {
  if (method != AAPDHG_METHOD_FAA) return nullptr;
  return partdot_.as<double>() + size_t(num_items_host(cap, AAPDHG_METHOD_FAA)) *
                                     size_t(std::max(std::max(ndot_tile_, num_sms_), 1));
}

IterBufs Problem::iter_bufs() {
  IterBufs B{};
  B.upool = upool_.as<double>();
  B.kxpool = kxpool_.as<double>();
  B.gpool = gpool_.as<double>();
  B.du = du_.as<double>();
  B.dg = dg_.as<double>();
  B.T = T_.as<double>();
  B.T2 = T2_.as<double>();
  B.part1 = part1_.as<double>();
  B.part2 = part2_.as<double>();
  B.c = c_.as<double>();
  B.q = q_.as<double>();
  B.l = l_.as<double>();
  B.u = u_.as<double>();
  return B;
}

void Problem::upload_iterate(int slot, const double* x, const double* y) {
  double* base = upool_.as<double>() + int64_t(slot) * N_;
  if (x) h2d(base, x, sizeof(double) * n_, stream_);
  else if (n_) AAPDHG_CUDA(cudaMemsetAsync(base, 0, sizeof(double) * n_, stream_));
  if (y) h2d(base + n_, y, sizeof(double) * m_, stream_);
  else if (m_) AAPDHG_CUDA(cudaMemsetAsync(base + n_, 0, sizeof(double) * m_, stream_));
}

// kkt_metrics (solver.cpp:64-110) of the iterate stored in upool slot `slot`.
void Problem::kkt_eval(int slot, bool serial, double* out_dev, double* lam_dev) {
  const double* x = upool_.as<double>() + int64_t(slot) * N_;
  const double* y = x + n_;
  if (serial) ensure_serial_norms();
  double* T = T_.as<double>();
  double* KX = pw_mx_.as<double>();
  if (n_) spmv(stream_, KTm(serial), vref(y), rout(T), serial, nullptr, 0, nullptr);
  if (m_) spmv(stream_, Km(serial), vref(x), rout(KX), serial, nullptr, 0, nullptr);
  const int64_t nbig = std::max<int64_t>(std::max<int64_t>(n_, m_), 1);
  const int nb = int((nbig + kThreads - 1) / kThreads);
  k_kkt_terms<<<nb, kThreads, 0, stream_>>>(x, y, T, KX, c_.as<double>(), q_.as<double>(),
                                            l_.as<double>(), u_.as<double>(), n_, m_, m1_,
                                            lam_dev, part_small_.as<double>(), nb);
  k_kkt_final<<<1, kCtrlThreads, 0, stream_>>>(
      x, y, T, KX, c_.as<double>(), q_.as<double>(), l_.as<double>(), u_.as<double>(), n_, m_,
      m1_, part_small_.as<double>(), nb, serial ? 1 : 0, nrm_q_[serial ? 0 : 1],
      nrm_c_[serial ? 0 : 1], out_dev);
  AAPDHG_CUDA(cudaGetLastError());
}

// ---- profiling ------------------------------------------------------------
void Problem::prof_begin(cudaStream_t s, const char* name) {
  if (!profiling_) return;
  cudaEvent_t a;
  if (event_pool_.empty()) {
    AAPDHG_CUDA(cudaEventCreate(&a));
  } else {
    a = event_pool_.back();
    event_pool_.pop_back();
  }
  AAPDHG_CUDA(cudaEventRecord(a, s));
  cur_name_ = name;
  cur_a_ = a;
}

void Problem::prof_end(cudaStream_t s) {
  if (!profiling_) return;
  cudaEvent_t b;
  if (event_pool_.empty()) {
    AAPDHG_CUDA(cudaEventCreate(&b));
  } else {
    b = event_pool_.back();
    event_pool_.pop_back();
  }
  AAPDHG_CUDA(cudaEventRecord(b, s));
  pending_.push_back({cur_name_, cur_a_, b});
}

void Problem::prof_collect() {
  for (auto& p : pending_) {
    float ms = 0.f;
    AAPDHG_CUDA(cudaEventSynchronize(p.b));
    AAPDHG_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    KernelStat& st = stats_[p.name];
    st.each.push_back(ms);
    event_pool_.push_back(p.a);
    event_pool_.push_back(p.b);
  }
  pending_.clear();
}

// cudaLaunchKernelEx, optionally with programmatic stream serialization
// (captured into the graph as a programmatic dependency edge).
template <typename... KArgs, typename... Args>
static void launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t s, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  AAPDHG_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

#define LAUNCH(name, ...)      \
  do {                         \
    prof_begin(s, name);       \
    __VA_ARGS__;               \
    prof_end(s);               \
    ++nodes;                   \
  } while (0)

// One solver iteration (solver.cpp:188-252) as three kernel segments:
//   core   K1, K2 (+ last-CTA control) or K1, K2, serial control
//   aa     the AA / FAA candidate: dots, small solve, mix, K x recache
//   commit role rotation and loop bookkeeping
// Eagerly the aa kernels are predicated on device flags; under graph replay
// they sit in an IF node the control sets, inside a WHILE node commit drives.
// K1 / K2 for a layout: the MULTI instantiation only for interleaved ones
template <bool SER, bool PUSH>
void launch_k1(const CsrDev& A, const IterBufs& B, const DevParams* P, DevState* S,
               cudaStream_t s) {
  if (A.interleave) k_dual_side<SER, PUSH, 0, true><<<A.grid(), kThreads, 0, s>>>(A, B, P, S);
  else k_dual_side<SER, PUSH><<<A.grid(), kThreads, 0, s>>>(A, B, P, S);
}
template <bool SER, bool PUSH>
auto k2_kernel(const CsrDev& A) {
  return A.interleave ? k_primal_side<SER, PUSH, 0, true> : k_primal_side<SER, PUSH>;
}

// the persistent plain-iteration grid for a push / reduction order
using PlainLoopKernel = void (*)(CsrDev, CsrDev, IterBufs, const DevParams*, DevState*, GridBar*,
                                 int, int, int, int, unsigned long long*);
static PlainLoopKernel plain_loop_kernel(bool push, bool serial) {
  return serial ? (push ? k_plain_loop<true, true> : k_plain_loop<false, true>)
                : (push ? k_plain_loop<true, false> : k_plain_loop<false, false>);
}

int Problem::launch_core(cudaStream_t s, const SolveSetup& su) {
  int nodes = 0;
  const bool ser = su.serial, push = su.push;
  if (su.persist) {  // co-resident grid: cooperative launch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(su.pgrid);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    auto kern = plain_loop_kernel(push, ser);
    LAUNCH("k_plain_loop", AAPDHG_CUDA(cudaLaunchKernelEx(&cfg, kern, su.pk1, su.pk2, su.B, su.P,
                                                          su.S, su.gb, su.pk1.grid(),
                                                          su.pk2.grid(), su.np1, su.np2,
                                                          su.bal)));
    return nodes;
  }
  if (su.split) {  // L2-blocked TREE: every block a pass, then the row-order epilogues
    if (n_ > 0) {
      nodes += launch_blocked_passes(s, ktb_, VecRef{nullptr, su.B.upool, U_CUR, N_, n_}, su.S, 0,
                                     nullptr, true);
    }
    // the dual epilogue per column block of K (xhat of block b) on s; K's
    // pass b on side_ right after it, beside the epilogue of block b + 1
    // (AAPDHG_EPI_PIPE=0: one epilogue launch, then the passes on s)
    const int nbk = kb_.nb();
    const bool pipe = su.epi_pipe && m_ > 0 && n_ > 0 && nbk <= kMaxPipe;
    if (n_ > 0) {
      const int parts = pipe ? nbk : 1;
      for (int b = 0; b < parts; ++b) {
        const int j0 = pipe ? int(int64_t(b) * kb_.width) : 0;
        const int j1 = pipe ? int(std::min<int64_t>(n_, int64_t(b + 1) * kb_.width)) : n_;
        const int off = b * su.epi;
        if (push) LAUNCH("k_dual_epi", (k_dual_epi<true><<<su.epi, kThreads, 0, s>>>(ktb_.partial.as<double>(), su.B, su.P, su.S, j0, j1, off, parts * su.epi)));
        else LAUNCH("k_dual_epi", (k_dual_epi<false><<<su.epi, kThreads, 0, s>>>(ktb_.partial.as<double>(), su.B, su.P, su.S, j0, j1, off, parts * su.epi)));
        if (pipe) AAPDHG_CUDA(cudaEventRecord(ev_blk_[b], s));
      }
    }
    if (pipe) {
      for (int b = 0; b < nbk; ++b) {
        AAPDHG_CUDA(cudaStreamWaitEvent(side_, ev_blk_[b], 0));
        prof_begin(side_, "k_spmv_pass");
        k_spmv_pass<<<kb_.blk[b].grid(), kThreads, 0, side_>>>(
            kb_.blk[b], VecRef{nullptr, su.B.upool, U_HAT, N_, 0}, kb_.partial.as<double>(),
            b == 0 ? 1 : pass_prefetch_, su.S, 0, nullptr);
        prof_end(side_);
        AAPDHG_CUDA(cudaGetLastError());
        ++nodes;
      }
      AAPDHG_CUDA(cudaEventRecord(ev_join_, side_));
      AAPDHG_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    }
    if (m_ > 0) {
      if (!pipe)
        nodes += launch_blocked_passes(s, kb_, VecRef{nullptr, su.B.upool, U_HAT, N_, 0}, su.S, 0,
                                       nullptr, true);
      if (push) LAUNCH("k_primal_epi", (k_primal_epi<true><<<su.epi, kThreads, 0, s>>>(kb_.partial.as<double>(), su.B, su.P, su.S)));
      else LAUNCH("k_primal_epi", (k_primal_epi<false><<<su.epi, kThreads, 0, s>>>(kb_.partial.as<double>(), su.B, su.P, su.S)));
    }
    if (su.B.fused_ctrl != 1)
      LAUNCH("k_control", k_control<<<1, kCtrlThreads, 0, s>>>(part1_.as<double>(), n_ > 0 ? su.B.nu1 : 0,
                                                              part2_.as<double>(), su.epi, su.P, su.S));
    AAPDHG_CUDA(cudaGetLastError());
    return nodes;
  }
  // TREE with L2 column blocking: the earlier column passes first, the last
  // block inside the fused kernel (rinit1 / rinit2 hold the partial sums)
  const bool b1 = !ser && ktb_.nb() > 1, b2 = !ser && kb_.nb() > 1;
  const CsrDev& K1m = b1 ? ktb_.blk.back() : KTm(ser);
  const CsrDev& K2m = b2 ? kb_.blk.back() : Km(ser);
  if (b1 && n_ > 0)
    nodes += launch_blocked_passes(s, ktb_, VecRef{nullptr, su.B.upool, U_CUR, N_, n_}, su.S);
  // K'y: products of K' with y = u_cur[n:], then the fused dual-side rows
  if (n_ > 0) {
    if (ser && push) LAUNCH("k_dual_side", (launch_k1<true, true>(K1m, su.B, su.P, su.S, s)));
    else if (ser) LAUNCH("k_dual_side", (launch_k1<true, false>(K1m, su.B, su.P, su.S, s)));
    else if (push && env_int("AAPDHG_K1VAR", 0) == 2) LAUNCH("k_dual_side", k_dual_side<false, true, 2><<<K1m.grid(), kThreads, 0, s>>>(K1m, su.B, su.P, su.S));
    else if (push) LAUNCH("k_dual_side", (launch_k1<false, true>(K1m, su.B, su.P, su.S, s)));
    else LAUNCH("k_dual_side", (launch_k1<false, false>(K1m, su.B, su.P, su.S, s)));
  }
  if (ser) {  // fork: the x-side serial chains run beside K2 on the side stream
    AAPDHG_CUDA(cudaEventRecord(ev_fork_, s));
    AAPDHG_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
    prof_begin(side_, "k_serial_xchains");
    k_serial_xchains<<<1, kSerThreads, kSerSmem, side_>>>(su.B, su.P, su.S);
    prof_end(side_);
    AAPDHG_CUDA(cudaGetLastError());
    AAPDHG_CUDA(cudaEventRecord(ev_join_, side_));
    ++nodes;
  }
  if (b2 && m_ > 0)
    nodes += launch_blocked_passes(s, kb_, VecRef{nullptr, su.B.upool, U_HAT, N_, 0}, su.S);
  // K xhat: products of K with xhat = u_hat[:n], then the fused dual step;
  // launched as a programmatic dependent of K1 (its CTAs load their slice
  // metadata while K1 drains, then wait for K1's xhat)
  if (m_ > 0) {
    const bool pdl = pdl_ && n_ > 0;
    const dim3 g(K2m.grid());
    auto kern = ser ? (push ? k2_kernel<true, true>(K2m) : k2_kernel<true, false>(K2m))
                    : (push ? (env_int("AAPDHG_K2VAR", 0) == 2 ? k_primal_side<false, true, 2>
                                                                : k2_kernel<false, true>(K2m))
                            : k2_kernel<false, false>(K2m));
    LAUNCH("k_primal_side", launch_ex(kern, g, dim3(kThreads), 0, s, pdl, K2m, su.B, su.P, su.S));
  }
  if (ser) {  // join, then the y-side chains and the control
    AAPDHG_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    LAUNCH("k_serial_control", k_serial_control<<<1, kSerThreads, kSerSmem, s>>>(su.B, su.P, su.S));
  } else if (su.B.fused_ctrl != 1) {  // (otherwise k_primal_side's last CTA)
    LAUNCH("k_control", k_control<<<1, kCtrlThreads, 0, s>>>(part1_.as<double>(), K1m.grid(),
                                                            part2_.as<double>(), K2m.grid(),
                                                            su.P, su.S));
  }
  AAPDHG_CUDA(cudaGetLastError());
  return nodes;
}

// The register-blocked Gram (k_gram_dots / FAA: k_gram_dots_dd, one CTA per
// SM or CTA pair) for TREE order and memories <= 10; k_tree_dots beyond.
bool use_gram_dots(int method, int cap, bool serial) {
  (void)method;
  return !serial && cap <= 10 && env_int("AAPDHG_GRAM_DOTS", 1) != 0;
}

int Problem::launch_aa(cudaStream_t s, const SolveSetup& su) {
  int nodes = 0;
  if (su.method == AAPDHG_METHOD_PDHG) return 0;
  if (use_gram_dots(su.method, su.cap, su.serial)) {  // g staged inside the register Gram
    const int c = su.cap <= 4 ? 4 : su.cap <= 6 ? 6 : su.cap <= 8 ? 8 : 10;
    if (su.method == AAPDHG_METHOD_FAA) {  // double-double Gram; CTA pairs for 8 / 10
      auto kern = c == 4 ? k_gram_dots_dd<4, 0> : c == 6 ? k_gram_dots_dd<6, 0>
                  : c == 8 ? k_gram_dots_dd<8, 1> : k_gram_dots_dd<10, 1>;
      const int grid = c >= 8 ? 2 * su.ndot_blk : su.ndot_blk;
      LAUNCH("k_gram_dots", kern<<<grid, kThreads, 0, s>>>(su.D, su.B.upool, su.P, su.S));
    } else if (su.ring) {  // g_k is in the ring already
      auto kern = c == 4 ? k_gram_dots_ring<4> : c == 6 ? k_gram_dots_ring<6>
                  : c == 8 ? k_gram_dots_ring<8> : k_gram_dots_ring<10>;
      LAUNCH("k_gram_dots", kern<<<su.ndot_blk, kThreads, 0, s>>>(su.D, su.P, su.S));
    } else {
      auto kern = c == 4 ? k_gram_dots<4, false> : c == 6 ? k_gram_dots<6, false>
                  : c == 8 ? k_gram_dots<8, false> : k_gram_dots<10, false>;
      LAUNCH("k_gram_dots", kern<<<su.ndot_blk, kThreads, 0, s>>>(su.D, su.B.upool, su.P, su.S));
    }
  } else {
    LAUNCH("k_stage_g", k_stage_g<<<grid_for(N_), kThreads, 0, s>>>(su.B.upool, su.B.gpool, su.P, su.S));
    if (su.serial) {
      const int blocks = (su.items_max * 32 + kThreads - 1) / kThreads;
      LAUNCH("k_serial_dots", k_serial_dots<<<blocks, kThreads, 0, s>>>(su.D, su.P, su.S));
    } else {
      LAUNCH("k_tree_dots", k_tree_dots<<<su.ndot_blk, kThreads, 0, s>>>(su.D, su.P, su.S));
    }
  }
  LAUNCH("k_aa_solve", k_aa_solve<<<1, 1024, aa_smem(su.cap), s>>>(su.D, su.P, su.S, 0));
  LAUNCH("k_mix", k_mix<<<grid_for(N_), kThreads, 0, s>>>(su.B, su.B.dg, su.P, su.S, 1));
  if (m_ > 0 && Km(su.serial).grid() > 0) {
    // K x recache of the accepted candidate, the commit in its last CTA
    RowsumArgs r{};
    r.out_pool = su.B.kxpool;
    r.out_role = KX_CAND;
    r.out_stride = m_;
    const VecRef xr{nullptr, su.B.upool, U_CAND, N_, 0};
    const bool blk = !su.serial && kb_.nb() > 1;  // L2-blocked K: passes, then the last block
    if (blk) {
      nodes += launch_blocked_passes(s, kb_, xr, su.S, 1);
      r.rinit = kb_.partial.as<double>();
    }
    const CsrDev& A = blk ? kb_.blk.back() : Km(su.serial);
    unsigned int* ticket = reinterpret_cast<unsigned int*>(ticket_.p);
    if (su.serial)
      LAUNCH("k_spmv", (k_spmv_commit<true><<<A.grid(), kThreads, 0, s>>>(A, xr, r, su.P, su.S, ticket)));
    else
      LAUNCH("k_spmv", (k_spmv_commit<false><<<A.grid(), kThreads, 0, s>>>(A, xr, r, su.P, su.S, ticket)));
  } else {
    LAUNCH("k_aa_commit", k_aa_commit<<<1, 128, 0, s>>>(su.P, su.S));
  }
  AAPDHG_CUDA(cudaGetLastError());
  return nodes;
}

int Problem::launch_iteration(cudaStream_t s, const SolveSetup& su) {
  return launch_core(s, su) + launch_aa(s, su);
}

// WHILE(batch) { core (+control); IF(aa_attempt) { aa (+commit) } } as one
// executable graph: the control kernel sets both conditions.
void Problem::build_graph(const SolveSetup& su) {
  const cudaStreamCaptureMode mode = cudaStreamCaptureModeThreadLocal;
  cudaStream_t s = stream_;
  cudaGraph_t g;
  AAPDHG_CUDA(cudaGraphCreate(&g, 0));
  AAPDHG_CUDA(cudaGraphConditionalHandleCreate(&cond_loop_, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = cond_loop_;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  AAPDHG_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];

  AAPDHG_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, mode));
  core_nodes_ = launch_core(s, su);
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  AAPDHG_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, nullptr, &deps, &ndeps));
  std::vector<cudaGraphNode_t> tail(deps, deps + ndeps);
  cudaGraph_t captured;
  AAPDHG_CUDA(cudaStreamEndCapture(s, &captured));

  cudaGraphNode_t after = nullptr;
  aa_nodes_ = 0;
  if (su.method != AAPDHG_METHOD_PDHG) {
    AAPDHG_CUDA(cudaGraphConditionalHandleCreate(&cond_aa_, body, 0, cudaGraphCondAssignDefault));
    cudaGraphNodeParams ip{};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = cond_aa_;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    AAPDHG_CUDA(cudaGraphAddNode(&after, body, tail.data(), tail.size(), &ip));
    cudaGraph_t ifbody = ip.conditional.phGraph_out[0];
    AAPDHG_CUDA(cudaStreamBeginCaptureToGraph(s, ifbody, nullptr, nullptr, 0, mode));
    aa_nodes_ = launch_aa(s, su);
    AAPDHG_CUDA(cudaStreamEndCapture(s, &captured));
  }
  (void)after;
  AAPDHG_CUDA(cudaGraphInstantiate(&graph_exec_, g, 0));
  cudaGraphDestroy(g);
}
#undef LAUNCH

// ---- step sizes -------------------------------------------------------------
void validate_config(const aapdhg_solve_params* c) {
  // validate, solver.cpp:25-38 (same messages)
  const char* msg = nullptr;
  if (c->m < 1) msg = "solver: m must be >= 1";
  else if (c->safeguard_d <= 0.0) msg = "solver: D must be > 0";
  else if (c->safeguard_eps <= 0.0) msg = "solver: eps must be > 0";
  else if (c->toll <= 0.0) msg = "solver: toll must be > 0";
  else if (c->kkt_eps <= 0.0) msg = "solver: kkt_eps must be > 0";
  else if (c->beta <= 0.0 || c->beta > 1.0) msg = "solver: beta must be in (0, 1]";
  else if (c->eta < 0.0) msg = "solver: eta must be >= 0";
  else if (c->c_s <= 0.0 || c->c_s > 1.0) msg = "solver: c_s must be in (0, 1]";
  else if (c->kappa_bar <= 0.0) msg = "solver: kappa_bar must be > 0";
  if (msg) throw StatusError(AAPDHG_ERR_INPUT, msg);
  if (c->method < AAPDHG_METHOD_PDHG || c->method > AAPDHG_METHOD_FAA)
    throw StatusError(AAPDHG_ERR_INPUT, "solver: unknown method");
  if (c->reduction < AAPDHG_REDUCE_AUTO || c->reduction > AAPDHG_REDUCE_TREE)
    throw StatusError(AAPDHG_ERR_INPUT, "solver: unknown reduction mode");
}

void Problem::run_power(const double* x0, int max_iters, double rel_tol, bool serial,
                        double* out, int* rounds) {
  double* x = pw_x_.as<double>();
  double* mx = pw_mx_.as<double>();
  double* mtmx = pw_mtmx_.as<double>();
  double* scal = scal_.as<double>();
  double* part = part_small_.as<double>();
  PowerState* ps = pw_state_.as<PowerState>();
  h2d(x, x0, sizeof(double) * n_, stream_);
  const int nb = grid_for(n_);
  if (!serial) k_sumsq_partials<<<nb, kThreads, 0, stream_>>>(x, nullptr, n_, part, nullptr);
  k_dot_final<<<1, kCtrlThreads, 0, stream_>>>(x, nullptr, n_, part, nb, serial, scal);
  k_power_init_norm<<<1, 1, 0, stream_>>>(x, scal);
  k_scale<<<grid_for(n_), kThreads, 0, stream_>>>(x, x, n_, nullptr, scal + 1);
  PowerState h{};
  h.max_iters = max_iters;
  h.rel_tol = rel_tol;
  h2d(ps, &h, sizeof h, stream_);
  PowerState hs{};
  for (;;) {
    for (int r = 0; r < kPowerBatch; ++r) {
      spmv_any(stream_, false, vref(x), rout(mx), serial, nullptr, &ps->done);
      spmv_any(stream_, true, vref(mx), rout(mtmx), serial, nullptr, &ps->done);
      if (!serial) k_sumsq_partials<<<nb, kThreads, 0, stream_>>>(mtmx, nullptr, n_, part, &ps->done);
      k_power_ctrl<<<1, kCtrlThreads, 0, stream_>>>(mtmx, n_, part, nb, serial, ps);
      k_scale<<<grid_for(n_), kThreads, 0, stream_>>>(x, mtmx, n_, ps, nullptr);
    }
    AAPDHG_CUDA(cudaGetLastError());
    d2h(&hs, ps, sizeof hs, stream_);
    sync();
    if (hs.done) break;
  }
  *out = hs.result;
  if (rounds) *rounds = hs.rounds;
}

// power_iteration_norm, sparse_linalg.cpp:95-123 (start vector drawn on the
// host with the same std::mt19937_64 + uniform_real_distribution(-1, 1)).
double Problem::power_norm(int max_iters, double rel_tol, uint64_t seed, bool serial,
                           int* rounds) {
  enter();
  if (rounds) *rounds = 0;
  if (all_zero_ || n_ == 0) return 0.0;
  if (max_iters <= 0) return 0.0;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(-1.0, 1.0);
  std::vector<double> x0(static_cast<size_t>(n_));
  for (double& v : x0) v = unif(rng);
  double out = 0.0;
  run_power(x0.data(), max_iters, rel_tol, serial, &out, rounds);
  return out;
}

// select_step_sizes, solver.cpp:112-123
void Problem::select_step_sizes(const aapdhg_solve_params* prm, double* tau, double* sigma) {
  if (prm->tau > 0.0 || prm->sigma > 0.0) {
    if (!(prm->tau > 0.0 && prm->sigma > 0.0))
      throw StatusError(AAPDHG_ERR_INPUT, "step sizes: override requires both tau and sigma");
    *tau = prm->tau;
    *sigma = prm->sigma;
    return;
  }
  const double k_norm = power_norm(5000, 1e-4, 12345u, resolve_serial(prm->reduction), nullptr);
  if (k_norm == 0.0) {
    *tau = *sigma = 1.0;
    return;
  }
  const double s = 0.9 / k_norm;
  *tau = *sigma = s;
}

// ---- solve ------------------------------------------------------------------
void Problem::solve(const aapdhg_solve_params* prm, const double* x0, const double* y0,
                    aapdhg_solve_result* res, double* x_out, double* y_out, double* lam_out,
                    aapdhg_record_sink sink, void* ctx) {
  const auto t_start = Clock::now();
  PhaseTimer ph;
  enter();
  validate_config(prm);
  if (!bounds_ok_) throw StatusError(AAPDHG_ERR_INPUT, "build_lambda_set: l > u");
  const int method = prm->method;
  if (method != AAPDHG_METHOD_PDHG && prm->m > uint64_t(kMaxMemory))
    throw StatusError(AAPDHG_ERR_UNSUPPORTED,
                      "solver: memory capacity m > " + std::to_string(kMaxMemory) +
                          " is not supported by the sm_100a path");
  if (prm->d_hat)
    for (int64_t i = 0; i < N_; ++i)
      if (prm->d_hat[i] <= 0.0) throw StatusError(AAPDHG_ERR_INPUT, "aa: d_hat entries must be > 0");
  double tau, sigma;
  select_step_sizes(prm, &tau, &sigma);
  ph("solve: step sizes");

  const bool serial = resolve_serial(prm->reduction);
  const int cap = method == AAPDHG_METHOD_PDHG ? 0 : int(prm->m);
  // AA-PDHG keeps its history as a ring of g (ring_push, pipeline.cuh;
  // AAPDHG_RING=0: the pushed du / dg columns)
  const bool ring = method == AAPDHG_METHOD_AA && env_int("AAPDHG_RING", 1) != 0;
  ensure_iter_buffers(method, std::max(cap, 1), ring);
  if (prm->d_hat) {
    dhat_.reserve(sizeof(double) * N_);
    h2d(dhat_.p, prm->d_hat, sizeof(double) * N_, stream_);
  }
  // executable graph, cached per launch layout
  // AAPDHG_EAGER=1 forces stream launches (ncu cannot profile kernels inside
  // graphs that hold conditional nodes)
  static const bool force_eager = [] {
    const char* e = std::getenv("AAPDHG_EAGER");
    return e && e[0] == '1';
  }();
  const bool use_graph = !profiling_ && !force_eager;
  // graph launches run up to `batch` iterations; the first one covers a
  // short solve whole (eager launching keeps small batches: every launched
  // iteration is issued even when predicated off)
  const uint64_t max_it_sat = prm->max_iters >= (UINT64_MAX >> 1) ? (UINT64_MAX >> 1)
                                                                   : prm->max_iters;
  const uint64_t ring_batch = std::min<uint64_t>(kMaxBatch, rec_cap_ / 2);
  int batch = use_graph ? int(std::min<uint64_t>(max_it_sat + 2, ring_batch)) : 8;
  // the safeguard's (i+1)^-(1+eps) for every i the first launch can reach
  if (method != AAPDHG_METHOD_PDHG)
    ensure_pow_table(prm->safeguard_eps, std::min<uint64_t>(max_it_sat, uint64_t(batch)) + 2);

  ph("solve: buffers + pow table");
  DevParams P{};
  P.method = method;
  P.serial = serial ? 1 : 0;
  P.m1 = m1_;
  P.kkt_terminate = prm->kkt_terminate ? 1 : 0;
  P.n = n_;
  P.mrows = m_;
  P.cap = cap;
  P.N = N_;
  P.Nglob = nglob_;
  P.safeguard_d = prm->safeguard_d;
  P.safeguard_eps = prm->safeguard_eps;
  P.beta = prm->beta;
  P.eta = prm->eta;
  P.c_s = prm->c_s;
  P.kappa_bar = prm->kappa_bar;
  P.toll = prm->toll;
  P.kkt_eps = prm->kkt_eps;
  P.tau = tau;
  P.sigma = sigma;
  P.max_iters = prm->max_iters;
  P.max_wall_s = prm->max_wall_seconds;
  if (serial) ensure_serial_norms();
  P.nrm_q = nrm_q_[serial ? 0 : 1];
  P.nrm_c = nrm_c_[serial ? 0 : 1];
  P.d_hat = prm->d_hat ? dhat_.as<double>() : nullptr;
  P.pow_tab = method == AAPDHG_METHOD_PDHG ? nullptr : pow_tab_.as<double>();
  P.pow_len = method == AAPDHG_METHOD_PDHG ? 0 : pow_len_;
  P.rec = rec_.as<aapdhg_record>();
  P.rec_cap = rec_cap_;
  // predicted stops in k_plain_loop (stop_likely, exact from the x part of
  // ||g_k||^2): measured a net loss on configs[1] AA-PDHG (52.0 -> 61.5 us
  // per iteration: ||g_x|| alone rarely rules an attempt out, so the workers
  // wait for most decisions; profiles/r02b/stop_predict.txt), so off unless
  // AAPDHG_STOP_PREDICT=1 (round 1's extrapolated prediction lost too)
  P.no_stop_predict = env_int("AAPDHG_STOP_PREDICT", 0) == 0 ? 1 : 0;
  // one-phase-ahead L2 prefetch of the slice streams (prefetch_slice_streams):
  // measured a loss on configs[1] (17.2k vs 18.6k it/s), opt-in experiment
  P.phase_prefetch = env_int("AAPDHG_PREFETCH", 0);
  P.ring = ring ? 1 : 0;
  const bool blk1 = !serial && ktb_.nb() > 1, blk2 = !serial && kb_.nb() > 1;
  const CsrDev& K1m = blk1 ? ktb_.blk.back() : KTm(serial);
  const CsrDev& K2m = blk2 ? kb_.blk.back() : Km(serial);
  P.nblk1 = K1m.grid();
  P.nblk2 = K2m.grid();
  // TREE with memory <= 10: one CTA per SM for the register Gram
  const int ndot = use_gram_dots(method, cap, serial) ? num_sms_ : ndot_tile_;
  P.ndot_blk = ndot;

  DevState S0{};
  S0.prev_plain = 1;
  for (int r = 0; r < 4; ++r) S0.u_idx[r] = r;
  for (int r = 0; r < 3; ++r) S0.kx_idx[r] = r;
  S0.g_idx[0] = 0;
  S0.g_idx[1] = 1;
  DevState* S = dstate_.as<DevState>();

  SolveSetup su;
  su.B = iter_bufs();
  su.B.nu1 = n_ > 0 ? K1m.grid() : 0;
  su.B.rinit1 = blk1 ? ktb_.partial.as<double>() : nullptr;
  su.B.rinit2 = blk2 ? kb_.partial.as<double>() : nullptr;
  su.B.fused_ctrl = (!serial && m_ > 0 && env_int("AAPDHG_FUSED", 1) != 0) ? 1 : 0;
  su.D = DotBufs{du_.as<double>(), dg_.as<double>(), gpool_.as<double>(),
                 partdot_.as<double>(), num_items_host(std::max(cap, 1), method)};
  su.D.part_lo = faa_part_lo(method, cap);
  su.W = SolveScratch{gram_.as<double>(), work_.as<double>(), vec_.as<double>()};
  su.P = dparams_.as<DevParams>();
  su.S = S;
  su.serial = serial;
  su.push = method != AAPDHG_METHOD_PDHG;
  su.ring = ring;
  su.method = method;
  su.cap = cap;
  su.nblk1 = K1m.grid();
  su.nblk2 = K2m.grid();
  su.ndot_blk = ndot;
  su.items_max = num_items_host(std::max(cap, 1), method);
  // L2-blocked TREE (configs[4]): the epilogues in row order after all the
  // column passes (AAPDHG_SPLIT_EPI=0: the last block fused with them)
  if (blk1 && blk2 && n_ > 0 && m_ > 0 && env_int("AAPDHG_SPLIT_EPI", 1) != 0) {
    su.split = true;
    su.epi = num_sms_ * kSpmvBlocksPerSM;
    su.epi_pipe = env_int("AAPDHG_EPI_PIPE", 1) != 0 && kb_.nb() <= kMaxPipe;
    su.B.nu1 = su.epi * (su.epi_pipe ? kb_.nb() : 1);
    su.nblk1 = su.B.nu1;
    su.nblk2 = su.epi;
    P.nblk1 = su.nblk1;
    P.nblk2 = su.epi;
  }

  // executable graph, cached per launch layout (use_graph above)
  // plain iterations in one persistent grid (AAPDHG_PERSIST=0: per-kernel graph)
  PersistLock plock;
  // (eager stream launches of it only on request, AAPDHG_PERSIST_EAGER=1: ncu
  // cannot profile kernels inside graphs that hold conditional nodes)
  const bool persist_ok = use_graph || (!profiling_ && env_int("AAPDHG_PERSIST_EAGER", 0) != 0);
  // (SERIAL too: the control CTA runs the index-ordered chains while the
  // workers run ahead; AAPDHG_SERIAL_PERSIST=0 keeps the per-kernel graph)
  const bool persist_mode =
      serial ? env_int("AAPDHG_SERIAL_PERSIST", 1) != 0 : su.B.fused_ctrl == 1;
  if (persist_ok && persist_mode && !blk1 && !blk2 && n_ > 0 && m_ > 0 &&
      env_int("AAPDHG_PERSIST", 1) != 0) {
    int per_sm = 0;
    AAPDHG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, plain_loop_kernel(su.push, serial), kThreads, 0));
    // one CTA of the co-resident grid is the control CTA: the short-row
    // slices spread over one CTA fewer when the layout fills the wave
    const int workers = per_sm * num_sms_ - 1;
    auto fit = [&](CsrDev d) {
      const int over = d.grid() - workers;
      if (over > 0) d.nblk_short = d.nblk_short > over ? d.nblk_short - over : 0;
      return d;
    };
    // (a warp owns one slice: every CTA keeps <= kWarps slices)
    auto fits = [&](const CsrDev& d) {
      return d.grid() <= workers &&
             (d.nslices == 0 || int64_t(d.nblk_short) * kWarps >= int64_t(d.nslices));
    };
    const CsrDev p1 = fit(K1m), p2 = fit(K2m);
    if (env_int("AAPDHG_VERBOSE", 0))
      std::fprintf(stderr, "aapdhg: k_plain_loop %d CTAs/SM, grids %d/%d -> %d/%d\n", per_sm,
                   K1m.grid(), K2m.grid(), p1.grid(), p2.grid());
    if (workers >= 1 && fits(p1) && fits(p2) && plock.try_lock(device_)) {
      gridbar_.reserve(sizeof(GridBar));
      su.persist = true;
      su.pk1 = p1;
      su.pk2 = p2;
      su.pgrid = std::max(p1.grid(), p2.grid()) + 1;
      su.gb = gridbar_.as<GridBar>();
      su.B.nu1 = p1.grid();
      su.np1 = p1.grid();
      su.np2 = p2.grid();
      // TREE: the calibrated partition over every worker CTA (no long rows,
      // not interleaved, more slices than workers; AAPDHG_BALANCE=0: off)
      auto plain = [&](const CsrDev& d) {
        return d.nlong == 0 && !d.interleave && d.nslices >= workers &&
               int64_t(d.nslices) <= int64_t(kWarps) * workers;
      };
      if (!serial && plain(p1) && plain(p2) && env_int("AAPDHG_BALANCE", 1) != 0) {
        bool measure = false;
        bal_setup(p1, p2, workers, &measure);
        part1_.reserve(sizeof(double) * P1_COUNT * size_t(p1.nslices));
        part2_.reserve(sizeof(double) * P2_COUNT * size_t(p2.nslices));
        su.B.part1 = part1_.as<double>();
        su.B.part2 = part2_.as<double>();
        su.pk1.sl_start = bal_start1_.as<int32_t>();
        su.pk2.sl_start = bal_start2_.as<int32_t>();
        su.pk1.nblk_short = su.pk2.nblk_short = workers;
        su.pgrid = workers + 1;
        su.B.nu1 = workers;
        su.np1 = p1.nslices;
        su.np2 = p2.nslices;
        su.bal = measure ? bal_stats_.as<unsigned long long>() : nullptr;
        bal_measuring_ = measure;
      }
    }
  }
  if (use_graph) {
    char key[256];
    std::snprintf(key, sizeof key, "%d/%d/%d/%d/%d/%d/%p/%p/%p/%p/%p/%p/%p/%p/%p/%p/%p/%p/%p", method,
                  int(serial), cap, int(su.persist), int(su.split), int(su.ring), upool_.p, gpool_.p, dg_.p, du_.p, partdot_.p, dparams_.p,
                  rec_.p, stream_, gridbar_.p, (const void*)su.pk1.sl_start, (void*)su.bal,
                  su.B.part1, su.B.part2);
    if (graph_key_ != key || !graph_exec_) {
      if (graph_exec_) {
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
      }
      build_graph(su);
      graph_key_ = key;
    }
  }
  ph("solve: graph");
  P.use_cond = use_graph ? 1 : 0;
  P.cond_aa = cond_aa_;
  P.cond_loop = cond_loop_;

  // start iterate P(u0) in slot 0, its K x cached in kx slot 0; fresh pools
  AAPDHG_CUDA(cudaMemsetAsync(upool_.p, 0, sizeof(double) * 4 * N_, stream_));
  if (method != AAPDHG_METHOD_PDHG && !ring) {  // (the ring's slots are written before read)
    AAPDHG_CUDA(cudaMemsetAsync(gpool_.p, 0, sizeof(double) * 2 * N_, stream_));
  }
  if (su.persist) AAPDHG_CUDA(cudaMemsetAsync(gridbar_.p, 0, sizeof(GridBar), stream_));
  upload_iterate(0, x0, y0);
  P.wall_offset_s = secs(t_start);
  h2d(dparams_.p, &P, sizeof P, stream_);
  h2d(S, &S0, sizeof S0, stream_);
  k_project_start<<<grid_for(N_, kThreads, 1 << 30), kThreads, 0, stream_>>>(
      upool_.as<double>(), l_.as<double>(), u_.as<double>(), n_, N_, m1_, S);
  // K x of the start: the default start P(0) has x = +0 when every box holds
  // 0, and then every row sum (started at +0, adding +-0 products) is +0
  if (m_ && !x0 && zero_start_ && env_int("AAPDHG_ZERO_START", 1) != 0)
    AAPDHG_CUDA(cudaMemsetAsync(kxpool_.p, 0, sizeof(double) * m_, stream_));
  else if (m_)
    spmv_any(stream_, false, vref(upool_.as<double>()), rout(kxpool_.as<double>()), serial,
             nullptr, nullptr);
  AAPDHG_CUDA(cudaGetLastError());

  ph("solve: start iterate");
  // Result download beside the last iteration (large LPs, page-locked x / y,
  // TREE, graph launches): the launches stop one iteration short of
  // max_iters. Every stop the last iteration can take finishes on its CUR
  // iterate (KKT of u_k, residual, max_iters, timeout: solver.cpp:182-199),
  // which is then known, so x / y cross PCIe on side_ while the device
  // computes its residual, KKT and lambda. A solve that stops earlier, or a
  // final role other than CUR, takes the usual downloads.
  const bool px_pin = x_out && n_ > 0 && host_is_pinned(x_out);
  const bool py_pin = y_out && m_ > 0 && host_is_pinned(y_out);
  const bool out_ovl = use_graph && !serial && (px_pin || py_pin) &&
                       max_it_sat < (UINT64_MAX >> 1) &&
                       int64_t(sizeof(double)) * N_ >= (int64_t(env_int("AAPDHG_OUT_OVERLAP_MB", 32)) << 20);
  if (out_ovl) batch = int(std::min<uint64_t>(max_it_sat + 1, ring_batch));
  int early_slot = -1;  // the slot whose x / y are on their way
  uint64_t flushed = 0, eager_launches = 0;
  std::vector<aapdhg_record> host_recs;
  const aapdhg_record* drec = rec_.as<aapdhg_record>();
  for (bool first = true;; first = false) {
    if (!first && out_ovl) {
      const uint64_t ij = h_state_->i + h_state_->j;
      if (ij >= prm->max_iters) {  // the next iteration is the last one
        batch = 1;
        if (early_slot < 0) {
          early_slot = h_state_->u_idx[U_CUR];
          const double* uc = upool_.as<double>() + int64_t(early_slot) * N_;
          AAPDHG_CUDA(cudaEventRecord(ev_out_, stream_));
          AAPDHG_CUDA(cudaStreamWaitEvent(side_, ev_out_, 0));
          if (px_pin)
            AAPDHG_CUDA(cudaMemcpyAsync(x_out, uc, sizeof(double) * n_, cudaMemcpyDeviceToHost, side_));
          if (py_pin)
            AAPDHG_CUDA(cudaMemcpyAsync(y_out, uc + n_, sizeof(double) * m_, cudaMemcpyDeviceToHost,
                                        side_));
          AAPDHG_CUDA(cudaEventRecord(ev_out_done_, side_));
        }
      } else {
        batch = int(std::min<uint64_t>(uint64_t(batch), prm->max_iters - ij));
      }
    }
    if (!first && method != AAPDHG_METHOD_PDHG) {
      // i grows by at most one per iteration: cover the next launch
      const uint64_t cap_before = pow_len_;
      const double* tab_before = pow_tab_.as<double>();
      ensure_pow_table(prm->safeguard_eps,
                       std::min<uint64_t>(max_it_sat, h_state_->i + uint64_t(batch)) + 2);
      if (pow_len_ != cap_before || pow_tab_.as<double>() != tab_before) {
        DevParams* Pd = dparams_.as<DevParams>();
        const double* tp = pow_tab_.as<double>();
        const uint64_t tl = pow_len_;
        h2d(&Pd->pow_tab, &tp, sizeof tp, stream_);
        h2d(&Pd->pow_len, &tl, sizeof tl, stream_);
      }
    }
    if (use_graph) {
      *h_batch_ = batch;
      h2d(&S->batch_left, h_batch_, sizeof(int32_t), stream_);
      AAPDHG_CUDA(cudaGraphLaunch(graph_exec_, stream_));
    } else {
      if (su.persist) {  // each launch runs until the control stops it
        *h_batch_ = batch;
        h2d(&S->batch_left, h_batch_, sizeof(int32_t), stream_);
      }
      for (int it = 0; it < batch; ++it) eager_launches += launch_iteration(stream_, su);
    }
    d2h(h_state_, S, sizeof(DevState), stream_);
    sync();
    ph("solve: launch + state");
    if (profiling_) prof_collect();
    // stream completed records out of the device ring
    const uint64_t done_recs = h_state_->rec_complete;
    if (done_recs > flushed) {
      const uint64_t cnt = done_recs - flushed;
      host_recs.resize(cnt);
      uint64_t got = 0;
      while (got < cnt) {
        const uint64_t pos = (flushed + got) % rec_cap_;
        const uint64_t chunk = std::min<uint64_t>(cnt - got, rec_cap_ - pos);
        d2h(host_recs.data() + got, drec + pos, chunk * sizeof(aapdhg_record), stream_);
        got += chunk;
      }
      sync();
      if (sink) sink(host_recs.data(), cnt, ctx);
      flushed = done_recs;
      ph("solve: records");
    }
    if (h_state_->done) break;
    // ring safety: a launch never runs further ahead than half the ring
    batch = int(std::min<uint64_t>(uint64_t(batch) * 2, ring_batch));
  }
  const DevState st = *h_state_;
  ph("solve: iterations");
  if (su.bal) bal_collect(su.pk1, su.pk2, su.pgrid - 1);

  // finish, solver.cpp:153-166
  const int slot = st.u_idx[st.final_role];
  const double* ufin = upool_.as<double>() + int64_t(slot) * N_;
  double kkt[4];
  // TREE: the final iterate is the CUR iterate of the last iteration, whose
  // KKT the fused kernels already reduced (DevState::kkt); only lambda needs
  // K'y again (CSR-ordered, so lambda is the reference's bit for bit). The
  // x / y downloads run while lambda is computed when the outputs are pinned.
  // SERIAL (and the fixed-point start): the index-ordered kkt_eval.
  const bool fast = !serial && st.final_role == U_CUR &&
                    st.status != AAPDHG_SOLVE_FIXED_POINT_START &&
                    env_int("AAPDHG_FAST_FINISH", 1) != 0;
  bool side_copies = early_slot >= 0;
  if (fast) {
    // page-locked x / y go over PCIe on side_ while lambda is computed (the
    // last iteration's CUR slot may already be on its way, above)
    const bool px = x_out && host_is_pinned(x_out), py = y_out && host_is_pinned(y_out);
    if ((px || py) && early_slot != slot) {
      if (early_slot >= 0) AAPDHG_CUDA(cudaStreamWaitEvent(stream_, ev_out_done_, 0));
      AAPDHG_CUDA(cudaEventRecord(ev_out_, stream_));
      AAPDHG_CUDA(cudaStreamWaitEvent(side_, ev_out_, 0));
      if (px) AAPDHG_CUDA(cudaMemcpyAsync(x_out, ufin, sizeof(double) * n_,
                                          cudaMemcpyDeviceToHost, side_));
      if (py) AAPDHG_CUDA(cudaMemcpyAsync(y_out, ufin + n_, sizeof(double) * m_,
                                          cudaMemcpyDeviceToHost, side_));
      AAPDHG_CUDA(cudaEventRecord(ev_out_done_, side_));
      side_copies = true;
    }
    if (lam_out && n_ > 0) {
      T_.reserve(sizeof(double) * std::max<int64_t>(n_, 1));
      // L2-blocked split iteration: the last evaluation's K' passes left the
      // finished K'y of its CUR iterate — this final iterate — in the row
      // partials (launch_core: every block a pass; nothing after the stop
      // writes them: the AA recache runs K's passes), the same sums in the
      // same block order spmv_any would form again (AAPDHG_LAMBDA_REUSE=0)
      const bool reuse = m_ > 0 && su.split && ktb_.nb() > 1 &&
                         env_int("AAPDHG_LAMBDA_REUSE", 1) != 0;
      const double* kty = reuse ? ktb_.partial.as<double>() : T_.as<double>();
      if (reuse) {
      } else if (m_ > 0) {
        spmv_any(stream_, true, vref(ufin + n_), rout(T_.as<double>()), false, nullptr, nullptr);
      } else {
        AAPDHG_CUDA(cudaMemsetAsync(T_.p, 0, sizeof(double) * n_, stream_));
      }
      k_lambda_from_T<<<grid_for(n_), kThreads, 0, stream_>>>(
          kty, c_.as<double>(), l_.as<double>(), u_.as<double>(), n_,
          lam_.as<double>());
      AAPDHG_CUDA(cudaGetLastError());
    }
    for (int q = 0; q < 4; ++q) kkt[q] = st.kkt[q];
    if (x_out && !px) d2h(x_out, ufin, sizeof(double) * n_, stream_);
    if (y_out && !py) d2h(y_out, ufin + n_, sizeof(double) * m_, stream_);
    if (lam_out) d2h(lam_out, lam_.as<double>(), sizeof(double) * n_, stream_);
    ph("solve: final lambda + downloads");
  } else {
    // (an early download of another slot must land before these copies)
    if (early_slot >= 0) AAPDHG_CUDA(cudaStreamWaitEvent(stream_, ev_out_done_, 0));
    double* kkt_dev = scal_.as<double>() + 8;
    kkt_eval(slot, serial, kkt_dev, lam_.as<double>());
    d2h(kkt, kkt_dev, sizeof kkt, stream_);
    ph("solve: final kkt");
    if (x_out) d2h(x_out, ufin, sizeof(double) * n_, stream_);
    if (y_out) d2h(y_out, ufin + n_, sizeof(double) * m_, stream_);
    if (lam_out) d2h(lam_out, lam_.as<double>(), sizeof(double) * n_, stream_);
  }
  if (side_copies) AAPDHG_CUDA(cudaStreamWaitEvent(stream_, ev_out_done_, 0));
  sync();
  std::memset(res, 0, sizeof *res);
  res->status = st.status;
  res->iterations = st.i + st.j;
  res->i = st.i;
  res->j = st.j;
  res->aa_failures = st.aa_failures;
  res->g_norm = st.g_final;
  res->r_gap = kkt[0];
  res->r_primal = kkt[1];
  res->r_dual = kkt[2];
  res->objective = kkt[3];
  res->tau = tau;
  res->sigma = sigma;
  res->wall_seconds = secs(t_start);
  last_loop_iters_ = st.loop_iters;
  last_plain_iters_ = st.plain_iters;
  last_plain_launches_ = st.loop_exits;
  last_plain_secs_ = double(st.plain_ns) * 1e-9;
  if (!use_graph)  // eager: every launch issued, predicated or not
    last_launches_ = eager_launches;
  else if (su.persist)
    last_launches_ = st.loop_exits + (st.i + st.aa_failures) * uint64_t(aa_nodes_);
  else
    last_launches_ = st.loop_iters * uint64_t(core_nodes_) +
                     (st.i + st.aa_failures) * uint64_t(aa_nodes_);
  ph("solve: finish");
}

// ---- single-op entry points ----------------------------------------------
void Problem::matvec(const double* x, double* out) {
  enter();
  h2d(pw_x_.p, x, sizeof(double) * n_, stream_);
  spmv(stream_, Ks_, vref(pw_x_.as<double>()), rout(pw_mx_.as<double>()), true, nullptr, 0,
       nullptr);
  d2h(out, pw_mx_.p, sizeof(double) * m_, stream_);
  sync();
}

void Problem::matvec_transpose(const double* y, double* out) {
  enter();
  h2d(pw_mx_.p, y, sizeof(double) * m_, stream_);
  spmv(stream_, KTs_, vref(pw_mx_.as<double>()), rout(pw_mtmx_.as<double>()), true, nullptr, 0,
       nullptr);
  d2h(out, pw_mtmx_.p, sizeof(double) * n_, stream_);
  sync();
}

static DevState identity_state() {
  DevState S{};
  S.prev_plain = 1;
  for (int r = 0; r < 4; ++r) S.u_idx[r] = r;
  for (int r = 0; r < 3; ++r) S.kx_idx[r] = r;
  S.g_idx[0] = 0;
  S.g_idx[1] = 1;
  return S;
}

// pdhg_step, pdhg_core.cpp:45-63, through the fused K1/K2 kernels
void Problem::pdhg_step(double tau, double sigma, const double* x, const double* y,
                        double* xn, double* yn) {
  enter();
  ensure_iter_buffers(AAPDHG_METHOD_PDHG, 1);
  upload_iterate(0, x, y);
  spmv(stream_, Ks_, vref(upool_.as<double>()), rout(kxpool_.as<double>()), true, nullptr, 0,
       nullptr);
  DevParams P{};
  P.method = AAPDHG_METHOD_PDHG;
  P.serial = 1;
  P.m1 = m1_;
  P.n = n_;
  P.mrows = m_;
  P.N = N_;
  P.Nglob = nglob_;
  P.tau = tau;
  P.sigma = sigma;
  P.nblk1 = KTs_.grid();
  P.nblk2 = Ks_.grid();
  const DevState S = identity_state();
  h2d(dparams_.p, &P, sizeof P, stream_);
  h2d(dstate_.p, &S, sizeof S, stream_);
  IterBufs B = iter_bufs();
  const DevParams* Pd = dparams_.as<DevParams>();
  DevState* Sd = dstate_.as<DevState>();
  if (n_) {
    launch_k1<true, false>(KTs_, B, Pd, Sd, stream_);
  }
  if (m_) {
    k2_kernel<true, false>(Ks_)<<<Ks_.grid(), kThreads, 0, stream_>>>(Ks_, B, Pd, Sd);
  }
  AAPDHG_CUDA(cudaGetLastError());
  const double* hat = upool_.as<double>() + 2 * N_;
  d2h(xn, hat, sizeof(double) * n_, stream_);
  d2h(yn, hat + n_, sizeof(double) * m_, stream_);
  sync();
}

void Problem::kkt_metrics(int reduction, const double* x, const double* y, double* kkt,
                          double* lam) {
  enter();
  ensure_iter_buffers(AAPDHG_METHOD_PDHG, 1);
  upload_iterate(0, x, y);
  double* kd = scal_.as<double>() + 16;
  kkt_eval(0, resolve_serial(reduction), kd, lam_.as<double>());
  d2h(kkt, kd, 4 * sizeof(double), stream_);
  if (lam) d2h(lam, lam_.p, sizeof(double) * n_, stream_);
  sync();
}

// aa_apply (anderson.cpp:106-135) or build_filtered_memory + filtered_aa_apply
// (filtering.cpp:140-181) through the solver's own kernels. Returns an
// aapdhg_status (AAPDHG_ERR_SINGULAR for the reference's SingularError).
int Problem::aa_apply(int reduction, bool filtered, int p, const double* du_cols,
                      const double* dg_cols, double beta, const double* d_hat, double eta,
                      double c_s, double kappa_bar, const double* u, const double* g,
                      double* out, int32_t* kept) {
  return aa_op(reduction, filtered, p, du_cols, dg_cols, beta, d_hat, eta, c_s, kappa_bar, 0, u,
               g, out, kept, nullptr, nullptr);
}

// The AA / FAA step on caller-supplied columns (per-op entries): dots,
// k_aa_solve, then the candidate (out != null), the FAA kept set (kept),
// and for economy_qr the kept columns' R (r_out, p x p column-major) and
// Q = F R^{-1} (q_out, N x kk column-major). faa_skip: kFaaSkip* stages.
// u / g may be null when no candidate is formed (zeros).
int Problem::aa_op(int reduction, bool filtered, int p, const double* du_cols,
                   const double* dg_cols, double beta, const double* d_hat, double eta,
                   double c_s, double kappa_bar, int faa_skip, const double* u, const double* g,
                   double* out, int32_t* kept, double* r_out, double* q_out) {
  enter();
  if (p < 0) throw StatusError(AAPDHG_ERR_DIMENSION, "aa_apply: negative memory size");
  if (p > kMaxMemory)
    throw StatusError(AAPDHG_ERR_UNSUPPORTED, "aa_apply: memory larger than supported");
  if (d_hat)
    for (int64_t i = 0; i < N_; ++i)
      if (d_hat[i] <= 0.0) throw StatusError(AAPDHG_ERR_INPUT, "aa: d_hat entries must be > 0");
  const int method = filtered ? AAPDHG_METHOD_FAA : AAPDHG_METHOD_AA;
  const bool serial = resolve_serial(reduction);
  ensure_iter_buffers(method, std::max(p, 1));
  if (du_cols) h2d(du_.p, du_cols, sizeof(double) * size_t(p) * N_, stream_);
  else AAPDHG_CUDA(cudaMemsetAsync(du_.p, 0, sizeof(double) * size_t(std::max(p, 1)) * N_, stream_));
  h2d(dg_.p, dg_cols, sizeof(double) * size_t(p) * N_, stream_);
  if (g) h2d(gpool_.p, g, sizeof(double) * N_, stream_);
  else AAPDHG_CUDA(cudaMemsetAsync(gpool_.p, 0, sizeof(double) * N_, stream_));
  if (u) h2d(upool_.p, u, sizeof(double) * N_, stream_);
  else AAPDHG_CUDA(cudaMemsetAsync(upool_.p, 0, sizeof(double) * N_, stream_));
  if (d_hat) {
    dhat_.reserve(sizeof(double) * N_);
    h2d(dhat_.p, d_hat, sizeof(double) * N_, stream_);
  }
  DevParams P{};
  P.method = method;
  P.serial = serial ? 1 : 0;
  P.m1 = m1_;
  P.n = n_;
  P.mrows = m_;
  P.cap = std::max(p, 1);
  P.N = N_;
  P.Nglob = nglob_;
  P.beta = beta;
  P.eta = eta;
  P.c_s = c_s;
  P.kappa_bar = kappa_bar;
  P.d_hat = d_hat ? dhat_.as<double>() : nullptr;
  P.rec = rec_.as<aapdhg_record>();
  P.rec_cap = rec_cap_;
  P.ndot_blk = ndot_tile_;
  P.faa_skip = faa_skip;
  if (r_out) {
    gram_.reserve(sizeof(double) * kMaxMemory * kMaxMemory);
    P.qr_r_out = gram_.as<double>();
  }
  DevState S = identity_state();
  S.aa_attempt = 1;
  S.mem_size = p;
  for (int t = 0; t < p; ++t) S.mem_slots[t] = t;
  h2d(dparams_.p, &P, sizeof P, stream_);
  h2d(dstate_.p, &S, sizeof S, stream_);
  DotBufs D{du_.as<double>(), dg_.as<double>(), gpool_.as<double>(), partdot_.as<double>(),
            num_items_host(std::max(p, 1), method)};
  D.part_lo = faa_part_lo(method, std::max(p, 1));
  SolveScratch W{gram_.as<double>(), work_.as<double>(), vec_.as<double>()};
  IterBufs B = iter_bufs();
  const DevParams* Pd = dparams_.as<DevParams>();
  DevState* Sd = dstate_.as<DevState>();
  const int items = num_items_host(p, method);
  if (items > 0) {
    if (serial) {
      k_serial_dots<<<(items * 32 + kThreads - 1) / kThreads, kThreads, 0, stream_>>>(D, Pd, Sd);
    } else {
      k_tree_dots<<<ndot_tile_, kThreads, 0, stream_>>>(D, Pd, Sd);
    }
  }
  k_aa_solve<<<1, 1024, aa_smem(std::max(p, 1)), stream_>>>(D, Pd, Sd, 1);
  if (out) k_mix<<<grid_for(N_), kThreads, 0, stream_>>>(B, dg_.as<double>(), Pd, Sd, 0);
  AAPDHG_CUDA(cudaGetLastError());
  d2h(h_state_, Sd, sizeof(DevState), stream_);
  sync();
  if (!h_state_->aa_ok) return AAPDHG_ERR_SINGULAR;
  if (out) d2h(out, upool_.as<double>() + 3 * N_, sizeof(double) * N_, stream_);
  const int kk = h_state_->mix_p;
  if (r_out && kk > 0) {
    d2h(r_out, gram_.p, sizeof(double) * size_t(kk) * kk, stream_);
    if (q_out) {  // Q = F_kept R^{-1}; the kept columns are memory slots mix_slots[]
      std::vector<int32_t> sl(h_state_->mix_slots, h_state_->mix_slots + kk);
      bool contiguous = true;
      for (int t = 0; t < kk; ++t) contiguous = contiguous && sl[size_t(t)] == t;
      if (!contiguous) throw StatusError(AAPDHG_ERR_INTERNAL, "economy_qr: columns were filtered");
      k_qr_q<<<grid_for(N_), kThreads, 0, stream_>>>(dg_.as<double>(), gram_.as<double>(), kk,
                                                      N_, du_.as<double>());
      AAPDHG_CUDA(cudaGetLastError());
      d2h(q_out, du_.p, sizeof(double) * size_t(kk) * N_, stream_);
    }
  }
  sync();
  if (kept) {
    for (int t = 0; t < p; ++t) kept[t] = 0;
    for (int t = 0; t < h_state_->mix_p; ++t) kept[h_state_->mix_slots[t]] = 1;
  }
  return AAPDHG_OK;
}

// ===========================================================================
// Sharded solve: one Problem per shard, phases driven in lockstep by
// ShardGroup (shard.cu) with all-gathers in between (shard.cuh)
// ===========================================================================

Problem::Problem(const ShardSpec& sp, int device) : device_(device) {
  init_device(device);
  shard_rank_ = sp.rank;
  n_ = sp.n_loc;
  m_ = sp.m_loc;
  m1_ = sp.m1_loc;
  nnz_ = sp.k_rp.empty() ? 0 : sp.k_rp.back();
  N_ = int64_t(n_) + m_;
  nglob_ = sp.n_glob + sp.m_glob;
  maxc_ = sp.maxc;
  maxr_ = sp.maxr;
  all_zero_ = sp.all_zero;
  bounds_ok_ = sp.bounds_ok;
  if (sp.dev) {  // blocks built on this device (shard_build.cu)
    nnz_ = sp.dev->k_nnz;
    upload_csr(sp.dev->k_rp.as<int32_t>(), sp.dev->k_ci.as<int32_t>(), sp.dev->k_v.as<double>(),
               m_, int(sp.world * sp.maxc), k_store_, Ks_, Kt_, sp.dev->k_nnz);
    upload_csr(sp.dev->t_rp.as<int32_t>(), sp.dev->t_ci.as<int32_t>(), sp.dev->t_v.as<double>(),
               n_, int(sp.world * sp.maxr), t_store_, KTs_, KTt_, sp.dev->t_nnz);
  } else {
    upload_csr(sp.k_rp.data(), sp.k_ci.data(), sp.k_v.data(), m_, int(sp.world * sp.maxc),
               k_store_, Ks_, Kt_);
    upload_csr(sp.t_rp.data(), sp.t_ci.data(), sp.t_v.data(), n_, int(sp.world * sp.maxr),
               t_store_, KTs_, KTt_);
  }
  // (relabelled indices stay ascending within a row: column blocks are in order)
  build_blocks(k_store_, m_, int(sp.world * sp.maxc), kb_);
  build_blocks(t_store_, n_, int(sp.world * sp.maxr), ktb_);
  upload_vectors(sp.c.data(), sp.q.data(), sp.l.data(), sp.u.data());
  init_vectors();
  nrm_q_[0] = nrm_q_[1] = sp.nrm_q;
  nrm_c_[0] = nrm_c_[1] = sp.nrm_c;
  serial_norms_ = true;
  const int64_t W = sp.world;
  xg_.reserve(sizeof(double) * W * maxc_);
  yg_.reserve(sizeof(double) * W * maxr_);
  lg_.reserve(sizeof(double) * W * maxc_);
  scal_all_.reserve(sizeof(double) * W * 8);
  // the dots exchange buffer at its largest (peers may hold its address)
  dots_all_.reserve(sizeof(double) * size_t(W) * size_t(num_items_host(kMaxMemory, AAPDHG_METHOD_FAA)));
  p2p_flags_.reserve(sizeof(unsigned long long) * 8 * kMaxPeers);
  AAPDHG_CUDA(cudaMemsetAsync(p2p_flags_.p, 0, p2p_flags_.bytes, stream_));
  AAPDHG_CUDA(cudaMemsetAsync(xg_.p, 0, xg_.bytes, stream_));
  AAPDHG_CUDA(cudaMemsetAsync(yg_.p, 0, yg_.bytes, stream_));
  AAPDHG_CUDA(cudaMemsetAsync(lg_.p, 0, lg_.bytes, stream_));
  AAPDHG_CUDA(cudaMemsetAsync(scal_all_.p, 0, scal_all_.bytes, stream_));
  shard_world_ = sp.world;
  sync();
}

ShardBufs Problem::shard_bufs() const {
  return ShardBufs{xg_.as<double>(),    yg_.as<double>(), lg_.as<double>(),
                   scal_all_.as<double>(), dots_all_.as<double>(),
                   p2p_flags_.as<unsigned long long>(), maxc_, maxr_, dot_stride_};
}

// P2P transports: every shard's exchange buffers, indexed by rank (this
// shard's own entry included). The producers then write this shard's chunk
// into all of them and the exchanges become flag barriers (k_p2p_barrier).
void Problem::sh_set_peers(const std::vector<ShardBufs>& peers, bool remote) {
  if (peers.size() > size_t(kMaxPeers))
    throw StatusError(AAPDHG_ERR_UNSUPPORTED, "p2p: more than 8 shards");
  peers_ = peers;
  peers_remote_ = remote;
}

void Problem::sh_p2p_barrier(int slot, int phase) {
  k_p2p_barrier<<<1, 32, 0, stream_>>>(sh_su_->P, sh_su_->S, slot, phase);
  AAPDHG_CUDA(cudaGetLastError());
  ++sh_launches_;
}

void Problem::sh_begin(const aapdhg_solve_params* prm, double tau, double sigma,
                       const double* x0, const double* y0, const double* d_hat,
                       double wall_offset) {
  enter();
  const int method = prm->method;
  const int cap = method == AAPDHG_METHOD_PDHG ? 0 : int(prm->m);
  ensure_iter_buffers(method, std::max(cap, 1));
  dot_stride_ = num_items_host(std::max(cap, 1), AAPDHG_METHOD_FAA);  // (<= the reserved stride)
  if (d_hat) {
    dhat_.reserve(sizeof(double) * std::max<int64_t>(N_, 1));
    h2d(dhat_.p, d_hat, sizeof(double) * N_, stream_);
  }
  // the safeguard table for every i the solve can reach (cached across solves)
  if (method != AAPDHG_METHOD_PDHG)
    ensure_pow_table(prm->safeguard_eps,
                     (prm->max_iters >= kPowTabMax ? kPowTabMax : prm->max_iters) + 1);
  DevParams P{};
  P.method = method;
  P.serial = 0;
  P.m1 = m1_;
  P.kkt_terminate = prm->kkt_terminate ? 1 : 0;
  P.n = n_;
  P.mrows = m_;
  P.cap = cap;
  P.N = N_;
  P.Nglob = nglob_;
  P.safeguard_d = prm->safeguard_d;
  P.safeguard_eps = prm->safeguard_eps;
  P.beta = prm->beta;
  P.eta = prm->eta;
  P.c_s = prm->c_s;
  P.kappa_bar = prm->kappa_bar;
  P.toll = prm->toll;
  P.kkt_eps = prm->kkt_eps;
  P.tau = tau;
  P.sigma = sigma;
  P.max_iters = prm->max_iters;
  P.max_wall_s = prm->max_wall_seconds;
  P.wall_offset_s = wall_offset;
  P.nrm_q = nrm_q_[1];
  P.nrm_c = nrm_c_[1];
  P.d_hat = d_hat ? dhat_.as<double>() : nullptr;
  P.pow_tab = method == AAPDHG_METHOD_PDHG ? nullptr : pow_tab_.as<double>();
  P.pow_len = method == AAPDHG_METHOD_PDHG ? 0 : pow_len_;
  P.rec = rec_.as<aapdhg_record>();
  P.rec_cap = rec_cap_;
  P.nblk1 = sh_k1m().grid();
  P.nblk2 = sh_k2m().grid();
  P.ndot_blk = ndot_tile_;
  P.use_cond = 0;
  P.xgather = xg_.as<double>();
  P.ygather = yg_.as<double>();
  // this shard's chunk of the exchange buffers: its own (then all-gathered)
  // or, P2P, every shard's (then a flag barrier)
  std::vector<ShardBufs> dst = peers_;
  if (dst.empty()) dst.push_back(shard_bufs());
  P.ndst = int32_t(dst.size());
  for (size_t q = 0; q < dst.size(); ++q) {
    P.xg_dst[q] = dst[q].xg + int64_t(shard_rank_) * maxc_;
    P.yg_dst[q] = dst[q].yg + int64_t(shard_rank_) * maxr_;
    P.scal_dst[q] = dst[q].scal + int64_t(shard_rank_) * 8;
    P.dots_dst[q] = dst[q].dots + int64_t(shard_rank_) * dot_stride_;
  }
  P.p2p_epoch = ++p2p_epoch_;
  P.p2p_fused = peers_.empty() ? 0 : 1;
  P.p2p_world = int32_t(peers_.size());
  P.p2p_rank = shard_rank_;
  for (size_t q = 0; q < peers_.size(); ++q) P.flag_peer[q] = peers_[q].flags;
  P.flag_own = p2p_flags_.as<unsigned long long>();
  P.p2p_sys = peers_remote_ && peers_.size() > 1 ? 1 : 0;
  P.store_T = 1;

  DevState S0 = DevState{};
  S0.prev_plain = 1;
  for (int r = 0; r < 4; ++r) S0.u_idx[r] = r;
  for (int r = 0; r < 3; ++r) S0.kx_idx[r] = r;
  S0.g_idx[0] = 0;
  S0.g_idx[1] = 1;
  DevState* S = dstate_.as<DevState>();

  if (!sh_su_) sh_su_ = new SolveSetup{};
  SolveSetup& su = *sh_su_;
  su.B = iter_bufs();
  su.B.nu1 = sh_k1m().grid();
  su.B.fused_ctrl = 2;  // K2's last CTA writes this shard's totals (P.scal_dst)
  su.B.p2p_sys = P.p2p_sys;
  su.B.rinit1 = ktb_.nb() > 1 ? ktb_.partial.as<double>() : nullptr;
  su.B.rinit2 = kb_.nb() > 1 ? kb_.partial.as<double>() : nullptr;
  su.D = DotBufs{du_.as<double>(), dg_.as<double>(), gpool_.as<double>(),
                 partdot_.as<double>(), num_items_host(std::max(cap, 1), method)};
  su.D.part_lo = faa_part_lo(method, cap);
  su.W = SolveScratch{gram_.as<double>(), work_.as<double>(), vec_.as<double>()};
  su.P = dparams_.as<DevParams>();
  su.S = S;
  su.serial = false;
  su.push = method != AAPDHG_METHOD_PDHG;
  su.method = method;
  su.cap = cap;
  su.nblk1 = sh_k1m().grid();
  su.nblk2 = sh_k2m().grid();
  su.ndot_blk = ndot_tile_;
  su.items_max = num_items_host(std::max(cap, 1), method);

  AAPDHG_CUDA(cudaMemsetAsync(upool_.p, 0, sizeof(double) * 4 * N_, stream_));
  if (method != AAPDHG_METHOD_PDHG)
    AAPDHG_CUDA(cudaMemsetAsync(gpool_.p, 0, sizeof(double) * 2 * N_, stream_));
  upload_iterate(0, x0, y0);
  sh_params_ = P;
  h2d(dparams_.p, &P, sizeof P, stream_);
  h2d(S, &S0, sizeof S0, stream_);
  k_project_start<<<grid_for(N_, kThreads, 1 << 30), kThreads, 0, stream_>>>(
      upool_.as<double>(), l_.as<double>(), u_.as<double>(), n_, N_, m1_, S);
  AAPDHG_CUDA(cudaGetLastError());
  sh_launches_ = 1;
}

// peers: into every P2P destination (else this shard's own buffer)
void Problem::sh_stage_x(int role, int mode, bool peers) {
  const bool to_peers = peers && !peers_.empty();
  const size_t nd = to_peers ? peers_.size() : 1;
  for (size_t q = 0; q < nd; ++q) {
    double* dst = to_peers ? peers_[q].xg : xg_.as<double>();
    k_stage<<<grid_for(n_), kThreads, 0, stream_>>>(upool_.as<double>(), role, N_, 0, n_,
                                                     dst + shard_rank_ * maxc_, sh_su_->S, mode);
    AAPDHG_CUDA(cudaGetLastError());
    ++sh_launches_;
  }
}

void Problem::sh_stage_y(int role, int mode, bool peers) {
  const bool to_peers = peers && !peers_.empty();
  const size_t nd = to_peers ? peers_.size() : 1;
  for (size_t q = 0; q < nd; ++q) {
    double* dst = to_peers ? peers_[q].yg : yg_.as<double>();
    k_stage<<<grid_for(m_), kThreads, 0, stream_>>>(upool_.as<double>(), role, N_, n_, m_,
                                                     dst + shard_rank_ * maxr_, sh_su_->S, mode);
    AAPDHG_CUDA(cudaGetLastError());
    ++sh_launches_;
  }
}

void Problem::sh_init_kx() {
  sh_launches_ += spmv(stream_, Kt_, vref(xg_.as<double>()), rout(kxpool_.as<double>()), false,
                       nullptr, 0, nullptr);
}

void Problem::sh_k1() {
  const SolveSetup& su = *sh_su_;
  if (ktb_.nb() > 1) sh_launches_ += launch_blocked_passes(stream_, ktb_, vref(yg_.as<double>()), su.S);
  const CsrDev& A = sh_k1m();
  if (su.push)
    launch_k1<false, true>(A, su.B, su.P, su.S, stream_);
  else
    launch_k1<false, false>(A, su.B, su.P, su.S, stream_);
  AAPDHG_CUDA(cudaGetLastError());
  ++sh_launches_;
}

void Problem::sh_k2_totals() {
  const SolveSetup& su = *sh_su_;
  if (kb_.nb() > 1) sh_launches_ += launch_blocked_passes(stream_, kb_, vref(xg_.as<double>()), su.S);
  const CsrDev& A = sh_k2m();
  if (su.push)
    k2_kernel<false, true>(A)<<<A.grid(), kThreads, 0, stream_>>>(A, su.B, su.P, su.S);
  else
    k2_kernel<false, false>(A)<<<A.grid(), kThreads, 0, stream_>>>(A, su.B, su.P, su.S);
  AAPDHG_CUDA(cudaGetLastError());
  ++sh_launches_;  // (its last CTA writes this shard's totals: fused_ctrl = 2)
}

// The sharded graph's IF (AA branch) / WHILE (batch) conditions, set by the
// replicated control of every shard (identical decisions on every shard).
void Problem::sh_set_conditions(cudaGraphConditionalHandle aa, cudaGraphConditionalHandle loop) {
  sh_params_.use_cond = (aa || loop) ? 1 : 0;
  sh_params_.cond_aa = aa;
  sh_params_.cond_loop = loop;
  h2d(dparams_.p, &sh_params_, sizeof sh_params_, stream_);
  sync();
}

void Problem::sh_set_batch(int32_t left) {
  h_batch_[0] = left;
  h2d(&sh_su_->S->batch_left, h_batch_, sizeof(int32_t), stream_);
}

void Problem::sh_control(int world) {
  k_control_dist<<<1, 128, 0, stream_>>>(scal_all_.as<double>(), world, sh_su_->P, sh_su_->S);
  AAPDHG_CUDA(cudaGetLastError());
  ++sh_launches_;
}

void Problem::sh_read_state(DevState* out) {
  d2h(h_state_, sh_su_->S, sizeof(DevState), stream_);
  sync();
  *out = *h_state_;
}

void Problem::sh_aa_dots() {
  const SolveSetup& su = *sh_su_;
  k_stage_g<<<grid_for(N_), kThreads, 0, stream_>>>(su.B.upool, su.B.gpool, su.P, su.S);
  ++sh_launches_;
  k_tree_dots<<<su.ndot_blk, kThreads, 0, stream_>>>(su.D, su.P, su.S);
  k_dot_totals<<<1, 1024, 0, stream_>>>(su.D, su.P, su.S);
  AAPDHG_CUDA(cudaGetLastError());
  sh_launches_ += 2;
}

void Problem::sh_aa_solve_mix(int world) {
  const SolveSetup& su = *sh_su_;
  k_aa_solve<<<1, 1024, aa_smem(su.cap), stream_>>>(su.D, su.P, su.S, 0, dots_all_.as<double>(),
                                                     world, int(dot_stride_));
  k_mix<<<grid_for(N_), kThreads, 0, stream_>>>(su.B, su.B.dg, su.P, su.S, 1);
  AAPDHG_CUDA(cudaGetLastError());
  sh_launches_ += 2;
  sh_stage_x(U_CAND, 2, true);  // an accepted candidate replaces xhat / yhat in
  sh_stage_y(U_CAND, 2, true);  // the exchange chunks (K1 / K2 wrote those)
}

void Problem::sh_aa_recache_commit() {
  const SolveSetup& su = *sh_su_;
  RowsumArgs r{};
  r.out_pool = su.B.kxpool;
  r.out_role = KX_CAND;
  r.out_stride = m_;
  sh_launches_ += spmv(stream_, Kt_, vref(xg_.as<double>()), r, false, su.S, 1, nullptr);
  k_aa_commit<<<1, 128, 0, stream_>>>(su.P, su.S);
  AAPDHG_CUDA(cudaGetLastError());
  ++sh_launches_;
}

void Problem::sh_lambda() {
  k_lambda_from_T<<<grid_for(n_), kThreads, 0, stream_>>>(
      T_.as<double>(), c_.as<double>(), l_.as<double>(), u_.as<double>(), n_,
      lg_.as<double>() + shard_rank_ * maxc_);
  AAPDHG_CUDA(cudaGetLastError());
}

void Problem::sh_records(uint64_t from, uint64_t cnt, aapdhg_record* out) {
  const aapdhg_record* drec = rec_.as<aapdhg_record>();
  uint64_t got = 0;
  while (got < cnt) {
    const uint64_t pos = (from + got) % rec_cap_;
    const uint64_t chunk = std::min<uint64_t>(cnt - got, rec_cap_ - pos);
    d2h(out + got, drec + pos, chunk * sizeof(aapdhg_record), stream_);
    got += chunk;
  }
  sync();
}

// power_iteration_norm (sparse_linalg.cpp:95-123) phases of one shard
void Problem::sh_pw_init(const double* x0_loc) {
  enter();
  double* x = pw_x_.as<double>();
  h2d(x, x0_loc, sizeof(double) * n_, stream_);
  const int nb = grid_for(n_);
  double* part = part_small_.as<double>();
  k_sumsq_partials<<<nb, kThreads, 0, stream_>>>(x, nullptr, n_, part, nullptr);
  k_dot_final<<<1, kCtrlThreads, 0, stream_>>>(x, nullptr, n_, part, nb, 0,
                                                scal_all_.as<double>() + shard_rank_ * 8);
  AAPDHG_CUDA(cudaGetLastError());
}

void Problem::sh_pw_div(double by) {
  h2d(scal_.as<double>(), &by, sizeof(double), stream_);
  k_scale<<<grid_for(n_), kThreads, 0, stream_>>>(pw_x_.as<double>(), pw_x_.as<double>(), n_,
                                                   nullptr, scal_.as<double>());
  AAPDHG_CUDA(cudaGetLastError());
}

void Problem::sh_pw_stage_x() {
  AAPDHG_CUDA(cudaMemcpyAsync(xg_.as<double>() + shard_rank_ * maxc_, pw_x_.p,
                              sizeof(double) * n_, cudaMemcpyDeviceToDevice, stream_));
}

void Problem::sh_pw_kx() {
  spmv(stream_, Kt_, vref(xg_.as<double>()), rout(yg_.as<double>() + shard_rank_ * maxr_), false,
       nullptr, 0, nullptr);
}

void Problem::sh_pw_ktkx() {
  double* v = pw_mtmx_.as<double>();
  spmv(stream_, KTt_, vref(yg_.as<double>()), rout(v), false, nullptr, 0, nullptr);
  const int nb = grid_for(n_);
  double* part = part_small_.as<double>();
  k_sumsq_partials<<<nb, kThreads, 0, stream_>>>(v, nullptr, n_, part, nullptr);
  k_dot_final<<<1, kCtrlThreads, 0, stream_>>>(v, nullptr, n_, part, nb, 0,
                                                scal_all_.as<double>() + shard_rank_ * 8);
  AAPDHG_CUDA(cudaGetLastError());
}

void Problem::sh_pw_update(double lam) {
  h2d(scal_.as<double>() + 1, &lam, sizeof(double), stream_);
  k_scale<<<grid_for(n_), kThreads, 0, stream_>>>(pw_x_.as<double>(), pw_mtmx_.as<double>(), n_,
                                                   nullptr, scal_.as<double>() + 1);
  AAPDHG_CUDA(cudaGetLastError());
}

double Problem::sh_read_scal(int world, int q) {
  std::vector<double> v(size_t(world) * 8);
  d2h(v.data(), scal_all_.p, sizeof(double) * v.size(), stream_);
  sync();
  double s = v[size_t(q)];
  for (int r = 1; r < world; ++r) s += v[size_t(r) * 8 + q];
  return s;
}

}  // namespace aapdhg_b200

#ifdef AAPDHG_PLAIN_STAMPS
// experiment build only: k_plain_loop phases averaged over workers and
// iterations (ns): K1, bar 1 wait, K2, bar 2 wait; then the maxima of K1 and
// K2 over all workers and iterations, and the count
extern "C" int aapdhg_cuda_plain_stamps(double* out) {
  unsigned long long v[8];
  if (cudaMemcpyFromSymbol(v, aapdhg_b200::g_plain_dbg, sizeof v) != cudaSuccess) return -1;
  const double c = v[4] ? double(v[4]) : 1.0;
  for (int i = 0; i < 4; ++i) out[i] = v[i] / c;
  out[4] = double(v[5]);
  out[5] = double(v[6]);
  out[6] = c;
  unsigned long long z[8] = {};
  cudaMemcpyToSymbol(aapdhg_b200::g_plain_dbg, z, sizeof z);
  return 0;
}
#endif

#ifdef AAPDHG_PLAIN_STAMPS
// experiment build only: per worker CTA (up to 1024) the K1 / K2 phase sums
// (ns), the iteration count and the SM it ran on; reset after the read
extern "C" int aapdhg_cuda_plain_stamps_cta(double* out) {
  static unsigned long long v[1024 * 4];
  if (cudaMemcpyFromSymbol(v, aapdhg_b200::g_plain_cta, sizeof v) != cudaSuccess) return -1;
  for (int i = 0; i < 1024 * 4; ++i) out[i] = double(v[i]);
  static unsigned long long z[1024 * 4] = {};
  cudaMemcpyToSymbol(aapdhg_b200::g_plain_cta, z, sizeof z);
  return 0;
}
#endif

#ifdef AAPDHG_TIMELINE
// experiment build only: the (kernel id, globaltimer ns) entry stamps since
// the last read; returns their count
extern "C" int aapdhg_cuda_timeline(double* out, int max) {
  unsigned n = 0;
  if (cudaMemcpyFromSymbol(&n, aapdhg_b200::g_tl_n, sizeof n) != cudaSuccess) return -1;
  n = n > 8192 ? 8192 : n;
  static unsigned long long v[2 * 8192];
  cudaMemcpyFromSymbol(v, aapdhg_b200::g_tl, sizeof(unsigned long long) * 2 * n);
  const int k = int(n) < max ? int(n) : max;
  for (int i = 0; i < 2 * k; ++i) out[i] = double(v[i]);
  unsigned z = 0;
  cudaMemcpyToSymbol(aapdhg_b200::g_tl_n, &z, sizeof z);
  return k;
}
#endif

#ifdef AAPDHG_TAIL_STAMPS
// experiment build only: averaged phase times (ns) of the fused control tail
extern "C" int aapdhg_cuda_debug_stamps(double* out) {
  unsigned long long v[16];
  if (cudaMemcpyFromSymbol(v, aapdhg_b200::g_dbg, sizeof v) != cudaSuccess) return -1;
  const double c = v[5] ? double(v[5]) : 1.0, c9 = v[9] ? double(v[9]) : 1.0;
  out[0] = v[11] / c;  // persistent: K1 phase + barrier (CTA 0)
  out[1] = v[1] / c;   // persistent: barrier passed (CTA 0) -> election won
  out[2] = v[2] / c;   // -> partials reduced
  out[3] = v[3] / c;   // -> decided
  out[4] = v[4] / c;   // -> end of tail
  out[5] = v[8] / c9;  // -> next K1 start (plain step)
  out[6] = v[14] ? v[13] / double(v[14]) : 0.0;  // -> next K1 start (after the AA branch)
  out[7] = c;
  out[8] = v[9];
  out[9] = v[14];
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(aapdhg_b200::g_dbg, z, sizeof z);
  return 0;
}
#endif
