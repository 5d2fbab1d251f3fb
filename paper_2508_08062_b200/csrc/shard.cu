// shard.cu — host side of the sharded (multi-GPU) AA-PDHG solve.
//
// The LP is split into `world` shards (plan_partition): shard r owns K's row
// block R_r and column block C_r. Each iteration runs the single-GPU kernels
// on every shard in lockstep with three all-gathers in between — y before
// K'y, xhat before K xhat, the 8 scalar totals before the control — plus,
// on AA attempts, the dot totals and the candidate x. The
// row sums of K and K' are the unsplit CSR rows, so only the scalar sums
// differ from one GPU (in rank order, identical on every shard).
//
// Transports: NCCL (one shard per process, one GPU each; ncclAllGather in
// place on the solver's stream, the library loaded at first use) and
// LOOPBACK (all shards in this process on one device; the all-gathers are
// device copies on one stream — a test vehicle for the partitioned kernels
// that needs no peer GPU and no kernel ever waits on another).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "shard.h"

namespace aapdhg_b200 {

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

// ---- NCCL, resolved at first use (single-GPU handles never load it) --------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString =
        reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy && a.GetErrorString;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  if (!api.ok) throw StatusError(AAPDHG_ERR_UNSUPPORTED, "NCCL unavailable: " + api.why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

void nccl_unique_id(uint8_t* out, size_t len) {
  if (len < sizeof(ncclUniqueId))
    throw StatusError(AAPDHG_ERR_INPUT, "nccl_id: buffer shorter than AAPDHG_NCCL_ID_BYTES");
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
}

// Greedy prefix split: bound r is the first index whose weight prefix
// reaches r/world of the total, nudged so every block is non-empty.
static std::vector<int32_t> split_weights(const std::vector<int64_t>& w, int world) {
  const int n = int(w.size());
  std::vector<int64_t> pre(size_t(n) + 1, 0);
  for (int i = 0; i < n; ++i) pre[i + 1] = pre[i] + w[i];
  std::vector<int32_t> b(size_t(world) + 1, 0);
  b[world] = n;
  int i = 0;
  for (int r = 1; r < world; ++r) {
    const int64_t target = (pre[n] * r + world / 2) / world;
    while (i < n && pre[i] < target) ++i;
    int v = std::max(i, b[r - 1] + 1);
    v = std::min(v, n - (world - r));
    b[r] = v;
  }
  return b;
}

// row weights from row_ptr (nnz + 4 per row), column weights given
Partition plan_partition_weights(const aapdhg_csr_view& k, const std::vector<int64_t>& wc,
                                 int world) {
  Partition p;
  std::vector<int64_t> wr(static_cast<size_t>(k.nrows));
  for (int r = 0; r < k.nrows; ++r) wr[r] = int64_t(k.row_ptr[r + 1] - k.row_ptr[r]) + 4;
  p.rows = split_weights(wr, world);
  p.cols = split_weights(wc, world);
  for (int r = 0; r < world; ++r) {
    p.maxr = std::max<int64_t>(p.maxr, p.rows[r + 1] - p.rows[r]);
    p.maxc = std::max<int64_t>(p.maxc, p.cols[r + 1] - p.cols[r]);
  }
  return p;
}

Partition plan_partition(const aapdhg_csr_view& k, int world) {
  Partition p;
  std::vector<int64_t> wr(static_cast<size_t>(k.nrows)), wc(static_cast<size_t>(k.ncols), 4);
  for (int r = 0; r < k.nrows; ++r) wr[r] = int64_t(k.row_ptr[r + 1] - k.row_ptr[r]) + 4;
  for (int64_t e = 0; e < k.nnz; ++e) wc[size_t(k.col_idx[e])] += 1;
  p.rows = split_weights(wr, world);
  p.cols = split_weights(wc, world);
  for (int r = 0; r < world; ++r) {
    p.maxr = std::max<int64_t>(p.maxr, p.rows[r + 1] - p.rows[r]);
    p.maxc = std::max<int64_t>(p.maxc, p.cols[r + 1] - p.cols[r]);
  }
  return p;
}

ShardGroup::ShardGroup(const aapdhg_problem_view* v, int device, const aapdhg_dist_view* d)
    : device_(device) {
  // the shards' blocks are built on the device (shard_build.cu) unless
  // AAPDHG_SHARD_HOST_BUILD=1 asks for the host builder below
  const char* hb = std::getenv("AAPDHG_SHARD_HOST_BUILD");
  const bool host_build = hb && hb[0] == '1';
  if (host_build) validate_problem_view(v);
  else validate_problem_header(v);
  if (!d) throw StatusError(AAPDHG_ERR_INPUT, "problem_create_dist: null dist");
  const aapdhg_csr_view& k = v->k;
  world_ = d->world;
  transport_ = d->transport;
  rank_ = d->rank;
  n_ = k.ncols;
  m_ = k.nrows;
  m1_ = v->m1;
  nnz_ = k.nnz;
  if (transport_ < AAPDHG_DIST_NCCL || transport_ > AAPDHG_DIST_LOOPBACK_P2P)
    throw StatusError(AAPDHG_ERR_INPUT, "problem_create_dist: unknown transport");
  multi_ = transport_ == AAPDHG_DIST_NCCL || transport_ == AAPDHG_DIST_P2P;
  p2p_ = transport_ == AAPDHG_DIST_P2P || transport_ == AAPDHG_DIST_LOOPBACK_P2P;
  if (p2p_ && world_ > kMaxPeers)
    throw StatusError(AAPDHG_ERR_UNSUPPORTED, "problem_create_dist: P2P transports take <= 8 shards");
  if (world_ < 1) throw StatusError(AAPDHG_ERR_INPUT, "problem_create_dist: world < 1");
  if (multi_ && (rank_ < 0 || rank_ >= world_))
    throw StatusError(AAPDHG_ERR_INPUT, "problem_create_dist: rank out of range");
  if (multi_ && !d->nccl_id)
    throw StatusError(AAPDHG_ERR_INPUT, "problem_create_dist: NCCL / P2P transports need nccl_id");
  if (world_ > std::min(n_, m_))
    throw StatusError(AAPDHG_ERR_UNSUPPORTED,
                      "problem_create_dist: every shard needs at least one row and one column");

  // device build: the whole CSR on this rank's GPU once (checked there),
  // column weights from a device histogram
  DeviceLp dlp;
  cudaStream_t bs = nullptr;
  if (!host_build) {
    AAPDHG_CUDA(cudaSetDevice(device));
    AAPDHG_CUDA(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking));
    dlp.upload(k, device, bs);
    part_ = plan_partition_weights(k, dlp.column_weights(bs), world_);
  } else {
    part_ = plan_partition(k, world_);
  }
  std::vector<int32_t> trp, tci;
  std::vector<double> tv;
  if (host_build) transpose_csr(k, trp, tci, tv);

  // ||q||, ||c|| once on the host (sequential): identical on every shard
  double qq = 0.0, cc = 0.0;
  for (int i = 0; i < m_; ++i) qq += v->q[i] * v->q[i];
  for (int j = 0; j < n_; ++j) cc += v->c[j] * v->c[j];
  all_zero_ = true;
  if (host_build)
    for (int64_t e = 0; e < nnz_ && all_zero_; ++e) all_zero_ = k.vals[e] == 0.0;
  else
    all_zero_ = dlp.all_zero;
  bounds_ok_ = true;
  for (int j = 0; j < n_; ++j)
    if (v->l[j] > v->u[j]) bounds_ok_ = false;

  // owner-relative indices in the padded all-gather buffers (host build)
  std::vector<int32_t> xmap(static_cast<size_t>(host_build ? n_ : 0)),
      ymap(static_cast<size_t>(host_build ? m_ : 0));
  for (int r = 0; r < world_ && host_build; ++r) {
    for (int j = part_.cols[r]; j < part_.cols[r + 1]; ++j)
      xmap[j] = int32_t(r * part_.maxc + (j - part_.cols[r]));
    for (int i = part_.rows[r]; i < part_.rows[r + 1]; ++i)
      ymap[i] = int32_t(r * part_.maxr + (i - part_.rows[r]));
  }
  if (int64_t(world_) * std::max(part_.maxc, part_.maxr) > INT32_MAX)
    throw StatusError(AAPDHG_ERR_UNSUPPORTED, "problem_create_dist: padded index overflow");

  std::vector<int> ranks;
  if (multi_) ranks.push_back(rank_);
  else
    for (int r = 0; r < world_; ++r) ranks.push_back(r);
  for (int r : ranks) {
    ShardSpec sp;
    sp.rank = r;
    sp.world = world_;
    const int r0 = part_.rows[r], r1 = part_.rows[r + 1];
    const int c0 = part_.cols[r], c1 = part_.cols[r + 1];
    sp.n_loc = c1 - c0;
    sp.m_loc = r1 - r0;
    sp.m1_loc = std::max(0, std::min(m1_ - r0, sp.m_loc));
    sp.maxc = part_.maxc;
    sp.maxr = part_.maxr;
    sp.n_glob = n_;
    sp.m_glob = m_;
    DeviceShardBlocks blocks;
    if (!host_build) {
      dlp.shard_blocks(part_, world_, r, bs, blocks);
      sp.dev = &blocks;
    }
    if (host_build) sp.k_rp.assign(size_t(sp.m_loc) + 1, 0);
    for (int i = r0; i < r1 && host_build; ++i) {
      for (int32_t e = k.row_ptr[i]; e < k.row_ptr[i + 1]; ++e) {
        sp.k_ci.push_back(xmap[size_t(k.col_idx[e])]);
        sp.k_v.push_back(k.vals[e]);
      }
      sp.k_rp[size_t(i - r0) + 1] = int32_t(sp.k_ci.size());
    }
    if (host_build) sp.t_rp.assign(size_t(sp.n_loc) + 1, 0);
    for (int j = c0; j < c1 && host_build; ++j) {
      for (int32_t e = trp[j]; e < trp[j + 1]; ++e) {
        sp.t_ci.push_back(ymap[size_t(tci[e])]);
        sp.t_v.push_back(tv[e]);
      }
      sp.t_rp[size_t(j - c0) + 1] = int32_t(sp.t_ci.size());
    }
    sp.c.assign(v->c + c0, v->c + c1);
    sp.l.assign(v->l + c0, v->l + c1);
    sp.u.assign(v->u + c0, v->u + c1);
    sp.q.assign(v->q + r0, v->q + r1);
    sp.nrm_q = std::sqrt(qq);
    sp.nrm_c = std::sqrt(cc);
    sp.all_zero = all_zero_;
    sp.bounds_ok = bounds_ok_;
    shards_.emplace_back(new Problem(sp, device));
  }
  if (bs) {
    cudaStreamSynchronize(bs);
    cudaStreamDestroy(bs);
  }
  AAPDHG_CUDA(cudaSetDevice(device));
  if (!multi_) {
    AAPDHG_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
    stream_ = own_stream_;
    each([&](Problem& s) { s.set_stream(stream_); });
  } else {
    stream_ = shards_[0]->stream();
    ncclUniqueId id;
    std::memcpy(&id, d->nccl_id, sizeof id);
    ncclComm_t comm = nullptr;
    nccl_check(nccl().CommInitRank(&comm, world_, id, rank_), "ncclCommInitRank");
    comm_ = comm;
  }
  if (p2p_) open_peers();
}

// P2P transports: every shard's exchange buffers as pointers this process can
// store to. Loopback: the other in-process shards' buffers. One shard per
// process: CUDA IPC handles of xg / yg / scal / dots / flags, all-gathered
// once over NCCL, opened with peer access (NVLink / NVSwitch).
void ShardGroup::open_peers() {
  std::vector<ShardBufs> peers;
  if (!multi_) {
    for (auto& s : shards_) peers.push_back(s->shard_bufs());
    each([&](Problem& s) { s.sh_set_peers(peers, false); });
    return;
  }
  const ShardBufs mine = shards_[0]->shard_bufs();
  constexpr int NB = 5;
  struct Handles {
    cudaIpcMemHandle_t h[NB];
  };
  Handles hm{};
  void* bases[NB] = {mine.xg, mine.yg, mine.scal, mine.dots, mine.flags};
  for (int b = 0; b < NB; ++b) AAPDHG_CUDA(cudaIpcGetMemHandle(&hm.h[b], bases[b]));
  DevBuf dh;
  dh.reserve(sizeof(Handles) * size_t(world_));
  uint8_t* d = dh.as<uint8_t>();
  AAPDHG_CUDA(cudaMemcpyAsync(d + rank_ * sizeof(Handles), &hm, sizeof(Handles),
                              cudaMemcpyHostToDevice, stream_));
  nccl_check(nccl().AllGather(d + rank_ * sizeof(Handles), d, sizeof(Handles), ncclUint8,
                              static_cast<ncclComm_t>(comm_), stream_),
             "ncclAllGather(ipc handles)");
  std::vector<Handles> all(static_cast<size_t>(world_));
  AAPDHG_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(Handles) * all.size(), cudaMemcpyDeviceToHost,
                              stream_));
  AAPDHG_CUDA(cudaStreamSynchronize(stream_));
  for (int q = 0; q < world_; ++q) {
    if (q == rank_) {
      peers.push_back(mine);
      continue;
    }
    void* p[NB];
    for (int b = 0; b < NB; ++b) {
      AAPDHG_CUDA(cudaIpcOpenMemHandle(&p[b], all[size_t(q)].h[b], cudaIpcMemLazyEnablePeerAccess));
      ipc_opened_.push_back(p[b]);
    }
    ShardBufs sb = mine;
    sb.xg = static_cast<double*>(p[0]);
    sb.yg = static_cast<double*>(p[1]);
    sb.scal = static_cast<double*>(p[2]);
    sb.dots = static_cast<double*>(p[3]);
    sb.flags = static_cast<unsigned long long*>(p[4]);
    sb.lg = nullptr;  // (not exchanged over peer memory)
    peers.push_back(sb);
  }
  shards_[0]->sh_set_peers(peers, true);
}

// The in-loop exchanges: P2P transports only synchronise (the producers
// wrote every shard's buffer); otherwise the all-gather.
void ShardGroup::exchange(Buf b) {
  if (!p2p_) {
    allgather(b);
    return;
  }
  const int slot = int(b);
  if (multi_) {
    shards_[0]->sh_p2p_barrier(slot, 3);
  } else {  // in-process shards: every arrival first, then the waits
    each([&](Problem& s) { s.sh_p2p_barrier(slot, 1); });
    each([&](Problem& s) { s.sh_p2p_barrier(slot, 2); });
  }
}

ShardGroup::~ShardGroup() {
  if (stream_) cudaStreamSynchronize(stream_);
  for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
  if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
  shards_.clear();
  if (own_stream_) cudaStreamDestroy(own_stream_);
}

void ShardGroup::set_stream(cudaStream_t s) {
  AAPDHG_CUDA(cudaStreamSynchronize(stream_));
  stream_ = s ? s : (own_stream_ ? own_stream_ : nullptr);
  each([&](Problem& p) { p.set_stream(stream_); });
  if (!stream_) stream_ = shards_[0]->stream();
}

void ShardGroup::allgather(Buf b) {
  auto pick = [&](const ShardBufs& sb, int64_t& chunk) -> double* {
    switch (b) {
      case XG:
      case XG2: chunk = sb.maxc; return sb.xg;
      case YG: chunk = sb.maxr; return sb.yg;
      case LG: chunk = sb.maxc; return sb.lg;
      case SCAL: chunk = 8; return sb.scal;
      default: chunk = sb.dot_stride; return sb.dots;
    }
  };
  if (multi_) {
    int64_t chunk = 0;
    double* buf = pick(shards_[0]->shard_bufs(), chunk);
    nccl_check(nccl().AllGather(buf + rank_ * chunk, buf, size_t(chunk), ncclDouble,
                                static_cast<ncclComm_t>(comm_), stream_),
               "ncclAllGather");
    return;
  }
  std::vector<double*> bufs;
  int64_t chunk = 0;
  for (auto& s : shards_) bufs.push_back(pick(s->shard_bufs(), chunk));
  for (int dst = 0; dst < world_; ++dst)
    for (int src = 0; src < world_; ++src)
      if (src != dst)
        AAPDHG_CUDA(cudaMemcpyAsync(bufs[dst] + src * chunk, bufs[src] + src * chunk,
                                    sizeof(double) * size_t(chunk), cudaMemcpyDeviceToDevice,
                                    stream_));
}

// power_iteration_norm, sparse_linalg.cpp:95-123, with x sharded by column
// block: K x needs the all-gathered x, K'(K x) the all-gathered K x.
double ShardGroup::power_norm(int max_iters, double rel_tol, uint64_t seed) {
  if (all_zero_ || n_ == 0 || max_iters <= 0) return 0.0;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unif(-1.0, 1.0);
  std::vector<double> x0(static_cast<size_t>(n_));
  for (double& v : x0) v = unif(rng);
  each([&](Problem& s) { s.sh_pw_init(x0.data() + part_.cols[s.shard_rank()]); });
  allgather(SCAL);
  double xn = std::sqrt(shards_[0]->sh_read_scal(world_, 0));
  if (xn == 0.0) {  // x = e_0: column 0 lives on shard 0
    std::vector<double> e0(size_t(part_.cols[1] - part_.cols[0]), 0.0);
    e0[0] = 1.0;
    each([&](Problem& s) {
      if (s.shard_rank() == 0) s.sh_pw_init(e0.data());
    });
    xn = 1.0;
  }
  each([&](Problem& s) { s.sh_pw_div(xn); });
  double est = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    each([&](Problem& s) { s.sh_pw_stage_x(); });
    allgather(XG);
    each([&](Problem& s) { s.sh_pw_kx(); });
    allgather(YG);
    each([&](Problem& s) { s.sh_pw_ktkx(); });
    allgather(SCAL);
    const double lam = std::sqrt(shards_[0]->sh_read_scal(world_, 0));
    const double next = std::sqrt(lam);
    if (lam == 0.0) return 0.0;
    each([&](Problem& s) { s.sh_pw_update(lam); });
    if (it > 0 && std::abs(next - est) < rel_tol * next) return next;
    est = next;
  }
  return est;
}

// select_step_sizes, solver.cpp:112-123
void ShardGroup::select_step_sizes(const aapdhg_solve_params* prm, double* tau, double* sigma) {
  if (prm->tau > 0.0 || prm->sigma > 0.0) {
    if (!(prm->tau > 0.0 && prm->sigma > 0.0))
      throw StatusError(AAPDHG_ERR_INPUT, "step sizes: override requires both tau and sigma");
    *tau = prm->tau;
    *sigma = prm->sigma;
    return;
  }
  const double k_norm = power_norm(5000, 1e-4, 12345u);
  if (k_norm == 0.0) {
    *tau = *sigma = 1.0;
    return;
  }
  *tau = *sigma = 0.9 / k_norm;
}

void ShardGroup::solve(const aapdhg_solve_params* prm, const double* x0, const double* y0,
                       aapdhg_solve_result* res, double* x_out, double* y_out, double* lam_out,
                       aapdhg_record_sink sink, void* ctx) {
  const auto t_start = Clock::now();
  AAPDHG_CUDA(cudaSetDevice(device_));
  validate_config(prm);
  if (!bounds_ok_) throw StatusError(AAPDHG_ERR_INPUT, "build_lambda_set: l > u");
  const int method = prm->method;
  if (method != AAPDHG_METHOD_PDHG && prm->m > uint64_t(kMaxMemory))
    throw StatusError(AAPDHG_ERR_UNSUPPORTED,
                      "solver: memory capacity m > " + std::to_string(kMaxMemory) +
                          " is not supported by the sm_100a path");
  const int64_t N = int64_t(n_) + m_;
  if (prm->d_hat)
    for (int64_t i = 0; i < N; ++i)
      if (prm->d_hat[i] <= 0.0) throw StatusError(AAPDHG_ERR_INPUT, "aa: d_hat entries must be > 0");
  double tau, sigma;
  select_step_sizes(prm, &tau, &sigma);

  const double wall_offset = secs(t_start);
  each([&](Problem& s) {
    const int r = s.shard_rank();
    const int c0 = part_.cols[r], c1 = part_.cols[r + 1], r0 = part_.rows[r], r1 = part_.rows[r + 1];
    std::vector<double> dh;
    if (prm->d_hat) {
      dh.assign(prm->d_hat + c0, prm->d_hat + c1);
      dh.insert(dh.end(), prm->d_hat + n_ + r0, prm->d_hat + n_ + r1);
    }
    s.sh_begin(prm, tau, sigma, x0 ? x0 + c0 : nullptr, y0 ? y0 + r0 : nullptr,
               prm->d_hat ? dh.data() : nullptr, wall_offset);
  });
  // K x of the projected start iterate (slot 0)
  each([&](Problem& s) { s.sh_stage_x(-1, 0); });
  allgather(XG);
  each([&](Problem& s) { s.sh_init_kx(); });

  // One iteration: the core, then the AA branch. Preferred form: the same
  // graph as on one GPU — WHILE(batch) { core; IF(attempt) { AA branch } },
  // both conditions set by the replicated control, NCCL all-gathers captured
  // in the bodies — so the host launches one graph per batch. If the driver
  // or NCCL cannot capture that, fall back to one captured graph per
  // iteration with the AA branch predicated on the device (its all-gathers
  // then always run).
  // (P2P transports: the producers store into every shard's buffer and each
  // exchange is a flag barrier; the exchange points are where every shard
  // has finished reading the buffer's previous contents — DESIGN.md §8)
  // P2P: the plain iteration has no exchange launches at all — K1 waits for
  // the YG arrivals and arrives at XG, K2 waits for XG and arrives at YG (its
  // yhat and totals), the control waits for YG (fused signals, pipeline.cuh).
  // The AA branch keeps barrier kernels and ends with a YG arrival, so the
  // next K1 also waits for every shard's candidate (and its recache reads).
  auto core = [&] {
    if (!p2p_) allgather(YG);
    each([&](Problem& s) { s.sh_k1(); });
    if (!p2p_) allgather(XG);
    each([&](Problem& s) { s.sh_k2_totals(); });
    if (!p2p_) allgather(SCAL);
    each([&](Problem& s) { s.sh_control(world_); });
  };
  auto aa_branch = [&] {
    each([&](Problem& s) { s.sh_aa_dots(); });
    exchange(DOTS);
    each([&](Problem& s) { s.sh_aa_solve_mix(world_); });
    exchange(XG2);
    each([&](Problem& s) { s.sh_aa_recache_commit(); });
    if (p2p_) each([&](Problem& s) { s.sh_p2p_barrier(int(YG), 1); });
  };
  // y of the start iterate; afterwards K2 (yhat) or the accepted candidate
  // writes each shard's chunk
  each([&](Problem& s) { s.sh_stage_y(-1, 0); });
  if (p2p_) {
    allgather(YG);  // the start iterate's y, then the first YG arrival
    exchange(YG);
  }
  const char* ge = std::getenv("AAPDHG_SHARD_GRAPH");
  const int mode = ge && *ge ? std::atoi(ge) : 2;  // 2 WHILE/IF, 1 per iteration, 0 eager
  cudaGraphExec_t exec = nullptr;
  bool cond_graph = false;
  uint64_t core_nodes = 0, aa_nodes = 0;
  auto launches = [&] {
    uint64_t t = 0;
    each([&](Problem& s) { t += s.sh_launches(); });
    return t;
  };
  if (mode == 2) {
    cudaGraph_t g = nullptr;
    try {
      const cudaStreamCaptureMode cm = cudaStreamCaptureModeThreadLocal;
      AAPDHG_CUDA(cudaGraphCreate(&g, 0));
      cudaGraphConditionalHandle h_loop = 0, h_aa = 0;
      AAPDHG_CUDA(cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams wp{};
      wp.type = cudaGraphNodeTypeConditional;
      wp.conditional.handle = h_loop;
      wp.conditional.type = cudaGraphCondTypeWhile;
      wp.conditional.size = 1;
      cudaGraphNode_t wnode;
      AAPDHG_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
      cudaGraph_t body = wp.conditional.phGraph_out[0];
      uint64_t l0 = launches();
      AAPDHG_CUDA(cudaStreamBeginCaptureToGraph(stream_, body, nullptr, nullptr, 0, cm));
      core();
      cudaStreamCaptureStatus cst;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      AAPDHG_CUDA(cudaStreamGetCaptureInfo(stream_, &cst, nullptr, nullptr, &deps, &ndeps));
      std::vector<cudaGraphNode_t> tail(deps, deps + ndeps);
      cudaGraph_t cap = nullptr;
      AAPDHG_CUDA(cudaStreamEndCapture(stream_, &cap));
      core_nodes = launches() - l0;
      AAPDHG_CUDA(cudaGraphConditionalHandleCreate(&h_aa, body, 0, cudaGraphCondAssignDefault));
      cudaGraphNodeParams ip{};
      ip.type = cudaGraphNodeTypeConditional;
      ip.conditional.handle = h_aa;
      ip.conditional.type = cudaGraphCondTypeIf;
      ip.conditional.size = 1;
      cudaGraphNode_t inode;
      AAPDHG_CUDA(cudaGraphAddNode(&inode, body, tail.data(), tail.size(), &ip));
      l0 = launches();
      AAPDHG_CUDA(cudaStreamBeginCaptureToGraph(stream_, ip.conditional.phGraph_out[0], nullptr,
                                                nullptr, 0, cm));
      aa_branch();
      AAPDHG_CUDA(cudaStreamEndCapture(stream_, &cap));
      aa_nodes = launches() - l0;
      AAPDHG_CUDA(cudaGraphInstantiate(&exec, g, 0));
      each([&](Problem& s) { s.sh_set_conditions(h_aa, h_loop); });
      cond_graph = true;
    } catch (const CudaError&) {
      cudaStreamCaptureStatus cst;
      if (cudaStreamIsCapturing(stream_, &cst) == cudaSuccess &&
          cst != cudaStreamCaptureStatusNone) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(stream_, &junk);
        if (junk) cudaGraphDestroy(junk);
      }
      cudaGetLastError();
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
    }
    if (g) cudaGraphDestroy(g);
  }
  // Every rank must issue the same collective sequence: the WHILE/IF graph
  // runs the AA branch's exchanges only on attempts, the per-iteration graph
  // on every iteration. A rank whose capture failed (or whose environment
  // asks for another mode) would hang the others, so the ranks agree on the
  // smallest mode any of them can run before the loop (one all-gather of a
  // flag through this rank's chunk of the SCAL exchange buffer, idle here).
  int agreed = cond_graph ? 2 : (mode >= 1 ? 1 : 0);
  if (multi_ && world_ > 1) {
    const ShardBufs sb = shards_[0]->shard_bufs();
    std::vector<double> chunk(8, 0.0), all(size_t(world_) * 8, 0.0);
    chunk[0] = double(agreed);
    AAPDHG_CUDA(cudaMemcpyAsync(sb.scal + size_t(rank_) * 8, chunk.data(), sizeof(double) * 8,
                                cudaMemcpyHostToDevice, stream_));
    allgather(SCAL);
    AAPDHG_CUDA(cudaMemcpyAsync(all.data(), sb.scal, sizeof(double) * all.size(),
                                cudaMemcpyDeviceToHost, stream_));
    AAPDHG_CUDA(cudaStreamSynchronize(stream_));
    for (int r = 0; r < world_; ++r) agreed = std::min(agreed, int(all[size_t(r) * 8]));
  }
  if (cond_graph && agreed < 2) {
    cudaGraphExecDestroy(exec);
    exec = nullptr;
    cond_graph = false;
    each([&](Problem& s) { s.sh_set_conditions(0, 0); });  // no conditional nodes
  }
  if (!cond_graph && agreed >= 1) {
    const uint64_t l0 = launches();
    AAPDHG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    core();
    aa_branch();
    cudaGraph_t g = nullptr;
    AAPDHG_CUDA(cudaStreamEndCapture(stream_, &g));
    AAPDHG_CUDA(cudaGraphInstantiate(&exec, g, 0));
    cudaGraphDestroy(g);
    core_nodes = launches() - l0;
  }
  DevState st{};
  uint64_t flushed = 0;
  std::vector<aapdhg_record> recs;
  uint64_t batch = 8;
  for (;;) {
    if (cond_graph) {
      each([&](Problem& s) { s.sh_set_batch(int32_t(batch)); });
      AAPDHG_CUDA(cudaGraphLaunch(exec, stream_));
    } else {
      for (uint64_t b = 0; b < batch; ++b) {
        if (exec) AAPDHG_CUDA(cudaGraphLaunch(exec, stream_));
        else {
          core();
          aa_branch();
        }
      }
    }
    shards_[0]->sh_read_state(&st);
    if (st.rec_complete > flushed) {
      const uint64_t cnt = st.rec_complete - flushed;
      recs.resize(cnt);
      shards_[0]->sh_records(flushed, cnt, recs.data());
      if (sink) sink(recs.data(), cnt, ctx);
      flushed = st.rec_complete;
    }
    if (st.done) break;
    batch = std::min<uint64_t>(batch * 2, 4096);  // <= half the device record ring
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (cond_graph) {  // plain control again for later solves
    each([&](Problem& s) { s.sh_set_conditions(0, 0); });
  }
  const uint64_t graph_launches =
      cond_graph ? st.loop_iters * core_nodes + (st.i + st.aa_failures) * aa_nodes
                 : (exec ? st.loop_iters * core_nodes : 0);

  // finish, solver.cpp:153-166: the final iterate, K'y-based lambda; the KKT
  // of the final iterate is the one its own control step evaluated
  const int fr = st.final_role;
  each([&](Problem& s) {
    s.sh_stage_x(fr, 0);
    s.sh_stage_y(fr, 0);
    s.sh_lambda();
  });
  allgather(XG);
  allgather(YG);
  allgather(LG);
  const ShardBufs sb = shards_[0]->shard_bufs();
  auto unpad = [&](const double* dev, int64_t chunk, const std::vector<int32_t>& bounds,
                   double* out) {
    std::vector<double> h(size_t(world_) * size_t(chunk));
    AAPDHG_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(double) * h.size(), cudaMemcpyDeviceToHost,
                                stream_));
    AAPDHG_CUDA(cudaStreamSynchronize(stream_));
    for (int r = 0; r < world_; ++r)
      std::copy(h.begin() + r * chunk, h.begin() + r * chunk + (bounds[r + 1] - bounds[r]),
                out + bounds[r]);
  };
  if (x_out) unpad(sb.xg, sb.maxc, part_.cols, x_out);
  if (y_out) unpad(sb.yg, sb.maxr, part_.rows, y_out);
  if (lam_out) unpad(sb.lg, sb.maxc, part_.cols, lam_out);
  AAPDHG_CUDA(cudaStreamSynchronize(stream_));

  std::memset(res, 0, sizeof *res);
  res->status = st.status;
  res->iterations = st.i + st.j;
  res->i = st.i;
  res->j = st.j;
  res->aa_failures = st.aa_failures;
  res->g_norm = st.g_final;
  res->r_gap = st.kkt[0];
  res->r_primal = st.kkt[1];
  res->r_dual = st.kkt[2];
  res->objective = st.kkt[3];
  res->tau = tau;
  res->sigma = sigma;
  res->wall_seconds = secs(t_start);
  last_loop_iters_ = st.loop_iters;
  last_launches_ = 0;
  each([&](Problem& s) { last_launches_ += s.sh_launches(); });
  last_launches_ += graph_launches;
}

}  // namespace aapdhg_b200
