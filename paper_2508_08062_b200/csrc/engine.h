// engine.h — host side of the sm_100a solver: one Problem per handle.
#pragma once

#include <atomic>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "memory.h"

namespace aapdhg_b200 {

// Device allocation that frees itself.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
  void reserve(size_t b);  // grows, never shrinks (contents lost on growth)
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct KernelStat {
  double ms = 0.0;
  uint64_t launches = 0;
  std::vector<float> each;  // per-launch ms (predicated-off launches filtered at read)
};

struct SolveSetup;

void validate_problem_view(const aapdhg_problem_view* v);    // header + deep (host)
// CSR from triplets on the device (triplets.cu); returns nnz
int64_t csr_from_triplets(int device, int nrows_in, int nrows_out, int ncols, int64_t count,
                          const aapdhg_triplet* trip, const int32_t* row_map,
                          const uint8_t* row_neg, int32_t* rp_out, int32_t* ci_out,
                          double* v_out);
void validate_problem_header(const aapdhg_problem_view* v);  // O(1) host checks
const char* csr_flag_message(int flags);  // kCsr* flags -> the error message, or null
void validate_config(const aapdhg_solve_params* c);
void transpose_csr(const aapdhg_csr_view& k, std::vector<int32_t>& trp, std::vector<int32_t>& tci,
                   std::vector<double>& tv);

// O(nnz) checks of a CSR on the device (kCsr* flags; ingest.cu)
int device_validate_csr(const int32_t* rp, const int32_t* ci, const double* v, int nrows,
                        int ncols, int64_t nnz, cudaStream_t s);

// A shard's device-built blocks (shard_build.cu): K[R_r, :] with padded
// column labels and K[:, C_r]' with padded row labels.
struct DeviceShardBlocks {
  DevBuf k_rp, k_ci, k_v, t_rp, t_ci, t_v;
  int64_t k_nnz = 0, t_nnz = 0;
};

struct Partition;
// The whole LP's CSR on one device, for building shards there.
struct DeviceLp {
  DevBuf rp, ci, v;
  int nrows = 0, ncols = 0;
  int64_t nnz = 0;
  bool all_zero = true;
  void upload(const aapdhg_csr_view& k, int device, cudaStream_t s);  // + device checks
  std::vector<int64_t> column_weights(cudaStream_t s) const;          // nnz per column + 4
  void shard_blocks(const Partition& part, int world, int r, cudaStream_t s,
                    DeviceShardBlocks& out) const;
};

// One shard of a row/column-partitioned LP (shard.cuh): K's
// rows R_r with column indices relabelled into the padded x all-gather
// buffer, K's columns C_r (rows of K') with row indices relabelled into the
// padded y buffer, and the local slices of c, l, u (C_r) and q (R_r).
struct ShardSpec {
  int rank = 0, world = 1;
  int n_loc = 0, m_loc = 0, m1_loc = 0;
  int64_t maxc = 0, maxr = 0;  // chunk lengths of the x / y all-gather buffers
  int64_t n_glob = 0, m_glob = 0;
  std::vector<int32_t> k_rp, k_ci, t_rp, t_ci;
  std::vector<double> k_v, t_v;
  // or the blocks already on this shard's device (shard_build.cu)
  const DeviceShardBlocks* dev = nullptr;
  std::vector<double> c, l, u, q;
  double nrm_q = 0.0, nrm_c = 0.0;
  bool all_zero = false, bounds_ok = true;
};

// Device buffers a shard exchanges with its peers: chunk r of each belongs
// to shard r (all-gathered in place).
struct ShardBufs {
  double* xg;    // world x maxc: x-space vectors (xhat, candidates, power x)
  double* yg;    // world x maxr: y-space vectors
  double* lg;    // world x maxc: lambda of the final iterate
  double* scal;  // world x 8: per-shard iteration totals / power-iteration norms
  double* dots;  // world x dot_stride: per-shard AA dot totals
  unsigned long long* flags;  // P2P barrier arrivals: 8 exchanges x kMaxPeers shards
  int64_t maxc, maxr, dot_stride;
};

class Problem {
 public:
  Problem(const aapdhg_problem_view* v, int device);
  Problem(const ShardSpec& sp, int device);  // one shard of a sharded solve
  ~Problem();

  // ---- sharded solve phases (driven by ShardGroup, in lockstep) -------------
  ShardBufs shard_bufs() const;
  cudaStream_t stream() const { return stream_; }
  int device() const { return device_; }
  int shard_rank() const { return shard_rank_; }
  void sh_begin(const aapdhg_solve_params* prm, double tau, double sigma, const double* x0,
                const double* y0, const double* d_hat, double wall_offset);
  // x-part of an iterate -> this shard's chunk of xg (peers: of every P2P peer's)
  void sh_stage_x(int role, int mode, bool peers = false);
  void sh_stage_y(int role, int mode, bool peers = false);  // y-part -> yg
  // P2P transports; remote: the peers are other processes' GPUs (IPC)
  void sh_set_peers(const std::vector<ShardBufs>& peers, bool remote);
  void sh_p2p_barrier(int slot, int phase);                  // k_p2p_barrier
  void sh_init_kx();                    // K x of the start iterate (after AG of xg)
  void sh_k1();                         // K'y + xhat (+ own chunk of xg)
  void sh_k2_totals();                  // K xhat + yhat, then own iteration totals
  void sh_control(int world);           // after AG of scal
  void sh_set_conditions(cudaGraphConditionalHandle aa, cudaGraphConditionalHandle loop);
  void sh_set_batch(int32_t left);       // iterations the next graph launch may run
  void sh_read_state(DevState* out);    // synchronous
  void sh_aa_dots();                    // own dot totals (AA attempt)
  void sh_aa_solve_mix(int world);      // after AG of dots; candidate x -> xg
  void sh_aa_recache_commit();          // after AG of xg
  void sh_lambda();                     // lambda of the final iterate -> lg
  void sh_records(uint64_t from, uint64_t cnt, aapdhg_record* out);
  void sh_pw_init(const double* x0_loc);  // power x; own ||x||^2 -> scal
  void sh_pw_div(double by);              // x /= by
  void sh_pw_stage_x();                   // x -> own chunk of xg
  void sh_pw_kx();                        // K xg -> own chunk of yg
  void sh_pw_ktkx();                      // K' yg -> mtmx; own ||mtmx||^2 -> scal
  void sh_pw_update(double lam);          // x = mtmx / lam
  double sh_read_scal(int world, int q);  // rank-ordered sum of scal[r][q] (sync)
  uint64_t sh_launches() const { return sh_launches_; }

  int n() const { return n_; }
  int m() const { return m_; }
  int m1() const { return m1_; }
  int64_t nnz() const { return nnz_; }

  void solve(const aapdhg_solve_params* prm, const double* x0, const double* y0,
             aapdhg_solve_result* res, double* x_out, double* y_out, double* lam_out,
             aapdhg_record_sink sink, void* ctx);
  void select_step_sizes(const aapdhg_solve_params* prm, double* tau, double* sigma);
  double power_norm(int max_iters, double rel_tol, uint64_t seed, bool serial, int* rounds);

  void matvec(const double* x, double* out);
  void matvec_transpose(const double* y, double* out);
  void pdhg_step(double tau, double sigma, const double* x, const double* y, double* xn,
                 double* yn);
  void kkt_metrics(int reduction, const double* x, const double* y, double* kkt, double* lam);
  int aa_apply(int reduction, bool filtered, int p, const double* du_cols,
               const double* dg_cols, double beta, const double* d_hat, double eta,
               double c_s, double kappa_bar, const double* u, const double* g, double* out,
               int32_t* kept);
  int aa_op(int reduction, bool filtered, int p, const double* du_cols, const double* dg_cols,
            double beta, const double* d_hat, double eta, double c_s, double kappa_bar,
            int faa_skip, const double* u, const double* g, double* out, int32_t* kept,
            double* r_out, double* q_out);

  void set_profiling(bool on) { profiling_ = on; }
  void enter();  // cudaSetDevice + this handle's streams for DevBuf growth (this thread)
  void set_stream(cudaStream_t s);
  const std::map<std::string, KernelStat>& kernel_stats() const { return stats_; }
  uint64_t last_launches() const { return last_launches_; }
  uint64_t last_loop_iters() const { return last_loop_iters_; }
  // k_plain_loop in the last solve: iterations, device seconds, launches
  void last_plain_stats(uint64_t* iters, double* secs, uint64_t* launches) const {
    *iters = last_plain_iters_;
    *secs = last_plain_secs_;
    *launches = last_plain_launches_;
  }

 private:
  bool resolve_serial(int reduction) const;
  double device_dot(const double* a, const double* b, int64_t n, bool serial);
  int spmv(cudaStream_t s, const CsrDev& A, const VecRef& x, const RowsumArgs& o, bool serial,
           const DevState* S, int pred, const int32_t* stop);
  static size_t aa_smem(int cap);
  struct SellStore {
    DevBuf sl_ptr, sl_len, sl_row, sl_cnt, sci, sv;
  };
  struct CsrStore {
    DevBuf rp, ci, v, longs;
    SellStore sell[2];
    DevBuf lt_row, lt_chunk, lt_base, lt_nch, lt_part, lt_ticket;  // chunked long rows (TREE)
  };
  // device-side ingestion (ingest.cu)
  // (s: the stream to build on, null = stream_; the K' build runs on side_
  // in a second host thread while K's layouts build on stream_)
  void finish_csr(int nrows, int ncols, int64_t nnz, CsrStore& st, CsrDev& ser, CsrDev& tree,
                  cudaStream_t s = nullptr);
  void device_sell(const int32_t* shorts, int nshort, const int32_t* len, int sf, CsrStore& st,
                   SellStore& ss, CsrDev& out, cudaStream_t s, bool sigma_global,
                   double short_mean);
  void device_transpose(const CsrStore& src, int nrows, int ncols, int64_t nnz, CsrStore& dst,
                        cudaStream_t s = nullptr);
  struct TransposeScratch {
    DevBuf perm, row_of;
  };
  void device_transpose_sort(const CsrStore& src, int nrows, int ncols, int64_t nnz,
                             CsrStore& dst, TransposeScratch& ts, cudaStream_t s = nullptr);
  void device_transpose_permute(const CsrStore& src, int64_t nnz, CsrStore& dst,
                                TransposeScratch& ts, cudaStream_t s = nullptr, int part = 3);
  // ingestion in two phases (page-locked values arrive while the structure is
  // built): with defer_fills_ the SELL fills and the blocks' value copies are
  // queued, flush_fills runs them once the values are on the device
  struct PendingFill {
    int kind;  // 0: SELL fill of st into ss; 1: the values of block st from src
    CsrStore* st;
    SellStore* ss;
    int nslices, sf;
    const CsrStore* src;
    int64_t c0;
    int nrows;
  };
  bool defer_fills_ = false;
  std::vector<PendingFill> pending_fills_;
  void flush_fills(cudaStream_t s = nullptr);
  void device_validate_values(const CsrStore& st, int64_t nnz);
  void device_block(const CsrStore& src, int nrows, int64_t c0, int64_t c1, CsrStore& dst,
                    int64_t* nnz_out);
  void upload_csr(const int32_t* rp, const int32_t* ci, const double* v, int nrows, int ncols,
                  CsrStore& st, CsrDev& ser, CsrDev& tree, int64_t nnz = -1);
  const CsrDev& Km(bool serial) const { return serial ? Ks_ : Kt_; }
  // a shard's fused-kernel matrices: the last column block when blocked
  const CsrDev& sh_k1m() const { return ktb_.nb() > 1 ? ktb_.blk.back() : KTt_; }
  const CsrDev& sh_k2m() const { return kb_.nb() > 1 ? kb_.blk.back() : Kt_; }
  const CsrDev& KTm(bool serial) const { return serial ? KTs_ : KTt_; }
  void ensure_iter_buffers(int method, int cap, bool ring = false);
  double* faa_part_lo(int method, int cap) const;
  void upload_iterate(int slot, const double* x, const double* y);
  IterBufs iter_bufs();

  void init_device(int device);
  void upload_vectors(const double* c, const double* q, const double* l, const double* u);
  void init_vectors();  // (after upload_vectors: joins its copies, the other buffers)
  bool vec_async_ = false;
  void kkt_eval(int slot, bool serial, double* kkt_dev_out, double* lam_dev);
  int launch_core(cudaStream_t s, const SolveSetup& su);
  int launch_aa(cudaStream_t s, const SolveSetup& su);
  int launch_iteration(cudaStream_t s, const SolveSetup& su);
  void build_graph(const SolveSetup& su);
  void run_power(const double* x0_host, int max_iters, double rel_tol, bool serial, double* out,
                 int* rounds);
  void sync();

  // profiling-aware launch bookkeeping
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  void prof_begin(cudaStream_t s, const char* name);
  void prof_end(cudaStream_t s);
  void prof_collect();
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> event_pool_;
  std::string cur_name_;
  cudaEvent_t cur_a_ = nullptr;

  int device_;
  int num_sms_ = 148;
  bool pdl_ = true;  // AAPDHG_PDL=0 disables programmatic dependent launch
  int pass_prefetch_ = 3;  // AAPDHG_PASS_PREFETCH: later column passes fetch their partial early (3: register, 2: L2, 0: off)
  cudaStream_t stream_ = nullptr;
  cudaStream_t own_stream_ = nullptr;
  cudaStream_t side_ = nullptr;  // SERIAL: x-side chains beside K2 (fork/join)
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  // the final iterate's x / y download on side_ beside the last iteration
  cudaEvent_t ev_out_ = nullptr, ev_out_done_ = nullptr;
  // L2-blocked TREE: k_dual_epi per column block of K on stream_, each K
  // column pass on side_ as soon as its block of xhat is out
  static constexpr int kMaxPipe = 16;
  cudaEvent_t ev_blk_[kMaxPipe] = {};
  int n_ = 0, m_ = 0, m1_ = 0;
  int64_t nnz_ = 0, N_ = 0, nglob_ = 0;
  // sharded solve
  int shard_rank_ = -1;  // -1: a whole-LP handle
  int shard_world_ = 1;
  int64_t maxc_ = 0, maxr_ = 0, dot_stride_ = 0;
  DevBuf xg_, yg_, lg_, scal_all_, dots_all_, p2p_flags_;
  std::vector<ShardBufs> peers_;  // P2P: every shard's exchange buffers (by rank)
  bool peers_remote_ = false;
  uint64_t p2p_epoch_ = 0;        // solves begun (barrier sequence base)
  SolveSetup* sh_su_ = nullptr;
  DevParams sh_params_{};
  uint64_t sh_launches_ = 0;
  bool all_zero_ = true;
  bool bounds_ok_ = true;
  bool zero_start_ = false;  // every [l_j, u_j] holds 0: the default start P(0) has x = 0
  CsrDev Ks_, Kt_, KTs_, KTt_;  // SERIAL (sf = 1) and TREE layouts
  CsrStore k_store_, t_store_;
  // L2 column blocking (TREE mode) of a matrix whose gathered vector exceeds
  // the L2 budget: the column blocks' CSRs, processed one pass each so the
  // gathers of a pass hit an L2-resident slice of the vector
  struct Blocked {
    std::vector<CsrDev> blk;
    std::vector<std::unique_ptr<CsrStore>> store;
    DevBuf partial;  // row partial sums between passes
    int64_t width = 0;  // columns per block (block b: [b width, (b + 1) width))
    int nb() const { return int(blk.size()); }
  };
  Blocked kb_, ktb_;  // K (gathers xhat, n) and K' (gathers y, m)
  void build_blocks(const CsrStore& src, int nrows, int ncols, Blocked& out,
                    const char* kb_env = "AAPDHG_L2_BLOCK_KB");
  int launch_blocked_passes(cudaStream_t s, const Blocked& bk, const VecRef& x,
                            const DevState* S, int pred_aa = 0, const int32_t* stop = nullptr,
                            bool all = false);
  int spmv_any(cudaStream_t s, bool transpose, const VecRef& x, RowsumArgs r, bool serial,
               const DevState* S, const int32_t* stop);
  std::atomic<size_t> sell_bytes_{0};
  bool building_blocks_ = false;  // device_sell: an L2 column block (never interleaved)
  DevBuf c_, q_, l_, u_;
  double nrm_q_[2] = {0, 0}, nrm_c_[2] = {0, 0};  // [serial, tree]
  bool serial_norms_ = false;
  double pow_eps_ = -1.0;            // the safeguard table's eps (NaN-free: validated)
  uint64_t pow_len_ = 0;             // entries valid on the device
  std::vector<double> pow_host_;
  void ensure_pow_table(double eps, uint64_t need);
  void ensure_serial_norms();
  // O(nnz) checks of the uploaded CSR, l <= u and the all-zero test on the
  // device (ingest.cu); throws the host validator's messages
  void device_validate(const CsrStore& st, int nrows, int ncols, int64_t nnz,
                       bool values = true);
  void device_flags_vectors();

  // iteration buffers
  int buf_method_ = -1, buf_cap_ = 0;
  DevBuf upool_, kxpool_, gpool_, du_, dg_, T_, T2_, part1_, part2_, partdot_,
      gram_, work_, vec_;
  DevBuf rec_, pow_tab_, dparams_, dstate_, dhat_, scal_, part_small_, lam_, pw_x_, pw_mx_,
      pw_mtmx_, pw_state_;
  int ndot_tile_ = 0;
  uint64_t rec_cap_ = 0;
  DevState* h_state_ = nullptr;  // pinned mirror

  // CUDA graph WHILE(batch){core; IF(aa){aa}; commit}, cached per layout
  cudaGraphExec_t graph_exec_ = nullptr;
  std::string graph_key_;
  cudaGraphConditionalHandle cond_loop_ = 0, cond_aa_ = 0;
  int core_nodes_ = 0, aa_nodes_ = 0;
  DevBuf gridbar_;  // k_plain_loop's barrier counters (GridBar)
  // k_plain_loop's calibrated partition (CsrDev::sl_start): slice starts per
  // worker CTA for K' and K, and the per-CTA phase times of the last launches
  DevBuf bal_start1_, bal_start2_, bal_stats_;
  bool bal_measuring_ = false;
  void bal_setup(const CsrDev& a, const CsrDev& b, int workers, bool* measure);
  void bal_collect(const CsrDev& a, const CsrDev& b, int workers);
  DevBuf ticket_;   // k_spmv_commit's last-CTA counter
  int32_t* h_batch_ = nullptr;  // pinned

  bool profiling_ = false;
  std::map<std::string, KernelStat> stats_;
  uint64_t last_launches_ = 0, last_loop_iters_ = 0;
  uint64_t last_plain_iters_ = 0, last_plain_launches_ = 0;
  double last_plain_secs_ = 0.0;
};

// k_plain_loop's calibrated partition (engine.cu): new slice starts per worker
// CTA from the current ones, each worker's mean phase time, its SM and the
// work of each slice (host only)
std::vector<int32_t> rebalance_partition(const std::vector<int32_t>& cur,
                                         const std::vector<double>& t, const std::vector<int>& sm,
                                         const std::vector<int32_t>& wt);

}  // namespace aapdhg_b200
