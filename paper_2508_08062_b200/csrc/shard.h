// shard.h — the sharded (multi-GPU) solve: row/column partition of K over
// `world` shards, one Problem per shard, all-gathers between the phases.
#pragma once

#include <memory>
#include <vector>

#include "engine.h"

namespace aapdhg_b200 {

// Contiguous blocks of K's rows and columns, balanced by (nnz + 4) per row /
// column; bounds have world + 1 entries. maxr / maxc: the largest block.
struct Partition {
  std::vector<int32_t> rows, cols;
  int64_t maxr = 0, maxc = 0;
};
Partition plan_partition(const aapdhg_csr_view& k, int world);
Partition plan_partition_weights(const aapdhg_csr_view& k, const std::vector<int64_t>& wc,
                                 int world);

class ShardGroup {
 public:
  ShardGroup(const aapdhg_problem_view* v, int device, const aapdhg_dist_view* d);
  ~ShardGroup();
  ShardGroup(const ShardGroup&) = delete;
  ShardGroup& operator=(const ShardGroup&) = delete;

  void solve(const aapdhg_solve_params* prm, const double* x0, const double* y0,
             aapdhg_solve_result* res, double* x_out, double* y_out, double* lam_out,
             aapdhg_record_sink sink, void* ctx);
  void select_step_sizes(const aapdhg_solve_params* prm, double* tau, double* sigma);
  void set_stream(cudaStream_t s);

  int n() const { return n_; }
  int m() const { return m_; }
  int m1() const { return m1_; }
  int64_t nnz() const { return nnz_; }
  uint64_t last_launches() const { return last_launches_; }
  uint64_t last_loop_iters() const { return last_loop_iters_; }

 private:
  // exchanged buffers (XG2: the candidate x of an AA step; also the P2P
  // barrier slot)
  enum Buf { XG, YG, LG, SCAL, DOTS, XG2 };
  void allgather(Buf b);
  void exchange(Buf b);
  void open_peers();
  double power_norm(int max_iters, double rel_tol, uint64_t seed);
  template <class F>
  void each(F&& f) {
    for (auto& s : shards_) f(*s);
  }

  int world_ = 1, transport_ = 0, rank_ = 0, device_ = 0;
  bool multi_ = false;  // one shard per process (NCCL / P2P)
  bool p2p_ = false;    // peer-memory exchanges (P2P / LOOPBACK_P2P)
  std::vector<void*> ipc_opened_;
  int n_ = 0, m_ = 0, m1_ = 0;
  int64_t nnz_ = 0;
  bool all_zero_ = false, bounds_ok_ = true;
  Partition part_;
  std::vector<std::unique_ptr<Problem>> shards_;
  cudaStream_t stream_ = nullptr;      // every shard launches on it
  cudaStream_t own_stream_ = nullptr;
  void* comm_ = nullptr;               // ncclComm_t (transport NCCL)
  uint64_t last_launches_ = 0, last_loop_iters_ = 0;
};

// 128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it).
void nccl_unique_id(uint8_t* out, size_t len);

}  // namespace aapdhg_b200
