// common.cuh — shared device/host definitions of the sm_100a AA-PDHG path.
//
// Layout of the iteration state in HBM:
//   upool[4][N]   stacked iterates u = (x[n]; y[m]); roles CUR/PREV/HAT/CAND
//                 are indices held in DevState and rotated on the device.
//   kxpool[3][m]  cached K*x for CUR / HAT (= K*xhat) / CAND.
//   gpool[2][N]   fixed-point residual g = T(u) - u for CUR / PREV.
//   du[cap][N], dg[cap][N]   difference memory ring (slot-major columns).
//   T[n]          K'y of the current iterate (serial reduction mode only).
// All arithmetic is IEEE fp64 compiled with -fmad=false: every product and
// sum is rounded exactly where the reference rounds it.
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "aapdhg_cuda.h"

namespace aapdhg_b200 {

constexpr int kThreads = 256;        // CTA size of the tile kernels
constexpr int kWarps = kThreads / 32;
constexpr int kMaxMemory = 64;       // largest AA memory capacity supported
constexpr int kDotChunk = 512;       // elements per CTA in the tree multi-dot
constexpr int kCtrlThreads = 1024;
constexpr int kMaxPeers = 8;         // shards of a peer-memory (P2P) sharded solve

// iterate roles
enum { U_CUR = 0, U_PREV = 1, U_HAT = 2, U_CAND = 3 };
enum { KX_CUR = 0, KX_HAT = 1, KX_CAND = 2 };
enum { G_CUR = 0, G_PREV = 1 };

// partial-sum quantities
enum { P1_GX2 = 0, P1_BOUND = 1, P1_DUALSQ = 2, P1_CX = 3, P1_COUNT = 4 };
enum { P2_GY2 = 0, P2_QY = 1, P2_INFEAS = 2, P2_COUNT = 3 };
// serial chain results (index into DevState::sres)
enum { S_G2 = 0, S_BOUND = 1, S_QY = 2, S_CX = 3, S_INFEAS = 4, S_DUALSQ = 5, S_COUNT = 6 };
constexpr int kSerThreads = 256;  // k_serial_control
constexpr int kSerChunk = 1024;   // elements staged per pass
constexpr size_t kSerSmem = sizeof(double) * S_COUNT * kSerChunk + kSerChunk;

// A CSR matrix on the device in the layout the SpMV kernels stream:
//   rp/ci/v        the CSR itself (row lengths; long rows read from here)
//   SELL-32        short rows (<= kLongRow nonzeros) grouped 32 per slice in
//                  row order; element k of the slice's lane-r row sits at
//                  sl_ptr[s] + 32 k + r of sci/sv; sl_row[32 s + r] = row
//                  (-1 = empty lane), sl_len[s] = longest row of the slice
//   long rows      row ids, one warp each
// Work units = slices then long rows, pulled by persistent warps.
struct CsrDev {
  int32_t nrows = 0, ncols = 0;
  int64_t nnz = 0;
  const int32_t* rp = nullptr;
  const int32_t* ci = nullptr;
  const double* v = nullptr;
  int32_t nslices = 0, nlong = 0;
  const int64_t* sl_ptr = nullptr;
  const int32_t* sl_len = nullptr;
  const int32_t* sl_row = nullptr;
  const int32_t* sl_cnt = nullptr;  // the lane's element count (no rp loads in the loop setup)
  const int32_t* sci = nullptr;
  const double* sv = nullptr;
  const int32_t* long_rows = nullptr;  // longest first
  int32_t nhuge = 0;  // TREE: the first nhuge long rows (>= kHugeRow) get a CTA each
  // TREE, many long rows: rows longer than 2 kLongChunk are cut into chunks of
  // kLongChunk entries, one warp each (task t: long row lt_row[t], chunk
  // lt_chunk[t]); a row's chunk sums go to lt_part[lt_base[row] + chunk] and
  // the chunk that finishes last (ticket lt_ticket[row]) adds them in chunk
  // order and owns the row's result. ntask = 0: a warp per long row.
  int32_t ntask = 0;
  const int32_t* lt_row = nullptr;
  const int32_t* lt_chunk = nullptr;
  const int32_t* lt_base = nullptr;
  const int32_t* lt_nch = nullptr;
  double* lt_part = nullptr;
  unsigned int* lt_ticket = nullptr;
  int32_t nblk_short = 0, nblk_long = 0;  // nblk_long = nhuge + ceil((nlong - nhuge) / 8)
  int32_t sf = 1;  // lanes per row in the slices (1 = CSR-ordered row sums)
  // more slices than one wave of warps: slice s belongs to CTA s % nblk_short
  // (one wave of CTAs), whose warps loop over theirs (row_sum `rep`)
  int32_t interleave = 0;
  // k_plain_loop with a calibrated partition (TREE, no long rows, not
  // interleaved): CTA b owns slices [sl_start[b], sl_start[b + 1]) (<= kWarps),
  // and the partial sums are per slice (part[q * nslices + slice]), so the
  // reduction does not depend on which CTA ran a slice
  const int32_t* sl_start = nullptr;
  int32_t grid() const { return nblk_short + nblk_long; }
};

// device validation flags (ingest.cu k_validate_*)
enum { kCsrBadRowPtr = 1, kCsrBadColumn = 2, kCsrUnsorted = 4, kCsrNonzero = 8, kBoundsBad = 16,
       kZeroOutside = 32 };  // (some [l_j, u_j] does not hold 0: the start P(0) is not 0)

constexpr int kLongRow = 256;        // rows longer than this get a warp each
constexpr int kHugeRow = 1024;       // TREE: rows at least this long get a CTA each
constexpr int kLongChunk = 512;      // TREE: long-row chunk per warp (CsrDev::ntask)
constexpr int kSpmvBlocksPerSM = 6;  // 48 warps/SM at <= 40 registers

constexpr int kGroup = 64;           // CTAs per first-level partial group

// Constant per solve (written before the loop starts).
struct DevParams {
  int32_t method, serial, m1, kkt_terminate;
  int32_t n, mrows, cap;
  int64_t N;
  double safeguard_d, safeguard_eps, beta, eta, c_s, kappa_bar, toll, kkt_eps;
  double tau, sigma;
  uint64_t max_iters;
  double max_wall_s;
  double wall_offset_s;   // host time already spent before the loop started
  double nrm_q, nrm_c;
  const double* d_hat;    // nullptr = identity
  const double* pow_tab;  // (i+1)^-(1+eps), host std::pow
  uint64_t pow_len;
  aapdhg_record* rec;     // ring of rec_cap records
  uint64_t rec_cap;
  int32_t nblk1, nblk2, ndot_blk, use_cond;
  cudaGraphConditionalHandle cond_aa;    // IF node of the AA branch
  cudaGraphConditionalHandle cond_loop;  // WHILE node of the iteration batch
  // sharded solve (nullptr / 0 on a single GPU): K1 gathers y from the
  // all-gathered ygather, K2 gathers xhat from xgather. The producers write
  // this shard's chunk of each exchanged buffer into ndst destinations: the
  // shard's own buffer (NCCL / copy transports: ndst = 1, the all-gather
  // follows), or every shard's buffer over peer memory (P2P transports:
  // ndst = world, a flag barrier follows) — K1 xhat -> xg_dst, K2 yhat ->
  // yg_dst, K2's last CTA the 8 shard totals -> scal_dst, the AA dot totals
  // -> dots_dst. K1 also keeps K'y in T.
  const double* xgather;
  const double* ygather;
  int32_t ndst, store_T;
  double* xg_dst[kMaxPeers];
  double* yg_dst[kMaxPeers];
  double* scal_dst[kMaxPeers];
  double* dots_dst[kMaxPeers];
  uint64_t p2p_epoch;  // barrier sequence base of this solve (high 32 bits)
  // P2P transports with fused signals: K1 waits for the YG arrivals and its
  // last CTA arrives at XG; K2 waits for XG and its last CTA arrives at YG
  // (ŷ and the shard totals); the control waits for YG. Arrival of shard r
  // at slot s: flag_peer[q][s * kMaxPeers + r] = (epoch << 32) + passes.
  int32_t p2p_fused, p2p_world, p2p_rank;
  int32_t p2p_sys;  // peers on other GPUs: system-scope fences before the arrivals
  unsigned long long* flag_peer[kMaxPeers];
  unsigned long long* flag_own;
  int64_t Nglob;  // n + m of the whole LP (FAA's QR row-count test)
  // per-op FAA entries (engine.cu faa_op): stages to skip (kFaaSkip*), and
  // where to write the kept columns' R (p x p column-major) when non-null
  int32_t faa_skip;
  int32_t no_stop_predict;  // k_plain_loop always speculates (AAPDHG_STOP_PREDICT=1: predicts)
  int32_t phase_prefetch;   // k_plain_loop: L2 bulk prefetch of the next phase's slice streams
  // ring history (AA-PDHG on one GPU, pipeline.cuh ring_free_slot): the
  // epilogues store g_k, the AA kernels difference it (0: du / dg pushed)
  int32_t ring;
  double* qr_r_out;
};
enum { kFaaSkipAngle = 1, kFaaSkipLength = 2 };

// Mutable solver state, device resident; the host reads it at polls.
struct DevState {
  int32_t done, status, final_role, aa_attempt;
  int32_t aa_ok, mem_size, push_slot, mix_p;
  uint64_t k, i, j, aa_failures;
  uint64_t rec_complete;
  double g0n, gkn, g_final;
  double kkt[4];  // r_gap, r_primal, r_dual, objective of CUR
  int32_t u_idx[4];
  int32_t kx_idx[3];
  int32_t g_idx[2];
  int32_t mem_slots[kMaxMemory];   // memory order, oldest first
  int32_t mix_slots[kMaxMemory];   // columns entering the mix (kept set)
  double w[kMaxMemory];
  double sres[8];                  // serial chain results
  double tot1[4];                  // K1 partial totals (TREE, fused control)
  uint64_t t0_ns;
  uint64_t loop_iters;             // iterations that did work (launch accounting)
  uint64_t loop_exits;             // k_plain_loop launches that ran (launch accounting)
  uint64_t plain_iters;            // iterations k_plain_loop completed
  uint64_t plain_ns;               // k_plain_loop time (globaltimer, launch start -> stop)
  uint32_t ticket;                 // last-CTA election in k_primal_side
  uint32_t ticket1;                // last-CTA election in k_dual_side (P2P arrival)
  int32_t prev_plain;              // the previous step was T(u_{k-1}) (not an AA candidate)
  int32_t batch_left;              // iterations left in this graph launch
  uint64_t p2p_seq[8];             // P2P flag barriers passed, per exchanged buffer
  // ring history (DevParams::ring): ring slots of g_{k-p}..g_k, oldest first
  // (gw_n = p + 1 entries once iteration 0 committed); gdux[q]: the column
  // ending at gw[q] has its du stored (u_t was an AA candidate)
  int32_t gw_n;
  int32_t gw[kMaxMemory + 1];
  uint8_t gdux[kMaxMemory + 3];
};

// Gathered vector: a plain pointer, or a role of the iterate pool resolved
// on the device (graph replay rotates roles).
struct VecRef {
  const double* p;      // used when pool == nullptr
  const double* pool;   // upool base
  int32_t role;
  int64_t stride;       // N
  int64_t offset;       // 0 for x, n for y
  __device__ __forceinline__ const double* get(const DevState* S) const {
    return pool ? pool + (int64_t)S->u_idx[role] * stride + offset : p;
  }
};

// out[r] = sum of row r's products (power iteration, K x recache, matvec).
struct RowsumArgs {
  double* out;           // used when out_pool == nullptr
  double* out_pool;      // kxpool base: out = out_pool + kx_idx[out_role]*out_stride
  int32_t out_role;
  int64_t out_stride;
  int32_t pred_aa_ok;
  const int32_t* stop;
  const double* rinit;  // L2-blocked: the earlier column passes' partial sums (or null)
};

struct IterBufs {
  double* upool;   // 4 x N
  double* kxpool;  // 3 x m
  double* gpool;   // 2 x N (ring history: cap + 2 slots of g)
  double* du;      // cap + 1 x N (ring history: cap + 2, indexed like gpool)
  double* dg;      // cap + 1 x N (unused by the ring history)
  double* T;       // n
  double* T2;      // n: SERIAL k_plain_loop, K'y of odd iterations (the control reads
                   // iteration k's while the speculative K1(k+1) writes the other)
  double* part1;   // P1_COUNT x nblk1 (per CTA)
  double* part2;   // P2_COUNT x nblk2
  const double* rinit1;  // L2-blocked K': partial K'y of the earlier column passes
  const double* rinit2;  // L2-blocked K: partial K xhat of the earlier passes
  int32_t nu1;        // K1 CTAs (rows of part1)
  int32_t fused_ctrl; // TREE: k_primal_side's last CTA runs the control (1) or,
                      // sharded, writes this shard's 8 totals to P->scal_dst (2)
  int32_t p2p_sys;    // = DevParams::p2p_sys (read before the params are staged)
  const double* c;
  const double* q;
  const double* l;
  const double* u;
};


struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StatusError : std::runtime_error {
  int code;
  StatusError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define AAPDHG_CUDA(call)                                                        \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      throw ::aapdhg_b200::CudaError(std::string(#call) + ": " +                 \
                                     cudaGetErrorString(e_));                   \
  } while (0)

// libstdc++ std::max / std::min semantics (signed zeros, NaN order).
__host__ __device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__host__ __device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }

// build_lambda_set + project_lambda (lp_model.cpp:293-306, pdhg_core.cpp:27-39)
__device__ __forceinline__ double project_lambda1(double v, double l, double u) {
  const bool lo = isfinite(l), hi = isfinite(u);
  if (!lo && !hi) return 0.0;
  if (!lo) return smin(v, 0.0);
  if (!hi) return smax(v, 0.0);
  return v;
}

// damp, anderson.cpp:10-20
__device__ __forceinline__ double damp1(double beta, const double* d_hat, int64_t i, double v) {
  return d_hat ? beta * d_hat[i] * v : beta * v;
}

#ifdef AAPDHG_TAIL_STAMPS
// experiment build only (make EXTRA=-DAAPDHG_TAIL_STAMPS): phase stamps of the
// fused control tail, read by aapdhg_cuda_debug_stamps
__device__ unsigned long long g_dbg[16];
#endif

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Experiment build only (EXTRA=-DAAPDHG_TIMELINE): CTA 0 of each kernel
// stamps (kernel id, globaltimer) on entry; aapdhg_cuda_timeline reads them.
#ifdef AAPDHG_TIMELINE
__device__ unsigned long long g_tl[2 * 8192];
__device__ unsigned int g_tl_n;
__device__ __forceinline__ void tl_mark(unsigned long long id) {
  const unsigned i = atomicAdd(&g_tl_n, 1u);
  if (i < 8192) {
    g_tl[2 * i] = id;
    g_tl[2 * i + 1] = globaltimer_ns();
  }
}
#define TL_MARK(id)                                          \
  do {                                                       \
    if (blockIdx.x == 0 && threadIdx.x == 0) tl_mark(id);    \
  } while (0)
#else
#define TL_MARK(id) \
  do {              \
  } while (0)
#endif

}  // namespace aapdhg_b200
