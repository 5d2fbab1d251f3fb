// pipeline.cuh — the per-iteration core of the sm_100a AA-PDHG solver.
//
// One iteration, evaluated at the current iterate u_k = (x, y):
//   k_dual_side     K'y warp-tile SpMV fused with the primal step
//                   xhat = P_X(x - tau (c - K'y)) and the dual-side KKT terms
//                   of u_k (lambda, bound terms, ||c - K'y - lambda||^2, c'x),
//                   plus the x-half of the history push (du, dg, g)
//                   — pdhg_core.cpp:49-53, solver.cpp:67-88,102-107,204-209
//   k_primal_side   K xhat warp-tile SpMV fused with the dual step
//                   yhat = P_Y(y + sigma (q - (2 K xhat - K x))) and the
//                   primal-side KKT terms of u_k, plus the y-half of the push
//                   — pdhg_core.cpp:55-60, solver.cpp:90-100
//                   TREE mode: its last CTA reduces every partial sum and runs
//                   the control logic (no extra launch).
//   k_serial_control SERIAL mode: all reductions as index-ordered chains, then
//                   the control logic.
// Control (solver.cpp:188-215,241-247): termination tests, trajectory
// records, memory push commit, safeguard — and, under graph replay, sets the
// IF condition of the AA branch.
//
// SpMV: CSR rows are grouped on the host into warp tiles of <= 32 rows and
// <= kWarpTile nonzeros (a longer row is a tile of its own). A warp streams
// its tile's (col, val) pairs coalesced, gathers x[col] through the read-only
// path, stages the products in its own shared-memory slice, and lane r sums
// row r sequentially in CSR order — bit-identical to the reference's
// row-serial matvec (sparse_linalg.cpp:60-69) and, on the transposed CSR
// (entries in ascending original row), to its row-ordered scatter
// matvec_transpose (sparse_linalg.cpp:77-87). No CTA barrier sits between a
// warp's loads and its sums, so warps stream independently; the epilogue
// operands of a lane's row are prefetched before the tile's loads.
#pragma once

#include "common.cuh"

namespace aapdhg_b200 {

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;  // identical in every lane (commutative butterfly)
}

// Fixed-shape block sum (warp xor tree, then warps in order); result valid in
// thread 0. Deterministic: the association never depends on timing.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) red[q * kWarps + warp] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = red[q * kWarps];
#pragma unroll
      for (int w = 1; w < kWarps; ++w) s += red[q * kWarps + w];
      v[q] = s;
    }
  }
  __syncthreads();
}

// Block-wide sum for any blockDim multiple of 32; result to all threads.
__device__ __forceinline__ double block_sum_dyn(double v, double* red32) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red32[warp] = v;
  __syncthreads();
  double s = red32[0];
  for (int w = 1; w < nw; ++w) s += red32[w];
  return s;
}

// Thread-strided sum of part[0..nb) with 8 independent loads in flight,
// then the fixed block tree. L1-bypassing loads: the partials were written
// by other CTAs of the same kernel.
__device__ __forceinline__ double reduce_partials(const double* part, int nb, double* red32) {
  double s = 0.0;
  int b = threadIdx.x;
  const int st = blockDim.x;
  for (; b + 7 * st < nb; b += 8 * st) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + b + u * st);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, v[u]);
  }
  for (; b < nb; b += st) s = __dadd_rn(s, __ldcg(part + b));
  return block_sum_dyn(s, red32);
}

// Index-ordered serial sums: the reference's vec.hpp:16-29 loops.
__device__ __forceinline__ double serial_dot(const double* __restrict__ a,
                                             const double* __restrict__ b, int64_t n) {
  double s = 0.0;
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    double p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = __dmul_rn(a[i + u], b[i + u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, p[u]);
  }
  for (; i < n; ++i) s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
  return s;
}

// ---------------------------------------------------------------------------
// pipelined warp-tile SpMV core
// ---------------------------------------------------------------------------
//
// Rows are grouped on the host into warp tiles (<= 32 rows, <= kWarpTile
// nonzeros; a longer row is a tile of its own) described by int4 metadata
// {r0, r1, e0, e1}. The tile kernels are persistent: warp w of the grid
// handles tiles w, w + W, w + 2W, ... and keeps two tiles in flight — while
// it gathers and sums tile t out of shared memory, cp.async is already
// streaming tile t+W's (val, col) slice, its row offsets and the epilogue
// operands of its rows (x, c, l, u, ...) into the other stage. In-flight
// data costs no registers, so ~2 tiles x 20 warps per SM keep HBM busy.

constexpr int kPipeWarps = 4;  // warps per CTA of the tile kernels
constexpr int kPipeThreads = 32 * kPipeWarps;
constexpr int kPipeBlocksPerSM = 5;  // 5 x 38 KB of stages per SM

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// One stage of a warp's pipeline. v/ci hold the 16-byte aligned superset of
// the tile's [e0, e1) slice (offsets e0 & 1 and e0 & 3); products overwrite v.
template <int NE>
struct __align__(16) WarpStage {
  double v[kWarpTile + 2];
  int32_t ci[kWarpTile + 8];
  int32_t rp[36];
  double epi[NE > 0 ? NE : 1][32];
};

__device__ __forceinline__ bool tile_is_long(const int4& m) {
  return (m.y - m.x == 1) && (m.w - m.z > kWarpTile);
}

// Starts the async copies of tile m into stage st (one commit group, empty
// for a long row, which is streamed synchronously when processed).
template <int NE>
__device__ __forceinline__ void issue_tile(const CsrDev& A, const int4& m, WarpStage<NE>& st,
                                           const double* const* src, int lane) {
  if (!tile_is_long(m)) {
    const int r0 = m.x, r1 = m.y, e0 = m.z, e1 = m.w;
    const int a0 = e0 & ~1, nv = (e1 - a0 + 1) >> 1;
    for (int k = lane; k < nv; k += 32) cp_async16(&st.v[2 * k], A.v + a0 + 2 * k);
    const int c0 = e0 & ~3, nc = (e1 - c0 + 3) >> 2;
    for (int k = lane; k < nc; k += 32) cp_async16(&st.ci[4 * k], A.ci + c0 + 4 * k);
    const int nr = r1 - r0;
    for (int i = lane; i <= nr; i += 32) cp_async4(&st.rp[i], A.rp + r0 + i);
    if (lane < nr)
#pragma unroll
      for (int q = 0; q < NE; ++q) cp_async8(&st.epi[q][lane], src[q] + r0 + lane);
  }
  cp_async_commit();
}

// wprod[t] = vals[e0+t] * x[col[e0+t]], t < cnt <= kWarpTile (register path,
// used for the chunks of long rows).
__device__ __forceinline__ void warp_stage(const CsrDev& A, const double* __restrict__ x,
                                           int64_t e0, int cnt, double* wprod, int lane) {
  constexpr int U = 4;
#pragma unroll 1
  for (int base = 0; base < cnt; base += 32 * U) {
    int c[U];
    double a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + lane + 32 * u;
      if (t < cnt) {
        c[u] = __ldcs(A.ci + e0 + t);
        a[u] = __ldcs(A.v + e0 + t);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + lane + 32 * u;
      if (t < cnt) wprod[t] = __dmul_rn(a[u], __ldg(x + c[u]));
    }
  }
}

// Sum of one long row (> kWarpTile nonzeros) by one warp, kWarpTile chunks;
// SERIAL adds every product in CSR order in lane 0 (bitwise = reference),
// TREE adds per-chunk warp trees in order. Valid in lane 0.
template <bool SERIAL>
__device__ double long_row_sum(const CsrDev& A, const double* __restrict__ x, int64_t e0,
                               int64_t e1, double* wprod, int lane) {
  double s = 0.0;
  for (int64_t c0 = e0; c0 < e1; c0 += kWarpTile) {
    const int cnt = (int)((e1 - c0) < kWarpTile ? (e1 - c0) : kWarpTile);
    warp_stage(A, x, c0, cnt, wprod, lane);
    __syncwarp();
    if (SERIAL) {
      if (lane == 0)
        for (int t = 0; t < cnt; ++t) s = __dadd_rn(s, wprod[t]);
    } else {
      double v = 0.0;
      for (int t = lane; t < cnt; t += 32) v = __dadd_rn(v, wprod[t]);
      s = __dadd_rn(s, warp_sum(v));
    }
    __syncwarp();
  }
  return s;
}

// Row sums of a staged tile: gathers x[col] (8 per lane in flight), products
// in place, then lane r adds row r0 + r in CSR order. Returns the lane's
// row (-1 if none); `s` valid there.
template <bool SERIAL, int NE>
__device__ __forceinline__ int tile_sums(const CsrDev& A, const int4& m, WarpStage<NE>& st,
                                         const double* __restrict__ x, int lane, double& s) {
  const int r0 = m.x, r1 = m.y, e0 = m.z, e1 = m.w;
  s = 0.0;
  if (tile_is_long(m)) {
    s = long_row_sum<SERIAL>(A, x, e0, e1, st.v, lane);
    return lane == 0 ? r0 : -1;
  }
  const int cnt = e1 - e0, vo = e0 & 1, co = e0 & 3;
  double g[kWarpTile / 32];
#pragma unroll
  for (int u = 0; u < kWarpTile / 32; ++u) {
    const int t = lane + 32 * u;
    if (t < cnt) g[u] = __ldg(x + st.ci[co + t]);
  }
#pragma unroll
  for (int u = 0; u < kWarpTile / 32; ++u) {
    const int t = lane + 32 * u;
    if (t < cnt) st.v[vo + t] = __dmul_rn(st.v[vo + t], g[u]);
  }
  __syncwarp();
  if (lane >= r1 - r0) return -1;
  const int a = st.rp[lane] - e0, z = st.rp[lane + 1] - e0;
  double acc = 0.0;
  for (int e = a; e < z; ++e) acc = __dadd_rn(acc, st.v[vo + e]);
  s = acc;
  return r0 + lane;
}

// Epilogue operand q of the lane's row: staged, or read directly for a long row.
template <int NE>
__device__ __forceinline__ double operand(const WarpStage<NE>& st, bool is_long,
                                          const double* const* src, int q, int row, int lane) {
  return is_long ? src[q][row] : st.epi[q][lane];
}

// out[r] = (A x)_r — power iteration, K x recache, per-op matvec.
struct SpmvArgs {
  const double* x;       // used when x_pool == nullptr
  double* out;           // used when out_pool == nullptr
  const double* x_pool;  // upool base: x = x_pool + u_idx[x_role]*x_stride
  double* out_pool;      // kxpool base: out = out_pool + kx_idx[out_role]*out_stride
  int32_t x_role, out_role;
  int64_t x_stride, out_stride;
  int32_t pred_aa_ok;    // run only when S->aa_ok
  const int32_t* stop;   // optional: skip when *stop != 0 (power iteration)
};

template <bool SERIAL>
__global__ void __launch_bounds__(kPipeThreads, kPipeBlocksPerSM)
    k_spmv(CsrDev A, SpmvArgs g, const DevState* S) {
  if (S) {
    if (S->done) return;
    if (g.pred_aa_ok && !S->aa_ok) return;
  }
  if (g.stop && *g.stop) return;
  __shared__ WarpStage<0> stage[kPipeWarps][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = gridDim.x * kPipeWarps;
  const double* x = g.x_pool ? g.x_pool + (int64_t)S->u_idx[g.x_role] * g.x_stride : g.x;
  double* out = g.out_pool ? g.out_pool + (int64_t)S->kx_idx[g.out_role] * g.out_stride : g.out;
  const double* const src[1] = {nullptr};
  int tile = blockIdx.x * kPipeWarps + warp;
  if (tile >= A.ntiles) return;
  int4 m = A.meta[tile];
  issue_tile<0>(A, m, stage[warp][0], src, lane);
  for (int buf = 0; tile < A.ntiles; buf ^= 1) {
    const int next = tile + W;
    int4 mn = m;
    if (next < A.ntiles) {
      mn = A.meta[next];
      issue_tile<0>(A, mn, stage[warp][buf ^ 1], src, lane);
    } else {
      cp_async_commit();
    }
    cp_async_wait<1>();
    __syncwarp();
    double s;
    const int row = tile_sums<SERIAL, 0>(A, m, stage[warp][buf], x, lane, s);
    if (row >= 0) out[row] = s;
    __syncwarp();
    tile = next;
    m = mn;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// the fused PDHG halves
// ---------------------------------------------------------------------------

struct IterBufs {
  double* upool;   // 4 x N
  double* kxpool;  // 3 x m
  double* gpool;   // 2 x N
  double* du;      // cap x N
  double* dg;      // cap x N
  double* T;       // n
  double* part1;   // P1_COUNT x nblk1
  double* part2;   // P2_COUNT x nblk2
  const double* c;
  const double* q;
  const double* l;
  const double* u;
};

// Adds the warps' acc[] in order into part[q * nb + blockIdx.x].
template <int NV>
__device__ __forceinline__ void block_partials(double (&acc)[NV], double (*wred)[NV],
                                               double* part, int nb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = warp_sum(acc[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) wred[warp][q] = acc[q];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = wred[0][q];
#pragma unroll
      for (int w = 1; w < kPipeWarps; ++w) s = __dadd_rn(s, wred[w][q]);
      part[q * nb + blockIdx.x] = s;
    }
}

// K1: t = (K'y)_j (row j of K' = column j of K), then
//   xhat_j = min(max(x_j - tau (c_j - t), l_j), u_j)      pdhg_core.cpp:49-53
//   lambda_j = P_Lambda(c_j - t)                           solver.cpp:67-71
//   partials: (xhat-x)^2, bound term, (c-t-lambda)^2, c_j x_j
//   PUSH: du_j = x_j - xprev_j, dg_j = g_j - gprev_j, g_j = xhat_j - x_j
// Per-lane partial sums run over the warp's tiles in a fixed order, so the
// CTA partials are deterministic.
template <bool SERIAL, bool PUSH>
__global__ void __launch_bounds__(kPipeThreads, kPipeBlocksPerSM)
    k_dual_side(CsrDev KT, IterBufs B, const DevParams* __restrict__ P, DevState* S) {
  if (S->done) return;
  constexpr int NE = PUSH ? 6 : 4;
  __shared__ WarpStage<NE> stage[kPipeWarps][2];
  __shared__ double wred[kPipeWarps][P1_COUNT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = gridDim.x * kPipeWarps;
  const int64_t N = P->N;
  const double* x = B.upool + (int64_t)S->u_idx[U_CUR] * N;
  const double* y = x + P->n;
  double* xh = B.upool + (int64_t)S->u_idx[U_HAT] * N;
  const double* xp = B.upool + (int64_t)S->u_idx[U_PREV] * N;
  const double* gp = PUSH ? B.gpool + (int64_t)S->g_idx[G_PREV] * N : nullptr;
  double* gc = PUSH ? B.gpool + (int64_t)S->g_idx[G_CUR] * N : nullptr;
  const int64_t slot = S->push_slot;
  double* du = PUSH ? B.du + slot * N : nullptr;
  double* dg = PUSH ? B.dg + slot * N : nullptr;
  const double tau = P->tau;
  const double* src[NE];
  src[0] = x;
  src[1] = B.c;
  src[2] = B.l;
  src[3] = B.u;
  if constexpr (PUSH) {
    src[4] = xp;
    src[5] = gp;
  }
  double acc[P1_COUNT] = {0.0, 0.0, 0.0, 0.0};
  int tile = blockIdx.x * kPipeWarps + warp;
  int4 m = tile < KT.ntiles ? KT.meta[tile] : make_int4(0, 0, 0, 0);
  if (tile < KT.ntiles) issue_tile<NE>(KT, m, stage[warp][0], src, lane);
  for (int buf = 0; tile < KT.ntiles; buf ^= 1) {
    const int next = tile + W;
    int4 mn = m;
    if (next < KT.ntiles) {
      mn = KT.meta[next];
      issue_tile<NE>(KT, mn, stage[warp][buf ^ 1], src, lane);
    } else {
      cp_async_commit();
    }
    cp_async_wait<1>();
    __syncwarp();
    WarpStage<NE>& st = stage[warp][buf];
    const bool lg = tile_is_long(m);
    double t;
    const int j = tile_sums<SERIAL, NE>(KT, m, st, y, lane, t);
    if (j >= 0) {
      const double xj = operand<NE>(st, lg, src, 0, j, lane);
      const double cj = operand<NE>(st, lg, src, 1, j, lane);
      const double lj = operand<NE>(st, lg, src, 2, j, lane);
      const double uj = operand<NE>(st, lg, src, 3, j, lane);
      double xn = __dsub_rn(xj, __dmul_rn(tau, __dsub_rn(cj, t)));
      xn = smin(smax(xn, lj), uj);
      xh[j] = xn;
      const double d = __dsub_rn(xn, xj);
      const double red_c = __dsub_rn(cj, t);
      const double lam = project_lambda1(red_c, lj, uj);
      double bt = 0.0;
      if (isfinite(lj) && lam > 0.0) bt = __dmul_rn(lj, lam);
      if (isfinite(uj) && lam < 0.0) bt = __dmul_rn(uj, lam);
      const double dv = __dsub_rn(red_c, lam);
      acc[P1_GX2] = __dadd_rn(acc[P1_GX2], __dmul_rn(d, d));
      acc[P1_BOUND] = __dadd_rn(acc[P1_BOUND], bt);
      acc[P1_DUALSQ] = __dadd_rn(acc[P1_DUALSQ], __dmul_rn(dv, dv));
      acc[P1_CX] = __dadd_rn(acc[P1_CX], __dmul_rn(cj, xj));
      if constexpr (PUSH) {
        du[j] = __dsub_rn(xj, operand<NE>(st, lg, src, 4, j, lane));
        dg[j] = __dsub_rn(d, operand<NE>(st, lg, src, 5, j, lane));
        gc[j] = d;
      }
      if (SERIAL) B.T[j] = t;
    }
    __syncwarp();
    tile = next;
    m = mn;
  }
  cp_async_wait<0>();
  if (!SERIAL) block_partials<P1_COUNT>(acc, wred, B.part1, P->nblk1);
}

__device__ __noinline__ void control_logic(const DevParams* P, DevState* S, double g2,
                                           double bound, double qy, double cx, double infeas,
                                           double dual_sq);

// TREE mode: reduce all partials of K1/K2 and run the control (one CTA).
__device__ __forceinline__ void control_from_partials(const IterBufs& B, const DevParams* P,
                                                      DevState* S) {
  __shared__ double red32[32];
  const double gx2 = reduce_partials(B.part1 + P1_GX2 * P->nblk1, P->nblk1, red32);
  const double gy2 = reduce_partials(B.part2 + P2_GY2 * P->nblk2, P->nblk2, red32);
  const double bound = reduce_partials(B.part1 + P1_BOUND * P->nblk1, P->nblk1, red32);
  const double qy = reduce_partials(B.part2 + P2_QY * P->nblk2, P->nblk2, red32);
  const double cx = reduce_partials(B.part1 + P1_CX * P->nblk1, P->nblk1, red32);
  const double inf = reduce_partials(B.part2 + P2_INFEAS * P->nblk2, P->nblk2, red32);
  const double dsq = reduce_partials(B.part1 + P1_DUALSQ * P->nblk1, P->nblk1, red32);
  if (threadIdx.x == 0) control_logic(P, S, __dadd_rn(gx2, gy2), bound, qy, cx, inf, dsq);
}

// K2: s = (K xhat)_i, then
//   yhat_i = y_i + sigma (q_i - (2 s - (K x)_i)), clamped >= 0 for i < m1
//                                                         pdhg_core.cpp:55-60
//   K xhat cached as the next K x (solver.cpp:90 / pdhg_core.cpp:56)
//   partials: (yhat-y)^2, q_i y_i, primal infeasibility of u_k
// TREE: the last CTA to finish reduces every partial and runs the control.
template <bool SERIAL, bool PUSH>
__global__ void __launch_bounds__(kPipeThreads, kPipeBlocksPerSM)
    k_primal_side(CsrDev K, IterBufs B, const DevParams* __restrict__ P, DevState* S) {
  if (S->done) return;
  constexpr int NE = PUSH ? 5 : 3;
  __shared__ WarpStage<NE> stage[kPipeWarps][2];
  __shared__ double wred[kPipeWarps][P2_COUNT];
  __shared__ int is_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = gridDim.x * kPipeWarps;
  const int64_t N = P->N;
  const int n = P->n, mr = P->mrows, m1 = P->m1;
  const double* xh = B.upool + (int64_t)S->u_idx[U_HAT] * N;
  const double* y = B.upool + (int64_t)S->u_idx[U_CUR] * N + n;
  double* yh = B.upool + (int64_t)S->u_idx[U_HAT] * N + n;
  const double* kx = B.kxpool + (int64_t)S->kx_idx[KX_CUR] * mr;
  double* kxh = B.kxpool + (int64_t)S->kx_idx[KX_HAT] * mr;
  const int64_t slot = S->push_slot;
  double* du = PUSH ? B.du + slot * N + n : nullptr;
  double* dg = PUSH ? B.dg + slot * N + n : nullptr;
  double* gc = PUSH ? B.gpool + (int64_t)S->g_idx[G_CUR] * N + n : nullptr;
  const double sigma = P->sigma;
  const double* src[NE];
  src[0] = y;
  src[1] = B.q;
  src[2] = kx;
  if constexpr (PUSH) {
    src[3] = B.upool + (int64_t)S->u_idx[U_PREV] * N + n;
    src[4] = B.gpool + (int64_t)S->g_idx[G_PREV] * N + n;
  }
  double acc[P2_COUNT] = {0.0, 0.0, 0.0};
  int tile = blockIdx.x * kPipeWarps + warp;
  int4 m = tile < K.ntiles ? K.meta[tile] : make_int4(0, 0, 0, 0);
  if (tile < K.ntiles) issue_tile<NE>(K, m, stage[warp][0], src, lane);
  for (int buf = 0; tile < K.ntiles; buf ^= 1) {
    const int next = tile + W;
    int4 mn = m;
    if (next < K.ntiles) {
      mn = K.meta[next];
      issue_tile<NE>(K, mn, stage[warp][buf ^ 1], src, lane);
    } else {
      cp_async_commit();
    }
    cp_async_wait<1>();
    __syncwarp();
    WarpStage<NE>& st = stage[warp][buf];
    const bool lg = tile_is_long(m);
    double s;
    const int i = tile_sums<SERIAL, NE>(K, m, st, xh, lane, s);
    if (i >= 0) {
      const double yi = operand<NE>(st, lg, src, 0, i, lane);
      const double qi = operand<NE>(st, lg, src, 1, i, lane);
      const double kxi = operand<NE>(st, lg, src, 2, i, lane);
      double yn =
          __dadd_rn(yi, __dmul_rn(sigma, __dsub_rn(qi, __dsub_rn(__dmul_rn(2.0, s), kxi))));
      if (i < m1) yn = smax(yn, 0.0);
      yh[i] = yn;
      kxh[i] = s;
      const double d = __dsub_rn(yn, yi);
      double v = __dsub_rn(qi, kxi);
      if (i < m1) v = smax(v, 0.0);
      acc[P2_GY2] = __dadd_rn(acc[P2_GY2], __dmul_rn(d, d));
      acc[P2_QY] = __dadd_rn(acc[P2_QY], __dmul_rn(qi, yi));
      acc[P2_INFEAS] = __dadd_rn(acc[P2_INFEAS], __dmul_rn(v, v));
      if constexpr (PUSH) {
        du[i] = __dsub_rn(yi, operand<NE>(st, lg, src, 3, i, lane));
        dg[i] = __dsub_rn(d, operand<NE>(st, lg, src, 4, i, lane));
        gc[i] = d;
      }
    }
    __syncwarp();
    tile = next;
    m = mn;
  }
  cp_async_wait<0>();
  if (SERIAL) return;
  block_partials<P2_COUNT>(acc, wred, B.part2, P->nblk2);
  // last CTA to finish reduces all partials and runs the control logic
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned tk = atomicAdd(&S->ticket, 1u);
    is_last = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  control_from_partials(B, P, S);
  if (threadIdx.x == 0) S->ticket = 0;
}

// ---------------------------------------------------------------------------
// SERIAL mode: every scalar reduction as one index-ordered chain
// (fixed_point_residual pdhg_core.cpp:65-74; kkt_metrics solver.cpp:64-110),
// one warp per chain (lane 0 sums), then the control logic.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(32 * S_COUNT)
    k_serial_control(IterBufs B, const DevParams* __restrict__ P, DevState* S) {
  if (S->done) {
    if (threadIdx.x == 0 && P->use_cond) cudaGraphSetConditional(P->cond_aa, 0);
    return;
  }
  __shared__ double res[S_COUNT];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    const int64_t N = P->N;
    const int n = P->n, mr = P->mrows, m1 = P->m1;
    const double* u = B.upool + (int64_t)S->u_idx[U_CUR] * N;
    const double* uh = B.upool + (int64_t)S->u_idx[U_HAT] * N;
    const double* kx = B.kxpool + (int64_t)S->kx_idx[KX_CUR] * mr;
    const double* T = B.T;
    double s = 0.0;
    switch (w) {
      case S_G2: {
        int64_t i = 0;
        for (; i + 8 <= N; i += 8) {
          double p[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const double d = __dsub_rn(uh[i + k], u[i + k]);
            p[k] = __dmul_rn(d, d);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) s = __dadd_rn(s, p[k]);
        }
        for (; i < N; ++i) {
          const double d = __dsub_rn(uh[i], u[i]);
          s = __dadd_rn(s, __dmul_rn(d, d));
        }
        break;
      }
      case S_BOUND:
        for (int j = 0; j < n; ++j) {
          const double lj = B.l[j], uj = B.u[j];
          const double lam = project_lambda1(__dsub_rn(B.c[j], T[j]), lj, uj);
          if (isfinite(lj) && lam > 0.0) s = __dadd_rn(s, __dmul_rn(lj, lam));
          if (isfinite(uj) && lam < 0.0) s = __dadd_rn(s, __dmul_rn(uj, lam));
        }
        break;
      case S_QY: s = serial_dot(B.q, u + n, mr); break;
      case S_CX: s = serial_dot(B.c, u, n); break;
      case S_INFEAS:
        for (int i = 0; i < mr; ++i) {
          double v = __dsub_rn(B.q[i], kx[i]);
          if (i < m1) v = smax(v, 0.0);
          s = __dadd_rn(s, __dmul_rn(v, v));
        }
        break;
      case S_DUALSQ:
        for (int j = 0; j < n; ++j) {
          const double rc = __dsub_rn(B.c[j], T[j]);
          const double v = __dsub_rn(rc, project_lambda1(rc, B.l[j], B.u[j]));
          s = __dadd_rn(s, __dmul_rn(v, v));
        }
        break;
    }
    res[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    control_logic(P, S, res[S_G2], res[S_BOUND], res[S_QY], res[S_CX], res[S_INFEAS],
                  res[S_DUALSQ]);
}

// KKT scalars of the CUR iterate from the reduced sums (solver.cpp:83-107).
__device__ __forceinline__ void kkt_from_sums(double nrm_q, double nrm_c, double bound,
                                              double qy, double cx, double infeas,
                                              double dual_sq, double* kkt) {
  const double dual_core = __dadd_rn(qy, bound);
  const double primal_obj = cx;
  kkt[0] = fabs(__dsub_rn(dual_core, primal_obj)) /
           __dadd_rn(__dadd_rn(1.0, fabs(dual_core)), fabs(primal_obj));
  kkt[1] = sqrt(infeas) / __dadd_rn(1.0, nrm_q);
  kkt[2] = sqrt(dual_sq) / __dadd_rn(1.0, nrm_c);
  kkt[3] = primal_obj;
}

__device__ __forceinline__ void finish_solve(DevState* S, int status, int role, double g) {
  S->status = status;
  S->final_role = role;
  S->g_final = g;
  S->done = 1;
}

// The scalar part of one iteration of solve() (solver.cpp:188-215,241-247),
// run by a single thread after every sum of the iteration is known.
__device__ __noinline__ void control_logic(const DevParams* P, DevState* S, double g2, double bound, double qy,
                              double cx, double infeas, double dual_sq) {
  double kkt[4];
  kkt_from_sums(P->nrm_q, P->nrm_c, bound, qy, cx, infeas, dual_sq, kkt);
  for (int q = 0; q < 4; ++q) S->kkt[q] = kkt[q];
  const double gkn = sqrt(g2);
  S->gkn = gkn;
  S->aa_attempt = 0;
  S->aa_ok = 0;
  const uint64_t k = S->k;
  const double elapsed = (double)(globaltimer_ns() - S->t0_ns) * 1e-9 + P->wall_offset_s;
  bool attempt = false;
  do {
    if (k == 0) {  // priming step, solver.cpp:168-172
      S->g0n = gkn;
      aapdhg_record* r = P->rec;
      r->k = 0;
      r->g_norm = gkn;
      r->aa_step = 0;
      r->i = 0;
      r->j = 0;
      break;
    }
    {  // the record of iterate k-1 takes the KKT of the produced iterate u_k
      aapdhg_record* r = P->rec + (k - 1) % P->rec_cap;
      r->r_gap = kkt[0];
      r->r_primal = kkt[1];
      r->r_dual = kkt[2];
      r->objective = kkt[3];
      r->elapsed_s = elapsed;
      S->rec_complete = k;
    }
    const double kmax = smax(smax(kkt[0], kkt[1]), kkt[2]);
    if (k == 1 && S->g0n == 0.0) { finish_solve(S, AAPDHG_SOLVE_FIXED_POINT_START, U_PREV, 0.0); break; }
    if (P->kkt_terminate && kmax <= P->kkt_eps) { finish_solve(S, AAPDHG_SOLVE_KKT_TOL, U_CUR, gkn); break; }
    if (gkn < P->toll) { finish_solve(S, AAPDHG_SOLVE_RESIDUAL_TOL, U_CUR, gkn); break; }
    if (S->i + S->j >= P->max_iters) { finish_solve(S, AAPDHG_SOLVE_MAX_ITERS, U_CUR, gkn); break; }
    if (elapsed >= P->max_wall_s) { finish_solve(S, AAPDHG_SOLVE_TIMEOUT, U_CUR, gkn); break; }

    if (P->method != AAPDHG_METHOD_PDHG) {  // memory_push / FaaState::push
      if (S->mem_size == P->cap) {
        for (int t = 1; t < S->mem_size; ++t) S->mem_slots[t - 1] = S->mem_slots[t];
        S->mem_slots[S->mem_size - 1] = S->push_slot;
      } else {
        S->mem_slots[S->mem_size++] = S->push_slot;
      }
    }
    aapdhg_record* r = P->rec + k % P->rec_cap;
    r->k = k;
    r->g_norm = gkn;
    r->aa_step = 0;
    r->i = S->i;
    r->j = S->j;
    if (P->method != AAPDHG_METHOD_PDHG) {
      // safeguard_pass, solver.cpp:59-62, with the host std::pow table
      const double pw = S->i < P->pow_len ? P->pow_tab[S->i]
                                          : pow((double)S->i + 1.0, -(1.0 + P->safeguard_eps));
      attempt = gkn <= __dmul_rn(__dmul_rn(P->safeguard_d, S->g0n), pw);
    }
    if (attempt) S->aa_attempt = 1;
    else S->j += 1;
  } while (false);
  if (P->use_cond) cudaGraphSetConditional(P->cond_aa, attempt ? 1u : 0u);
}

}  // namespace aapdhg_b200
