// pipeline.cuh — the per-iteration core of the sm_100a AA-PDHG solver.
//
// One iteration, evaluated at the current iterate u_k = (x, y):
//   k_dual_side     K'y SpMV fused with the primal step
//                   xhat = P_X(x - tau (c - K'y)) and the dual-side KKT terms
//                   of u_k (lambda, bound terms, ||c - K'y - lambda||^2, c'x),
//                   plus the x-half of the history push (du, dg, g)
//                   — pdhg_core.cpp:49-53, solver.cpp:67-88,102-107,204-209
//   k_primal_side   K xhat SpMV fused with the dual step
//                   yhat = P_Y(y + sigma (q - (2 K xhat - K x))) and the
//                   primal-side KKT terms of u_k, plus the y-half of the push
//                   — pdhg_core.cpp:55-60, solver.cpp:90-100
//                   TREE mode: its last CTA sums every partial and runs the
//                   control logic (no launch of its own).
//   k_serial_control SERIAL mode: all reductions as index-ordered chains, then
//                   the control logic.
// Control (solver.cpp:188-215,241-247): termination tests, trajectory
// records, memory push commit, safeguard — and, under graph replay, the
// conditions of the AA branch and of the iteration loop.
//
// SpMV layout (SELL-32, built in engine.cu): rows in slices of 32 lanes;
// element k of the row in lane r sits at sl_ptr[slice] + 32 k + r, so a
// warp's loads of (col, val) are coalesced. One warp per slice, the slices
// spread evenly over exactly one wave of CTAs. Each lane adds its row's
// products in CSR order (split factor sf = 1): bit-identical to the
// reference's row-serial matvec (sparse_linalg.cpp:60-69) and, on the
// transposed CSR (entries in ascending original row), to its row-ordered
// matvec_transpose (sparse_linalg.cpp:77-87). sf > 1 (TREE layout of a
// matrix with few rows) splits a row over sf lanes joined by a fixed xor
// tree. Rows longer than kLongRow get a warp each. No FMA anywhere
// (-fmad=false, __dmul_rn / __dadd_rn).
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
// red must hold NV * kWarps doubles; any blockDim multiple of 32 <= 256.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red) {
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) red[q * kWarps + warp] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = red[q * kWarps];
      for (int w = 1; w < nw; ++w) s += red[q * kWarps + w];
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

// The iteration state is tiny (~1.3 KB) but a single thread walking it in
// global memory pays one L2 round trip per field; the scalar kernels stage it
// in shared memory with one coalesced block-wide copy each way.
__device__ __forceinline__ void state_load(DevState* sm, const DevState* g) {
  constexpr int W = sizeof(DevState) / 4;
  const int* s = reinterpret_cast<const int*>(g);
  int* d = reinterpret_cast<int*>(sm);
  for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = __ldcg(s + i);
  __syncthreads();
}
__device__ __forceinline__ void params_load(DevParams* sm, const DevParams* g) {
  constexpr int W = sizeof(DevParams) / 4;
  const int* s = reinterpret_cast<const int*>(g);
  int* d = reinterpret_cast<int*>(sm);
  for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = __ldg(s + i);
  // (the caller's state_load provides the barrier)
}
__device__ __forceinline__ void state_store(DevState* g, const DevState* sm) {
  constexpr int W = sizeof(DevState) / 4;
  __syncthreads();
  const int* s = reinterpret_cast<const int*>(sm);
  int* d = reinterpret_cast<int*>(g);
  for (int i = threadIdx.x; i < W; i += blockDim.x) d[i] = s[i];
}

// Ring history (DevParams::ring; AA-PDHG on one GPU). Every iteration k
// stores g_k = T(u_k) - u_k (the K1 / K2 epilogues, both halves) into ring
// slot push_slot instead of pushing the pair (du_k, dg_k) (solver.cpp:
// 204-209): with the window gw[0..p] = slots of g_{k-p}..g_k, column t of
// the memory is dg_t = g_t - g_{t-1} and du_t = u_t - u_{t-1}, which is
// g_{t-1} bit for bit after a plain step (u_t = T(u_{t-1})) and is stored by
// k_mix (in du, at g_t's slot) after an accepted candidate — the same
// roundings as the pushed pair. A plain iteration writes 8 bytes per element
// instead of reading u_{k-1} and writing 16. cap + 2 slots: the window holds
// up to cap + 1, and the speculative K1(k+1) of k_plain_loop writes the next
// one before iteration k is decided. The next slot: the first one outside
// the window.
__device__ __forceinline__ int ring_free_slot(const DevParams* P, const DevState* S) {
  int slot = 0;
  for (; slot < P->cap + 1; ++slot) {
    bool used = false;
    for (int q = 0; q < S->gw_n; ++q) used |= S->gw[q] == slot;
    if (!used) break;
  }
  return slot;
}

// memory_push of the ring (control_commit): g_k's slot joins the window, the
// oldest leaves a full one (cap + 1 entries = cap columns)
__device__ __forceinline__ void ring_push(const DevParams* P, DevState* S) {
  int n = S->gw_n;
  if (n == P->cap + 1) {
    for (int q = 1; q < n; ++q) {
      S->gw[q - 1] = S->gw[q];
      S->gdux[q - 1] = S->gdux[q];
    }
    --n;
  }
  S->gw[n] = S->push_slot;
  S->gdux[n] = S->prev_plain ? 0 : 1;
  S->gw_n = n + 1;
  S->mem_size = n;
}

// Role rotation at the end of an iteration (solver.cpp:249-251) and the
// next push slot: u_prev <- u, u <- u_next (the AA candidate or T(u)).
__device__ __forceinline__ void advance(const DevParams* P, DevState* S) {
  int* U = S->u_idx;
  int* KX = S->kx_idx;
  const int old_prev = U[U_PREV];
  U[U_PREV] = U[U_CUR];
  const int okx = KX[KX_CUR];
  if (S->aa_ok) {
    U[U_CUR] = U[U_CAND];
    U[U_CAND] = old_prev;
    KX[KX_CUR] = KX[KX_CAND];
    KX[KX_CAND] = okx;
  } else {
    U[U_CUR] = U[U_HAT];
    U[U_HAT] = old_prev;
    KX[KX_CUR] = KX[KX_HAT];
    KX[KX_HAT] = okx;
  }
  if (P->ring) {
    S->push_slot = ring_free_slot(P, S);
  } else if (P->method != AAPDHG_METHOD_PDHG) {
    const int t = S->g_idx[G_CUR];
    S->g_idx[G_CUR] = S->g_idx[G_PREV];
    S->g_idx[G_PREV] = t;
    // the first of the cap + 1 history slots not in the memory: the slot the
    // next push evicts stays intact until the push commits (k_plain_loop
    // writes the next push while the control still decides this iteration)
    int slot = 0;
    for (; slot < P->cap; ++slot) {
      bool used = false;
      for (int q = 0; q < S->mem_size; ++q) used |= S->mem_slots[q] == slot;
      if (!used) break;
    }
    S->push_slot = slot;
  }
  S->prev_plain = S->aa_ok ? 0 : 1;
  S->aa_attempt = 0;
  S->aa_ok = 0;
  S->k += 1;
  S->loop_iters += 1;
}


// ---------------------------------------------------------------------------
// SpMV core: SELL-32 slices, one per warp
// ---------------------------------------------------------------------------
//
// Random-column SpMVs on B200 are bound by the L1TEX gather rate (~1.2
// cycles per random 8-byte gather per SM with thousands of gathers in flight;
// measured, profiles/microbench/gather_bench.cu). The matrix is stored once,
// on upload, in 32-lane slices (SELL-32): with split factor sf a slice holds
// 32 / sf consecutive short rows, and element k of the slice's row rho sits at
// sl_ptr[s] + 32 (k / sf) + rho sf + (k % sf). A warp owns a slice: its
// (col, val) loads are coalesced, each lane issues all loads of a group of
// kUnroll steps before using them (kUnroll gathers x[col] in flight per lane)
// and adds its share of the row in CSR order; the sf lanes of a row meet in a
// fixed xor tree. sf = 1 (the SERIAL layout) keeps each row in one lane —
// bit-identical to the reference's row-serial matvec (sparse_linalg.cpp:60-69)
// and, on the transposed CSR (entries in ascending original row), to its
// row-ordered scatter matvec_transpose (sparse_linalg.cpp:77-87). The TREE
// layout uses sf > 1 only for matrices with too few rows to fill the GPU.
// Rows longer than kLongRow get a warp each (CTAs after the slice CTAs).

constexpr int kUnroll = 4;

// cp.async (LDGSTS): global -> shared without a register round trip
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Programmatic dependent launch (no-ops when the kernel was launched without
// the attribute): a dependent kernel's CTAs may become resident while the
// primary drains; they load their slice metadata, then wait here until the
// primary grid has completed and its writes are visible.
__device__ __forceinline__ void grid_dependency_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

__device__ __forceinline__ bool skip_launch(const DevState* S, int pred_aa_ok,
                                            const int32_t* stop) {
  if (S) {
    if (S->done) return true;
    if (pred_aa_ok && !S->aa_ok) return true;
  }
  return stop && *stop;
}

// Sum of the row this lane owns in this CTA's work; returns the row (-1 if
// none): the sum is valid in the owning lane only.
struct NoPre {
  __device__ __forceinline__ void operator()(int) const {}
};
__device__ __forceinline__ void l2_prefetch(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// One phase ahead (k_plain_loop): lane 0 of each warp asks L2 for the
// (column, value) stream of the warp's slice of the OTHER matrix, so the
// next phase's dependent stream -> gather chains start from L2 instead of
// DRAM. A slice's streams are contiguous: 32 L int32 and 32 L doubles at a
// 32-element-aligned offset (bulk prefetches need 16-byte granules).
__device__ __forceinline__ void prefetch_slice_streams(const CsrDev& A, int bid) {
  if ((threadIdx.x & 31) != 0 || bid < A.nblk_long || A.interleave) return;
  const int b = bid - A.nblk_long, warp = threadIdx.x >> 5;
  const int sl = int(int64_t(b) * A.nslices / A.nblk_short) + warp;
  if (sl >= int(int64_t(b + 1) * A.nslices / A.nblk_short)) return;
  const int L = __ldg(A.sl_len + sl);
  const int64_t base = __ldg(A.sl_ptr + sl);
  if (L <= 0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.sci + base),
               "r"(uint32_t(128 * L)) : "memory");
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A.sv + base),
               "r"(uint32_t(256 * L)) : "memory");
}

// pre(row): called in the row's owning lane right after the metadata loads
// when the whole slice is one unroll group (short rows): the fused kernels
// prefetch their epilogue operands into L2 so the epilogue does not pay a
// DRAM round trip after the (short) SpMV chain.
//
// COH (the persistent loop, k_plain_loop): the gathered vector changes while
// the kernel runs, so it is read with ld.global.ca (L1 invalidated by the
// grid barrier's acquire) instead of the read-only ld.global.nc path. bid is
// the CTA's index in the layout (blockIdx.x unless the caller remaps it).
template <bool COH>
__device__ __forceinline__ double ldx(const double* p) {
  if constexpr (COH) return __ldca(p);
  else return __ldg(p);
}

// Calibrated partition (CsrDev::sl_start): the warp's slice terms, summed by a
// fixed warp tree, stored as the slice's partial row (lane 0).
template <int NQ>
__device__ __forceinline__ void slice_partials(const CsrDev& A, int b, double (&acc)[NQ],
                                               double* part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sl = __ldg(A.sl_start + b) + warp;
  const bool own = sl < __ldg(A.sl_start + b + 1);
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double v = warp_sum(acc[q]);
    if (lane == 0 && own) part[q * A.nslices + sl] = v;
  }
}

// rep: the warp's rep-th slice of an interleaved layout (returns -2 when the
// warp has no more); otherwise only rep 0 exists.
template <bool SERIAL, int UNROLL = kUnroll, bool COH = false, bool BAL = true,
          class Pre = NoPre, bool PRE_ALL = false>
__device__ __forceinline__ int row_sum(const CsrDev& A, const double* __restrict__ x, double& s,
                                       Pre pre = Pre{}, int bid = -1, int rep = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (bid < 0) bid = int(blockIdx.x);
  s = 0.0;
  if (rep > 0 && (!A.interleave || bid < A.nblk_long)) return -2;
  if (bid >= A.nblk_long) {
    const int b = bid - A.nblk_long;
    int sl;
    if (A.interleave) {  // slices b + nblk * (warp + kWarps * rep)
      sl = int(b + int64_t(A.nblk_short) * (warp + kWarps * rep));
      if (sl >= A.nslices) return -2;
    } else if (BAL && A.sl_start) {  // calibrated partition (k_plain_loop)
      sl = __ldg(A.sl_start + b) + warp;
      if (sl >= __ldg(A.sl_start + b + 1)) return -1;
    } else {  // CTA b owns slices [b * ns / nblk, (b + 1) * ns / nblk): <= kWarps each
      sl = int(int64_t(b) * A.nslices / A.nblk_short) + warp;
      if (sl >= int(int64_t(b + 1) * A.nslices / A.nblk_short)) return -1;
    }
    const int sf = A.sf, j = lane & (sf - 1);
    const int L = __ldg(A.sl_len + sl);
    const int64_t sbase = __ldg(A.sl_ptr + sl);
    const int row = __ldg(A.sl_row + sl * 32 + lane);
    const int cnt = __ldg(A.sl_cnt + sl * 32 + lane);  // this lane's elements
    if ((PRE_ALL || L <= UNROLL) && row >= 0 && j == 0) pre(row);
    const int64_t base = sbase + lane;
    const int32_t* __restrict__ cp = A.sci + base;
    const double* __restrict__ vp = A.sv + base;
    grid_dependency_wait();  // x may be the previous kernel's output (PDL)
    double acc = 0.0;
    for (int t0 = 0; t0 < L; t0 += UNROLL) {
      int c[UNROLL];
      double v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const bool on = t0 + u < cnt;
        c[u] = on ? __ldcs(cp + 32 * (t0 + u)) : 0;
        v[u] = on ? __ldcs(vp + 32 * (t0 + u)) : 0.0;
      }
      double g[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) g[u] = t0 + u < cnt ? ldx<COH>(x + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (t0 + u < cnt) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
    }
    for (int off = sf >> 1; off > 0; off >>= 1)
      acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
    s = acc;
    return (row >= 0 && j == 0) ? row : -1;
  }
  if (!SERIAL && bid < A.nhuge) {
    // a huge row per CTA: thread-strided products, warp trees, then the 8
    // warp sums in warp order (fixed shape: deterministic)
    const int row = __ldg(A.long_rows + bid);
    const int64_t e0 = __ldg(A.rp + row), e1 = __ldg(A.rp + row + 1);
    grid_dependency_wait();
    double acc = 0.0;
    for (int64_t c0 = e0 + threadIdx.x; c0 < e1; c0 += kThreads * kUnroll) {
      double pr[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e = c0 + kThreads * u;
        pr[u] = e < e1 ? __dmul_rn(__ldcs(A.v + e), ldx<COH>(x + __ldcs(A.ci + e))) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) acc = __dadd_rn(acc, pr[u]);
    }
    acc = warp_sum(acc);
    __shared__ double hw[kWarps];
    if (lane == 0) hw[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = hw[0];
      for (int w = 1; w < kWarps; ++w) t = __dadd_rn(t, hw[w]);
      s = t;
    }
    return threadIdx.x == 0 ? row : -1;
  }
  if (!SERIAL && A.ntask > 0) {
    // chunked long rows: a warp per chunk; the chunk that finishes its row
    // last adds the row's chunk sums in chunk order (deterministic)
    const int t = (bid - A.nhuge) * kWarps + warp;
    if (t >= A.ntask) return -1;
    const int lr = __ldg(A.lt_row + t), ch = __ldg(A.lt_chunk + t);
    const int nch = __ldg(A.lt_nch + lr);
    const int row = __ldg(A.long_rows + lr);
    const int64_t r0 = __ldg(A.rp + row), r1 = __ldg(A.rp + row + 1);
    const int64_t e0 = r0 + int64_t(ch) * kLongChunk;  // (one chunk: the whole row)
    const int64_t e1 = nch > 1 && e0 + kLongChunk < r1 ? e0 + kLongChunk : r1;
    grid_dependency_wait();
    double acc = 0.0;
    for (int64_t c0 = e0 + lane; c0 < e1; c0 += 32 * kUnroll) {
      double pr[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e = c0 + 32 * u;
        pr[u] = e < e1 ? __dmul_rn(__ldcs(A.v + e), ldx<COH>(x + __ldcs(A.ci + e))) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) acc = __dadd_rn(acc, pr[u]);
    }
    acc = warp_sum(acc);
    if (nch == 1) {
      s = acc;
      return lane == 0 ? row : -1;
    }
    unsigned last = 0;
    if (lane == 0) {
      const int base = __ldg(A.lt_base + lr);
      __stcg(A.lt_part + base + ch, acc);
      __threadfence();
      last = atomicAdd(A.lt_ticket + lr, 1u) == unsigned(nch - 1);
      if (last) {
        __threadfence();
        double t2 = __ldcg(A.lt_part + base);
        for (int c = 1; c < nch; ++c) t2 = __dadd_rn(t2, __ldcg(A.lt_part + base + c));
        A.lt_ticket[lr] = 0u;  // (ready for the next launch)
        s = t2;
      }
    }
    return (lane == 0 && last) ? row : -1;
  }
  // the other long rows: a warp each, 8 per CTA, after the huge rows' CTAs
  const int lr = A.nhuge + (bid - A.nhuge) * kWarps + warp;
  if (lr >= A.nlong) return -1;
  const int row = __ldg(A.long_rows + lr);
  const int64_t e0 = __ldg(A.rp + row), e1 = __ldg(A.rp + row + 1);
  grid_dependency_wait();
  double acc = 0.0;
  if (SERIAL) {  // CSR order through lane 0
    for (int64_t c0 = e0; c0 < e1; c0 += 32) {
      const int64_t e = c0 + lane;
      const double pr = e < e1 ? __dmul_rn(__ldcs(A.v + e), ldx<COH>(x + __ldcs(A.ci + e))) : 0.0;
      const int n = (e1 - c0) < 32 ? (int)(e1 - c0) : 32;
      for (int q = 0; q < n; ++q) {
        const double t = __shfl_sync(0xffffffffu, pr, q);
        if (lane == 0) acc = __dadd_rn(acc, t);
      }
    }
  } else {
    for (int64_t c0 = e0 + lane; c0 < e1; c0 += 32 * kUnroll) {
      double pr[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e = c0 + 32 * u;
        pr[u] = e < e1 ? __dmul_rn(__ldcs(A.v + e), ldx<COH>(x + __ldcs(A.ci + e))) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) acc = __dadd_rn(acc, pr[u]);
    }
    acc = warp_sum(acc);
  }
  s = acc;
  return lane == 0 ? row : -1;
}


// ---------------------------------------------------------------------------
// peer-memory exchange flags (sharded solve, P2P transports; shard.cuh)
// ---------------------------------------------------------------------------
// Slots of the exchanged buffers (ShardGroup::Buf, shard.h).
enum { P2P_XG = 0, P2P_YG = 1, P2P_SCAL = 3, P2P_DOTS = 4, P2P_XG2 = 5 };

// This shard arrives at exchange `slot` on every shard: one more pass, a
// system-scope fence (cumulative over the stores this thread has observed —
// the caller's CTA barrier / last-CTA ticket brings every store of the
// kernel in), then the sequence number into every shard's flag array.
// Thread 0 only.
__device__ __forceinline__ void p2p_arrive(const DevParams* P, DevState* S, int slot) {
  const unsigned long long seq = (P->p2p_epoch << 32) | (++S->p2p_seq[slot]);
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int q = 0; q < P->p2p_world; ++q)
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P->flag_peer[q] + slot * kMaxPeers +
                                                             P->p2p_rank),
                 "l"(seq)
                 : "memory");
}

// Waits until every shard has arrived at `slot` as often as this one (its own
// arrival came earlier in the stream). A shard that never arrives (crashed
// rank) traps after 30 s instead of hanging the GPU. Thread 0 only; the
// caller's CTA barrier then orders the CTA's reads after the acquire.
__device__ __forceinline__ void p2p_wait(const DevParams* P, const DevState* S, int slot) {
  const unsigned long long seq = (P->p2p_epoch << 32) | S->p2p_seq[slot];
  const uint64_t t0 = globaltimer_ns();
  for (int r = 0; r < P->p2p_world; ++r) {
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];"
                   : "=l"(v) : "l"(P->flag_own + slot * kMaxPeers + r) : "memory");
      if (v >= seq) break;
      if (globaltimer_ns() - t0 > 30000000000ull) asm volatile("trap;");
    }
  }
}

template <bool SERIAL>
__global__ void __launch_bounds__(kThreads, kSpmvBlocksPerSM)
    k_spmv(CsrDev A, VecRef xr, RowsumArgs o, const DevState* S) {
  TL_MARK(14);
  if (skip_launch(S, o.pred_aa_ok, o.stop)) return;
  const double* x = xr.get(S);
  double* out = o.out_pool ? o.out_pool + (int64_t)S->kx_idx[o.out_role] * o.out_stride : o.out;
  for (int rep = 0;; ++rep) {
    double s;
    const int row = row_sum<SERIAL, kUnroll, false, false>(A, x, s, NoPre{}, -1, rep);
    if (row == -2) break;
    if (row >= 0) out[row] = o.rinit ? __dadd_rn(o.rinit[row], s) : s;
  }
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
// in four pieces so the fused TREE tail can run them on two warps:
//   control_kkt_records  KKT of u_k (kept for the finish), the KKT fields of
//                        record k-1, the base fields of record k
//   control_decide       termination (FIXED_POINT -> KKT_TOL -> RESIDUAL_TOL
//                        -> MAX_ITERS -> TIMEOUT), safeguard, batch count
//   control_commit       memory push, plain-step counter, role rotation
//   control_setcond      the graph's IF / WHILE conditions
// control_logic runs them in sequence (one thread). Records are read by the
// host only below rec_complete, so record k's base fields may be written
// even when the iteration terminates.
struct Decision {
  int attempt, left;
};

__device__ __noinline__ void control_kkt_records(const DevParams* P, DevState* S, uint64_t k,
                                                    double g2, double bound, double qy, double cx,
                                                    double infeas, double dual_sq,
                                                    double elapsed_in) {
  double kkt[4];
  kkt_from_sums(P->nrm_q, P->nrm_c, bound, qy, cx, infeas, dual_sq, kkt);
  for (int q = 0; q < 4; ++q) S->kkt[q] = kkt[q];
  const uint64_t mask = P->rec_cap - 1;  // rec_cap is a power of two
  if (k > 0) {  // the record of iterate k-1 takes the KKT of the produced iterate u_k
    aapdhg_record* r = P->rec + ((k - 1) & mask);
    r->r_gap = kkt[0];
    r->r_primal = kkt[1];
    r->r_dual = kkt[2];
    r->objective = kkt[3];
    r->elapsed_s = elapsed_in >= 0.0
                       ? elapsed_in
                       : (double)(globaltimer_ns() - S->t0_ns) * 1e-9 + P->wall_offset_s;
  }
  aapdhg_record* r = P->rec + (k & mask);
  r->k = k;
  r->g_norm = sqrt(g2);
  r->aa_step = 0;
  r->i = S->i;  // counters before this iteration's step
  r->j = S->j;
}

__device__ __noinline__ Decision control_decide(const DevParams* P, DevState* S, uint64_t k,
                                                   double g2, double bound, double qy, double cx,
                                                   double infeas, double dual_sq,
                                                   double elapsed_in, double pw_in) {
  const double gkn = sqrt(g2);
  S->gkn = gkn;
  S->aa_attempt = 0;
  S->aa_ok = 0;
  const double elapsed = elapsed_in >= 0.0
                             ? elapsed_in
                             : (double)(globaltimer_ns() - S->t0_ns) * 1e-9 + P->wall_offset_s;
  bool attempt = false;
  do {
    if (k == 0) {  // priming step, solver.cpp:168-172
      S->g0n = gkn;
      break;
    }
    S->rec_complete = k;
    if (k == 1 && S->g0n == 0.0) { finish_solve(S, AAPDHG_SOLVE_FIXED_POINT_START, U_PREV, 0.0); break; }
    if (P->kkt_terminate) {
      double kkt[4];
      kkt_from_sums(P->nrm_q, P->nrm_c, bound, qy, cx, infeas, dual_sq, kkt);
      if (smax(smax(kkt[0], kkt[1]), kkt[2]) <= P->kkt_eps) {
        finish_solve(S, AAPDHG_SOLVE_KKT_TOL, U_CUR, gkn);
        break;
      }
    }
    if (gkn < P->toll) { finish_solve(S, AAPDHG_SOLVE_RESIDUAL_TOL, U_CUR, gkn); break; }
    if (S->i + S->j >= P->max_iters) { finish_solve(S, AAPDHG_SOLVE_MAX_ITERS, U_CUR, gkn); break; }
    if (elapsed >= P->max_wall_s) { finish_solve(S, AAPDHG_SOLVE_TIMEOUT, U_CUR, gkn); break; }
    if (P->method != AAPDHG_METHOD_PDHG) {
      // safeguard_pass, solver.cpp:59-62, with the host std::pow table
      const double pw = pw_in >= 0.0           ? pw_in
                        : S->i < P->pow_len ? P->pow_tab[S->i]
                                          : pow((double)S->i + 1.0, -(1.0 + P->safeguard_eps));
      attempt = gkn <= __dmul_rn(__dmul_rn(P->safeguard_d, S->g0n), pw);
    }
  } while (false);
  Decision d;
  d.attempt = attempt ? 1 : 0;
  d.left = S->done ? 0 : --S->batch_left;
  return d;
}

__device__ __noinline__ void control_commit(const DevParams* P, DevState* S, uint64_t k,
                                               Decision d) {
  if (S->done) return;
  if (P->ring) ring_push(P, S);  // (g_0 opens the window at k = 0)
  if (k > 0) {
    if (P->method != AAPDHG_METHOD_PDHG && !P->ring) {  // memory_push / FaaState::push
      if (S->mem_size == P->cap) {
        for (int t = 1; t < S->mem_size; ++t) S->mem_slots[t - 1] = S->mem_slots[t];
        S->mem_slots[S->mem_size - 1] = S->push_slot;
      } else {
        S->mem_slots[S->mem_size++] = S->push_slot;
      }
    }
    if (d.attempt) S->aa_attempt = 1;
    else S->j += 1;
  }
  // no AA attempt: the iteration ends here (the AA branch commits otherwise)
  if (!d.attempt) advance(P, S);
}

__device__ __noinline__ void control_setcond(const DevParams* P, Decision d) {
  if (P->use_cond) {
    cudaGraphSetConditional(P->cond_aa, d.attempt ? 1u : 0u);
    cudaGraphSetConditional(P->cond_loop, d.left > 0 ? 1u : 0u);
  }
}

// elapsed_in >= 0: the wall clock agreed by all shards (sharded solve)
__device__ __noinline__ void control_logic(const DevParams* P, DevState* S, double g2,
                                           double bound, double qy, double cx, double infeas,
                                           double dual_sq, double elapsed_in = -1.0,
                                           double pw_in = -1.0) {
  const uint64_t k = S->k;
  control_kkt_records(P, S, k, g2, bound, qy, cx, infeas, dual_sq, elapsed_in);
  const Decision d = control_decide(P, S, k, g2, bound, qy, cx, infeas, dual_sq, elapsed_in, pw_in);
  control_commit(P, S, k, d);
  control_setcond(P, d);
}

// ---------------------------------------------------------------------------
// TREE-mode control without a launch of its own
// ---------------------------------------------------------------------------

// Sums NQ rows of per-CTA partials (row q at part[q * nu]) in a fixed shape:
// thread-strided in CTA order, warp xor tree, warps in order. Result in
// thread 0 of the calling CTA. red holds NQ * 32 doubles.
template <int NQ>
__device__ __forceinline__ void reduce_partial_rows(const double* part, int nu, double (&t)[NQ],
                                                    double* red) {
  double v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = 0.0;
  // groups of 4 strides: every load of a group is in flight before the adds
  // (the adds keep the CTA order b, b + blockDim, ...)
  for (int b0 = threadIdx.x; b0 < nu; b0 += 4 * blockDim.x) {
    double x[4][NQ];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int b = b0 + u * blockDim.x;
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[u][q] = b < nu ? __ldcg(part + q * nu + b) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b0 + u * int(blockDim.x) < nu)
#pragma unroll
        for (int q = 0; q < NQ; ++q) v[q] = __dadd_rn(v[q], x[u][q]);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) red[q * 32 + warp] = v[q];
  __syncthreads();
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double s = red[q * 32];
      for (int w = 1; w < nw; ++w) s = __dadd_rn(s, red[q * 32 + w]);
      t[q] = s;
    }
}

// Fused TREE-mode control of k_primal_side (threadFenceReduction pattern).
// tail_prefetch() runs in every CTA right after its rows: cp.async copies of
// the state, the parameters and the safeguard power (i+1)^-(1+eps) into
// shared memory, landing while the CTA reduces and elects. CTA 0 folds K1's
// per-CTA partials (complete: K1 finished before K2 started) into S->tot1.
// The last CTA to finish (acq_rel ticket) then needs one round trip — the
// K2 partials — before it runs the control logic on its shared copy. Sums
// have a fixed shape whichever CTA is last: deterministic.
struct TailSmem {
  DevState st;
  DevParams pr;
  double pw;
};


__device__ __forceinline__ void tail_prefetch(TailSmem& ts, const DevParams* P,
                                              const DevState* S) {
  constexpr int WS = sizeof(DevState) / 8, WP = sizeof(DevParams) / 8;
  static_assert(sizeof(DevState) % 8 == 0 && sizeof(DevParams) % 8 == 0, "8-byte copies");
  for (int i = threadIdx.x; i < WS; i += blockDim.x)
    cp_async8(reinterpret_cast<uint64_t*>(&ts.st) + i, reinterpret_cast<const uint64_t*>(S) + i);
  for (int i = threadIdx.x; i < WP; i += blockDim.x)
    cp_async8(reinterpret_cast<uint64_t*>(&ts.pr) + i, reinterpret_cast<const uint64_t*>(P) + i);
  if (threadIdx.x == 0) {
    // S->i is constant during K2; the table lookup of the safeguard
    const uint64_t i = S->i;
    if (P->pow_tab && i < P->pow_len) cp_async8(&ts.pw, P->pow_tab + i);
    else ts.pw = -1.0;
  }
}

// K1's per-CTA partials folded into S->tot1 by CTA 0 of k_primal_side (K1
// finished before K2 started).
__device__ __forceinline__ void tail_fold_k1(const IterBufs& B, DevState* S, double* red) {
  double t1[P1_COUNT];
  reduce_partial_rows<P1_COUNT>(B.part1, B.nu1, t1, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < P1_COUNT; ++q) S->tot1[q] = B.nu1 > 0 ? t1[q] : 0.0;
}

// The last CTA's part of the fused control: K2 partials (nu2 rows), then the
// control logic on the prefetched shared copy of the state. persist: the
// caller is k_plain_loop, which only hands the graph conditions over when it
// stops (AA attempt, batch end, termination). Returns true when it stops.
__device__ __noinline__ bool tail_control(const IterBufs& B, DevState* S, TailSmem& ts, int nu2,
                                          bool persist, double* red) {
#ifdef AAPDHG_TAIL_STAMPS
  const uint64_t ts0 = globaltimer_ns();
  if (threadIdx.x == 0 && persist) g_dbg[1] += ts0 - g_dbg[10];  // K2 phase -> election won
#endif
  double t2[P2_COUNT];
  reduce_partial_rows<P2_COUNT>(B.part2, nu2, t2, red);
  cp_async_wait_all();
  __syncthreads();
#ifdef AAPDHG_TAIL_STAMPS
  const uint64_t ts1 = globaltimer_ns();
#endif
  if (B.fused_ctrl == 2) {  // sharded: this shard's totals (k_local_totals' layout)
    if (threadIdx.x == 0) {
      double own[8];
      own[0] = __ldcg(&S->tot1[P1_GX2]);
      own[1] = __ldcg(&S->tot1[P1_BOUND]);
      own[2] = __ldcg(&S->tot1[P1_CX]);
      own[3] = __ldcg(&S->tot1[P1_DUALSQ]);
      own[4] = t2[P2_GY2];
      own[5] = t2[P2_QY];
      own[6] = t2[P2_INFEAS];
      own[7] = (double)(globaltimer_ns() - ts.st.t0_ns) * 1e-9 + ts.pr.wall_offset_s;
      for (int q = 0; q < ts.pr.ndst; ++q)  // own chunk / every peer's chunk
#pragma unroll
        for (int t = 0; t < 8; ++t) ts.pr.scal_dst[q][t] = own[t];
      S->ticket = 0;
      // P2P: publish yhat (every CTA's stores) and the totals
      if (ts.pr.p2p_fused) p2p_arrive(&ts.pr, S, P2P_YG);
    }
    return true;
  }
  // the control on two warps: KKT + records (warp 1) beside the decision and
  // the graph conditions (warp 0); the commit needs the decision
  __shared__ double sums[7];
  __shared__ Decision dec;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < P1_COUNT; ++q) sums[q] = __ldcg(&S->tot1[q]);
#pragma unroll
    for (int q = 0; q < P2_COUNT; ++q) sums[P1_COUNT + q] = t2[q];
  }
  __syncthreads();
  DevState& sm = ts.st;
  const uint64_t k = sm.k;
  const double g2 = __dadd_rn(sums[P1_GX2], sums[P1_COUNT + P2_GY2]);
  const double bound = sums[P1_BOUND], qy = sums[P1_COUNT + P2_QY], cx = sums[P1_CX];
  const double infeas = sums[P1_COUNT + P2_INFEAS], dsq = sums[P1_DUALSQ];
  if (threadIdx.x == 32)
    control_kkt_records(&ts.pr, &sm, k, g2, bound, qy, cx, infeas, dsq, -1.0);
  if (threadIdx.x == 0) {
    sm.ticket = 0;
    dec = control_decide(&ts.pr, &sm, k, g2, bound, qy, cx, infeas, dsq, -1.0, ts.pw);
  }
  __syncthreads();
#ifdef AAPDHG_TAIL_STAMPS
  const uint64_t ts2 = globaltimer_ns();
#endif
  const bool stop = !persist || dec.attempt || dec.left <= 0;
  if (threadIdx.x == 0 && stop) {
    control_setcond(&ts.pr, dec);
    if (persist) sm.loop_exits += 1;
  }
  if (threadIdx.x == 32) control_commit(&ts.pr, &sm, k, dec);
  state_store(S, &ts.st);
#ifdef AAPDHG_TAIL_STAMPS
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t ts3 = globaltimer_ns();
    g_dbg[2] += ts1 - ts0;  // K2 partials reduced
    g_dbg[3] += ts2 - ts1;  // kkt/records + decide
    g_dbg[4] += ts3 - ts2;  // setcond + commit + state store
    g_dbg[5] += 1;
    g_dbg[6] = ts3;
    g_dbg[12] = dec.attempt;
  }
#endif
  return stop;
}

// Fused TREE-mode control of k_primal_side: CTA 0 folds K1's partials, the
// last CTA to finish (acq_rel ticket) runs tail_control.
__device__ __forceinline__ void fused_control_tail(const IterBufs& B, DevState* S, TailSmem& ts) {
  __shared__ double red[P1_COUNT * 32];
  __shared__ int last;
  if (blockIdx.x == 0) tail_fold_k1(B, S, red);
  if (threadIdx.x == 0) {
    if (B.p2p_sys) __threadfence_system();  // P2P across GPUs: this CTA's peer stores first
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(&S->ticket) : "memory");
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  tail_control(B, S, ts, gridDim.x, false, red);
}

// One column pass of an L2-blocked SpMV: part[row] (+)= the row's products
// with the columns of this block (passes in block order: deterministic).
template <int U>
__device__ __forceinline__ void spmv_pass_body(const CsrDev& A, const VecRef& xr,
                                               double* __restrict__ part, int first,
                                               const DevState* S, int pred_aa,
                                               const int32_t* stop) {
  TL_MARK(20);
  if (skip_launch(S, 0, stop)) return;
  if (S && pred_aa == 1 && (!S->aa_attempt || !S->aa_ok)) return;  // (AA recache passes)
  const double* x = xr.get(S);
  for (int rep = 0;; ++rep) {
    double s;
    // later passes (first = 0): mode 2 asks the row's partial into L2 with the
    // metadata, mode 3 loads it into a register there, so the read-add-store
    // after the gather chain does not wait for a DRAM round trip
    double prev = 0.0;
    auto pre = [&](int r) {
      if (first == 2) l2_prefetch(part + r);
      else if (first == 3) prev = __ldcs(part + r);
    };
    const int row = row_sum<false, U, false, false, decltype(pre), true>(A, x, s, pre, -1, rep);
    if (row == -2) break;
    if (row >= 0)
      __stcs(part + row, first == 1 ? s : __dadd_rn(first == 3 ? prev : __ldcs(part + row), s));
  }
}


__global__ void __launch_bounds__(kThreads, kSpmvBlocksPerSM)
    k_spmv_pass(CsrDev A, VecRef xr, double* __restrict__ part, int first, const DevState* S,
                int pred_aa, const int32_t* stop) {
  spmv_pass_body<kUnroll>(A, xr, part, first, S, pred_aa, stop);
}

// ---------------------------------------------------------------------------
// the fused PDHG halves
// ---------------------------------------------------------------------------

// K1 on K' (row j of K' = column j of K), t = (K'y)_j:
//   xhat_j = min(max(x_j - tau (c_j - t), l_j), u_j)      pdhg_core.cpp:49-53
//   lambda_j = P_Lambda(c_j - t)                           solver.cpp:67-71
//   per-CTA partials: (xhat-x)^2, bound term, (c-t-lambda)^2, c_j x_j
//   PUSH: du_j = x_j - xprev_j, dg_j = g_j - gprev_j, g_j = xhat_j - x_j
// VAR 2 (experiment, AAPDHG_K1VAR=2): the SpMV alone, no epilogue.
// CTA bid of nb; red holds P1_COUNT * kWarps doubles.
// dual_epilogue: column j given t = (K'y)_j; the terms of u_k are assigned
// to acc[].
template <bool SERIAL, bool PUSH>
__device__ __forceinline__ void dual_epilogue(int j, double t, const double* __restrict__ x,
                                              const IterBufs& B, const DevParams* __restrict__ P,
                                              const DevState* S, double (&acc)[P1_COUNT]) {
  const int64_t N = P->N;
  const double xj = x[j], cj = __ldg(B.c + j), lj = __ldg(B.l + j), uj = __ldg(B.u + j);
  double xn = __dsub_rn(xj, __dmul_rn(P->tau, __dsub_rn(cj, t)));
  xn = smin(smax(xn, lj), uj);
  B.upool[(int64_t)S->u_idx[U_HAT] * N + j] = xn;
  for (int q = 0; q < P->ndst; ++q) P->xg_dst[q][j] = xn;  // sharded: own / peers' chunks
  const double d = __dsub_rn(xn, xj);
  const double red_c = __dsub_rn(cj, t);
  const double lam = project_lambda1(red_c, lj, uj);
  double bt = 0.0;
  if (isfinite(lj) && lam > 0.0) bt = __dmul_rn(lj, lam);
  if (isfinite(uj) && lam < 0.0) bt = __dmul_rn(uj, lam);
  const double dv = __dsub_rn(red_c, lam);
  acc[P1_GX2] = __dmul_rn(d, d);
  acc[P1_BOUND] = bt;
  acc[P1_DUALSQ] = __dmul_rn(dv, dv);
  acc[P1_CX] = __dmul_rn(cj, xj);
  if (PUSH && P->ring) {  // ring history: g_k only
    B.gpool[(int64_t)S->push_slot * N + j] = d;
  } else if constexpr (PUSH) {
    // after a plain step u_k = T(u_{k-1}) bit for bit, so g_{k-1} = u_k -
    // u_{k-1} = du: g is only materialized (k_stage_g) for AA attempts
    const int64_t slot = S->push_slot;
    const double xp = B.upool[(int64_t)S->u_idx[U_PREV] * N + j];
    const double dx = __dsub_rn(xj, xp);
    const double gp = S->prev_plain ? dx : B.gpool[(int64_t)S->g_idx[G_PREV] * N + j];
    B.du[slot * N + j] = dx;
    B.dg[slot * N + j] = __dsub_rn(d, gp);
  }
  if (SERIAL || P->store_T) B.T[j] = t;
}

template <bool SERIAL, bool PUSH, int VAR = 0, bool COH = false, bool MULTI = false>
__device__ __forceinline__ void dual_side_rows(const CsrDev& KT, const IterBufs& B,
                                               const DevParams* __restrict__ P, DevState* S,
                                               int bid, int nb, double* red) {
  const int64_t N = P->N;
  const double* x = B.upool + (int64_t)S->u_idx[U_CUR] * N;
  double acc[P1_COUNT] = {0.0, 0.0, 0.0, 0.0};
  bool first = true;  // one row per thread: the terms themselves (no add)
  for (int rep = 0;; ++rep) {
    double t;
    const int j = row_sum<SERIAL, kUnroll, COH, !MULTI>(
        KT, P->ygather ? P->ygather : x + P->n, t, [&](int r) {
          l2_prefetch(x + r);
          l2_prefetch(B.c + r);
          l2_prefetch(B.l + r);
          l2_prefetch(B.u + r);
          if (PUSH && !P->ring) l2_prefetch(B.upool + (int64_t)S->u_idx[U_PREV] * N + r);
        }, bid, rep);
    if (j == -2) break;
    if (B.rinit1 && j >= 0) t = __dadd_rn(B.rinit1[j], t);  // earlier column passes
    if (VAR == 2) {  // experiment: SpMV only
      if (j >= 0) B.T[j] = t;
      continue;
    }
    if (j >= 0) {
      double term[P1_COUNT];
      dual_epilogue<SERIAL, PUSH>(j, t, x, B, P, S, term);
#pragma unroll
      for (int q = 0; q < P1_COUNT; ++q) acc[q] = first ? term[q] : __dadd_rn(acc[q], term[q]);
      first = false;
    }
    if constexpr (!MULTI) break;  // (one slice per warp: no loop state)
  }
  if (VAR == 2) return;
  if constexpr (!SERIAL && !MULTI) {
    if (KT.sl_start) {
      slice_partials<P1_COUNT>(KT, bid, acc, B.part1);
      return;
    }
  }
  if (!SERIAL) {
    block_sum<P1_COUNT>(acc, red);
    if (threadIdx.x == 0)
#pragma unroll
      for (int q = 0; q < P1_COUNT; ++q) B.part1[q * nb + bid] = acc[q];
  }
}

// MULTI: the layout is interleaved (several slices per warp, CsrDev)
template <bool SERIAL, bool PUSH, int VAR = 0, bool MULTI = false>
#ifndef AAPDHG_K12_MINBLOCKS
#define AAPDHG_K12_MINBLOCKS kSpmvBlocksPerSM
#endif
__global__ void __launch_bounds__(kThreads, AAPDHG_K12_MINBLOCKS)
    k_dual_side(CsrDev KT, IterBufs B, const DevParams* __restrict__ P, DevState* S) {
  TL_MARK(16);
  launch_dependents();  // k_primal_side may start its prologue (PDL)
  if (S->done) return;
#ifdef AAPDHG_TAIL_STAMPS
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_dbg[6]) {
    const int a = g_dbg[12] ? 13 : 8;  // after an AA branch / a plain step
    g_dbg[a] += globaltimer_ns() - g_dbg[6];  // K2 tail end -> next K1 CTA 0 start
    g_dbg[a + 1] += 1;
    g_dbg[6] = 0;
  }
#endif
  __shared__ double red[P1_COUNT * kWarps];
  const bool fused = !SERIAL && P->p2p_fused;
  if (fused) {  // y of u_k: every shard's K2 (or AA branch) stored its chunk here
    if (threadIdx.x == 0) p2p_wait(P, S, P2P_YG);
    __syncthreads();
  }
  dual_side_rows<SERIAL, PUSH, VAR, false, MULTI>(KT, B, P, S, int(blockIdx.x), int(gridDim.x), red);
  if (fused) {  // the last CTA publishes xhat (every CTA stored its chunk to every shard)
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
      // peers on other GPUs: this CTA's remote stores drain before the ticket
      // (in-process peers: the ticket's gpu-scope release covers them)
      if (P->p2p_sys) __threadfence_system();
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(prev) : "l"(&S->ticket1) : "memory");
      last = prev == gridDim.x - 1;
      if (last) {
        S->ticket1 = 0;
        p2p_arrive(P, S, P2P_XG);
      }
    }
  }
}

// K2 on K, s = (K xhat)_i:
//   yhat_i = y_i + sigma (q_i - (2 s - (K x)_i)), clamped >= 0 for i < m1
//                                                         pdhg_core.cpp:55-60
//   K xhat cached as the next K x (solver.cpp:90 / pdhg_core.cpp:56)
//   per-CTA partials: (yhat-y)^2, q_i y_i, primal infeasibility of u_k
// The rows and epilogue; acc gets this thread's share of the partials.
// primal_epilogue: row i given s = (K xhat)_i; the terms of u_k are
// assigned to acc[].
template <bool PUSH>
__device__ __forceinline__ void primal_epilogue(int i, double s, const IterBufs& B,
                                                const DevParams* __restrict__ P, const DevState* S,
                                                double (&acc)[P2_COUNT]) {
  const int64_t N = P->N;
  const int n = P->n, mr = P->mrows;
  const double yi = B.upool[(int64_t)S->u_idx[U_CUR] * N + n + i];
  const double qi = __ldg(B.q + i);
  const double kxi = B.kxpool[(int64_t)S->kx_idx[KX_CUR] * mr + i];
  double yn =
      __dadd_rn(yi, __dmul_rn(P->sigma, __dsub_rn(qi, __dsub_rn(__dmul_rn(2.0, s), kxi))));
  if (i < P->m1) yn = smax(yn, 0.0);
  B.upool[(int64_t)S->u_idx[U_HAT] * N + n + i] = yn;
  for (int q = 0; q < P->ndst; ++q) P->yg_dst[q][i] = yn;
  B.kxpool[(int64_t)S->kx_idx[KX_HAT] * mr + i] = s;
  const double d = __dsub_rn(yn, yi);
  double v = __dsub_rn(qi, kxi);
  if (i < P->m1) v = smax(v, 0.0);
  acc[P2_GY2] = __dmul_rn(d, d);
  acc[P2_QY] = __dmul_rn(qi, yi);
  acc[P2_INFEAS] = __dmul_rn(v, v);
  if (PUSH && P->ring) {  // ring history: g_k only
    B.gpool[(int64_t)S->push_slot * N + n + i] = d;
  } else if constexpr (PUSH) {
    const int64_t slot = S->push_slot;
    const double yp = B.upool[(int64_t)S->u_idx[U_PREV] * N + n + i];
    const double dy = __dsub_rn(yi, yp);
    const double gp = S->prev_plain ? dy : B.gpool[(int64_t)S->g_idx[G_PREV] * N + n + i];
    B.du[slot * N + n + i] = dy;
    B.dg[slot * N + n + i] = __dsub_rn(d, gp);
  }
}

template <bool SERIAL, bool PUSH, bool COH = false, bool MULTI = false>
__device__ __forceinline__ void primal_side_rows(const CsrDev& K, const IterBufs& B,
                                                 const DevParams* __restrict__ P, DevState* S,
                                                 int bid, double (&acc)[P2_COUNT]) {
  const int64_t N = P->N;
  bool first = true;  // one row per thread: the terms themselves (no add)
  for (int rep = 0;; ++rep) {
    double s;
    const int i = row_sum<SERIAL, kUnroll, COH, !MULTI>(
        K, P->xgather ? P->xgather : B.upool + (int64_t)S->u_idx[U_HAT] * N, s, NoPre{}, bid,
        rep);
    if (i == -2) break;
    if (B.rinit2 && i >= 0) s = __dadd_rn(B.rinit2[i], s);  // earlier column passes
    if (i >= 0) {
      double term[P2_COUNT];
      primal_epilogue<PUSH>(i, s, B, P, S, term);
#pragma unroll
      for (int q = 0; q < P2_COUNT; ++q) acc[q] = first ? term[q] : __dadd_rn(acc[q], term[q]);
      first = false;
    }
    if constexpr (!MULTI) break;  // (one slice per warp: no loop state)
  }
}

// VAR 2 (experiment, AAPDHG_K2VAR=2): the SpMV alone, no epilogue or control
template <bool SERIAL, bool PUSH, int VAR = 0, bool MULTI = false>
__global__ void __launch_bounds__(kThreads, AAPDHG_K12_MINBLOCKS)
    k_primal_side(CsrDev K, IterBufs B, const DevParams* __restrict__ P, DevState* S) {
  TL_MARK(17);
  if (S->done) return;
  if constexpr (VAR == 2) {
    double s;
    const int i = row_sum<SERIAL, kUnroll, false, false>(K, B.upool + (int64_t)S->u_idx[U_HAT] * P->N, s);
    if (i >= 0) B.kxpool[(int64_t)S->kx_idx[KX_HAT] * P->mrows + i] = s;
    return;
  }
  __shared__ double red[P2_COUNT * kWarps];
  double acc[P2_COUNT] = {0.0, 0.0, 0.0};
  if (!SERIAL && P->p2p_fused) {  // xhat: every shard's K1 stored its chunk here
    if (threadIdx.x == 0) p2p_wait(P, S, P2P_XG);
    __syncthreads();
  }
  primal_side_rows<SERIAL, PUSH, false, MULTI>(K, B, P, S, int(blockIdx.x), acc);
  if (!SERIAL) {
    __shared__ __align__(16) TailSmem ts;
    if (B.fused_ctrl) tail_prefetch(ts, P, S);
    block_sum<P2_COUNT>(acc, red);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < P2_COUNT; ++q) B.part2[q * gridDim.x + blockIdx.x] = acc[q];
    }
    if (B.fused_ctrl) fused_control_tail(B, S, ts);
  }
}

// ---------------------------------------------------------------------------
// L2-blocked TREE layouts (configs[4]): every column block of K' and of K runs
// as a plain pass (k_spmv_pass; the last one leaves the finished sums, added
// in block order as the fused kernels add them), then the epilogues in row
// order over those sums: the vector operands stream coalesced instead of in
// the slices' length-sorted order, and no block's gathers share L2 with them.
// Grid-stride rows; each thread's terms in row order, then the fixed CTA tree.
// ---------------------------------------------------------------------------
template <bool PUSH>
__global__ void __launch_bounds__(kThreads)
    k_dual_epi(const double* __restrict__ T, IterBufs B, const DevParams* __restrict__ P,
               DevState* S, int j0, int j1, int part_off, int part_rows) {
  TL_MARK(26);
  if (S->done) return;
  __shared__ double red[P1_COUNT * kWarps];
  const double* x = B.upool + (int64_t)S->u_idx[U_CUR] * P->N;
  double acc[P1_COUNT] = {0.0, 0.0, 0.0, 0.0};
  bool first = true;
  for (int64_t j = j0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < j1;
       j += (int64_t)gridDim.x * blockDim.x) {
    double term[P1_COUNT];
    dual_epilogue<false, PUSH>(int(j), T[j], x, B, P, S, term);
#pragma unroll
    for (int q = 0; q < P1_COUNT; ++q) acc[q] = first ? term[q] : __dadd_rn(acc[q], term[q]);
    first = false;
  }
  block_sum<P1_COUNT>(acc, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < P1_COUNT; ++q) B.part1[q * part_rows + part_off + blockIdx.x] = acc[q];
}

template <bool PUSH>
__global__ void __launch_bounds__(kThreads)
    k_primal_epi(const double* __restrict__ Kx, IterBufs B, const DevParams* __restrict__ P,
                 DevState* S) {
  TL_MARK(27);
  if (S->done) return;
  __shared__ double red[P2_COUNT * kWarps];
  double acc[P2_COUNT] = {0.0, 0.0, 0.0};
  bool first = true;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P->mrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    double term[P2_COUNT];
    primal_epilogue<PUSH>(int(i), Kx[i], B, P, S, term);
#pragma unroll
    for (int q = 0; q < P2_COUNT; ++q) acc[q] = first ? term[q] : __dadd_rn(acc[q], term[q]);
    first = false;
  }
  __shared__ __align__(16) TailSmem ts;
  if (B.fused_ctrl) tail_prefetch(ts, P, S);
  block_sum<P2_COUNT>(acc, red);
  if (threadIdx.x == 0)
#pragma unroll
    for (int q = 0; q < P2_COUNT; ++q) B.part2[q * gridDim.x + blockIdx.x] = acc[q];
  if (B.fused_ctrl) fused_control_tail(B, S, ts);
}

// ---------------------------------------------------------------------------
// the persistent plain-step loop (TREE, fused control, graph replay)
// ---------------------------------------------------------------------------
//
// Under graph replay every iteration otherwise pays the WHILE/IF node
// overhead between K2's control and the next K1, and the last CTA's control
// (~5 us) sits between K2 and the next K1 (globaltimer stamps,
// profiles/exp_tail_stamps.py). k_plain_loop runs consecutive plain
// iterations in one co-resident grid (cooperative launch): CTAs 0..W-1 are
// workers that run K1 and K2 of each iteration (the same rows, epilogues and
// partial layout as k_dual_side / k_primal_side), CTA W is the control CTA.
// Per iteration k:
//   workers   K1(k) | barrier 1 | K2(k) | barrier 2 | K1(k+1) ...
//   control          barrier 1 -> fold K1 partials | barrier 2 -> K2 partials,
//                    control(k) -> arrives at barrier 1 of k+1
// A worker starts K1(k+1) right after barrier 2 on the roles of a plain step,
// which it derives itself (control_commit + advance on its own copy of the
// state), while the control CTA decides iteration k: the control leaves the
// critical path. When the control stops the loop (AA attempt -> the graph's
// IF branch, batch end, termination) it raises a flag with its barrier-1
// arrival; the workers drop the speculative K1(k+1) and return. Nothing that
// K1(k+1) wrote is read before it is rewritten: x-hat goes to the buffer of
// u_{k-1} (no consumer after iteration k; at k = 1 the only exception, the
// fixed-point start, rewrites u_0 with the identical T_x(u_0)), the x-half of
// the push to the spare history slot (advance keeps cap + 1 slots), and the
// K1 partials, which the control CTA folded before barrier 2. Results are
// bit-identical to the per-kernel graph with the same CTA layout.
#ifdef AAPDHG_PLAIN_STAMPS
__device__ unsigned long long g_plain_dbg[8];
// experiment build: per CTA (k_plain_loop worker) K1 / K2 phase sums, count, SM id
__device__ unsigned long long g_plain_cta[1024 * 4];
#endif
struct GridBar {
  unsigned long long arrive1;  // barrier 1: arrivals (low 40 bits) + stops (high bits)
  unsigned long long arrive2;  // barrier 2: arrivals
  // predicted stops: the control publishes, after its barrier-1 arrival,
  // decided = k + 1 for iteration k; before its barrier-2 arrival, maystop =
  // (k << 1) | flag: flag 0 when the x part of ||g_k||^2 alone already rules
  // out an AA attempt and the residual tolerance (stop_likely)
  unsigned long long decided;
  unsigned long long maystop;
  double g_last, g_prev, thr, pad1;
};
constexpr unsigned long long kBarCount = (1ull << 40) - 1;
constexpr unsigned long long kBarStop = 1ull << 40;

__device__ __forceinline__ unsigned long long atom_add_acq_rel(unsigned long long* p,
                                                               unsigned long long v) {
  unsigned long long prev;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;"
               : "=l"(prev) : "l"(p), "l"(v) : "memory");
  return prev;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Arrive at a barrier of nb participants and wait for the instance to fill.
// Spins with relaxed loads (an acquire load invalidates the SM's L1 — under
// CTAs still gathering — on every poll), then acquires once. Thread 0 only.
__device__ __forceinline__ unsigned long long bar_arrive_wait(unsigned long long* p,
                                                              unsigned long long add,
                                                              unsigned long long nb) {
  const unsigned long long prev = atom_add_acq_rel(p, add);
  const unsigned long long target = ((prev & kBarCount) / nb + 1) * nb;
  while ((ld_relaxed(p) & kBarCount) < target) {
  }
  return ld_acquire(p);
}

// A worker's guess, after barrier 2 of iteration k = st.k, that the control
// will stop the launch after k (st: the state before k's commit; wp:
// iterations already decided in this launch). Exact for the batch end and
// max_iters; for the safeguard and the residual tolerance the control CTA
// publishes before barrier 2 whether the x part of ||g_k||^2 (known since
// barrier 1) leaves them possible: ||g_k|| >= ||g_x|| (a sum of non-negative
// terms), so flag 0 is exact. Only then do the workers wait for the decision;
// the rare KKT / wall-clock stops stay speculative (a dropped K1).
__device__ __forceinline__ bool stop_likely(const DevParams* P, const GridBar* gb,
                                            const DevState& st, int wp) {
  if (P->no_stop_predict) return false;
  if (st.batch_left - (wp + 1) <= 0) return true;
  if (st.k > 0 && st.i + st.j >= P->max_iters) return true;
  if (st.k < 2) return true;  // priming / fixed-point start
  const unsigned long long ms = ld_relaxed(&gb->maystop);
  return (ms >> 1) != st.k || (ms & 1ull);
}

// The control CTA's maystop flag of iteration k (stop_likely): can the
// decision be an AA attempt or the residual tolerance, given the x part gx2
// of ||g_k||^2? Thread 0.
__device__ __forceinline__ void publish_maystop(const DevParams& pr, const DevState& sm,
                                                GridBar* gb, double gx2) {
  const double gx = sqrt(gx2);
  bool may = gx < pr.toll;
  if (pr.method != AAPDHG_METHOD_PDHG) {
    const double pw = sm.i < pr.pow_len ? pr.pow_tab[sm.i]
                                        : pow((double)sm.i + 1.0, -(1.0 + pr.safeguard_eps));
    may = may || gx <= __dmul_rn(__dmul_rn(pr.safeguard_d, sm.g0n), pw);
  }
  gb->maystop = (sm.k << 1) | (may ? 1ull : 0ull);
}

// The control CTA of k_plain_loop: state and parameters in shared memory for
// the whole launch (it is the only writer of the state until it stops).
// One lane adds tm[0..cnt) to s in index order (a dependent chain; each
// group's 8 shared-memory loads are issued before its adds).
__device__ __forceinline__ double chain_add(double s, const double* tm, int cnt) {
  int k = 0;
  for (; k + 8 <= cnt; k += 8) {
    double p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = tm[k + q];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dadd_rn(s, p[q]);
  }
  for (; k < cnt; ++k) s = __dadd_rn(s, tm[k]);
  return s;
}

// SERIAL-order chains, by a whole CTA: the elementwise terms of a chunk of CH
// entries are formed by all threads into shared memory, then one lane per
// quantity adds them in index order (fixed_point_residual pdhg_core.cpp:
// 65-74, kkt_metrics solver.cpp:64-110; vec.hpp dot). Roles from `st`.
// x side: out[0] ||xhat - x||^2, [1] bound term, [2] c'x, [3] ||c - K'y - lambda||^2
// The chunks are double-buffered: while the chain lanes (lane 0 of warps
// 0..3 / 0..2) add chunk c, warps 4.. stage chunk c + 1 into the other half
// of `terms` (two buffers of CH / 2 entries per quantity).
template <int CH>
__device__ __forceinline__ void stage_x_terms(const IterBufs& B, const double* __restrict__ T,
                                              const double* u, const double* uh, int n, int c0,
                                              double* buf, int t0, int nt) {
  constexpr int H = CH / 2;
  for (int t = t0; t < H; t += nt) {
    const int i = c0 + t;
    if (i < n) {
      const double d = __dsub_rn(uh[i], u[i]);
      buf[0 * H + t] = __dmul_rn(d, d);
      const double lj = B.l[i], uj = B.u[i], cj = B.c[i];
      const double rc = __dsub_rn(cj, T[i]);
      const double lam = project_lambda1(rc, lj, uj);
      // kkt_metrics adds l*lambda / u*lambda only where they apply; a
      // skipped term is -0.0, the exact identity of IEEE addition (x + -0 =
      // x for every x, -0 included), so the chain adds unconditionally
      double bt = -0.0;
      if (isfinite(lj) && lam > 0.0) bt = __dmul_rn(lj, lam);
      if (isfinite(uj) && lam < 0.0) bt = __dmul_rn(uj, lam);
      buf[1 * H + t] = bt;
      buf[2 * H + t] = __dmul_rn(cj, u[i]);
      const double v = __dsub_rn(rc, lam);
      buf[3 * H + t] = __dmul_rn(v, v);
    }
  }
}

template <int CH>
__device__ void serial_xchains_cta(const IterBufs& B, const double* __restrict__ T,
                                   const DevParams* __restrict__ P, const DevState& st,
                                   double* terms, unsigned char* take, double* out) {
  constexpr int H = CH / 2;
  const int64_t N = P->N;
  const int n = P->n;
  const double* u = B.upool + (int64_t)st.u_idx[U_CUR] * N;
  const double* uh = B.upool + (int64_t)st.u_idx[U_HAT] * N;
  const int w = threadIdx.x >> 5;
  const bool chain = (threadIdx.x & 31) == 0 && w < 4;
  const int nw = blockDim.x >> 5;
  const bool stager = w >= 4 && nw > 4;
  double s = 0.0;
  const int nch = (n + H - 1) / H;
  stage_x_terms<CH>(B, T, u, uh, n, 0, terms, threadIdx.x, blockDim.x);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    double* cur = terms + (c & 1) * 4 * H;
    if (chain) {
      const int c0 = c * H;
      const int cnt = n - c0 < H ? n - c0 : H;
      s = chain_add(s, cur + w * H, cnt);
    } else if (stager && c + 1 < nch) {
      stage_x_terms<CH>(B, T, u, uh, n, (c + 1) * H, terms + ((c + 1) & 1) * 4 * H,
                        threadIdx.x - 128, blockDim.x - 128);
    }
    __syncthreads();
    if (nw <= 4 && c + 1 < nch) {  // (no spare warps: stage after the chain)
      stage_x_terms<CH>(B, T, u, uh, n, (c + 1) * H, terms + ((c + 1) & 1) * 4 * H, threadIdx.x,
                        blockDim.x);
      __syncthreads();
    }
  }
  if (chain) out[w] = s;  // 0 G2x, 1 BOUND, 2 CX, 3 DUALSQ
  __syncthreads();
}

// y side: out[0] ||ghat||^2 continued from the x part g2x, [1] q'y,
// [2] primal infeasibility ||((h - Gx)_+; b - Ax)||^2
template <int CH>
__device__ __forceinline__ void stage_y_terms(const IterBufs& B, const double* u, const double* uh,
                                              const double* kx, int n, int mr, int m1, int c0,
                                              double* buf, int t0, int nt) {
  constexpr int H = CH / 2;
  for (int t = t0; t < H; t += nt) {
    const int i = c0 + t;
    if (i < mr) {
      const double d = __dsub_rn(uh[n + i], u[n + i]);
      buf[0 * H + t] = __dmul_rn(d, d);
      buf[1 * H + t] = __dmul_rn(B.q[i], u[n + i]);
      double v = __dsub_rn(B.q[i], kx[i]);
      if (i < m1) v = smax(v, 0.0);
      buf[2 * H + t] = __dmul_rn(v, v);
    }
  }
}

template <int CH>
__device__ void serial_ychains_cta(const IterBufs& B, const DevParams* __restrict__ P,
                                   const DevState& st, double g2x, double* terms, double* out) {
  constexpr int H = CH / 2;
  const int64_t N = P->N;
  const int n = P->n, mr = P->mrows, m1 = P->m1;
  const double* u = B.upool + (int64_t)st.u_idx[U_CUR] * N;
  const double* uh = B.upool + (int64_t)st.u_idx[U_HAT] * N;
  const double* kx = B.kxpool + (int64_t)st.kx_idx[KX_CUR] * mr;
  const int w = threadIdx.x >> 5;
  const bool chain = (threadIdx.x & 31) == 0 && w < 3;
  const int nw = blockDim.x >> 5;
  const bool stager = w >= 4 && nw > 4;
  double s = (chain && w == 0) ? g2x : 0.0;
  const int nch = (mr + H - 1) / H;
  stage_y_terms<CH>(B, u, uh, kx, n, mr, m1, 0, terms, threadIdx.x, blockDim.x);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    double* cur = terms + (c & 1) * 4 * H;
    if (chain) {
      const int c0 = c * H;
      const int cnt = mr - c0 < H ? mr - c0 : H;
      s = chain_add(s, cur + w * H, cnt);
    } else if (stager && c + 1 < nch) {
      stage_y_terms<CH>(B, u, uh, kx, n, mr, m1, (c + 1) * H, terms + ((c + 1) & 1) * 4 * H,
                        threadIdx.x - 128, blockDim.x - 128);
    }
    __syncthreads();
    if (nw <= 4 && c + 1 < nch) {
      stage_y_terms<CH>(B, u, uh, kx, n, mr, m1, (c + 1) * H, terms + ((c + 1) & 1) * 4 * H,
                        threadIdx.x, blockDim.x);
      __syncthreads();
    }
  }
  if (chain) out[w] = s;
  __syncthreads();
}

constexpr int kPlainSerChunk = 1024;  // SERIAL control CTA: terms staged per chain pass (33 KB)

template <bool SERIAL>
__device__ __noinline__ void plain_loop_control(const IterBufs& B, const DevParams* P, DevState* S,
                                                GridBar* gb, int nb1, int nb2, DevState& sm,
                                                DevParams& pr, double* red) {
  const unsigned long long G = gridDim.x;
  __shared__ double t1s[P1_COUNT], t2s[P2_COUNT];
  // SERIAL: the index-ordered chains of iteration k by this CTA (x side after
  // barrier 1, y side after barrier 2) while the workers run ahead
  __shared__ double sterms[SERIAL ? 4 * kPlainSerChunk : 1];
  __shared__ unsigned char stake[SERIAL ? kPlainSerChunk : 1];
  __shared__ double xres[4], yres[3];
  __shared__ Decision dec;
  params_load(&pr, P);
  __syncthreads();
  const uint64_t t_start = globaltimer_ns();
  uint64_t passes = 0;
  unsigned long long target1 = 0;  // barrier-1 instance this CTA arrived at early (0: none)
  for (;;) {
    // barrier 1 of iteration k: K1(k) done -> fold its partials (after a
    // plain decision the control has already arrived: it only waits)
    if (threadIdx.x == 0) {
      if (target1) {
        while ((ld_relaxed(&gb->arrive1) & kBarCount) < target1) {
        }
        ld_acquire(&gb->arrive1);
      } else {
        bar_arrive_wait(&gb->arrive1, 1, G);
      }
    }
    __syncthreads();
    if constexpr (SERIAL) {
      serial_xchains_cta<kPlainSerChunk>(B, (sm.k & 1) ? B.T2 : B.T, &pr, sm, sterms, stake,
                                         xres);
    } else {
      double t1[P1_COUNT];
      reduce_partial_rows<P1_COUNT>(B.part1, nb1, t1, red);
      if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < P1_COUNT; ++q) t1s[q] = t1[q];
    }
    // barrier 2: K2(k) done (the workers start K1(k+1) on plain-step roles,
    // or wait for the decision when maystop says it can stop the loop)
    if (!pr.no_stop_predict) {  // (opt-in, stop_likely)
      __syncthreads();
      if (threadIdx.x == 0) publish_maystop(pr, sm, gb, SERIAL ? xres[0] : t1s[P1_GX2]);
    }
    if (threadIdx.x == 0) bar_arrive_wait(&gb->arrive2, 1, G);
    __syncthreads();
    if constexpr (SERIAL) {
      serial_ychains_cta<kPlainSerChunk>(B, &pr, sm, xres[0], sterms, yres);
    } else {
      double t2[P2_COUNT];
      reduce_partial_rows<P2_COUNT>(B.part2, nb2, t2, red);
      if (threadIdx.x == 0)
#pragma unroll
        for (int q = 0; q < P2_COUNT; ++q) t2s[q] = t2[q];
    }
    __syncthreads();
    const uint64_t k = sm.k;
    // (SERIAL: ||g||^2 is the x chain continued over y, as solver.cpp's)
    const double g2 = SERIAL ? yres[0] : __dadd_rn(t1s[P1_GX2], t2s[P2_GY2]);
    const double bound = SERIAL ? xres[1] : t1s[P1_BOUND];
    const double qy = SERIAL ? yres[1] : t2s[P2_QY];
    const double cx = SERIAL ? xres[2] : t1s[P1_CX];
    const double infeas = SERIAL ? yres[2] : t2s[P2_INFEAS];
    const double dsq = SERIAL ? xres[3] : t1s[P1_DUALSQ];
    if (threadIdx.x == 32) control_kkt_records(&pr, &sm, k, g2, bound, qy, cx, infeas, dsq, -1.0);
    if (threadIdx.x == 0) dec = control_decide(&pr, &sm, k, g2, bound, qy, cx, infeas, dsq, -1.0, -1.0);
    __syncthreads();
    const bool stop = dec.attempt || dec.left <= 0;
    ++passes;
    if (threadIdx.x == 0 && stop) {
      control_setcond(&pr, dec);
      sm.loop_exits += 1;
      sm.plain_iters += passes;
      sm.plain_ns += globaltimer_ns() - t_start;
    }
    if (threadIdx.x == 32) control_commit(&pr, &sm, k, dec);
    if (threadIdx.x == 0 && !sm.done) {  // for the workers' stop prediction
      const double pw = sm.i < pr.pow_len ? pr.pow_tab[sm.i]
                                          : pow((double)sm.i + 1.0, -(1.0 + pr.safeguard_eps));
      gb->g_prev = gb->g_last;
      gb->g_last = sm.gkn;
      gb->thr = pr.method != AAPDHG_METHOD_PDHG ? __dmul_rn(__dmul_rn(pr.safeguard_d, sm.g0n), pw)
                                                : 0.0;
    }
    __syncthreads();
    if (stop) {
      // release the workers (they drop K1(k+1), or skip it on a predicted
      // stop), then hand the state over
      if (threadIdx.x == 0) {
        atom_add_acq_rel(&gb->arrive1, 1 + kBarStop);
        st_release(&gb->decided, k + 1);
      }
      state_store(S, &sm);
      return;
    }
    if (threadIdx.x == 0) {  // plain: arrive at barrier 1 of k+1 now, then publish
      const unsigned long long prev = atom_add_acq_rel(&gb->arrive1, 1);
      target1 = ((prev & kBarCount) / G + 1) * G;
      st_release(&gb->decided, k + 1);
    }
  }
}

template <bool PUSH, bool SERIAL = false>
__global__ void __launch_bounds__(kThreads, kSpmvBlocksPerSM)
    k_plain_loop(CsrDev KT, CsrDev K, IterBufs B, const DevParams* __restrict__ P, DevState* S,
                 GridBar* gb, int nb1, int nb2, int np1, int np2,
                 unsigned long long* __restrict__ bal) {
  __shared__ __align__(16) DevState st;  // worker: roles of its iteration; control: the state
  __shared__ double red[P1_COUNT * 32];
  __shared__ int s_stop;
  const int G = int(gridDim.x), W = G - 1, bid = int(blockIdx.x);
  TL_MARK(1);
  state_load(&st, S);
#ifdef AAPDHG_TIMELINE
  if (bid == 0 && threadIdx.x == 0) tl_mark(4);  // state loaded
#endif
  if (st.done || st.batch_left <= 0) return;  // (eager launches past the batch)
  if (bid == W) {
    __shared__ __align__(16) DevParams pr;
    plain_loop_control<SERIAL>(B, P, S, gb, np1, np2, st, pr, red);
#ifdef AAPDHG_TIMELINE
    if (threadIdx.x == 0) tl_mark(2);
#endif
    return;
  }
  unsigned long long h0 = 0;  // stop flags raised before this launch
  if (threadIdx.x == 0) h0 = ld_relaxed(&gb->arrive1) >> 40;
  int wp = 0;  // iterations decided in this launch (thread 0)
#ifdef AAPDHG_PLAIN_STAMPS
  // experiment build only: per worker and iteration, the K1 phase, the bar 1
  // wait, the K2 phase, the bar 2 wait (summed, aapdhg_cuda_plain_stamps)
  uint64_t ps0 = globaltimer_ns(), ps1 = 0, ps2 = 0, ps3 = 0;
#endif
  const bool pf = P->phase_prefetch != 0;
  // calibration (bal): this CTA's K1 / K2 phase times (start of its rows to
  // its barrier arrival), iterations and SM, for the host's partition
  uint64_t tb0 = 0, tb1 = 0, tb2 = 0;
  if (bal && threadIdx.x == 0) tb0 = globaltimer_ns();
  for (;;) {
    if (pf && bid < nb2) prefetch_slice_streams(K, bid);  // K2's streams, one phase ahead
    if constexpr (SERIAL) {  // K'y of iteration k into its parity buffer (the control's chains)
      IterBufs Bk = B;
      Bk.T = (st.k & 1) ? B.T2 : B.T;
      if (bid < nb1) dual_side_rows<true, PUSH, 0, true>(KT, Bk, P, &st, bid, nb1, red);
    } else {
      if (bid < nb1) dual_side_rows<false, PUSH, 0, true>(KT, B, P, &st, bid, nb1, red);
    }
    __syncthreads();
#ifdef AAPDHG_PLAIN_STAMPS
    if (threadIdx.x == 0) ps1 = globaltimer_ns();
#endif
    if (bal && threadIdx.x == 0) tb1 = globaltimer_ns();
    if (threadIdx.x == 0) s_stop = (bar_arrive_wait(&gb->arrive1, 1, G) >> 40) != h0;
    __syncthreads();
    if (s_stop) return;  // the control stopped after the previous iteration
#ifdef AAPDHG_TIMELINE
    if (bid == 0 && threadIdx.x == 0 && wp == 0) tl_mark(3);  // first barrier 1 passed
#endif
    if (bal && threadIdx.x == 0) tb2 = globaltimer_ns();
#ifdef AAPDHG_PLAIN_STAMPS
    if (threadIdx.x == 0) ps2 = globaltimer_ns();
#endif
    if (pf && bid < nb1) prefetch_slice_streams(KT, bid);  // the next K1's streams
    double acc[P2_COUNT] = {0.0, 0.0, 0.0};
    if (bid < nb2) {
      primal_side_rows<SERIAL, PUSH, true>(K, B, P, &st, bid, acc);
      if constexpr (!SERIAL) {
        if (K.sl_start) {
          slice_partials<P2_COUNT>(K, bid, acc, B.part2);
        } else {
          block_sum<P2_COUNT>(acc, red);
          if (threadIdx.x == 0)
#pragma unroll
            for (int q = 0; q < P2_COUNT; ++q) B.part2[q * nb2 + bid] = acc[q];
        }
      }
    }
    __syncthreads();
    if (bal && threadIdx.x == 0) {
      const uint64_t t3 = globaltimer_ns();
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      bal[4 * bid + 0] += tb1 - tb0;
      bal[4 * bid + 1] += t3 - tb2;
      bal[4 * bid + 2] += 1;
      bal[4 * bid + 3] = smid;
    }
#ifdef AAPDHG_PLAIN_STAMPS
    if (threadIdx.x == 0) ps3 = globaltimer_ns();
#endif
    if (threadIdx.x == 0) {
      bar_arrive_wait(&gb->arrive2, 1, G);
      s_stop = 0;
      // Predicted stop: the control is about to end the launch after
      // iteration k (batch end, max_iters, or ||g_k|| extrapolated from the
      // last two reaching the safeguard threshold — an AA attempt — or the
      // tolerance). Then K1(k+1) would be dropped: wait for the decision
      // instead (decided >= k + 1), and leave if it is a stop.
      if (stop_likely(P, gb, st, wp)) {
        while (ld_acquire(&gb->decided) < st.k + 1) {
        }
        if ((ld_relaxed(&gb->arrive1) >> 40) != h0) {
          atom_add_acq_rel(&gb->arrive1, 1);  // (keeps the barrier count whole)
          s_stop = 1;
        }
      }
      ++wp;
      // the roles of iteration k+1 if iteration k is a plain step
      st.aa_ok = 0;
      control_commit(P, &st, st.k, Decision{0, 1});
    }
    __syncthreads();
    if (s_stop) return;
    if (bal && threadIdx.x == 0) tb0 = globaltimer_ns();
#ifdef AAPDHG_PLAIN_STAMPS
    if (threadIdx.x == 0) {
      const uint64_t ps4 = globaltimer_ns();
      atomicAdd(&g_plain_dbg[0], ps1 - ps0);
      atomicAdd(&g_plain_dbg[1], ps2 - ps1);
      atomicAdd(&g_plain_dbg[2], ps3 - ps2);
      atomicAdd(&g_plain_dbg[3], ps4 - ps3);
      atomicAdd(&g_plain_dbg[4], 1ull);
      if (bid < 1024) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_plain_cta[bid * 4 + 0] += ps1 - ps0;
        g_plain_cta[bid * 4 + 1] += ps3 - ps2;
        g_plain_cta[bid * 4 + 2] += 1;
        g_plain_cta[bid * 4 + 3] = smid;
      }
      atomicMax(&g_plain_dbg[5], ps1 - ps0);
      atomicMax(&g_plain_dbg[6], ps3 - ps2);
      ps0 = ps4;
    }
#endif
  }
}

// ---------------------------------------------------------------------------
// TREE mode control: add the per-CTA partials of K1 (nu1 CTAs) and K2 (nu2)
// in CTA order (thread-strided + fixed block tree), then run the control
// logic on a shared-memory copy of the state.
__global__ void __launch_bounds__(kCtrlThreads)
    k_control(const double* __restrict__ part1, int nu1, const double* __restrict__ part2,
              int nu2, const DevParams* __restrict__ P, DevState* S) {
  if (S->done) {
    if (threadIdx.x == 0 && P->use_cond) {
      cudaGraphSetConditional(P->cond_aa, 0);
      cudaGraphSetConditional(P->cond_loop, 0);
    }
    return;
  }
  __shared__ double red[P1_COUNT * 32];
  double t1[P1_COUNT], t2[P2_COUNT];
  reduce_partial_rows<P1_COUNT>(part1, nu1, t1, red);
  reduce_partial_rows<P2_COUNT>(part2, nu2, t2, red);
  __shared__ DevState sm;
  __shared__ DevParams sp;
  params_load(&sp, P);
  state_load(&sm, S);
  if (threadIdx.x == 0) {
    if (nu1 == 0) t1[P1_GX2] = t1[P1_BOUND] = t1[P1_CX] = t1[P1_DUALSQ] = 0.0;
    if (nu2 == 0) t2[P2_GY2] = t2[P2_QY] = t2[P2_INFEAS] = 0.0;
    control_logic(&sp, &sm, __dadd_rn(t1[P1_GX2], t2[P2_GY2]), t1[P1_BOUND], t2[P2_QY],
                  t1[P1_CX], t2[P2_INFEAS], t1[P1_DUALSQ]);
  }
  state_store(S, &sm);
}

// ---------------------------------------------------------------------------
// SERIAL mode: every scalar reduction as one index-ordered chain
// (fixed_point_residual pdhg_core.cpp:65-74; kkt_metrics solver.cpp:64-110),
// one warp per chain (lane 0 sums), then the control logic.
// ---------------------------------------------------------------------------
// SERIAL mode, x side (runs beside K2: it needs only K1's outputs): the
// index-ordered chains over j < n of ||xhat - x||^2 (the first part of
// ||g||^2), the bound terms, c'x and ||c - K'y - lambda||^2 -> S->sres.
// The elementwise terms of a chunk are formed by all threads in shared
// memory; one lane per quantity adds them in order (bit for bit the
// reference's loops, fixed_point_residual pdhg_core.cpp:65-74 and
// kkt_metrics solver.cpp:64-110).
__global__ void __launch_bounds__(kSerThreads)
    k_serial_xchains(IterBufs B, const DevParams* __restrict__ P, DevState* S) {
  if (S->done) return;
  extern __shared__ double terms[];  // S_COUNT x kSerChunk
  unsigned char* take = reinterpret_cast<unsigned char*>(terms + S_COUNT * kSerChunk);
  __shared__ double out[4];
  __shared__ DevState st;
  state_load(&st, S);
  serial_xchains_cta<kSerChunk>(B, B.T, P, st, terms, take, out);
  if (threadIdx.x < 4) S->sres[threadIdx.x] = out[threadIdx.x];  // G2x, BOUND, CX, DUALSQ
}

// SERIAL mode, y side + control (after K2 and k_serial_xchains): ||g||^2
// continues the x-part chain over the y entries, then q'y and the primal
// infeasibility, each in index order.
__global__ void __launch_bounds__(kSerThreads)
    k_serial_control(IterBufs B, const DevParams* __restrict__ P, DevState* S) {
  if (S->done) {
    if (threadIdx.x == 0 && P->use_cond) {
      cudaGraphSetConditional(P->cond_aa, 0);
      cudaGraphSetConditional(P->cond_loop, 0);
    }
    return;
  }
  extern __shared__ double terms[];  // 3 x kSerChunk used
  __shared__ double res[3];
  __shared__ DevState sm;
  __shared__ DevParams sp;
  params_load(&sp, P);
  state_load(&sm, S);  // (syncs; sres[] from k_serial_xchains)
  serial_ychains_cta<kSerChunk>(B, P, sm, sm.sres[0], terms, res);
  if (threadIdx.x == 0)
    control_logic(&sp, &sm, res[0], sm.sres[1], res[1], sm.sres[2], res[2], sm.sres[3]);
  state_store(S, &sm);
}


}  // namespace aapdhg_b200
