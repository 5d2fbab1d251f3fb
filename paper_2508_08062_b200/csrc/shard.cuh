// shard.cuh — kernels of the sharded (multi-GPU) solve.
//
// Layout: shard r owns a contiguous block R_r of K's rows
// (its y, q, K x slices) and a block C_r of K's columns (its x, c, l, u
// slices). It stores K[R_r, :] for K xhat and K[:, C_r]' (rows of K') for
// (K'y)[C_r], with column indices relabelled into the padded all-gather
// buffers (chunk r of xgather holds x[C_r], chunk r of ygather y[R_r]).
// Every row sum is still the full CSR-ordered row of K or K', so the SpMVs
// match the single-GPU ones bit for bit; only the scalar sums meet across
// shards, in rank order. The control logic runs replicated on every shard
// from identical all-gathered scalars, so all shards take the same branch.
#pragma once

#include "aa.cuh"

namespace aapdhg_b200 {

// dst[t] = (vector of role `role`, or of slot `-role - 1` when role < 0)
// [off + t], t < len — into this shard's chunk of an all-gather buffer.
// mode 0: always; 1: while the solve runs; 2: only after an accepted AA step.
__global__ void k_stage(const double* __restrict__ upool, int role, int64_t N, int64_t off,
                        int64_t len, double* __restrict__ dst, const DevState* S, int mode) {
  if (mode >= 1 && S->done) return;
  if (mode == 2 && !S->aa_ok) return;
  const int r = role >= 0 ? S->u_idx[role] : -role - 1;
  const double* src = upool + (int64_t)r * N + off;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < len;
       t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[t];
}

// Sums the all-gathered shard totals in rank order (elapsed: the maximum, so
// a TIMEOUT is taken by every shard at the same iteration) and runs the
// control logic.
__global__ void __launch_bounds__(128)
    k_control_dist(const double* __restrict__ all, int nranks, const DevParams* __restrict__ P,
                   DevState* S) {
  if (S->done) return;
  if (P->p2p_fused && threadIdx.x == 0) p2p_wait(P, S, P2P_YG);  // every shard's totals
  __syncthreads();
  __shared__ DevState sm;
  __shared__ DevParams sp;
  params_load(&sp, P);
  state_load(&sm, S);
  if (threadIdx.x == 0) {
    double t[7];
    double el = all[7];
    for (int q = 0; q < 7; ++q) t[q] = all[q];
    for (int r = 1; r < nranks; ++r) {
      for (int q = 0; q < 7; ++q) t[q] = __dadd_rn(t[q], all[r * 8 + q]);
      el = smax(el, all[r * 8 + 7]);
    }
    control_logic(&sp, &sm, __dadd_rn(t[0], t[4]), t[1], t[5], t[2], t[6], t[3], el);
  }
  state_store(S, &sm);
}

// This shard's Gram / rhs / column-norm partial dots (k_tree_dots per-CTA
// partials, summed in CTA order like k_aa_solve does) into its chunk of the
// dots exchange buffer of every destination (P->dots_dst).
__global__ void __launch_bounds__(1024)
    k_dot_totals(DotBufs D, const DevParams* __restrict__ P, const DevState* S) {
  if (S->done || !S->aa_attempt) return;
  const int nit = num_items(S->mem_size, P->method);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int it = warp; it < nit; it += nw) {
    const double* pp = D.part + (int64_t)it * P->ndot_blk;
    double s = 0.0;
    if (D.part_lo) {  // FAA: the double-double partials, rounded once per shard
      const double* pl = D.part_lo + (int64_t)it * P->ndot_blk;
      dd t = {0.0, 0.0};
      for (int b = lane; b < P->ndot_blk; b += 32) t = dd_add(t, dd{pp[b], pl[b]});
      s = warp_sum_dd(t).hi;
    } else {
      for (int b = lane; b < P->ndot_blk; b += 32) s = __dadd_rn(s, pp[b]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    }
    if (lane == 0)
      for (int q = 0; q < P->ndst; ++q) P->dots_dst[q][it] = s;
  }
}

// Peer-memory (P2P) exchange barrier, for the exchanges that are not fused
// into K1 / K2 / the control (the AA branch, the start iterate). The
// producers already stored this shard's chunk into every shard's buffer
// (P->*_dst); this publishes that and waits until every shard has published
// the same exchange (p2p_arrive / p2p_wait, pipeline.cuh). phase 1: arrive,
// 2: wait, 3: both (one shard per process). In-process loopback shards
// arrive all first, then wait (no kernel spins on a shard that has not been
// launched).
__global__ void k_p2p_barrier(const DevParams* __restrict__ P, DevState* S, int slot, int phase) {
  if (threadIdx.x != 0) return;
  if (phase & 1) p2p_arrive(P, S, slot);
  if (phase & 2) p2p_wait(P, S, slot);
}

// lambda = P_Lambda(c - K'y) of the final iterate from the K'y kept by K1
// (project_lambda, pdhg_core.cpp:27-39), into this shard's chunk.
__global__ void k_lambda_from_T(const double* __restrict__ T, const double* __restrict__ c,
                                const double* __restrict__ l, const double* __restrict__ u,
                                int n, double* __restrict__ lam) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
    lam[t] = project_lambda1(__dsub_rn(c[t], T[t]), l[t], u[t]);
}

}  // namespace aapdhg_b200
