// aa.cuh — AA / FAA step kernels, role rotation, setup and power-iteration
// helpers of the sm_100a solver (see pipeline.cuh for the iteration core).
#pragma once

#include "pipeline.cuh"

namespace aapdhg_b200 {

// ---------------------------------------------------------------------------
// AA / FAA: dots over the memory columns
__device__ __forceinline__ int num_items(int p, int method) {
  return p * (p + 1) / 2 + p + (method == AAPDHG_METHOD_FAA ? p : 0);
}

// item -> (kind, a, b); kind 0 pair, 1 rhs, 2 e-norm
__device__ __forceinline__ void decode_item(int item, int p, int& kind, int& a, int& b) {
  const int npair = p * (p + 1) / 2;
  if (item < npair) {
    int r = 0, rem = item;
    while (rem >= p - r) { rem -= p - r; ++r; }
    kind = 0; a = r; b = r + rem;
  } else if (item < npair + p) {
    kind = 1; a = b = item - npair;
  } else {
    kind = 2; a = b = item - npair - p;
  }
}

struct DotBufs {
  const double* du;
  const double* dg;
  const double* gpool;
  double* part;     // items x ndot_blk (tree) or items (serial)
  int32_t max_items;
};

__device__ __forceinline__ void item_vectors(const DotBufs& D, const DevParams* P,
                                             const DevState* S, int item, int p,
                                             const double*& va, const double*& vb) {
  int kind, a, b;
  decode_item(item, p, kind, a, b);
  const int64_t N = P->N;
  const int sa = S->mem_slots[a], sb = S->mem_slots[b];
  if (kind == 0) { va = D.dg + sa * N; vb = D.dg + sb * N; }
  else if (kind == 1) { va = D.dg + sa * N; vb = D.gpool + (int64_t)S->g_idx[G_CUR] * N; }
  else { va = D.du + sa * N; vb = va; }
}

// SERIAL: one index-ordered chain per item (vec.hpp dot) — warp lane 0.
__global__ void k_serial_dots(DotBufs D, const DevParams* __restrict__ P, const DevState* S) {
  if (S->done || !S->aa_attempt) return;
  const int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if ((threadIdx.x & 31) != 0) return;
  const int p = S->mem_size;
  if (item >= num_items(p, P->method)) return;
  const double *va, *vb;
  item_vectors(D, P, S, item, p, va, vb);
  D.part[item] = serial_dot(va, vb, P->N);
}

// TREE: CTA b covers elements [b*kDotChunk, ...); warp w takes items w, w+8..
// Column chunks are re-read from L1 across items; HBM sees each once.
__global__ void __launch_bounds__(kThreads)
    k_tree_dots(DotBufs D, const DevParams* __restrict__ P, const DevState* S) {
  if (S->done || !S->aa_attempt) return;
  // the memory's slot table once per CTA (not a dependent global load per item)
  __shared__ int slots[kMaxMemory];
  __shared__ int sh_p, sh_g;
  if (threadIdx.x < kMaxMemory) slots[threadIdx.x] = S->mem_slots[threadIdx.x];
  if (threadIdx.x == 0) {
    sh_p = S->mem_size;
    sh_g = S->g_idx[G_CUR];
  }
  __syncthreads();
  const int p = sh_p;
  const int nit = num_items(p, P->method);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * kDotChunk;
  const int64_t N = P->N;
  const int cnt = (int)((N - base) < kDotChunk ? (N - base) : kDotChunk);
  constexpr int kPer = kDotChunk / 32;
  for (int item = warp; item < nit; item += kThreads / 32) {
    int kind, ia, ib;
    decode_item(item, p, kind, ia, ib);
    const double *va, *vb;
    if (kind == 0) { va = D.dg + slots[ia] * N; vb = D.dg + slots[ib] * N; }
    else if (kind == 1) { va = D.dg + slots[ia] * N; vb = D.gpool + (int64_t)sh_g * N; }
    else { va = D.du + slots[ia] * N; vb = va; }
    // every load of the lane's share in flight before the adds (same order:
    // t = lane, lane + 32, ...)
    double x[kPer], y[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int t = lane + 32 * u;
      x[u] = t < cnt ? va[base + t] : 0.0;
      y[u] = t < cnt ? vb[base + t] : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < kPer; ++u)
      if (lane + 32 * u < cnt) s = __dadd_rn(s, __dmul_rn(x[u], y[u]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) D.part[(int64_t)item * P->ndot_blk + blockIdx.x] = s;
  }
}

// TREE, memory capacity <= CAP (<= 10): the whole Gram / rhs / column-norm
// set in registers. Each thread loads the p + 1 (FAA: 2p + 1) vectors at its
// elements once — grid-stride, element order — and accumulates every item;
// the CTA then reduces each item over its warps in a fixed shape into
// part[item * gridDim.x + blockIdx.x]. One HBM read of each column instead of
// one L1 read per item that uses it (k_tree_dots). Also stages g = T(u) - u
// (k_stage_g), which the mix reads next.
template <int CAP, bool FAA>
__global__ void __launch_bounds__(kThreads, 1)
    k_gram_dots(DotBufs D, double* __restrict__ upool, const DevParams* __restrict__ P,
                const DevState* S) {
  if (S->done || !S->aa_attempt) return;
  constexpr int NPAIR = CAP * (CAP + 1) / 2;
  constexpr int NACC = NPAIR + CAP + (FAA ? CAP : 0);
  __shared__ int slots[CAP];
  __shared__ int sh_p, sh_g, sh_h, sh_c;
  if (threadIdx.x < CAP) slots[threadIdx.x] = S->mem_slots[threadIdx.x];
  if (threadIdx.x == 0) {
    sh_p = S->mem_size;
    sh_g = S->g_idx[G_CUR];
    sh_h = S->u_idx[U_HAT];
    sh_c = S->u_idx[U_CUR];
  }
  __syncthreads();
  const int p = sh_p;
  const int64_t N = P->N;
  const double* dgc[CAP];
  const double* duc[CAP];
#pragma unroll
  for (int a = 0; a < CAP; ++a) {
    dgc[a] = D.dg + (int64_t)(a < p ? slots[a] : 0) * N;
    duc[a] = D.du + (int64_t)(a < p ? slots[a] : 0) * N;
  }
  const double* uh = upool + (int64_t)sh_h * N;
  const double* uc = upool + (int64_t)sh_c * N;
  double* g = const_cast<double*>(D.gpool) + (int64_t)sh_g * N;
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double gt = __dsub_rn(uh[t], uc[t]);
    g[t] = gt;
    double v[CAP];
#pragma unroll
    for (int a = 0; a < CAP; ++a) v[a] = a < p ? dgc[a][t] : 0.0;
    int q = 0;
#pragma unroll
    for (int a = 0; a < CAP; ++a)
#pragma unroll
      for (int b = a; b < CAP; ++b, ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v[a], v[b]));
#pragma unroll
    for (int a = 0; a < CAP; ++a) acc[NPAIR + a] = __dadd_rn(acc[NPAIR + a], __dmul_rn(v[a], gt));
    if constexpr (FAA) {
#pragma unroll
      for (int a = 0; a < CAP; ++a) {
        const double e = a < p ? duc[a][t] : 0.0;
        acc[NPAIR + CAP + a] = __dadd_rn(acc[NPAIR + CAP + a], __dmul_rn(e, e));
      }
    }
  }
  // fixed-shape CTA reduction of every live item, written in p-space order
  __shared__ double red[kWarps][NACC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NACC; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = s;
  }
  __syncthreads();
  const int np = p * (p + 1) / 2;
  for (int q = threadIdx.x; q < NACC; q += blockDim.x) {
    double s = red[0][q];
    for (int w = 1; w < kWarps; ++w) s = __dadd_rn(s, red[w][q]);
    int item = -1;
    if (q < NPAIR) {  // (a, b) in CAP space -> p space
      int a = 0, rem = q;
      while (rem >= CAP - a) { rem -= CAP - a; ++a; }
      const int b = a + rem;
      if (b < p) item = a * p - a * (a - 1) / 2 + (b - a);
    } else if (q < NPAIR + CAP) {
      const int a = q - NPAIR;
      if (a < p) item = np + a;
    } else {
      const int a = q - NPAIR - CAP;
      if (a < p) item = np + p + a;
    }
    if (item >= 0) D.part[(int64_t)item * gridDim.x + blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// AA / FAA small solve (one CTA; the p x p algebra runs in thread 0)
// ---------------------------------------------------------------------------

// cholesky_solve, anderson.cpp:26-51 (a: p x p column-major, overwritten)
__device__ bool dev_cholesky_solve(int p, double* a, double* rhs) {
#define A_(i, j) a[(j) * p + (i)]
  for (int j = 0; j < p; ++j) {
    double d = A_(j, j);
    for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(A_(j, k), A_(j, k)));
    if (d <= 0.0) return false;
    d = sqrt(d);
    A_(j, j) = d;
    for (int i = j + 1; i < p; ++i) {
      double s = A_(i, j);
      for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(A_(i, k), A_(j, k)));
      A_(i, j) = s / d;
    }
  }
  for (int i = 0; i < p; ++i) {
    double s = rhs[i];
    for (int k = 0; k < i; ++k) s = __dsub_rn(s, __dmul_rn(A_(i, k), rhs[k]));
    rhs[i] = s / A_(i, i);
  }
  for (int i = p - 1; i >= 0; --i) {
    double s = rhs[i];
    for (int k = i + 1; k < p; ++k) s = __dsub_rn(s, __dmul_rn(A_(k, i), rhs[k]));
    rhs[i] = s / A_(i, i);
  }
#undef A_
  return true;
}

// dev_cholesky_solve on a whole CTA (a, rhs in shared memory; every thread
// calls it). Each entry sees exactly the operations of the one-thread
// version in the same order — the row updates of a column run in parallel,
// the forward substitution is applied column by column (each rhs_k still
// subtracts A_k0 r0, A_k1 r1, ... in that order), the backward one stays
// row by row — so the result is bit for bit the same.
__device__ bool block_cholesky_solve(int p, double* a, double* rhs) {
#define A_(i, j) a[(j) * p + (i)]
  __shared__ double dsh;
  __shared__ int bad;
  for (int j = 0; j < p; ++j) {
    if (threadIdx.x == 0) {
      double d = A_(j, j);
      for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(A_(j, k), A_(j, k)));
      bad = d <= 0.0;
      if (!bad) {
        d = sqrt(d);
        A_(j, j) = d;
      }
      dsh = d;
    }
    __syncthreads();
    if (bad) return false;
    for (int i = j + 1 + int(threadIdx.x); i < p; i += blockDim.x) {
      double s = A_(i, j);
      for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(A_(i, k), A_(j, k)));
      A_(i, j) = s / dsh;
    }
    __syncthreads();
  }
  for (int i = 0; i < p; ++i) {
    if (threadIdx.x == 0) rhs[i] = rhs[i] / A_(i, i);
    __syncthreads();
    for (int k = i + 1 + int(threadIdx.x); k < p; k += blockDim.x)
      rhs[k] = __dsub_rn(rhs[k], __dmul_rn(A_(k, i), rhs[i]));
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int i = p - 1; i >= 0; --i) {
      double s = rhs[i];
      for (int k = i + 1; k < p; ++k) s = __dsub_rn(s, __dmul_rn(A_(k, i), rhs[k]));
      rhs[i] = s / A_(i, i);
    }
  __syncthreads();
#undef A_
  return true;
}

// length_bounds, filtering.cpp:92-114 (fn_sq of the kept columns, newest first)
__device__ void dev_length_bounds(int m, const double* fn_sq, double c_s, double* b) {
  if (m == 0) return;
  const double cs2 = __dmul_rn(c_s, c_s);
  const double ct = sqrt(smax(0.0, __dsub_rn(1.0, cs2)));
  const double ct2 = __dmul_rn(ct, ct);
  b[0] = 1.0 / fn_sq[0];
  for (int jj = 1; jj < m; ++jj) {
    const int j = jj + 1;
    double acc = __dmul_rn(ct2, pow(__dadd_rn(ct, c_s) / c_s, 2.0 * (j - 2))) / fn_sq[0];
    for (int i = 2; i <= j - 1; ++i)
      acc = __dadd_rn(acc, __dmul_rn(ct2, pow(__dadd_rn(ct, c_s), 2.0 * (j - i - 1))) /
                               __dmul_rn(fn_sq[i - 1], pow(c_s, 2.0 * (j - i))));
    acc = __dadd_rn(acc, 1.0 / fn_sq[jj]);
    b[jj] = acc / cs2;
  }
}

struct SolveScratch {
  double* gram;  // kMaxMemory^2
  double* work;  // kMaxMemory^2
  double* vec;   // 8 * kMaxMemory
};

// Reduces the dot partials, then:
//  AA : Gram + eta*tr(Gram) I, Cholesky, w            (anderson.cpp:106-128)
//  FAA: angle filter on the newest-first Cholesky diagonal of F'F
//       (= |diag R| of its Householder QR), length filter, then
//       w = R^{-1} R^{-T} F'g with R = chol(F_kept'F_kept) and the
//       back_substitute singularity floor      (filtering.cpp:69-181,
//                                               sparse_linalg.cpp:200-218)
// Success: S->aa_ok, weights and mix columns set, i += 1.
// SingularError: plain step, j += 1, aa_failures += 1 (solver.cpp:229-235).
__global__ void __launch_bounds__(1024)
    k_aa_solve(DotBufs D, const DevParams* __restrict__ P, DevState* Sg, int per_op,
               const double* __restrict__ rank_tot = nullptr, int nranks = 0,
               int rank_stride = 0) {
  if (Sg->done || !Sg->aa_attempt) return;
  __shared__ DevState smS;
  state_load(&smS, Sg);
  DevState* S = &smS;
  // p x p Gram and factor in dynamic shared memory (2 * cap^2 doubles)
  extern __shared__ double dyn_smem[];
  __shared__ double vecs[8 * kMaxMemory];
  const SolveScratch W{dyn_smem, dyn_smem + P->cap * P->cap, vecs};
  const int p = S->mem_size;
  const int nit = num_items(p, P->method);
  __shared__ double vals[kMaxMemory * (kMaxMemory + 1) / 2 + 2 * kMaxMemory];
  if (rank_tot) {  // sharded: per-shard totals summed in rank order
    for (int it = threadIdx.x; it < nit; it += blockDim.x) {
      double s = rank_tot[it];
      for (int r = 1; r < nranks; ++r) s = __dadd_rn(s, rank_tot[(int64_t)r * rank_stride + it]);
      vals[it] = s;
    }
  } else if (P->serial) {
    for (int it = threadIdx.x; it < nit; it += blockDim.x) vals[it] = D.part[it];
  } else {
    // warp per item, lanes stride over the CTAs' partials, fixed tree
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int it = warp; it < nit; it += nw) {
      const double* pp = D.part + (int64_t)it * P->ndot_blk;
      double s = 0.0;
      // groups of 8 strides: the loads of a group are in flight together,
      // the adds keep the order b, b + 32, ...
      for (int b0 = lane; b0 < P->ndot_blk; b0 += 32 * 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = b0 + 32 * u < P->ndot_blk ? __ldcg(pp + b0 + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (b0 + 32 * u < P->ndot_blk) s = __dadd_rn(s, x[u]);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) vals[it] = s;
    }
  }
  __syncthreads();
  const int npair = p * (p + 1) / 2;
  double* G = W.gram;  // p x p column-major, full symmetric (item (a<=b) row-major upper)
  for (int t = threadIdx.x; t < p * p; t += blockDim.x) {
    const int r = t % p, c = t / p, lo = r < c ? r : c, hi = r < c ? c : r;
    G[t] = vals[lo * p - lo * (lo - 1) / 2 + (hi - lo)];
  }
  __syncthreads();
  // AA: G + eta tr(G) I, factored by the whole CTA (anderson.cpp:106-128)
  __shared__ int aa_solved;
  if (P->method == AAPDHG_METHOD_AA) {
    __shared__ double eta_eff_sh;
    if (threadIdx.x == 0) {
      double frob_sq = 0.0;
      for (int i = 0; i < p; ++i) frob_sq = __dadd_rn(frob_sq, G[i * p + i]);
      eta_eff_sh = __dmul_rn(P->eta, frob_sq);
    }
    __syncthreads();
    double* A = W.work;
    for (int t = threadIdx.x; t < p * p; t += blockDim.x)
      A[t] = (t % p == t / p) ? __dadd_rn(G[t], eta_eff_sh) : G[t];
    for (int i = threadIdx.x; i < p; i += blockDim.x) W.vec[i] = vals[npair + i];
    __syncthreads();
    const bool solved = block_cholesky_solve(p, A, W.vec);
    if (threadIdx.x == 0) aa_solved = solved ? 1 : 0;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
  const double* rhs = vals + npair;
  double* w = W.vec;  // p
  bool ok = true;
  int pm = 0;         // mixed columns
  if (P->method == AAPDHG_METHOD_AA) {
    ok = aa_solved != 0;
    if (ok) {
      pm = p;
      for (int t = 0; t < p; ++t) S->mix_slots[t] = S->mem_slots[t];
    }
  } else {
    const double* en2 = vals + npair + p;
    // angle filter on the newest-first order: Gr(s,t) = G(p-1-s, p-1-t);
    // upper R with R'R = Gr row by row; |R(j,j)| = |diag| of the Householder
    // QR of the reversed F (qr_diagonal, filtering.cpp:25-50). Dependent
    // columns (pivot <= 0) get a zero diagonal like a zero Householder step.
    double* R = W.work;  // row-major p x p
    int* keep = (int*)(W.vec + 2 * kMaxMemory);
    for (int j = 0; j < p; ++j) {
      const int gj = p - 1 - j;
      double d = G[gj * p + gj];
      for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(R[k * p + j], R[k * p + j]));
      const double rjj = d > 0.0 ? sqrt(d) : 0.0;
      R[j * p + j] = rjj;
      for (int i = j + 1; i < p; ++i) {
        const int gi = p - 1 - i;
        double s = G[gi * p + gj];
        for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(R[k * p + j], R[k * p + i]));
        R[j * p + i] = rjj > 0.0 ? s / rjj : 0.0;
      }
      const double fn = sqrt(G[gj * p + gj]);
      const double sine = ((int64_t)j < P->Nglob && fn > 0.0) ? rjj / fn : 0.0;
      keep[j] = 1;
      if (j == 0) {
        if (fn == 0.0) ok = false;  // zero leading column -> SingularError
        continue;
      }
      if (sine < P->c_s) keep[j] = 0;
    }
    if (ok) {
      // length filter over kept (newest first)
      int idx[kMaxMemory];
      int m = 0;
      for (int t = 0; t < p; ++t)
        if (keep[t]) idx[m++] = p - 1 - t;  // memory positions, newest first
      double* fn_sq = W.vec + 3 * kMaxMemory;
      double* bb = W.vec + 4 * kMaxMemory;
      for (int t = 0; t < m; ++t) fn_sq[t] = G[idx[t] * p + idx[t]];
      dev_length_bounds(m, fn_sq, P->c_s, bb);
      double ep = 0.0, bp = 0.0;
      const double cap = __dmul_rn(P->kappa_bar, P->kappa_bar);
      int kk = 0;
      double epre[kMaxMemory + 1], bpre[kMaxMemory + 1];
      epre[0] = bpre[0] = 0.0;
      for (int t = 0; t < m; ++t) {
        ep = __dadd_rn(ep, en2[idx[t]]);
        bp = __dadd_rn(bp, bb[t]);
        epre[t + 1] = ep;
        bpre[t + 1] = bp;
      }
      for (int t = m; t >= 1; --t)
        if (__dmul_rn(epre[t], bpre[t]) <= cap) { kk = t; break; }
      // kept positions back in memory (oldest-first) order
      int kpos[kMaxMemory];
      for (int t = 0; t < kk; ++t) kpos[t] = idx[kk - 1 - t];
      pm = kk;
      if (kk > 0) {
        // R = chol(F_kept' F_kept) (upper), then w = R^{-1} R^{-T} F'g
        double* Rm = W.work;  // reuse (angle-filter R no longer needed)
        for (int a = 0; a < kk; ++a)
          for (int b = 0; b < kk; ++b) Rm[b * kk + a] = G[kpos[b] * p + kpos[a]];
        // Cholesky: Rm lower = L, L L^T = Gk; R = L^T
        for (int j = 0; j < kk && ok; ++j) {
          double d = Rm[j * kk + j];
          for (int k2 = 0; k2 < j; ++k2) d = __dsub_rn(d, __dmul_rn(Rm[k2 * kk + j], Rm[k2 * kk + j]));
          if (d <= 0.0) { ok = false; break; }
          d = sqrt(d);
          Rm[j * kk + j] = d;
          for (int i = j + 1; i < kk; ++i) {
            double s = Rm[j * kk + i];
            for (int k2 = 0; k2 < j; ++k2) s = __dsub_rn(s, __dmul_rn(Rm[k2 * kk + i], Rm[k2 * kk + j]));
            Rm[j * kk + i] = s / d;
          }
        }
        if (ok) {
          // back_substitute floor: |r_ii| <= 1e-14 ||R||_F -> SingularError
          double fro = 0.0;
          for (int j = 0; j < kk; ++j)
            for (int i = j; i < kk; ++i) fro = __dadd_rn(fro, __dmul_rn(Rm[j * kk + i], Rm[j * kk + i]));
          const double floor_v = 1e-14 * sqrt(fro);
          for (int i = 0; i < kk; ++i)
            if (fabs(Rm[i * kk + i]) <= floor_v) ok = false;
        }
        if (ok) {
          // forward: L z = F'g ; back: L^T w = z
          for (int i = 0; i < kk; ++i) {
            double s = rhs[kpos[i]];
            for (int k2 = 0; k2 < i; ++k2) s = __dsub_rn(s, __dmul_rn(Rm[k2 * kk + i], w[k2]));
            w[i] = s / Rm[i * kk + i];
          }
          for (int i = kk - 1; i >= 0; --i) {
            double s = w[i];
            for (int k2 = i + 1; k2 < kk; ++k2) s = __dsub_rn(s, __dmul_rn(Rm[i * kk + k2], w[k2]));
            w[i] = s / Rm[i * kk + i];
          }
        }
      }
      if (ok) {
        for (int t = 0; t < kk; ++t) S->mix_slots[t] = S->mem_slots[kpos[t]];
        if (!per_op) {
          // carried memory replaced only on success (solver.cpp:221-224)
          for (int t = 0; t < kk; ++t) S->mem_slots[t] = S->mix_slots[t];
          S->mem_size = kk;
        }
      }
    }
  }
  if (ok) {
    S->mix_p = pm;
    for (int t = 0; t < pm; ++t) S->w[t] = w[t];
    S->aa_ok = 1;
    S->i += 1;
    if (!per_op) (P->rec + (S->k & (P->rec_cap - 1)))->aa_step = 1;
  } else {
    S->aa_ok = 0;
    S->j += 1;
    S->aa_failures += 1;
  }
  }  // thread 0
  state_store(Sg, &smS);
}

// cand = P_feasible(u + damp(g) - sum_j w_j (du_j + damp(dg_j)))
// (anderson.cpp:109,130-133 / filtering.cpp:165,176-179; solver.cpp:226)
__global__ void __launch_bounds__(kThreads)
    k_mix(IterBufs B, const double* __restrict__ dg, const DevParams* __restrict__ P,
          const DevState* S, int project) {
  if (S->done || !S->aa_ok) return;
  const int64_t N = P->N;
  const int n = P->n;
  const double* u = B.upool + (int64_t)S->u_idx[U_CUR] * N;
  const double* g = B.gpool + (int64_t)S->g_idx[G_CUR] * N;
  double* out = B.upool + (int64_t)S->u_idx[U_CAND] * N;
  const int pm = S->mix_p;
  const double beta = P->beta;
  const double* dh = P->d_hat;
  __shared__ double nw[kMaxMemory];
  __shared__ int64_t sls[kMaxMemory];
  for (int jj = threadIdx.x; jj < pm; jj += blockDim.x) {
    nw[jj] = -S->w[jj];
    sls[jj] = S->mix_slots[jj];
  }
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (int64_t)gridDim.x * blockDim.x) {
    double o = __dadd_rn(u[t], damp1(beta, dh, t, g[t]));
    for (int jj = 0; jj < pm; ++jj) {
      const int64_t sl = sls[jj];
      const double a = nw[jj];
      o = __dadd_rn(o, __dmul_rn(a, B.du[sl * N + t]));
      o = __dadd_rn(o, __dmul_rn(a, damp1(beta, dh, t, dg[sl * N + t])));
    }
    if (project) {
      if (t < n) o = smin(smax(o, B.l[t]), B.u[t]);
      else if (t - n < P->m1) o = smax(o, 0.0);
    }
    out[t] = o;
  }
}

// g_k = T(u_k) - u_k of an iteration that attempts an AA step (the Gram
// rhs and the mix read it; the next iteration's push reads it as g_{k-1}
// when the candidate is accepted). K1/K2 do not store g: after a plain step
// the push derives g_{k-1} from du (solver.cpp:204-209).
__global__ void k_stage_g(const double* __restrict__ upool, double* __restrict__ gpool,
                          const DevParams* __restrict__ P, const DevState* S) {
  if (S->done || !S->aa_attempt) return;
  const int64_t N = P->N;
  const double* uh = upool + (int64_t)S->u_idx[U_HAT] * N;
  const double* u = upool + (int64_t)S->u_idx[U_CUR] * N;
  double* g = gpool + (int64_t)S->g_idx[G_CUR] * N;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (int64_t)gridDim.x * blockDim.x)
    g[t] = __dsub_rn(uh[t], u[t]);
}

// End of an iteration that attempted an AA step (the IF body of the graph):
// rotate to the candidate (or to T(u) after a SingularError fallback).
__global__ void k_aa_commit(const DevParams* __restrict__ P, DevState* S) {
  if (S->done || !S->aa_attempt) return;
  __shared__ DevState sm;
  state_load(&sm, S);
  if (threadIdx.x == 0) advance(P, &sm);
  state_store(S, &sm);
}

// ---------------------------------------------------------------------------
// setup / finishing / power iteration helpers
// ---------------------------------------------------------------------------

// u0 -> P_feasible(u0) in place (pdhg_core.cpp:41-43); records t0.
__global__ void k_project_start(double* u, const double* l, const double* uu, int n,
                                int64_t N, int m1, DevState* S) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0 && S) S->t0_ns = globaltimer_ns();
  if (t >= N) return;
  if (t < n) u[t] = smin(smax(u[t], l[t]), uu[t]);
  else if (t - n < m1) u[t] = smax(u[t], 0.0);
}

// elementwise KKT terms + lambda from T = K'y and KX = K x (tree partials)
__global__ void __launch_bounds__(kThreads)
    k_kkt_terms(const double* x, const double* y, const double* T, const double* KX,
                const double* c, const double* q, const double* l, const double* uu, int n,
                int mr, int m1, double* lambda, double* part, int nb) {
  __shared__ double red[5 * (kThreads / 32)];
  double acc[5] = {0, 0, 0, 0, 0};
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    const double rc = __dsub_rn(c[t], T[t]);
    const double lam = project_lambda1(rc, l[t], uu[t]);
    if (lambda) lambda[t] = lam;
    if (isfinite(l[t]) && lam > 0.0) acc[0] = __dmul_rn(l[t], lam);
    if (isfinite(uu[t]) && lam < 0.0) acc[0] = __dmul_rn(uu[t], lam);
    const double dv = __dsub_rn(rc, lam);
    acc[1] = __dmul_rn(dv, dv);
    acc[2] = __dmul_rn(c[t], x[t]);
  }
  if (t < mr) {
    acc[3] = __dmul_rn(q[t], y[t]);
    double v = __dsub_rn(q[t], KX[t]);
    if (t < m1) v = smax(v, 0.0);
    acc[4] = __dmul_rn(v, v);
  }
  block_sum<5>(acc, red);
  if (threadIdx.x == 0)
    for (int k = 0; k < 5; ++k) part[k * nb + blockIdx.x] = acc[k];
}

// final KKT: tree partials or serial chains (computed here, thread 0)
__global__ void __launch_bounds__(kCtrlThreads)
    k_kkt_final(const double* x, const double* y, const double* T, const double* KX,
                const double* c, const double* q, const double* l, const double* uu, int n,
                int mr, int m1, const double* part, int nb, int serial, double nrm_q,
                double nrm_c, double* out) {
  __shared__ double red32[32];
  double s[5];
  if (!serial)
    for (int k = 0; k < 5; ++k) s[k] = reduce_partials(part + k * nb, nb, red32);
  if (threadIdx.x != 0) return;
  if (serial) {
    double bound = 0.0, dual_sq = 0.0, infeas = 0.0;
    for (int j = 0; j < n; ++j) {
      const double lam = project_lambda1(__dsub_rn(c[j], T[j]), l[j], uu[j]);
      if (isfinite(l[j]) && lam > 0.0) bound = __dadd_rn(bound, __dmul_rn(l[j], lam));
      if (isfinite(uu[j]) && lam < 0.0) bound = __dadd_rn(bound, __dmul_rn(uu[j], lam));
    }
    for (int j = 0; j < n; ++j) {
      const double rc = __dsub_rn(c[j], T[j]);
      const double v = __dsub_rn(rc, project_lambda1(rc, l[j], uu[j]));
      dual_sq = __dadd_rn(dual_sq, __dmul_rn(v, v));
    }
    for (int i = 0; i < mr; ++i) {
      double v = __dsub_rn(q[i], KX[i]);
      if (i < m1) v = smax(v, 0.0);
      infeas = __dadd_rn(infeas, __dmul_rn(v, v));
    }
    s[0] = bound;
    s[1] = dual_sq;
    s[2] = serial_dot(c, x, n);
    s[3] = serial_dot(q, y, mr);
    s[4] = infeas;
  }
  kkt_from_sums(nrm_q, nrm_c, s[0], s[3], s[2], s[4], s[1], out);
}

// sum of squares: tree partials per CTA (grid-stride, fixed)
__global__ void __launch_bounds__(kThreads)
    k_sumsq_partials(const double* v, const double* w, int64_t n, double* part,
                     const int32_t* stop) {
  if (stop && *stop) return;
  __shared__ double red[kThreads / 32];
  double acc[1] = {0.0};
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    acc[0] = __dadd_rn(acc[0], __dmul_rn(v[t], w ? w[t] : v[t]));
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}

// dot / sum of squares: serial chain (thread 0) or partial reduce; out[0]
__global__ void __launch_bounds__(kCtrlThreads)
    k_dot_final(const double* v, const double* w, int64_t n, const double* part, int nb,
                int serial, double* out) {
  __shared__ double red32[32];
  double s = 0.0;
  if (!serial) s = reduce_partials(part, nb, red32);
  if (threadIdx.x != 0) return;
  if (serial) s = serial_dot(v, w ? w : v, n);
  out[0] = s;
}

struct PowerState {
  int32_t done, it, max_iters, rounds;
  double est, lam, result, rel_tol;
};

// power_iteration_norm loop body control (sparse_linalg.cpp:111-122)
__global__ void __launch_bounds__(kCtrlThreads)
    k_power_ctrl(const double* mtmx, int64_t n, const double* part, int nb, int serial,
                 PowerState* ps) {
  if (ps->done) return;
  __shared__ double red32[32];
  double s = 0.0;
  if (!serial) s = reduce_partials(part, nb, red32);
  if (threadIdx.x != 0) return;
  if (serial) s = serial_dot(mtmx, mtmx, n);
  const double lam = sqrt(s);
  const double next = sqrt(lam);
  const int it = ps->it;
  ps->rounds = it + 1;
  ps->lam = lam;
  if (lam == 0.0) { ps->result = 0.0; ps->done = 1; return; }
  if (it > 0 && fabs(__dsub_rn(next, ps->est)) < __dmul_rn(ps->rel_tol, next)) {
    ps->result = next;
    ps->done = 1;
    return;
  }
  ps->est = next;
  ps->it = it + 1;
  if (ps->it >= ps->max_iters) { ps->result = ps->est; ps->done = 1; }
}

// power_iteration_norm start: xn = ||x0|| (x0 = e_0 when zero), scal[1] = xn
// (sparse_linalg.cpp:106-108)
__global__ void k_power_init_norm(double* x, double* scal) {
  double xn = sqrt(scal[0]);
  if (xn == 0.0) {
    x[0] = 1.0;
    xn = 1.0;
  }
  scal[1] = xn;
}

// x = v / lam (or / ps->lam) — skipped once the iteration has stopped
__global__ void k_scale(double* x, const double* v, int64_t n, const PowerState* ps,
                        const double* lam_ptr) {
  if (ps && ps->done) return;
  const double lam = lam_ptr ? *lam_ptr : ps->lam;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    x[t] = v[t] / lam;
}

}  // namespace aapdhg_b200
