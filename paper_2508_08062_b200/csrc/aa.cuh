// aa.cuh — AA / FAA step kernels, role rotation, setup and power-iteration
// helpers of the sm_100a solver (see pipeline.cuh for the iteration core).
#pragma once

#include "dd.cuh"
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
  // FAA: the low parts of double-double partials (dd.cuh), same layout;
  // null for AA (whose reference solve is itself the Gram's Cholesky)
  double* part_lo = nullptr;
};

// index-ordered Dot2 chain (FAA, SERIAL order)
__device__ __forceinline__ dd serial_dot_dd(const double* a, const double* b, int64_t n) {
  double hi = 0.0, lo = 0.0;
  for (int64_t t = 0; t < n; ++t) dot2_acc(hi, lo, a[t], b[t]);
  return dd_norm(hi, lo);
}

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
  if (P->ring) {  // ring history: dg_a = g(a+1) - g(a) in the chain, the same order
    int kind, a, b;
    decode_item(item, p, kind, a, b);
    const int64_t N = P->N;
    const double* a1 = D.gpool + (int64_t)S->gw[a + 1] * N;
    const double* a0 = D.gpool + (int64_t)S->gw[a] * N;
    const double* b1 = D.gpool + (int64_t)S->gw[kind == 0 ? b + 1 : p] * N;
    const double* b0 = D.gpool + (int64_t)S->gw[b] * N;
    double s = 0.0;
    for (int64_t t = 0; t < N; ++t) {
      const double x = __dsub_rn(a1[t], a0[t]);
      const double y = kind == 0 ? __dsub_rn(b1[t], b0[t]) : b1[t];
      s = __dadd_rn(s, __dmul_rn(x, y));
    }
    D.part[item] = s;
    return;
  }
  const double *va, *vb;
  item_vectors(D, P, S, item, p, va, vb);
  if (D.part_lo) {
    const dd v = serial_dot_dd(va, vb, P->N);
    D.part[item] = v.hi;
    D.part_lo[item] = v.lo;
  } else {
    D.part[item] = serial_dot(va, vb, P->N);
  }
}

// TREE: CTA b covers elements [b*kDotChunk, ...); warp w takes items w, w+8..
// Column chunks are re-read from L1 across items; HBM sees each once.
__global__ void __launch_bounds__(kThreads)
    k_tree_dots(DotBufs D, const DevParams* __restrict__ P, const DevState* S) {
  TL_MARK(19);
  if (S->done || !S->aa_attempt) return;
  // the memory's slot table once per CTA (not a dependent global load per item)
  __shared__ int slots[kMaxMemory + 1];
  __shared__ int sh_p, sh_g;
  const bool ring = P->ring != 0;
  if (threadIdx.x < kMaxMemory + 1)
    slots[threadIdx.x] = ring ? S->gw[threadIdx.x] : threadIdx.x < kMaxMemory ? S->mem_slots[threadIdx.x] : 0;
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
    double x[kPer], y[kPer];
    if (ring) {  // ring history: the differences of the window's g columns
      const double* a1 = D.gpool + (int64_t)slots[ia + 1] * N + base;
      const double* a0 = D.gpool + (int64_t)slots[ia] * N + base;
      const double* b1 = D.gpool + (int64_t)slots[kind == 0 ? ib + 1 : p] * N + base;
      const double* b0 = D.gpool + (int64_t)slots[ib] * N + base;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int t = lane + 32 * u;
        x[u] = t < cnt ? __dsub_rn(a1[t], a0[t]) : 0.0;
        y[u] = t < cnt ? (kind == 0 ? __dsub_rn(b1[t], b0[t]) : b1[t]) : 0.0;
      }
    } else {
      if (kind == 0) { va = D.dg + slots[ia] * N; vb = D.dg + slots[ib] * N; }
      else if (kind == 1) { va = D.dg + slots[ia] * N; vb = D.gpool + (int64_t)sh_g * N; }
      else { va = D.du + slots[ia] * N; vb = va; }
      // every load of the lane's share in flight before the adds (same order:
      // t = lane, lane + 32, ...)
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int t = lane + 32 * u;
        x[u] = t < cnt ? va[base + t] : 0.0;
        y[u] = t < cnt ? vb[base + t] : 0.0;
      }
    }
    if (D.part_lo) {  // FAA: double-double partials
      double hi = 0.0, lo = 0.0;
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (lane + 32 * u < cnt) dot2_acc(hi, lo, x[u], y[u]);
      const dd v = warp_sum_dd(dd_norm(hi, lo));
      if (lane == 0) {
        D.part[(int64_t)item * P->ndot_blk + blockIdx.x] = v.hi;
        D.part_lo[(int64_t)item * P->ndot_blk + blockIdx.x] = v.lo;
      }
      continue;
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

// CAP-space accumulator q of the register Gram -> p-space item (-1: unused):
// q < NPAIR pairs (a <= b), then the rhs items, then the e-norms
__device__ __forceinline__ int gram_item(int q, int cap, int p, int np) {
  const int npair = cap * (cap + 1) / 2;
  if (q < npair) {
    int a = 0, rem = q;
    while (rem >= cap - a) { rem -= cap - a; ++a; }
    const int b = a + rem;
    return b < p ? a * p - a * (a - 1) / 2 + (b - a) : -1;
  }
  if (q < npair + cap) return q - npair < p ? np + (q - npair) : -1;
  return q - npair - cap < p ? np + p + (q - npair - cap) : -1;
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
  TL_MARK(10);
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
  // software-pipelined (AA): the next element's loads are in flight while
  // this one accumulates (the same element order, so the same sums)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double nv[CAP], nh = 0.0, nc = 0.0;
  if (!FAA && t < N) {
    nh = uh[t];
    nc = uc[t];
#pragma unroll
    for (int a = 0; a < CAP; ++a) nv[a] = a < p ? dgc[a][t] : 0.0;
  }
  for (; t < N; t += stride) {
    double v[CAP];
    double gt;
    if constexpr (!FAA) {
      gt = __dsub_rn(nh, nc);
#pragma unroll
      for (int a = 0; a < CAP; ++a) v[a] = nv[a];
      const int64_t tn = t + stride;
      if (tn < N) {
        nh = uh[tn];
        nc = uc[tn];
#pragma unroll
        for (int a = 0; a < CAP; ++a) nv[a] = a < p ? dgc[a][tn] : 0.0;
      }
    } else {
      gt = __dsub_rn(uh[t], uc[t]);
#pragma unroll
      for (int a = 0; a < CAP; ++a) v[a] = a < p ? dgc[a][t] : 0.0;
    }
    g[t] = gt;
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
    const int item = gram_item(q, CAP, p, np);
    if (item >= 0) D.part[(int64_t)item * gridDim.x + blockIdx.x] = s;
  }
}

// k_gram_dots of the ring history (DevParams::ring, AA): the p + 1 window
// columns g_{k-p}..g_k are loaded per element (one HBM read each, software
// pipelined like k_gram_dots) and differenced in registers, dg_a = g(a+1) -
// g(a) — the pushed dg bit for bit; the rhs item is dg_a . g_k. Nothing is
// staged: the epilogues stored g_k.
template <int CAP>
__global__ void __launch_bounds__(kThreads, 1)
    k_gram_dots_ring(DotBufs D, const DevParams* __restrict__ P, const DevState* S) {
  TL_MARK(10);
  if (S->done || !S->aa_attempt) return;
  constexpr int NPAIR = CAP * (CAP + 1) / 2;
  constexpr int NACC = NPAIR + CAP;
  __shared__ int slots[CAP + 1];
  __shared__ int sh_p;
  if (threadIdx.x <= CAP) slots[threadIdx.x] = S->gw[threadIdx.x];
  if (threadIdx.x == 0) sh_p = S->mem_size;
  __syncthreads();
  const int p = sh_p;
  const int64_t N = P->N;
  const double* gc[CAP + 1];
#pragma unroll
  for (int a = 0; a <= CAP; ++a) gc[a] = D.gpool + (int64_t)(a <= p ? slots[a] : slots[0]) * N;
  double acc[NACC];
#pragma unroll
  for (int q = 0; q < NACC; ++q) acc[q] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double nv[CAP + 1];
#pragma unroll
  for (int a = 0; a <= CAP; ++a) nv[a] = (a <= p && t < N) ? gc[a][t] : 0.0;
  for (; t < N; t += stride) {
    double w[CAP + 1];
#pragma unroll
    for (int a = 0; a <= CAP; ++a) w[a] = nv[a];
    const int64_t tn = t + stride;
    if (tn < N) {
#pragma unroll
      for (int a = 0; a <= CAP; ++a) nv[a] = a <= p ? gc[a][tn] : 0.0;
    }
    double v[CAP];
    double gt = 0.0;
#pragma unroll
    for (int a = 0; a < CAP; ++a) v[a] = a < p ? __dsub_rn(w[a + 1], w[a]) : 0.0;
#pragma unroll
    for (int a = 0; a <= CAP; ++a)
      if (a == p) gt = w[a];
    int q = 0;
#pragma unroll
    for (int a = 0; a < CAP; ++a)
#pragma unroll
      for (int b = a; b < CAP; ++b, ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v[a], v[b]));
#pragma unroll
    for (int a = 0; a < CAP; ++a) acc[NPAIR + a] = __dadd_rn(acc[NPAIR + a], __dmul_rn(v[a], gt));
  }
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
    const int item = gram_item(q, CAP, p, np);
    if (item >= 0) D.part[(int64_t)item * gridDim.x + blockIdx.x] = s;
  }
}

// FAA, memory capacity <= CAP (<= 10): the Gram F'F and the rhs F'g as
// double-double partials (Dot2, dd.cuh), the e-norms in double, in one pass
// over the columns with g staged (k_stage_g). With SPLIT the dd items are
// shared by a pair of CTAs over the same elements (CTA 2b: the even items,
// 2b + 1: the odd ones and the e-norms), so each keeps half the
// accumulators in registers (memory 8 and 10 would spill); the pair reads
// the same columns at the same time, the second read hits L2.
template <int CAP, int SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    k_gram_dots_dd(DotBufs D, double* __restrict__ upool, const DevParams* __restrict__ P,
                   const DevState* S) {
  TL_MARK(11);
  if (S->done || !S->aa_attempt) return;
  constexpr int NPAIR = CAP * (CAP + 1) / 2;
  constexpr int NDD = NPAIR + CAP;                        // Gram + rhs items (dd)
  constexpr int NH = SPLIT ? (NDD + 1) / 2 : NDD;         // this CTA's dd items
  const int half = SPLIT ? int(blockIdx.x & 1) : 0;
  const int eblk = SPLIT ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int nblk = SPLIT ? int(gridDim.x >> 1) : int(gridDim.x);
  const bool enorms = !SPLIT || half == 1;
  __shared__ int64_t soff[CAP];
  __shared__ int sh_p, sh_g, sh_h, sh_c;
  if (threadIdx.x == 0) {
    sh_p = S->mem_size;
    sh_g = S->g_idx[G_CUR];
    sh_h = S->u_idx[U_HAT];
    sh_c = S->u_idx[U_CUR];
  }
  __syncthreads();
  const int p = sh_p;
  const int64_t N = P->N;
  if (threadIdx.x < CAP)
    soff[threadIdx.x] = (int64_t)(int(threadIdx.x) < p ? S->mem_slots[threadIdx.x] : 0) * N;
  __syncthreads();
  const double* uh = upool + (int64_t)sh_h * N;
  const double* uc = upool + (int64_t)sh_c * N;
  double* g = const_cast<double*>(D.gpool) + (int64_t)sh_g * N;
  double hi[NH], lo[NH], en[CAP];
#pragma unroll
  for (int k = 0; k < NH; ++k) hi[k] = lo[k] = 0.0;
#pragma unroll
  for (int a = 0; a < CAP; ++a) en[a] = 0.0;
  for (int64_t t = (int64_t)eblk * blockDim.x + threadIdx.x; t < N;
       t += (int64_t)nblk * blockDim.x) {
    const double gt = __dsub_rn(uh[t], uc[t]);
    if (half == 0) g[t] = gt;
    double v[CAP];
#pragma unroll
    for (int a = 0; a < CAP; ++a) v[a] = a < p ? D.dg[soff[a] + t] : 0.0;
    int q = 0;
#pragma unroll
    for (int a = 0; a < CAP; ++a)
#pragma unroll
      for (int b = a; b < CAP; ++b, ++q)
        if (!SPLIT || (q & 1) == half) dot2_acc(hi[q >> SPLIT], lo[q >> SPLIT], v[a], v[b]);
#pragma unroll
    for (int a = 0; a < CAP; ++a, ++q)
      if (!SPLIT || (q & 1) == half) dot2_acc(hi[q >> SPLIT], lo[q >> SPLIT], v[a], gt);
    if (enorms) {
#pragma unroll
      for (int a = 0; a < CAP; ++a) {
        const double e = a < p ? D.du[soff[a] + t] : 0.0;
        en[a] = __dadd_rn(en[a], __dmul_rn(e, e));
      }
    }
  }
  // fixed-shape CTA reduction: warp xor trees, then the warps in order
  __shared__ double red_hi[kWarps][NH], red_lo[kWarps][NH], red_en[kWarps][CAP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NH; ++k) {
    const dd sv = warp_sum_dd(dd_norm(hi[k], lo[k]));
    if (lane == 0) {
      red_hi[warp][k] = sv.hi;
      red_lo[warp][k] = sv.lo;
    }
  }
  if (enorms) {
#pragma unroll
    for (int a = 0; a < CAP; ++a) {
      const double sv = warp_sum(en[a]);
      if (lane == 0) red_en[warp][a] = sv;
    }
  }
  __syncthreads();
  const int np = p * (p + 1) / 2;
  for (int k = threadIdx.x; k < NH; k += blockDim.x) {
    const int q = SPLIT ? 2 * k + half : k;
    if (q >= NDD) continue;
    dd sd = dd{red_hi[0][k], red_lo[0][k]};
    for (int w = 1; w < kWarps; ++w) sd = dd_add(sd, dd{red_hi[w][k], red_lo[w][k]});
    const int item = gram_item(q, CAP, p, np);
    if (item < 0) continue;
    D.part[(int64_t)item * nblk + eblk] = sd.hi;
    D.part_lo[(int64_t)item * nblk + eblk] = sd.lo;
  }
  if (enorms)
    for (int a = threadIdx.x; a < p; a += blockDim.x) {
      double sv = red_en[0][a];
      for (int w = 1; w < kWarps; ++w) sv = __dadd_rn(sv, red_en[w][a]);
      D.part[(int64_t)(np + p + a) * nblk + eblk] = sv;
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
// p <= 32: the same factorization and solves by warp 0 alone (lane i owns row
// i; the operation order of every element is the one above, so the bits are
// too), with warp shuffles instead of CTA barriers between the columns.
__device__ bool warp_cholesky_solve(int p, double* a, double* rhs) {
#define A_(i, j) a[(j) * p + (i)]
  __shared__ int ok_sh;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    bool ok = true;
    for (int j = 0; j < p && ok; ++j) {
      double d = 0.0;
      int bad = 0;
      if (lane == 0) {
        d = A_(j, j);
        for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(A_(j, k), A_(j, k)));
        bad = d <= 0.0;
        if (!bad) {
          d = sqrt(d);
          A_(j, j) = d;
        }
      }
      d = __shfl_sync(0xffffffffu, d, 0);
      bad = __shfl_sync(0xffffffffu, bad, 0);
      __syncwarp();
      if (bad) {
        ok = false;
        break;
      }
      const int i = j + 1 + lane;
      if (i < p) {
        double s = A_(i, j);
        for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(A_(i, k), A_(j, k)));
        A_(i, j) = s / d;
      }
      __syncwarp();
    }
    if (ok) {
      double r = lane < p ? rhs[lane] : 0.0;  // lane k holds rhs[k]
      for (int i = 0; i < p; ++i) {
        double ri = __shfl_sync(0xffffffffu, r, i);
        ri = ri / A_(i, i);
        if (lane == i) r = ri;
        if (lane > i && lane < p) r = __dsub_rn(r, __dmul_rn(A_(lane, i), ri));
      }
      if (lane < p) rhs[lane] = r;
      __syncwarp();
      if (lane == 0)
        for (int i = p - 1; i >= 0; --i) {
          double t = rhs[i];
          for (int k = i + 1; k < p; ++k) t = __dsub_rn(t, __dmul_rn(A_(k, i), rhs[k]));
          rhs[i] = t / A_(i, i);
        }
    }
    if (lane == 0) ok_sh = ok ? 1 : 0;
  }
  __syncthreads();
#undef A_
  return ok_sh != 0;
}

__device__ bool block_cholesky_solve(int p, double* a, double* rhs) {
  if (p <= 32) return warp_cholesky_solve(p, a, rhs);
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
  TL_MARK(12);
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
  // FAA: the low parts of the Gram / rhs items (double-double, dd.cuh)
  __shared__ double vlo[kMaxMemory * (kMaxMemory + 1) / 2 + kMaxMemory];
  const int ndd = (P->method == AAPDHG_METHOD_FAA && D.part_lo) ? p * (p + 1) / 2 + p : 0;
  for (int it = threadIdx.x; it < p * (p + 1) / 2 + p; it += blockDim.x) vlo[it] = 0.0;
  __syncthreads();
  if (rank_tot) {  // sharded: per-shard totals summed in rank order
    for (int it = threadIdx.x; it < nit; it += blockDim.x) {
      double s = rank_tot[it];
      for (int r = 1; r < nranks; ++r) s = __dadd_rn(s, rank_tot[(int64_t)r * rank_stride + it]);
      vals[it] = s;
    }
  } else if (P->serial) {
    for (int it = threadIdx.x; it < nit; it += blockDim.x) {
      vals[it] = D.part[it];
      if (it < ndd) vlo[it] = D.part_lo[it];
    }
  } else if (ndd > 0) {
    // FAA: warp per item, the CTAs' double-double partials added in a fixed
    // shape (lane-strided, then the xor tree)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int it = warp; it < nit; it += nw) {
      const double* pp = D.part + (int64_t)it * P->ndot_blk;
      const double* pl = D.part_lo + (int64_t)it * P->ndot_blk;
      const bool two = it < ndd;
      dd s = {0.0, 0.0};
      for (int b = lane; b < P->ndot_blk; b += 32)
        s = dd_add(s, dd{__ldcg(pp + b), two ? __ldcg(pl + b) : 0.0});
      s = warp_sum_dd(s);
      if (lane == 0) {
        vals[it] = s.hi;
        if (two) vlo[it] = s.lo;
      }
    }
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
  TL_MARK(24);
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
    TL_MARK(25);
  }
  // FAA (filtering.cpp:140-181): angle filter on the newest-first order,
  // length filter, then the least-squares weights of the kept columns, all
  // from the double-double Gram F'F and rhs F'g (dd.cuh) by the whole CTA:
  //   * the angle filter's |R(j,j)| / ||f_j|| is the Householder QR diagonal
  //     of the reversed F (qr_diagonal, filtering.cpp:25-50): the Cholesky
  //     factor of the reversed Gram, row by row; a dependent column (pivot
  //     <= 0) gets a zero diagonal and a zero row, like a skipped reflection;
  //   * w = R^{-1} R^{-T} F'g with R'R = F_kept'F_kept (= R^{-1} Q'g of the
  //     economy QR, sparse_linalg.cpp:131-227, with the 1e-14 ||R||_F
  //     singularity floor of back_substitute).
  __shared__ int faa_ok, faa_kk;
  __shared__ int faa_kpos[kMaxMemory];
  __shared__ double faa_w[kMaxMemory];
  if (P->method == AAPDHG_METHOD_FAA) {
    double* Rh = W.work;            // p x p row-major (angle filter), then kk x kk
    double* Rl = W.work + P->cap * P->cap;  // its low parts (third cap^2 block, aa_smem)
    __shared__ double dsh_hi, dsh_lo;
    __shared__ int keep[kMaxMemory];
    auto gdd = [&](int r, int c) {  // Gram item (r, c) as double-double
      const int lo = r < c ? r : c, hi = r < c ? c : r;
      const int it = lo * p - lo * (lo - 1) / 2 + (hi - lo);
      return dd{vals[it], vlo[it]};
    };
    if (threadIdx.x == 0) faa_ok = 1;
    __syncthreads();
    for (int j = 0; j < p; ++j) {
      const int gj = p - 1 - j;
      if (threadIdx.x == 0) {
        dd d = gdd(gj, gj);
        for (int k = 0; k < j; ++k) {
          const dd r = dd{Rh[k * p + j], Rl[k * p + j]};
          d = dd_sub(d, dd_mul(r, r));
        }
        const dd rjj = d.hi > 0.0 ? dd_sqrt(d) : dd{0.0, 0.0};
        Rh[j * p + j] = rjj.hi;
        Rl[j * p + j] = rjj.lo;
        dsh_hi = rjj.hi;
        dsh_lo = rjj.lo;
        const dd fn = dd_sqrt(gdd(gj, gj));
        const double sine =
            ((int64_t)j < P->Nglob && fn.hi > 0.0) ? dd_div(rjj, fn).hi : 0.0;
        keep[j] = 1;
        if (P->faa_skip & kFaaSkipAngle) {
          // (per-op length_filter / QR: every column goes on)
        } else if (j == 0) {
          if (fn.hi == 0.0) faa_ok = 0;  // zero leading column -> SingularError
        } else if (sine < P->c_s) {
          keep[j] = 0;
        }
      }
      __syncthreads();
      const dd rjj = dd{dsh_hi, dsh_lo};
      for (int i2 = j + 1 + int(threadIdx.x); i2 < p; i2 += blockDim.x) {
        const int gi = p - 1 - i2;
        dd sv = gdd(gi, gj);
        for (int k = 0; k < j; ++k)
          sv = dd_sub(sv, dd_mul(dd{Rh[k * p + j], Rl[k * p + j]}, dd{Rh[k * p + i2], Rl[k * p + i2]}));
        const dd r = rjj.hi > 0.0 ? dd_div(sv, rjj) : dd{0.0, 0.0};
        Rh[j * p + i2] = r.hi;
        Rl[j * p + i2] = r.lo;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      int kk = 0;
      if (faa_ok) {
        // length filter over the kept columns (newest first), filtering.cpp:116-138
        const double* en2 = vals + npair + p;
        int idx[kMaxMemory];
        int m = 0;
        for (int t = 0; t < p; ++t)
          if (keep[t]) idx[m++] = p - 1 - t;  // memory positions, newest first
        double* fn_sq = W.vec + 3 * kMaxMemory;
        double* bb = W.vec + 4 * kMaxMemory;
        for (int t = 0; t < m; ++t) fn_sq[t] = vals[idx[t] * p - idx[t] * (idx[t] - 1) / 2];
        dev_length_bounds(m, fn_sq, P->c_s, bb);
        double ep = 0.0, bp = 0.0;
        const double cap = __dmul_rn(P->kappa_bar, P->kappa_bar);
        double epre[kMaxMemory + 1], bpre[kMaxMemory + 1];
        epre[0] = bpre[0] = 0.0;
        for (int t = 0; t < m; ++t) {
          ep = __dadd_rn(ep, en2[idx[t]]);
          bp = __dadd_rn(bp, bb[t]);
          epre[t + 1] = ep;
          bpre[t + 1] = bp;
        }
        if (P->faa_skip & kFaaSkipLength) kk = m;
        else
          for (int t = m; t >= 1; --t)
            if (__dmul_rn(epre[t], bpre[t]) <= cap) { kk = t; break; }
        // kept positions back in memory (oldest-first) order
        for (int t = 0; t < kk; ++t) faa_kpos[t] = idx[kk - 1 - t];
      }
      faa_kk = kk;
    }
    __syncthreads();
    const int kk = faa_kk;
    if (faa_ok && kk > 0) {
      // R'R = G_kept (upper R, row-major kk x kk), the whole CTA per column
      for (int j = 0; j < kk; ++j) {
        if (threadIdx.x == 0) {
          dd d = gdd(faa_kpos[j], faa_kpos[j]);
          for (int k = 0; k < j; ++k) {
            const dd r = dd{Rh[k * kk + j], Rl[k * kk + j]};
            d = dd_sub(d, dd_mul(r, r));
          }
          if (!(d.hi > 0.0)) {
            faa_ok = 0;
            d = dd{1.0, 0.0};
          }
          const dd r = dd_sqrt(d);
          Rh[j * kk + j] = r.hi;
          Rl[j * kk + j] = r.lo;
          dsh_hi = r.hi;
          dsh_lo = r.lo;
        }
        __syncthreads();
        if (!faa_ok) break;
        const dd rjj = dd{dsh_hi, dsh_lo};
        for (int i2 = j + 1 + int(threadIdx.x); i2 < kk; i2 += blockDim.x) {
          dd sv = gdd(faa_kpos[i2], faa_kpos[j]);
          for (int k = 0; k < j; ++k)
            sv = dd_sub(sv, dd_mul(dd{Rh[k * kk + j], Rl[k * kk + j]},
                                   dd{Rh[k * kk + i2], Rl[k * kk + i2]}));
          const dd r = dd_div(sv, rjj);
          Rh[j * kk + i2] = r.hi;
          Rl[j * kk + i2] = r.lo;
        }
        __syncthreads();
      }
      if (threadIdx.x == 0 && faa_ok) {
        // back_substitute floor: |r_ii| <= 1e-14 ||R||_F -> SingularError
        double fro = 0.0;
        for (int j = 0; j < kk; ++j)
          for (int i2 = j; i2 < kk; ++i2) fro = __dadd_rn(fro, __dmul_rn(Rh[j * kk + i2], Rh[j * kk + i2]));
        const double floor_v = 1e-14 * sqrt(fro);
        for (int i2 = 0; i2 < kk; ++i2)
          if (fabs(Rh[i2 * kk + i2]) <= floor_v) faa_ok = 0;
        if (faa_ok) {
          // forward R' z = F'g, back R w = z, in double-double
          dd z[kMaxMemory];
          for (int i2 = 0; i2 < kk; ++i2) {
            const int it = npair + faa_kpos[i2];
            dd sv = dd{vals[it], vlo[it]};
            for (int k2 = 0; k2 < i2; ++k2)
              sv = dd_sub(sv, dd_mul(dd{Rh[k2 * kk + i2], Rl[k2 * kk + i2]}, z[k2]));
            z[i2] = dd_div(sv, dd{Rh[i2 * kk + i2], Rl[i2 * kk + i2]});
          }
          for (int i2 = kk - 1; i2 >= 0; --i2) {
            dd sv = z[i2];
            for (int k2 = i2 + 1; k2 < kk; ++k2)
              sv = dd_sub(sv, dd_mul(dd{Rh[i2 * kk + k2], Rl[i2 * kk + k2]}, z[k2]));
            z[i2] = dd_div(sv, dd{Rh[i2 * kk + i2], Rl[i2 * kk + i2]});
          }
          for (int i2 = 0; i2 < kk; ++i2) faa_w[i2] = z[i2].hi;
        }
      }
      // per-op economy_qr: R of the kept columns (column-major, diag >= 0)
      if (P->qr_r_out && faa_ok)
        for (int t = threadIdx.x; t < kk * kk; t += blockDim.x) {
          const int r = t % kk, c = t / kk;
          P->qr_r_out[t] = r <= c ? Rh[r * kk + c] : 0.0;
        }
    }
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
    // FAA: the CTA's double-double solve above
    ok = faa_ok != 0;
    const int kk = faa_kk;
    pm = kk;
    if (ok) {
      for (int t = 0; t < kk; ++t) w[t] = faa_w[t];
      for (int t = 0; t < kk; ++t) S->mix_slots[t] = S->mem_slots[faa_kpos[t]];
      if (!per_op) {
        // carried memory replaced only on success (solver.cpp:221-224)
        for (int t = 0; t < kk; ++t) S->mem_slots[t] = S->mix_slots[t];
        S->mem_size = kk;
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
  TL_MARK(23);
}

constexpr int kMixGroup = 4;  // k_mix: history columns whose loads are in flight together

// cand = P_feasible(u + damp(g) - sum_j w_j (du_j + damp(dg_j)))
// (anderson.cpp:109,130-133 / filtering.cpp:165,176-179; solver.cpp:226)
__global__ void __launch_bounds__(kThreads)
    k_mix(IterBufs B, const double* __restrict__ dg, const DevParams* __restrict__ P,
          const DevState* S, int project) {
  TL_MARK(13);
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
  if (P->ring) {
    // ring history: du_j / dg_j from the window (pipeline.cuh ring_push), and
    // the candidate's own du_{k+1} = cand - u_k into du at the slot g_{k+1}
    // takes (ring_free_slot), used when the candidate is accepted
    __shared__ int64_t gsl[kMaxMemory + 1];
    __shared__ uint8_t gx[kMaxMemory + 1];
    __shared__ int64_t nxt;
    for (int q = threadIdx.x; q <= pm; q += blockDim.x) {
      gsl[q] = (int64_t)S->gw[q] * N;
      gx[q] = S->gdux[q];
    }
    if (threadIdx.x == 0) nxt = (int64_t)ring_free_slot(P, S) * N;
    __syncthreads();
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
         t += (int64_t)gridDim.x * blockDim.x) {
      const double gk = B.gpool[gsl[pm] + t];
      const double ut = u[t];
      double o = __dadd_rn(ut, damp1(beta, dh, t, gk));
      double gp = B.gpool[gsl[0] + t];
      // columns in groups of kMixGroup: the group's loads are all issued
      // before its (ordered) adds, so a thread keeps up to 2 kMixGroup loads
      // in flight instead of one (same operations in the same order)
      for (int j0 = 0; j0 < pm; j0 += kMixGroup) {
        double gc[kMixGroup], dv[kMixGroup];
#pragma unroll
        for (int q = 0; q < kMixGroup; ++q) {
          const int jj = j0 + q;
          gc[q] = 0.0;
          dv[q] = 0.0;
          if (jj < pm) {
            if (jj + 1 < pm) gc[q] = B.gpool[gsl[jj + 1] + t];
            if (gx[jj + 1]) dv[q] = B.du[gsl[jj + 1] + t];
          }
        }
#pragma unroll
        for (int q = 0; q < kMixGroup; ++q) {
          const int jj = j0 + q;
          if (jj < pm) {
            const double a = nw[jj];
            const double gcq = jj + 1 == pm ? gk : gc[q];
            const double du = gx[jj + 1] ? dv[q] : gp;
            o = __dadd_rn(o, __dmul_rn(a, du));
            o = __dadd_rn(o, __dmul_rn(a, damp1(beta, dh, t, __dsub_rn(gcq, gp))));
            gp = gcq;
          }
        }
      }
      if (project) {
        if (t < n) o = smin(smax(o, B.l[t]), B.u[t]);
        else if (t - n < P->m1) o = smax(o, 0.0);
      }
      out[t] = o;
      B.du[nxt + t] = __dsub_rn(o, ut);
    }
    return;
  }
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (int64_t)gridDim.x * blockDim.x) {
    double o = __dadd_rn(u[t], damp1(beta, dh, t, g[t]));
    for (int j0 = 0; j0 < pm; j0 += kMixGroup) {  // (grouped loads, as above)
      double uv[kMixGroup], gv[kMixGroup];
#pragma unroll
      for (int q = 0; q < kMixGroup; ++q) {
        const int jj = j0 + q;
        uv[q] = jj < pm ? B.du[sls[jj] * N + t] : 0.0;
        gv[q] = jj < pm ? dg[sls[jj] * N + t] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kMixGroup; ++q) {
        const int jj = j0 + q;
        if (jj < pm) {
          const double a = nw[jj];
          o = __dadd_rn(o, __dmul_rn(a, uv[q]));
          o = __dadd_rn(o, __dmul_rn(a, damp1(beta, dh, t, gv[q])));
        }
      }
    }
    if (project) {
      if (t < n) o = smin(smax(o, B.l[t]), B.u[t]);
      else if (t - n < P->m1) o = smax(o, 0.0);
    }
    out[t] = o;
  }
}

// economy_qr's Q = F R^{-1} (per-op): row t of Q solves q R = f_t by
// forward substitution over R's columns (R upper, column-major kk x kk, in
// shared memory); F's columns are the memory slots 0..kk-1 of dg.
__global__ void __launch_bounds__(kThreads)
    k_qr_q(const double* __restrict__ f, const double* __restrict__ r, int kk, int64_t N,
           double* __restrict__ q) {
  __shared__ double rs[kMaxMemory * kMaxMemory];
  for (int t = threadIdx.x; t < kk * kk; t += blockDim.x) rs[t] = r[t];
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N;
       t += (int64_t)gridDim.x * blockDim.x) {
    double row[kMaxMemory];
    for (int j = 0; j < kk; ++j) {
      double s = f[(int64_t)j * N + t];
      for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(row[k], rs[j * kk + k]));
      row[j] = s / rs[j * kk + j];
      q[(int64_t)j * N + t] = row[j];
    }
  }
}

// g_k = T(u_k) - u_k of an iteration that attempts an AA step (the Gram
// rhs and the mix read it; the next iteration's push reads it as g_{k-1}
// when the candidate is accepted). K1/K2 do not store g: after a plain step
// the push derives g_{k-1} from du (solver.cpp:204-209).
__global__ void k_stage_g(const double* __restrict__ upool, double* __restrict__ gpool,
                          const DevParams* __restrict__ P, const DevState* S) {
  TL_MARK(18);
  if (S->done || !S->aa_attempt || P->ring) return;  // (the ring holds g_k)
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
  TL_MARK(21);
  if (S->done || !S->aa_attempt) return;
  __shared__ DevState sm;
  state_load(&sm, S);
  if (threadIdx.x == 0) advance(P, &sm);
  state_store(S, &sm);
}

// The K x recache of an accepted candidate with the AA branch's commit in
// its last CTA (one launch instead of k_spmv + k_aa_commit). Every CTA
// reads the roles when it starts; the last one to finish (ticket) rotates
// them, so no reader sees the new roles. A SingularError fallback has no
// candidate: CTA 0 only commits.
template <bool SERIAL>
__global__ void __launch_bounds__(kThreads, kSpmvBlocksPerSM)
    k_spmv_commit(CsrDev A, VecRef xr, RowsumArgs o, const DevParams* __restrict__ P,
                  DevState* S, unsigned int* ticket) {
  TL_MARK(15);
  if (S->done || !S->aa_attempt) return;
  __shared__ DevState sm;
  if (!S->aa_ok) {
    if (blockIdx.x == 0) {
      state_load(&sm, S);
      if (threadIdx.x == 0) advance(P, &sm);
      state_store(S, &sm);
    }
    return;
  }
  const double* x = xr.get(S);
  double* out = o.out_pool + (int64_t)S->kx_idx[o.out_role] * o.out_stride;
  for (int rep = 0;; ++rep) {
    double v;
    const int row = row_sum<SERIAL, kUnroll, false, false>(A, x, v, NoPre{}, -1, rep);
    if (row == -2) break;
    if (row >= 0) out[row] = o.rinit ? __dadd_rn(o.rinit[row], v) : v;
  }
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) *ticket = 0u;
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
  TL_MARK(22);
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
