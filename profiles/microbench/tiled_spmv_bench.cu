// tiled_spmv_bench.cu — microbenchmark (not product code): 2-D tiled SpMV
// y = A x for the config-1 shapes, against the one-slice-per-warp SELL-32
// global-gather SpMV the solver uses today.
//
// Tiled: rows split into R groups, columns into C blocks. One CTA per tile
// (r, c) copies x[block c] into shared memory (cp.async.bulk), then runs a
// tile-local SELL-32 (u16 column, f64 value) with shared-memory gathers and
// writes the tile's row partials P[c][row]. A second kernel sums the C
// partials of each row in block order. Random gathers move from L1TEX/L2
// sectors (32 B per 8-byte gather, the ceiling of the global path) to shared
// memory; the price is R copies of x and 2*C*M*8 bytes of partials.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tiled_spmv_bench tiled_spmv_bench.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

struct Csr {
  int M, N;
  std::vector<int> rp, ci;
  std::vector<double> v;
};

static Csr planted(int m, int n, int per_col, uint64_t seed) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> nd;
  std::vector<std::vector<std::pair<int, double>>> rows(m);
  std::vector<int> pick;
  for (int j = 0; j < n; ++j) {
    pick.clear();
    while ((int)pick.size() < per_col) {
      int r = (int)(g() % (uint64_t)m);
      if (std::find(pick.begin(), pick.end(), r) == pick.end()) pick.push_back(r);
    }
    for (int r : pick) rows[r].push_back({j, nd(g)});
  }
  Csr a;
  a.M = m;
  a.N = n;
  a.rp.assign(m + 1, 0);
  for (int i = 0; i < m; ++i) {
    a.rp[i + 1] = a.rp[i] + (int)rows[i].size();
    for (auto& e : rows[i]) {
      a.ci.push_back(e.first);
      a.v.push_back(e.second);
    }
  }
  return a;
}

static Csr transpose(const Csr& a) {
  Csr t;
  t.M = a.N;
  t.N = a.M;
  t.rp.assign(a.N + 1, 0);
  for (int c : a.ci) t.rp[c + 1]++;
  for (int j = 0; j < a.N; ++j) t.rp[j + 1] += t.rp[j];
  t.ci.resize(a.ci.size());
  t.v.resize(a.v.size());
  std::vector<int> pos(t.rp.begin(), t.rp.end() - 1);
  for (int i = 0; i < a.M; ++i)
    for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
      int p = pos[a.ci[k]]++;
      t.ci[p] = i;
      t.v[p] = a.v[k];
    }
  return t;
}

// ---- baseline: global SELL-32, one slice per warp ------------------------------------------
struct GSell {
  std::vector<int> sl_ptr, sl_len, row;  // per slice; row[32*s+lane] (-1 pad)
  std::vector<int> ci;
  std::vector<double> v;
};

static GSell build_gsell(const Csr& a) {
  GSell s;
  std::vector<int> ord(a.M);
  std::iota(ord.begin(), ord.end(), 0);
  // SELL-sigma: sort by length inside windows of 8 slices
  const int W = 256;
  for (int w = 0; w < a.M; w += W) {
    int e = std::min(a.M, w + W);
    std::stable_sort(ord.begin() + w, ord.begin() + e, [&](int x, int y) {
      return a.rp[x + 1] - a.rp[x] > a.rp[y + 1] - a.rp[y];
    });
  }
  int ns = (a.M + 31) / 32;
  for (int sl = 0; sl < ns; ++sl) {
    int L = 0;
    for (int l = 0; l < 32; ++l) {
      int k = sl * 32 + l;
      int r = k < a.M ? ord[k] : -1;
      s.row.push_back(r);
      if (r >= 0) L = std::max(L, a.rp[r + 1] - a.rp[r]);
    }
    s.sl_ptr.push_back((int)s.ci.size());
    s.sl_len.push_back(L);
    for (int k = 0; k < L; ++k)
      for (int l = 0; l < 32; ++l) {
        int r = s.row[sl * 32 + l];
        bool ok = r >= 0 && k < a.rp[r + 1] - a.rp[r];
        s.ci.push_back(ok ? a.ci[a.rp[r] + k] : 0);
        s.v.push_back(ok ? a.v[a.rp[r] + k] : 0.0);
      }
  }
  return s;
}

__global__ void __launch_bounds__(256) k_gsell(const int* __restrict__ sl_ptr,
                                               const int* __restrict__ sl_len,
                                               const int* __restrict__ row,
                                               const int* __restrict__ ci,
                                               const double* __restrict__ v,
                                               const double* __restrict__ x, double* __restrict__ y,
                                               int ns) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = warp; s < ns; s += nw) {
    const int base = sl_ptr[s] + lane, L = sl_len[s];
    double acc = 0.0;
    int k = 0;
    for (; k + 4 <= L; k += 4) {
      int c[4];
      double a[4], g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = __ldcs(ci + base + 32 * (k + u));
        a[u] = __ldcs(v + base + 32 * (k + u));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) g[u] = __ldg(x + c[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = __dadd_rn(acc, __dmul_rn(a[u], g[u]));
    }
    for (; k < L; ++k)
      acc = __dadd_rn(acc, __dmul_rn(__ldcs(v + base + 32 * k), __ldg(x + __ldcs(ci + base + 32 * k))));
    const int r = row[32 * s + lane];
    if (r >= 0) y[r] = acc;
  }
}

// ---- tiled -------------------------------------------------------------------------------------
struct Tiled {
  int R, C, BW, M;
  std::vector<int> tile_sl0;  // first slice of tile t = r*C + c (size R*C+1)
  std::vector<int> tile_c0;   // first column of the block of tile t
  std::vector<int> tile_bw;   // block width of tile t
  std::vector<int> sl_ptr, sl_len, row;
  std::vector<uint16_t> ci;
  std::vector<double> v;
  std::vector<int> rg;  // row group bounds (R+1)
};

static bool g_skip_empty = true;
static Tiled build_tiled(const Csr& a, int R, int C) {
  Tiled t;
  t.R = R;
  t.C = C;
  t.M = a.M;
  t.BW = ((a.N + C - 1) / C + 1) & ~1;
  // balanced-nnz row groups
  t.rg.push_back(0);
  const long long tot = a.rp[a.M];
  for (int r = 1; r < R; ++r) {
    long long tgt = tot * r / R;
    int i = (int)(std::lower_bound(a.rp.begin(), a.rp.end(), (int)tgt) - a.rp.begin());
    t.rg.push_back(std::max(i, t.rg.back()));
  }
  t.rg.push_back(a.M);
  for (int r = 0; r < R; ++r) {
    const int r0 = t.rg[r], r1 = t.rg[r + 1];
    // per row, split points by block
    for (int c = 0; c < C; ++c) {
      const int c0 = c * t.BW, c1 = std::min(a.N, c0 + t.BW);
      std::vector<int> lo(r1 - r0), len(r1 - r0);
      for (int i = r0; i < r1; ++i) {
        auto b = a.ci.begin() + a.rp[i], e = a.ci.begin() + a.rp[i + 1];
        auto p = std::lower_bound(b, e, c0), q = std::lower_bound(b, e, c1);
        lo[i - r0] = (int)(p - a.ci.begin());
        len[i - r0] = (int)(q - p);
      }
      std::vector<int> ord;
      for (int i = 0; i < r1 - r0; ++i)
        if (len[i] > 0 || !g_skip_empty) ord.push_back(i);  // empty rows: P slot stays 0
      std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return len[x] > len[y]; });
      t.tile_sl0.push_back((int)t.sl_len.size());
      t.tile_c0.push_back(c0);
      t.tile_bw.push_back(c1 - c0);
      const int nr = (int)ord.size();
      for (int s0 = 0; s0 < nr; s0 += 32) {
        int L = 0;
        for (int l = 0; l < 32; ++l) {
          int k = s0 + l;
          int rr = k < nr ? ord[k] : -1;
          t.row.push_back(rr >= 0 ? rr + r0 : -1);
          if (rr >= 0) L = std::max(L, len[rr]);
        }
        t.sl_ptr.push_back((int)t.ci.size());
        t.sl_len.push_back(L);
        for (int k = 0; k < L; ++k)
          for (int l = 0; l < 32; ++l) {
            int kk = s0 + l;
            int rr = kk < nr ? ord[kk] : -1;
            bool ok = rr >= 0 && k < len[rr];
            t.ci.push_back(ok ? (uint16_t)(a.ci[lo[rr] + k] - c0) : 0);
            t.v.push_back(ok ? a.v[lo[rr] + k] : 0.0);
          }
      }
    }
  }
  t.tile_sl0.push_back((int)t.sl_len.size());
  return t;
}

__global__ void k_reduce(const double* __restrict__ P, double* __restrict__ y, int C, int M);
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int NT>
__global__ void __launch_bounds__(NT) k_tile(const int* __restrict__ tile_sl0,
                                             const int* __restrict__ tile_c0,
                                             const int* __restrict__ tile_bw,
                                             const int* __restrict__ sl_ptr,
                                             const int* __restrict__ sl_len,
                                             const int* __restrict__ row,
                                             const uint16_t* __restrict__ ci,
                                             const double* __restrict__ v,
                                             const double* __restrict__ x, double* __restrict__ P,
                                             int C, int M, int ntiles) {
  extern __shared__ __align__(128) double xs[];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned phase = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = tile_c0[t], bw = tile_bw[t];
    const int c = t % C;
    if (threadIdx.x == 0) {
      const unsigned bytes = unsigned(bw) * 8u;  // multiple of 16: bw even (asserted on host)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                   "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(xs)),
          "l"(x + c0), "r"(bytes), "r"(smem_u32(&bar))
          : "memory");
    }
    const int s0 = tile_sl0[t], s1 = tile_sl0[t + 1];
    // prefetch the first slice's metadata before waiting on the fill
    asm volatile(
        "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(&bar)),
        "r"(phase)
        : "memory");
    phase ^= 1;
    for (int s = s0 + wid; s < s1; s += NT / 32) {
      const int base = sl_ptr[s] + lane, L = sl_len[s];
      double acc = 0.0;
      int k = 0;
      for (; k + 4 <= L; k += 4) {
        int cc[4];
        double a[4], g[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cc[u] = __ldcs(ci + base + 32 * (k + u));
          a[u] = __ldcs(v + base + 32 * (k + u));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) g[u] = xs[cc[u]];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc = __dadd_rn(acc, __dmul_rn(a[u], g[u]));
      }
      for (; k < L; ++k)
        acc = __dadd_rn(acc, __dmul_rn(__ldcs(v + base + 32 * k), xs[__ldcs(ci + base + 32 * k)]));
      const int r = row[32 * s + lane];
      if (r >= 0) P[(size_t)c * M + r] = acc;
    }
    __syncthreads();  // xs reused by the next tile
  }
}

__global__ void k_reduce(const double* __restrict__ P, double* __restrict__ y, int C, int M) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < C; ++c) s = __dadd_rn(s, P[(size_t)c * M + i]);
    y[i] = s;
  }
}


// v2: the warp's slices are walked two at a time; up to 8 elements of each are
// loaded (predicated) before any gather, and the first pair is loaded before
// waiting on the x-block fill.
template <int NT>
__global__ void __launch_bounds__(NT) k_tile2(const int* __restrict__ tile_sl0,
                                              const int* __restrict__ tile_c0,
                                              const int* __restrict__ tile_bw,
                                              const int* __restrict__ sl_ptr,
                                              const int* __restrict__ sl_len,
                                              const int* __restrict__ row,
                                              const uint16_t* __restrict__ ci,
                                              const double* __restrict__ v,
                                              const double* __restrict__ x, double* __restrict__ P,
                                              int C, int M, int ntiles, int mode) {
  extern __shared__ __align__(128) double xs[];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned phase = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  constexpr int E = 6;
  const bool nofill = mode & 1, slot = mode & 2, nogather = mode & 4;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c0 = tile_c0[t], bw = tile_bw[t];
    const int c = t % C;
    if (threadIdx.x == 0 && !nofill) {
      const unsigned bytes = unsigned(bw) * 8u;
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                   "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(xs)),
          "l"(x + c0), "r"(bytes), "r"(smem_u32(&bar))
          : "memory");
    }
    const int s0 = tile_sl0[t], s1 = tile_sl0[t + 1];
    bool waited = false;
    for (int s = s0 + 2 * wid; s < s1; s += 2 * (NT / 32)) {
      const bool two = s + 1 < s1;
      const int b0 = sl_ptr[s] + lane, L0 = sl_len[s];
      const int b1 = two ? sl_ptr[s + 1] + lane : 0, L1 = two ? sl_len[s + 1] : 0;
      const int r0 = row[32 * s + lane], r1 = two ? row[32 * (s + 1) + lane] : -1;
      int c_a[E], c_b[E];
      double v_a[E], v_b[E];
#pragma unroll
      for (int u = 0; u < E; ++u) {
        c_a[u] = u < L0 ? __ldcs(ci + b0 + 32 * u) : 0;
        v_a[u] = u < L0 ? __ldcs(v + b0 + 32 * u) : 0.0;
        c_b[u] = u < L1 ? __ldcs(ci + b1 + 32 * u) : 0;
        v_b[u] = u < L1 ? __ldcs(v + b1 + 32 * u) : 0.0;
      }
      if (!waited && !nofill) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
            "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
            "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(&bar)),
            "r"(phase)
            : "memory");
        waited = true;
      }
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int u = 0; u < E; ++u) {
        if (u < L0) a0 = __dadd_rn(a0, __dmul_rn(v_a[u], nogather ? double(c_a[u]) : xs[c_a[u]]));
        if (u < L1) a1 = __dadd_rn(a1, __dmul_rn(v_b[u], nogather ? double(c_b[u]) : xs[c_b[u]]));
      }
      for (int k = E; k < L0; ++k)
        a0 = __dadd_rn(a0, __dmul_rn(__ldcs(v + b0 + 32 * k), xs[__ldcs(ci + b0 + 32 * k)]));
      for (int k = E; k < L1; ++k)
        a1 = __dadd_rn(a1, __dmul_rn(__ldcs(v + b1 + 32 * k), xs[__ldcs(ci + b1 + 32 * k)]));
      if (slot) {
        P[(size_t)c * M + ((32 * s + lane) % M)] = a0;
        P[(size_t)c * M + ((32 * s + 32 + lane) % M)] = a1;
      } else {
        if (r0 >= 0) P[(size_t)c * M + r0] = a0;
        if (r1 >= 0) P[(size_t)c * M + r1] = a1;
      }
    }
    if (!waited && !nofill)
      asm volatile(
          "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
          "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
          "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(&bar)),
          "r"(phase)
          : "memory");
    phase ^= 1;
    __syncthreads();  // xs reused by the next tile
  }
}

template <int C>
__global__ void k_reduceT(const double* __restrict__ P, double* __restrict__ y, int M) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    double p[C];
#pragma unroll
    for (int c = 0; c < C; ++c) p[c] = __ldcg(P + (size_t)c * M + i);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) s = __dadd_rn(s, p[c]);
    y[i] = s;
  }
}
static void reduce_launch(int sms, const double* P, double* y, int C, int M) {
  const int g = (M + 255) / 256;
  switch (C) {
    case 4: k_reduceT<4><<<g, 256>>>(P, y, M); break;
    case 8: k_reduceT<8><<<g, 256>>>(P, y, M); break;
    case 16: k_reduceT<16><<<g, 256>>>(P, y, M); break;
    default: k_reduce<<<sms * 4, 256>>>(P, y, C, M);
  }
}


// v3: each tile's stream is cut into chunks of whole slices (<= CH elements,
// <= MS slices) that the TMA engine copies into a 2-stage shared-memory ring
// (values, u16 columns, the slices' 32 row ids and a 16-byte descriptor per
// slice). Warps walk the staged slices; no global load sits on a warp's
// critical path.
constexpr int CH = 4096, MS = 128;
struct Chunks {
  std::vector<int> tile_q0;          // first chunk of tile t
  std::vector<int> q_sl0, q_e0;      // first slice / element of chunk q
  std::vector<int4> desc;            // per slice: {elem offset in chunk, L, 0, 0}
};
static Chunks build_chunks(const Tiled& t) {
  Chunks q;
  const int nt = (int)t.tile_sl0.size() - 1;
  for (int ti = 0; ti < nt; ++ti) {
    q.tile_q0.push_back((int)q.q_sl0.size());
    int s = t.tile_sl0[ti];
    while (s < t.tile_sl0[ti + 1]) {
      int e0 = t.sl_ptr[s], s1 = s;
      while (s1 < t.tile_sl0[ti + 1] && s1 - s < MS && t.sl_ptr[s1] + 32 * t.sl_len[s1] - e0 <= CH) ++s1;
      if (s1 == s) { printf("slice too long\n"); exit(1); }
      q.q_sl0.push_back(s);
      q.q_e0.push_back(e0);
      s = s1;
    }
  }
  q.tile_q0.push_back((int)q.q_sl0.size());
  q.q_sl0.push_back(t.tile_sl0[nt]);
  q.q_e0.push_back((int)t.ci.size());
  for (size_t s = 0; s < t.sl_len.size(); ++s) q.desc.push_back({0, t.sl_len[s], 0, 0});
  for (size_t c = 0; c + 1 < q.q_sl0.size(); ++c)
    for (int s = q.q_sl0[c]; s < q.q_sl0[c + 1]; ++s) q.desc[s].x = t.sl_ptr[s] - q.q_e0[c];
  return q;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(b)),
      "r"(ph)
      : "memory");
}

template <int NT>
__global__ void __launch_bounds__(NT) k_tile3(const int* __restrict__ tile_q0,
                                              const int* __restrict__ tile_c0,
                                              const int* __restrict__ tile_bw,
                                              const int* __restrict__ q_sl0,
                                              const int* __restrict__ q_e0,
                                              const int4* __restrict__ desc,
                                              const int* __restrict__ row,
                                              const uint16_t* __restrict__ ci,
                                              const double* __restrict__ v,
                                              const double* __restrict__ x, double* __restrict__ P,
                                              int C, int M, int ntiles, int BWmax, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* xs = reinterpret_cast<double*>(sm);
  constexpr int STG = CH * 8 + CH * 2 + MS * 128 + MS * 16;
  unsigned char* stg = sm + ((size_t(BWmax) * 8 + 127) / 128) * 128;
  __shared__ __align__(8) uint64_t bx, bf[2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool nogather = mode & 4;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bx)));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bf[0])));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bf[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned phx = 0, ph[2] = {0, 0};
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int q0 = tile_q0[t], q1 = tile_q0[t + 1];
    const int c = t % C;
    auto issue = [&](int q) {
      unsigned char* b = stg + (q - q0) % 2 * STG;
      const int sl0 = q_sl0[q], sl1 = q_sl0[q + 1];
      const int e0 = q_e0[q], cnt = q_e0[q + 1] - e0;  // multiple of 32
      const int nsl = sl1 - sl0;
      uint64_t* bar = &bf[(q - q0) % 2];
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"(unsigned(cnt * 10 + nsl * 144))
                   : "memory");
      bulk_g2s(b, v + e0, cnt * 8, bar);
      bulk_g2s(b + CH * 8, ci + e0, cnt * 2, bar);
      bulk_g2s(b + CH * 10, row + 32 * sl0, nsl * 128, bar);
      bulk_g2s(b + CH * 10 + MS * 128, desc + sl0, nsl * 16, bar);
    };
    if (threadIdx.x == 0) {
      if (!(mode & 1)) {
        const unsigned bytes = unsigned(tile_bw[t]) * 8u;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bx)), "r"(bytes)
                     : "memory");
        bulk_g2s(xs, x + tile_c0[t], bytes, &bx);
      }
      for (int q = q0; q < q1 && q < q0 + 2; ++q) issue(q);
    }
    if (!(mode & 1)) { mbar_wait(&bx, phx); phx ^= 1; }
    for (int q = q0; q < q1; ++q) {
      const int st = (q - q0) % 2;
      mbar_wait(&bf[st], ph[st]);
      ph[st] ^= 1;
      const unsigned char* b = stg + st * STG;
      const double* sv = reinterpret_cast<const double*>(b);
      const uint16_t* sc = reinterpret_cast<const uint16_t*>(b + CH * 8);
      const int* sr = reinterpret_cast<const int*>(b + CH * 10);
      const int4* sd = reinterpret_cast<const int4*>(b + CH * 10 + MS * 128);
      const int nsl = q_sl0[q + 1] - q_sl0[q];
      for (int s = wid; s < nsl; s += NT / 32) {
        const int4 d = sd[s];
        const int base = d.x + lane;
        double acc = 0.0;
        for (int k = 0; k < d.y; ++k) {
          const int cc = sc[base + 32 * k];
          acc = __dadd_rn(acc, __dmul_rn(sv[base + 32 * k], nogather ? double(cc) : xs[cc]));
        }
        const int r = sr[32 * s + lane];
        if (r >= 0) P[(size_t)c * M + r] = acc;
      }
      __syncthreads();
      if (threadIdx.x == 0 && q + 2 < q1) issue(q + 2);
    }
    __syncthreads();
  }
}


// v4: flat per-warp streams. The tile's slices are cut into 32 contiguous
// per-warp ranges (<= MJ slices each, balanced by elements). A warp streams
// its element range in batches of U independent (col, val) loads that do not
// depend on any metadata; slice ends (held one per lane, read by shfl) tell
// every lane at once when to store its row partial. The tile's row ids are
// staged in shared memory as u16 offsets inside the row group.
constexpr int MJ = 8, U4 = 8;
struct WarpSched {
  std::vector<int> w_sl0;  // per tile, 33 entries (slice bounds of the 32 warps)
  std::vector<uint16_t> lrow;  // per slice 32 local rows (0xFFFF pad)
  std::vector<int> tile_r0;
};
static bool build_wsched(const Tiled& t, WarpSched& w) {
  const int nt = (int)t.tile_sl0.size() - 1;
  w.lrow.resize(t.row.size());
  for (int ti = 0; ti < nt; ++ti) {
    const int r = ti / t.C;
    const int r0 = t.rg[r];
    w.tile_r0.push_back(r0);
    const int s0 = t.tile_sl0[ti], s1 = t.tile_sl0[ti + 1];
    for (int s = s0; s < s1; ++s)
      for (int l = 0; l < 32; ++l) {
        int rr = t.row[32 * s + l];
        if (rr >= 0 && rr - r0 >= 65535) return false;
        w.lrow[32 * s + l] = rr < 0 ? 0xFFFF : (uint16_t)(rr - r0);
      }
    const long long tot = t.sl_ptr[s1 - 1] + 32ll * t.sl_len[s1 - 1] - t.sl_ptr[s0];
    int s = s0;
    for (int wi = 0; wi < 32; ++wi) {
      w.w_sl0.push_back(s);
      const long long tgt = tot * (wi + 1) / 32;
      int cnt = 0;
      while (s < s1 && cnt < MJ && (t.sl_ptr[s] - t.sl_ptr[s0] < tgt || s1 - s > MJ * (31 - wi))) { ++s; ++cnt; }
    }
    if (s != s1) return false;
    w.w_sl0.push_back(s1);
  }
  return true;
}

__global__ void __launch_bounds__(1024, 1) k_tile4(const int* __restrict__ w_sl0,
                                                  const int* __restrict__ tile_c0,
                                                  const int* __restrict__ tile_bw,
                                                  const int* __restrict__ tile_r0,
                                                  const int* __restrict__ sl_ptr,
                                                  const int* __restrict__ sl_len,
                                                  const uint16_t* __restrict__ lrow,
                                                  const uint16_t* __restrict__ ci,
                                                  const double* __restrict__ v,
                                                  const double* __restrict__ x, double* __restrict__ P,
                                                  int C, int M, int ntiles, int BWmax, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* xs = reinterpret_cast<double*>(sm);
  uint16_t* srow = reinterpret_cast<uint16_t*>(sm + size_t(BWmax) * 8);  // 32 warps x MJ x 32
  __shared__ __align__(8) uint64_t bx;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool nogather = mode & 4;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bx)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned phx = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int c = t % C;
    if (threadIdx.x == 0 && !(mode & 1)) {
      const unsigned bytes = unsigned(tile_bw[t]) * 8u;
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bx)), "r"(bytes)
                   : "memory");
      bulk_g2s(xs, x + tile_c0[t], bytes, &bx);
    }
    const int sa = w_sl0[33 * t + wid], sb = w_sl0[33 * t + wid + 1];
    const int nsl = sb - sa;
    const int e_beg = nsl > 0 ? sl_ptr[sa] : 0;
    const int my_end = lane < nsl ? sl_ptr[sa + lane] + 32 * sl_len[sa + lane] : 0x7fffffff;
    const int e_end = nsl > 0 ? __shfl_sync(~0u, my_end, nsl - 1) : 0;
    uint16_t* wr = srow + wid * MJ * 32;
#pragma unroll
    for (int j = 0; j < MJ; ++j)
      if (j < nsl) wr[32 * j + lane] = lrow[32 * (sa + j) + lane];
    __syncwarp();
    const size_t pbase = (size_t)c * M + tile_r0[t];
    int j = 0, endj = __shfl_sync(~0u, my_end, 0);
    double acc = 0.0;
    bool waited = (mode & 1);
    // zero-length slices at the start
    while (j < nsl && endj <= e_beg) {
      const int r = wr[32 * j + lane];
      if (r != 0xFFFF) P[pbase + r] = acc;
      ++j;
      endj = __shfl_sync(~0u, my_end, j < 32 ? j : 31);
    }
    for (int e = e_beg; e < e_end; e += 32 * U4) {
      int cc[U4];
      double vv[U4];
#pragma unroll
      for (int u = 0; u < U4; ++u) {
        const bool in = e + 32 * u < e_end;
        cc[u] = in ? __ldcs(ci + e + 32 * u + lane) : 0;
        vv[u] = in ? __ldcs(v + e + 32 * u + lane) : 0.0;
      }
      if (!waited) {
        mbar_wait(&bx, phx);
        waited = true;
      }
#pragma unroll
      for (int u = 0; u < U4; ++u) {
        const int p = e + 32 * u;
        if (p < e_end) {
          while (p >= endj) {
            const int r = wr[32 * j + lane];
            if (r != 0xFFFF) P[pbase + r] = acc;
            acc = 0.0;
            ++j;
            endj = __shfl_sync(~0u, my_end, j < 32 ? j : 31);
          }
          acc = __dadd_rn(acc, __dmul_rn(vv[u], nogather ? double(cc[u]) : xs[cc[u]]));
        }
      }
    }
    while (j < nsl) {
      const int r = wr[32 * j + lane];
      if (r != 0xFFFF) P[pbase + r] = acc;
      acc = 0.0;
      ++j;
    }
    if (!waited) { mbar_wait(&bx, phx); }
    phx ^= (mode & 1) ? 0 : 1;
    __syncthreads();
  }
}


// v5: persistent emulation. Each CTA owns one tile for the whole launch (as a
// persistent solver grid would): its schedule (per-warp element ranges, slice
// ends, the tile's u16 row ids in shared memory) is loaded once, then NREP
// SpMVs run back to back, each on another copy of the (col, val) stream so
// the stream comes from DRAM. 512 threads, 2 CTAs per SM.
constexpr int NW5 = 16, MJ5 = 16;
static bool build_wsched5(const Tiled& t, WarpSched& w) {
  const int nt = (int)t.tile_sl0.size() - 1;
  w.lrow.resize(t.row.size());
  for (int ti = 0; ti < nt; ++ti) {
    const int r0 = t.rg[ti / t.C];
    w.tile_r0.push_back(r0);
    const int s0 = t.tile_sl0[ti], s1 = t.tile_sl0[ti + 1];
    for (int s = s0; s < s1; ++s)
      for (int l = 0; l < 32; ++l) {
        int rr = t.row[32 * s + l];
        if (rr >= 0 && rr - r0 >= 65535) return false;
        w.lrow[32 * s + l] = rr < 0 ? 0xFFFF : (uint16_t)(rr - r0);
      }
    const long long tot = s1 > s0 ? t.sl_ptr[s1 - 1] + 32ll * t.sl_len[s1 - 1] - t.sl_ptr[s0] : 0;
    int s = s0;
    for (int wi = 0; wi < NW5; ++wi) {
      w.w_sl0.push_back(s);
      const long long tgt = tot * (wi + 1) / NW5;
      int cnt = 0;
      while (s < s1 && cnt < MJ5 && (t.sl_ptr[s] - t.sl_ptr[s0] < tgt || s1 - s > MJ5 * (NW5 - 1 - wi))) { ++s; ++cnt; }
    }
    if (s != s1) return false;
    w.w_sl0.push_back(s1);
  }
  return true;
}

template <int U>
__global__ void __launch_bounds__(512, 2) k_tile5(const int* __restrict__ w_sl0,
                                                 const int* __restrict__ tile_c0,
                                                 const int* __restrict__ tile_bw,
                                                 const int* __restrict__ tile_r0,
                                                 const int* __restrict__ sl_ptr,
                                                 const int* __restrict__ sl_len,
                                                 const uint16_t* __restrict__ lrow,
                                                 const uint16_t* const* __restrict__ cis,
                                                 const double* const* __restrict__ vs, int ncopies,
                                                 const double* __restrict__ x, double* __restrict__ P,
                                                 int C, int M, int BWmax, int nrep, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* xs = reinterpret_cast<double*>(sm);
  uint16_t* srow = reinterpret_cast<uint16_t*>(sm + size_t(BWmax) * 8);
  __shared__ __align__(8) uint64_t bx;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool nogather = mode & 4;
  const int t = blockIdx.x;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bx)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int c = t % C;
  const int sa = w_sl0[(NW5 + 1) * t + wid], sb = w_sl0[(NW5 + 1) * t + wid + 1];
  const int nsl = sb - sa;
  const int e_beg = nsl > 0 ? sl_ptr[sa] : 0;
  const int my_end = lane < nsl ? sl_ptr[sa + lane] + 32 * sl_len[sa + lane] : 0x7fffffff;
  const int e_end = nsl > 0 ? __shfl_sync(~0u, my_end, nsl - 1) : 0;
  uint16_t* wr = srow + wid * MJ5 * 32;
  for (int j = 0; j < nsl; ++j) wr[32 * j + lane] = lrow[32 * (sa + j) + lane];
  const size_t pbase = (size_t)c * M + tile_r0[t];
  const double* xsrc = x + tile_c0[t];
  const unsigned xbytes = unsigned(tile_bw[t]) * 8u;
  __syncthreads();
  unsigned phx = 0;
  for (int rep = 0; rep < nrep; ++rep) {
    const uint16_t* __restrict__ ci = cis[rep % ncopies];
    const double* __restrict__ v = vs[rep % ncopies];
    if (threadIdx.x == 0 && !(mode & 1)) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bx)), "r"(xbytes)
                   : "memory");
      bulk_g2s(xs, xsrc, xbytes, &bx);
    }
    int j = 0, endj = __shfl_sync(~0u, my_end, 0);
    double acc = 0.0;
    bool waited = (mode & 1);
    for (int e = e_beg; e < e_end; e += 32 * U) {
      int cc[U];
      double vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool in = e + 32 * u < e_end;
        cc[u] = in ? __ldcs(ci + e + 32 * u + lane) : 0;
        vv[u] = in ? __ldcs(v + e + 32 * u + lane) : 0.0;
      }
      if (!waited) {
        mbar_wait(&bx, phx);
        waited = true;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = e + 32 * u;
        if (p < e_end) {
          while (p >= endj) {
            const int r = wr[32 * j + lane];
            if (r != 0xFFFF) P[pbase + r] = acc;
            acc = 0.0;
            ++j;
            endj = __shfl_sync(~0u, my_end, j < 32 ? j : 31);
          }
          acc = __dadd_rn(acc, __dmul_rn(vv[u], nogather ? double(cc[u]) : xs[cc[u]]));
        }
      }
    }
    while (j < nsl) {
      const int r = wr[32 * j + lane];
      if (r != 0xFFFF) P[pbase + r] = acc;
      acc = 0.0;
      ++j;
    }
    if (!waited) mbar_wait(&bx, phx);
    if (!(mode & 1)) phx ^= 1;
    __syncthreads();
  }
}

// persistent-style baseline: the global SELL-32 on rotating stream copies
__global__ void __launch_bounds__(256) k_gsell_rep(const int* __restrict__ sl_ptr,
                                                   const int* __restrict__ sl_len,
                                                   const int* __restrict__ row,
                                                   const int* const* __restrict__ cis,
                                                   const double* const* __restrict__ vs, int ncopies,
                                                   const double* __restrict__ x, double* __restrict__ y,
                                                   int ns, int nrep) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int rep = 0; rep < nrep; ++rep) {
    const int* __restrict__ ci = cis[rep % ncopies];
    const double* __restrict__ v = vs[rep % ncopies];
    for (int s = warp; s < ns; s += nw) {
      const int base = sl_ptr[s] + lane, L = sl_len[s];
      double acc = 0.0;
      int k = 0;
      for (; k + 8 <= L; k += 8) {
        int c[8];
        double a[8], g[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          c[u] = __ldcs(ci + base + 32 * (k + u));
          a[u] = __ldcs(v + base + 32 * (k + u));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) g[u] = __ldg(x + c[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(a[u], g[u]));
      }
      for (; k < L; ++k)
        acc = __dadd_rn(acc, __dmul_rn(__ldcs(v + base + 32 * k), __ldg(x + __ldcs(ci + base + 32 * k))));
      const int r = row[32 * s + lane];
      if (r >= 0) y[r] = acc;
    }
  }
}

__global__ void k_empty() {}
__global__ void k_readsum(const double* __restrict__ a, size_t n, double* out) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    s += __ldcs(a + i);
  if (s == 1234.5) out[0] = s;
}
__global__ void k_flush(double* b, size_t n) {
  double s = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    s += __ldcg(b + i);
  if (s == 1234.5) b[0] = s;  // read-only flush: no dirty lines left in L2
}

template <class T>
static T* up(const std::vector<T>& h) {
  T* d;
  CK(cudaMalloc(&d, sizeof(T) * std::max<size_t>(1, h.size())));
  CK(cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  return d;
}

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const Csr K = planted(100000, 200000, 20, 2508080621ull);
  const Csr Kt = transpose(K);
  const size_t FL = 64ull << 20;  // 512 MB flush buffer
  double* flush;
  CK(cudaMalloc(&flush, FL * 8));
  CK(cudaMemset(flush, 0, FL * 8));
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  for (int which = 0; which < 2; ++which) {
    const Csr& A = which == 0 ? K : Kt;
    const char* nm = which == 0 ? "K  (K2: 100k x 200k)" : "K' (K1: 200k x 100k)";
    std::vector<double> hx(A.N);
    std::mt19937_64 g(5);
    std::normal_distribution<double> nd;
    for (auto& z : hx) z = nd(g);
    std::vector<double> yref(A.M);
    for (int i = 0; i < A.M; ++i) {
      double s = 0;
      for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) s += A.v[k] * hx[A.ci[k]];
      yref[i] = s;
    }
    double* dx = up(hx);
    double* dy;
    CK(cudaMalloc(&dy, 8 * A.M));
    auto check = [&](const char* what) {
      std::vector<double> hy(A.M);
      CK(cudaMemcpy(hy.data(), dy, 8 * A.M, cudaMemcpyDeviceToHost));
      double err = 0, nrm = 0;
      for (int i = 0; i < A.M; ++i) {
        err = std::max(err, std::abs(hy[i] - yref[i]));
        nrm = std::max(nrm, std::abs(yref[i]));
      }
      if (err > 1e-12 * nrm) printf("  !! %s mismatch: max err %.3e (|y| %.3e)\n", what, err, nrm);
    };
    auto timed = [&](auto launchA, auto launchB, float* ta, float* tb) {
      float sa = 0, sb = 0;
      const int reps = 20;
      for (int r = 0; r < reps + 2; ++r) {
        k_flush<<<sms * 4, 512>>>(flush, FL);
        // warm the gathered vector into L2 (the solver's producer just wrote it)
        CK(cudaMemcpyAsync(dy, dy, 8, cudaMemcpyDeviceToDevice));
        cudaEventRecord(e0);
        launchA();
        cudaEventRecord(e1);
        launchB();
        cudaEventRecord(e2);
        CK(cudaEventSynchronize(e2));
        float a, b;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        if (r >= 2) {
          sa += a;
          sb += b;
        }
      }
      *ta = 1000 * sa / reps;
      *tb = 1000 * sb / reps;
    };

    const int NREP = 40, NCOPY = 4;
    auto timed_rep = [&](auto launch) {
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float a;
      cudaEventElapsedTime(&a, e0, e1);
      return 1000.f * a / NREP;
    };
    {
      GSell s = build_gsell(A);
      int *sp = up(s.sl_ptr), *sl = up(s.sl_len), *rw = up(s.row);
      std::vector<int*> hc;
      std::vector<double*> hv;
      for (int k = 0; k < NCOPY; ++k) { hc.push_back(up(s.ci)); hv.push_back(up(s.v)); }
      int** dc = up(hc);
      double** dv = up(hv);
      const int ns = (int)s.sl_len.size();
      for (int cps : {4, 6, 8}) {
        float us = timed_rep([&] { k_gsell_rep<<<sms * cps, 256>>>(sp, sl, rw, dc, dv, NCOPY, dx, dy, ns, NREP); });
        check("gsell_rep");
        printf("%s  [persistent x%d] global SELL-32 unroll 8 (%d CTAs/SM)   %7.2f us/SpMV\n", nm, NREP, cps, us);
      }
      for (int k = 0; k < NCOPY; ++k) { cudaFree(hc[k]); cudaFree(hv[k]); }
      cudaFree(sp); cudaFree(sl); cudaFree(rw); cudaFree(dc); cudaFree(dv);
    }
    std::vector<std::pair<int, int>> rc5 = which == 0
        ? std::vector<std::pair<int, int>>{{18, 16}, {9, 32}, {16, 18}, {12, 24}, {8, 37}, {4, 74}}
        : std::vector<std::pair<int, int>>{{37, 8}, {36, 8}, {18, 16}, {24, 12}, {74, 4}};
    for (auto [R, C] : rc5) {
      Tiled t = build_tiled(A, R, C);
      WarpSched w;
      if (!build_wsched5(t, w)) { printf("%s  v5 schedule does not fit R=%d C=%d\n", nm, R, C); continue; }
      const int ntiles = R * C;
      const size_t sm5 = size_t(t.BW) * 8 + NW5 * MJ5 * 32 * 2;
      if (sm5 > 227 * 1024) continue;
      int *ws = up(w.w_sl0), *tr = up(w.tile_r0), *tc = up(t.tile_c0), *tw = up(t.tile_bw),
          *sp = up(t.sl_ptr), *sl = up(t.sl_len);
      uint16_t* lr = up(w.lrow);
      std::vector<uint16_t*> hc;
      std::vector<double*> hv;
      for (int k = 0; k < NCOPY; ++k) { hc.push_back(up(t.ci)); hv.push_back(up(t.v)); }
      uint16_t** dc = up(hc);
      double** dv = up(hv);
      double* P;
      CK(cudaMalloc(&P, 8ull * C * A.M));
      CK(cudaMemset(P, 0, 8ull * C * A.M));
      for (int U : {4, 8}) {
        auto kern = U == 4 ? k_tile5<4> : k_tile5<8>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm5));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, sm5));
        if (occ * sms < ntiles) { printf("%s  v5 R=%d C=%d: %d tiles > %d resident\n", nm, R, C, ntiles, occ * sms); continue; }
        for (int mode : {0, 5}) {
          float us = timed_rep([&] {
            kern<<<ntiles, 512, sm5>>>(ws, tc, tw, tr, sp, sl, lr, dc, dv, NCOPY, dx, P, C, A.M, t.BW, NREP, mode);
          });
          float ta, tb;
          if (mode == 0) {
            timed([] {}, [&] { reduce_launch(sms, P, dy, C, A.M); }, &ta, &tb);
            check("tiled5");
          }
          printf("%s  [persistent x%d] tiled v5 U=%d %s R=%3d C=%2d (%3d KB smem, occ %d, %d tiles)  %7.2f us/SpMV (+ reduce pass, %.1f MB partials)\n",
                 nm, NREP, U, mode ? "stream only" : "full       ", R, C, (int)(sm5 / 1024), occ, ntiles, us,
                 2.0 * 8 * C * A.M / 1e6);
        }
      }
      for (int k = 0; k < NCOPY; ++k) { cudaFree(hc[k]); cudaFree(hv[k]); }
      cudaFree(ws); cudaFree(tr); cudaFree(tc); cudaFree(tw); cudaFree(sp); cudaFree(sl); cudaFree(lr);
      cudaFree(dc); cudaFree(dv); cudaFree(P);
    }
    cudaFree(dx);
    cudaFree(dy);
    continue;
    {
      float ta, tb;
      timed([&] { k_empty<<<1, 32>>>(); }, [&] { k_empty<<<1, 32>>>(); }, &ta, &tb);
      printf("harness: empty kernel %.2f us, second empty %.2f us\n", ta, tb);
      timed([&] { k_readsum<<<sms * 8, 256>>>(flush + (FL - (5ull << 20)), 5ull << 20, dy); }, [&] { k_empty<<<1, 32>>>(); }, &ta, &tb);
      printf("harness: coalesced read of 40 MB %.2f us (%.0f GB/s)\n", ta, 40.0 * 1.048576e6 / ta / 1e3);
      timed([&] { k_readsum<<<sms * 8, 256>>>(flush + (FL - (20ull << 20)), 20ull << 20, dy); }, [&] { k_empty<<<1, 32>>>(); }, &ta, &tb);
      printf("harness: coalesced read of 160 MB %.2f us (%.0f GB/s)\n", ta, 160.0 * 1.048576e6 / ta / 1e3);
    }
    {
      GSell s = build_gsell(A);
      int *sp = up(s.sl_ptr), *sl = up(s.sl_len), *rw = up(s.row), *ci = up(s.ci);
      double* v = up(s.v);
      const int ns = (int)s.sl_len.size();
      float ta, tb;
      for (int cps : {6, 8}) {
        timed([&] { k_gsell<<<sms * cps, 256>>>(sp, sl, rw, ci, v, dx, dy, ns); }, [] {}, &ta, &tb);
        check("gsell");
        printf("%s  global SELL-32 (%d CTAs/SM)             %7.2f us  stream %.1f MB\n", nm, cps, ta,
               (s.ci.size() * 12.0) / 1e6);
      }
      cudaFree(sp); cudaFree(sl); cudaFree(rw); cudaFree(ci); cudaFree(v);
    }
    std::vector<std::pair<int, int>> rcs = which == 0
        ? std::vector<std::pair<int, int>>{{18, 16}, {24, 16}, {37, 16}, {18, 17}, {24, 17}, {37, 17}, {37, 32}}
        : std::vector<std::pair<int, int>>{{18, 8}, {24, 8}, {37, 8}, {18, 9}, {37, 9}, {37, 16}};
    for (auto [R, C] : rcs) {
      Tiled t = build_tiled(A, R, C);
      if (t.BW % 2) continue;
      if (t.BW > 65536) continue;
      int *ts = up(t.tile_sl0), *tc = up(t.tile_c0), *tw = up(t.tile_bw), *sp = up(t.sl_ptr),
          *sl = up(t.sl_len), *rw = up(t.row);
      uint16_t* ci = up(t.ci);
      double* v = up(t.v);
      double* P;
      CK(cudaMalloc(&P, 8ull * C * A.M));
      CK(cudaMemset(P, 0, 8ull * C * A.M));
      const int ntiles = R * C;
      const size_t smem = 8ull * t.BW;
      if (smem > 227 * 1024) continue;
      CK(cudaFuncSetAttribute(k_tile<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaFuncSetAttribute(k_tile<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int occ1024 = 0, occ512 = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1024, k_tile<1024>, 1024, smem));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ512, k_tile<512>, 512, smem));
      float ta, tb;
      CK(cudaFuncSetAttribute(k_tile2<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CK(cudaFuncSetAttribute(k_tile2<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      {
        Chunks q = build_chunks(t);
        int *tq = up(q.tile_q0), *qs = up(q.q_sl0), *qe = up(q.q_e0);
        int4* dd = up(q.desc);
        const int STG = CH * 8 + CH * 2 + MS * 128 + MS * 16;
        const size_t sm3 = ((size_t(t.BW) * 8 + 127) / 128) * 128 + 2 * STG;
        if (sm3 <= 227 * 1024) {
          CK(cudaFuncSetAttribute(k_tile3<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3));
          CK(cudaFuncSetAttribute(k_tile3<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3));
          for (int nt : {1024}) {
            int occ3 = 0;
            if (nt == 1024) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_tile3<1024>, 1024, sm3));
            else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_tile3<512>, 512, sm3));
            const int grid = std::min(ntiles, sms * occ3);
            for (int mode : {0, 5}) {
              timed([&] {
                if (nt == 1024) k_tile3<1024><<<grid, 1024, sm3>>>(tq, tc, tw, qs, qe, dd, rw, ci, v, dx, P, C, A.M, ntiles, t.BW, mode);
                else k_tile3<512><<<grid, 512, sm3>>>(tq, tc, tw, qs, qe, dd, rw, ci, v, dx, P, C, A.M, ntiles, t.BW, mode);
              }, [&] { reduce_launch(sms, P, dy, C, A.M); }, &ta, &tb);
              if (mode == 0) check("tiled3");
              printf("%s  tiled v3 %s R=%3d C=%2d (%3d KB smem, %d thr, occ %d, grid %d, %d chunks)  tile %7.2f us + reduce %6.2f us = %7.2f us\n",
                     nm, mode ? "stream only" : "full       ", R, C, (int)(sm3 / 1024), nt, occ3, grid,
                     (int)q.q_e0.size() - 1, ta, tb, ta + tb);
            }
          }
        }
        cudaFree(tq); cudaFree(qs); cudaFree(qe); cudaFree(dd);
      }
      {
        WarpSched w;
        if (build_wsched(t, w)) {
          int *ws = up(w.w_sl0), *tr = up(w.tile_r0);
          uint16_t* lr = up(w.lrow);
          const size_t sm4 = size_t(t.BW) * 8 + 32 * MJ * 32 * 2;
          if (sm4 <= 227 * 1024) {
            CK(cudaFuncSetAttribute(k_tile4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4));
            int occ4 = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, k_tile4, 1024, sm4));
            const int grid = std::min(ntiles, sms * occ4);
            for (int mode : {0, 5}) {
              timed([&] {
                k_tile4<<<grid, 1024, sm4>>>(ws, tc, tw, tr, sp, sl, lr, ci, v, dx, P, C, A.M, ntiles, t.BW, mode);
              }, [&] { reduce_launch(sms, P, dy, C, A.M); }, &ta, &tb);
              if (mode == 0) check("tiled4");
              printf("%s  tiled v4 %s R=%3d C=%2d (%3d KB smem, occ %d, grid %d)  tile %7.2f us + reduce %6.2f us = %7.2f us   [harness-corrected: %6.2f]\n",
                     nm, mode ? "stream only" : "full       ", R, C, (int)(sm4 / 1024), occ4, grid, ta, tb, ta + tb, ta + tb - 12.0);
            }
          }
          cudaFree(ws); cudaFree(tr); cudaFree(lr);
        } else {
          printf("%s  v4 schedule does not fit R=%d C=%d\n", nm, R, C);
        }
      }
      for (int variant = 1; variant < 9; variant += 7) {
        const int nt = 1024;
        const int mode = variant - 1;
        const int occ = nt == 1024 ? occ1024 : occ512;
        const int grid = std::min(ntiles, sms * occ);
        timed(
            [&] {
              if (variant == 0)
                k_tile<1024><<<grid, 1024, smem>>>(ts, tc, tw, sp, sl, rw, ci, v, dx, P, C, A.M, ntiles);
              else
                k_tile2<1024><<<grid, 1024, smem>>>(ts, tc, tw, sp, sl, rw, ci, v, dx, P, C, A.M, ntiles, mode);
            },
            [&] { reduce_launch(sms, P, dy, C, A.M); }, &ta, &tb);
        if (mode == 0) check("tiled");
        printf("%s  tiled%s R=%3d C=%2d BW=%6d (%2d KB smem, %d thr, occ %d, grid %d)  tile %7.2f us + reduce %6.2f us = %7.2f us  stream %.1f MB  pad %.2f\n",
               nm, mode == 0 ? "v2 full     " : mode == 1 ? "v2 nofill   " : mode == 2 ? "v2 slotstore" : mode == 3 ? "v2 nofill+slot" : mode==4 ? "v2 nogather " : mode==5 ? "v2 nofill+nogather": mode==6?"v2 nogath+slot":"v2 stream only", R, C, t.BW, (int)(smem / 1024), nt, occ, grid, ta, tb, ta + tb,
               t.ci.size() * 10.0 / 1e6, double(t.ci.size()) / A.ci.size());
      }
      cudaFree(ts); cudaFree(tc); cudaFree(tw); cudaFree(sp); cudaFree(sl); cudaFree(rw);
      cudaFree(ci); cudaFree(v); cudaFree(P);
    }
    cudaFree(dx);
    cudaFree(dy);
  }
  return 0;
}
