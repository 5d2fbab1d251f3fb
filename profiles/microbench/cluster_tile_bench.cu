// cluster_tile_bench.cu — microbenchmark (not product code): x-stationary
// tiled SpMV for the configs[1] shapes with the row partials reduced inside
// a thread-block cluster through distributed shared memory, so a SpMV phase
// needs no extra grid barrier and no global partial vector.
//
// Rows are cut into G groups (one cluster each), columns into C*S blocks.
// The CTA of cluster rank c walks blocks c*S .. c*S+S-1: it copies the x
// block into shared memory, streams the tile's entries (u32 = row_local<<16
// | col_local, f64 value; CSR order, perfectly coalesced, no padding) one
// entry per lane, gathers from shared memory and adds the products of each
// row with a segmented warp scan (rows are sorted; each warp's range is cut
// at row boundaries, so every row's partial has one writer). After a cluster
// barrier CTA c sums rows [c*R/C, (c+1)*R/C) of the group over the C CTAs'
// partials (DSMEM, fixed rank order) and writes y. Persistent: P phases,
// alternating y = K' x and x = K y, separated by a grid barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o cluster_tile_bench cluster_tile_bench.cu
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); exit(1); } \
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
    for (int r : pick) rows[r].push_back({j, nd(g) / 30.0});
  }
  Csr a;
  a.M = m;
  a.N = n;
  a.rp.assign(m + 1, 0);
  for (int i = 0; i < m; ++i) {
    std::sort(rows[i].begin(), rows[i].end());
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

// ---- cluster-tiled layout ---------------------------------------------------------------
struct Layout {
  int M, N, G, C, S, W;  // W warps per CTA
  int bw;                // block width (columns)
  int rows_max;          // max rows per group
  std::vector<int> grp;  // G+1 row bounds
  // tile t = (g*C + c)*S + s: warp w's entry range [woff[t*(W+1)+w], woff[t*(W+1)+w+1])
  std::vector<int64_t> woff;
  std::vector<uint32_t> rc;
  std::vector<double> v;
};

static Layout build(const Csr& a, int G, int C, int S, int W) {
  Layout L;
  L.M = a.M;
  L.N = a.N;
  L.G = G;
  L.C = C;
  L.S = S;
  L.W = W;
  const int nb = C * S;
  L.bw = ((a.N + nb - 1) / nb + 1) & ~1;
  L.grp.resize(G + 1);
  for (int g = 0; g <= G; ++g) L.grp[g] = int((int64_t)a.M * g / G);
  L.rows_max = 0;
  for (int g = 0; g < G; ++g) L.rows_max = std::max(L.rows_max, L.grp[g + 1] - L.grp[g]);
  if (L.rows_max > 65535 || L.bw > 65535) { printf("layout does not fit u16\n"); exit(1); }
  for (int g = 0; g < G; ++g) {
    const int r0 = L.grp[g], r1 = L.grp[g + 1];
    for (int b = 0; b < nb; ++b) {
      const int c0 = b * L.bw, c1 = std::min(a.N, c0 + L.bw);
      // entries of the tile in CSR order, with the row start offsets
      std::vector<int> rstart;  // index (in tile) of each row's first entry, rows with entries
      const int64_t t0 = (int64_t)L.rc.size();
      for (int i = r0; i < r1; ++i) {
        auto bb = a.ci.begin() + a.rp[i], ee = a.ci.begin() + a.rp[i + 1];
        auto p = std::lower_bound(bb, ee, c0), q = std::lower_bound(bb, ee, c1);
        if (p != q) rstart.push_back(int((int64_t)L.rc.size() - t0));
        for (auto it = p; it != q; ++it) {
          const int k = int(it - a.ci.begin());
          L.rc.push_back((uint32_t(i - r0) << 16) | uint32_t(a.ci[k] - c0));
          L.v.push_back(a.v[k]);
        }
      }
      const int64_t E = (int64_t)L.rc.size() - t0;
      // warp ranges: cut at the row start nearest w*E/W
      for (int w = 0; w <= W; ++w) {
        int64_t cut;
        if (w == 0) cut = 0;
        else if (w == W) cut = E;
        else {
          const int64_t tgt = E * w / W;
          auto it = std::lower_bound(rstart.begin(), rstart.end(), (int)tgt);
          cut = it == rstart.end() ? E : *it;
        }
        L.woff.push_back(t0 + cut);
      }
    }
  }
  return L;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void grid_bar(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
    }
  }
  __syncthreads();
}

struct Dev {
  const int64_t* woff;
  const uint32_t* rc;
  const double* v;
  int bw, rows_max, G, C, S, W, M, N;
  const int* grp;
};

// one SpMV phase of one CTA: y[group rows] = A x
template <int U>
__device__ void tile_phase(const Dev& d, const double* __restrict__ x, double* __restrict__ y,
                           double* xs, double* part, cg::cluster_group& cl, int mode) {
  const int g = blockIdx.x / d.C, c = blockIdx.x % d.C;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = d.grp[g], nrows = d.grp[g + 1] - r0;
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) part[i] = 0.0;
  for (int s = 0; s < d.S; ++s) {
    const int b = c * d.S + s;
    const int c0 = b * d.bw, c1 = min(d.N, c0 + d.bw);
    // fill the x block (L2-resident, written by the previous phase)
    if (!(mode & 1)) {
      const double2* src = reinterpret_cast<const double2*>(x + c0);
      double2* dst = reinterpret_cast<double2*>(xs);
      const int n2 = (c1 - c0) >> 1;
      for (int i = threadIdx.x; i < n2; i += blockDim.x) dst[i] = __ldcg(src + i);
      if (((c1 - c0) & 1) && threadIdx.x == 0) xs[c1 - c0 - 1] = __ldcg(x + c1 - 1);
    }
    __syncthreads();
    const int t = (g * d.C + c) * d.S + s;
    const int64_t e0 = d.woff[(int64_t)t * (d.W + 1) + w], e1 = d.woff[(int64_t)t * (d.W + 1) + w + 1];
    int crow = -1;
    double carry = 0.0;
    for (int64_t base = e0; base < e1; base += 32 * U) {
      uint32_t q[U];
      double a[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = base + 32 * u + lane;
        q[u] = e < e1 ? __ldcs(d.rc + e) : 0xffffffffu;
        a[u] = e < e1 ? __ldcs(d.v + e) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (base + 32 * u >= e1) break;
        const int row = int(q[u] >> 16);
        double p = q[u] == 0xffffffffu ? 0.0 : __dmul_rn(a[u], (mode & 2) ? 1.0 : xs[q[u] & 0xffff]);
        // segmented inclusive scan (rows ascending inside the warp's range)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double pv = __shfl_up_sync(0xffffffffu, p, o);
          const int rv = __shfl_up_sync(0xffffffffu, row, o);
          if (lane >= o && rv == row) p = __dadd_rn(p, pv);
        }
        if (row == crow) p = __dadd_rn(carry, p);
        // the previous chunk's last row ended with that chunk: flush it
        const int row0 = __shfl_sync(0xffffffffu, row, 0);
        if (lane == 0 && crow >= 0 && crow != 0xffff && row0 != crow)
          part[crow] = __dadd_rn(part[crow], carry);
        const int nrow = __shfl_down_sync(0xffffffffu, row, 1);
        const bool tail = lane == 31 || nrow != row;
        // the chunk's last segment may continue in the next chunk
        const double lastp = __shfl_sync(0xffffffffu, p, 31);
        const int lastrow = __shfl_sync(0xffffffffu, row, 31);
        if (tail && lane != 31 && q[u] != 0xffffffffu) part[row] = __dadd_rn(part[row], p);
        crow = lastrow;
        carry = lastp;
      }
    }
    if (lane == 0 && crow >= 0 && crow != 0xffff) part[crow] = __dadd_rn(part[crow], carry);
    __syncthreads();
  }
  cl.sync();
  // reduce my share of the group's rows over the cluster, in rank order
  const int q0 = int((int64_t)nrows * c / d.C), q1 = int((int64_t)nrows * (c + 1) / d.C);
  for (int i = q0 + threadIdx.x; i < q1; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < d.C; ++k) {
      const double* rp = cl.map_shared_rank(part, k);
      s = __dadd_rn(s, rp[i]);
    }
    y[r0 + i] = s;
  }
}

template <int U>
__global__ void __launch_bounds__(512, 1)
    k_cluster_spmv(Dev a, Dev b, double* x, double* y, unsigned* bar, int phases, int mode,
                   int which, unsigned long long* stamps) {
  extern __shared__ __align__(16) double smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int bw_pad = (max(a.bw, b.bw) + 1) & ~1;
  double* xs = smem;
  double* part = smem + bw_pad;
  unsigned target = 0;
  for (int ph = 0; ph < phases; ++ph) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    // which: 0 alternate K' / K, 1 only A, 2 only B
    const bool useA = which == 1 || (which == 0 && (ph & 1) == 0);
    if (useA) tile_phase<U>(a, y, x, xs, part, cl, mode);   // x = A y   (A = K', M = n)
    else tile_phase<U>(b, x, y, xs, part, cl, mode);        // y = B x   (B = K, M = m)
    target += gridDim.x;
    grid_bar(bar, target);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0 && stamps) stamps[(size_t)ph * gridDim.x + blockIdx.x] = t1 - t0;
  }
}

static void cpu_spmv(const Csr& a, const std::vector<double>& x, std::vector<double>& y) {
  y.assign(a.M, 0.0);
  for (int i = 0; i < a.M; ++i) {
    double s = 0.0;
    for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) s += a.v[k] * x[a.ci[k]];
    y[i] = s;
  }
}

struct DevLayout {
  Dev d;
  void* bufs[4];
};
static DevLayout upload(const Layout& L) {
  DevLayout D{};
  int64_t *woff;
  uint32_t* rc;
  double* v;
  int* grp;
  CK(cudaMalloc(&woff, L.woff.size() * 8));
  CK(cudaMalloc(&rc, L.rc.size() * 4));
  CK(cudaMalloc(&v, L.v.size() * 8));
  CK(cudaMalloc(&grp, L.grp.size() * 4));
  CK(cudaMemcpy(woff, L.woff.data(), L.woff.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(rc, L.rc.data(), L.rc.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(v, L.v.data(), L.v.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(grp, L.grp.data(), L.grp.size() * 4, cudaMemcpyHostToDevice));
  D.d = Dev{woff, rc, v, L.bw, L.rows_max, L.G, L.C, L.S, L.W, L.M, L.N, grp};
  D.bufs[0] = woff;
  D.bufs[1] = rc;
  D.bufs[2] = v;
  D.bufs[3] = grp;
  return D;
}

template <int U>
static void run(const Csr& K, const Csr& Kt, int G, int C, int SA, int SB, int phases, int mode,
                int which, bool check) {
  const int W = 16;
  Layout LA = build(Kt, G, C, SA, W), LB = build(K, G, C, SB, W);
  DevLayout A = upload(LA), B = upload(LB);
  const int bw_pad = (std::max(LA.bw, LB.bw) + 1) & ~1;
  const size_t smem = sizeof(double) * (bw_pad + std::max(LA.rows_max, LB.rows_max));
  auto kern = k_cluster_spmv<U>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (C > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(G * C);
  cfg.blockDim = dim3(32 * W);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int maxc = 0;
  CK(cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg));
  if (maxc < G) {
    printf("G=%d C=%d: only %d clusters co-resident (smem %zu)\n", G, C, maxc, smem);
    return;
  }
  double *x, *y;
  unsigned* bar;
  unsigned long long* st;
  CK(cudaMalloc(&x, sizeof(double) * K.N));
  CK(cudaMalloc(&y, sizeof(double) * K.M));
  CK(cudaMalloc(&bar, 4));
  CK(cudaMalloc(&st, sizeof(unsigned long long) * phases * G * C));
  std::vector<double> hx(K.N), hy(K.M);
  std::mt19937_64 rg(7);
  std::normal_distribution<double> nd;
  for (auto& e : hy) e = nd(rg);
  CK(cudaMemcpy(y, hy.data(), sizeof(double) * K.M, cudaMemcpyHostToDevice));
  if (check) {  // one A phase then one B phase, against the CPU
    CK(cudaMemset(bar, 0, 4));
    int ph = 2;
    int md = 0, wh = 0;
    unsigned long long* ns = nullptr;
    void* args[] = {&A.d, &B.d, &x, &y, &bar, &ph, &md, &wh, &ns};
    CK(cudaLaunchKernelExC(&cfg, (const void*)kern, args));
    CK(cudaDeviceSynchronize());
    std::vector<double> gx(K.N), gy(K.M), cx, cy;
    CK(cudaMemcpy(gx.data(), x, sizeof(double) * K.N, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(gy.data(), y, sizeof(double) * K.M, cudaMemcpyDeviceToHost));
    cpu_spmv(Kt, hy, cx);
    cpu_spmv(K, gx, cy);
    double ex = 0, ey = 0, nx = 0, ny = 0;
    for (int i = 0; i < K.N; ++i) { ex = std::max(ex, std::fabs(gx[i] - cx[i])); nx = std::max(nx, std::fabs(cx[i])); }
    for (int i = 0; i < K.M; ++i) { ey = std::max(ey, std::fabs(gy[i] - cy[i])); ny = std::max(ny, std::fabs(cy[i])); }
    printf("check: K'y max err %.3e (|.| %.3e), Kx max err %.3e (|.| %.3e)\n", ex, nx, ey, ny);
    CK(cudaMemcpy(y, hy.data(), sizeof(double) * K.M, cudaMemcpyHostToDevice));
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaMemset(bar, 0, 4));
    void* args[] = {&A.d, &B.d, &x, &y, &bar, &phases, &mode, &which, &st};
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelExC(&cfg, (const void*)kern, args));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  std::vector<unsigned long long> hs((size_t)phases * G * C);
  CK(cudaMemcpy(hs.data(), st, hs.size() * 8, cudaMemcpyDeviceToHost));
  double avg = 0;
  for (auto v : hs) avg += v;
  avg /= hs.size();
  printf("U=%d G=%2d C=%2d SA=%d SB=%d bw=%5d/%5d rows=%5d smem=%6zu mode=%d which=%d: %7.2f us/phase (launch %d phases), "
         "stamp avg %.2f us, maxclusters %d\n",
         U, G, C, SA, SB, LA.bw, LB.bw, std::max(LA.rows_max, LB.rows_max), smem, mode, which,
         1e3 * best / phases, phases, avg / 1e3, maxc);
  cudaFree(x);
  cudaFree(y);
  cudaFree(bar);
  cudaFree(st);
  for (int i = 0; i < 4; ++i) { cudaFree(A.bufs[i]); cudaFree(B.bufs[i]); }
}

int main(int argc, char** argv) {
  const int m = 100000, n = 200000;
  Csr K = planted(m, n, 20, 1);
  Csr Kt = transpose(K);
  printf("K %d x %d, nnz %d\n", K.M, K.N, (int)K.ci.size());
  int phases = 40;
  // (G, C, SA, SB)
  struct Cfg { int G, C, SA, SB; };
  std::vector<Cfg> cfgs = {{15, 8, 1, 2}, {33, 4, 2, 4}, {74, 2, 4, 8}};
  bool first = true;
  for (auto c : cfgs) {
    run<4>(K, Kt, c.G, c.C, c.SA, c.SB, phases, 0, 0, first);
    first = false;
  }
  for (auto c : cfgs) {
    run<4>(K, Kt, c.G, c.C, c.SA, c.SB, phases, 0, 1, false);
    run<4>(K, Kt, c.G, c.C, c.SA, c.SB, phases, 0, 2, false);
  }
  // mode 1: no fill, mode 2: no gather
  for (int md = 1; md < 4; ++md) {
    run<4>(K, Kt, 15, 8, 1, 2, phases, md, 0, false);
    run<4>(K, Kt, 74, 2, 4, 8, phases, md, 0, false);
  }
  run<8>(K, Kt, 15, 8, 1, 2, phases, 0, 0, false);
  run<2>(K, Kt, 15, 8, 1, 2, phases, 0, 0, false);
  return 0;
}
