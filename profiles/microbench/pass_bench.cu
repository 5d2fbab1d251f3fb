// pass_bench.cu — microbenchmark (not product code): one configs[4] column
// pass as the solver runs it (k_spmv_pass): 20M rows with ~4 entries each in
// the column block (uniform 0..8), SELL-32 slices sorted by decreasing length
// inside 256-row windows (sl_ptr / sl_len per slice, sl_row / sl_cnt per
// lane), gathers from an S-MB block of x, row partials read + written.
// Variants (argv[1] bit mask):
//   1: metadata (sl_row / sl_cnt) loaded evict-first (ld.global.cs)
//   2: gathers with an L2 evict_last cache policy
//   4: an L2 persisting access-policy window over the x block (+ set-aside)
//   8: whole slice in flight (unroll 8, the partial load issued first)
//  16: partial stores with an L2 evict_first policy (st.global.L2::cache_hint)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pass_bench pass_bench.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

struct Sell {
  int nslices;
  const int64_t* sl_ptr;
  const int* sl_len;
  const int* sl_row;
  const int* sl_cnt;
  const int* sci;
  const double* sv;
};

template <int V, int U>
__global__ void __launch_bounds__(256, 6) pass(Sell A, const double* __restrict__ x,
                                               double* __restrict__ part, int first) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sl = blockIdx.x * 8 + warp;
  if (sl >= A.nslices) return;
  uint64_t plast = 0, pfirst = 0;
  if (V & 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(plast));
  if (V & 16) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pfirst));
  uint64_t sfirst = 0;
  if (V & 64) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(sfirst));
  const int L = __ldg(A.sl_len + sl);
  const int64_t sbase = __ldg(A.sl_ptr + sl);
  int row, cnt;
  if (V & 1) {
    row = __ldcs(A.sl_row + sl * 32 + lane);
    cnt = __ldcs(A.sl_cnt + sl * 32 + lane);
  } else {
    row = __ldg(A.sl_row + sl * 32 + lane);
    cnt = __ldg(A.sl_cnt + sl * 32 + lane);
  }
  const int* cp = A.sci + sbase + lane;
  const double* vp = A.sv + sbase + lane;
  double prev = 0.0;
  if ((V & 8) && !first && row >= 0) prev = __ldcs(part + row);
  double acc = 0.0;
  for (int t0 = 0; t0 < L; t0 += U) {
    int c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool on = t0 + u < cnt;
      if (V & 64) {
        int ci = 0;
        double vi = 0.0;
        if (on) {
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
                       : "=r"(ci) : "l"(cp + 32 * (t0 + u)), "l"(sfirst));
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                       : "=d"(vi) : "l"(vp + 32 * (t0 + u)), "l"(sfirst));
        }
        c[u] = ci;
        v[u] = vi;
      } else {
        c[u] = on ? __ldcs(cp + 32 * (t0 + u)) : 0;
        v[u] = on ? __ldcs(vp + 32 * (t0 + u)) : 0.0;
      }
    }
    double g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (t0 + u < cnt) {
        if (V & 2)
          asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                       : "=d"(g[u]) : "l"(x + c[u]), "l"(plast));
        else
          g[u] = __ldg(x + c[u]);
      } else {
        g[u] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (t0 + u < cnt) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
  }
  if (row < 0) return;
  if (!first) acc = __dadd_rn((V & 8) ? prev : __ldcs(part + row), acc);
  if (V & 16)
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(part + row), "d"(acc),
                 "l"(pfirst));
  else
    __stcs(part + row, acc);
}

template <int V>
void launch(const Sell& A, const double* x, double* part, int first, cudaStream_t st) {
  const int grid = (A.nslices + 7) / 8;
  if (V & 8) pass<V, 8><<<grid, 256, 0, st>>>(A, x, part, first);
  else pass<V, 4><<<grid, 256, 0, st>>>(A, x, part, first);
}


// Persistent pass: one wave of CTAs, warp w owns the contiguous slices
// [w * spw, (w + 1) * spw). STAGES = 2: the next slice's metadata loads are in
// flight while this slice streams and gathers; STAGES = 3: the next slice's
// (column, value) stream is loaded too before this slice's gathers.
struct Meta {
  int L, row, cnt;
  int64_t base;
};
__device__ __forceinline__ Meta load_meta(const Sell& A, int sl, int lane) {
  Meta m;
  m.L = __ldg(A.sl_len + sl);
  m.base = __ldg(A.sl_ptr + sl);
  m.row = __ldcs(A.sl_row + sl * 32 + lane);
  m.cnt = __ldcs(A.sl_cnt + sl * 32 + lane);
  return m;
}
template <int U>
__device__ __forceinline__ void load_stream(const Sell& A, const Meta& m, int lane, int* c,
                                            double* v) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool on = u < m.cnt;
    c[u] = on ? __ldcs(A.sci + m.base + lane + 32 * u) : 0;
    v[u] = on ? __ldcs(A.sv + m.base + lane + 32 * u) : 0.0;
  }
}
template <int U>
__device__ __forceinline__ double finish_slice(const Sell& A, const Meta& m, int lane,
                                               const int* c, const double* v,
                                               const double* __restrict__ x) {
  double g[U];
#pragma unroll
  for (int u = 0; u < U; ++u) g[u] = u < m.cnt ? __ldg(x + c[u]) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (u < m.cnt) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
  for (int t = U; t < m.L; ++t)  // rows longer than U (rare in a pass)
    if (t < m.cnt)
      acc = __dadd_rn(acc, __dmul_rn(__ldcs(A.sv + m.base + lane + 32 * t),
                                     __ldg(x + __ldcs(A.sci + m.base + lane + 32 * t))));
  return acc;
}
template <int STAGES, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) pass2(Sell A, const double* __restrict__ x,
                                                  double* __restrict__ part, int first, int spw) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int s0 = gw * spw, s1 = min(A.nslices, s0 + spw);
  if (s0 >= s1) return;
  Meta m = load_meta(A, s0, lane);
  int c[U];
  double v[U];
  if (STAGES == 3) load_stream<U>(A, m, lane, c, v);
  for (int s = s0; s < s1; ++s) {
    if (STAGES == 2) load_stream<U>(A, m, lane, c, v);
    const double prev = (!first && m.row >= 0) ? __ldcs(part + m.row) : 0.0;
    Meta mn = m;
    if (s + 1 < s1) mn = load_meta(A, s + 1, lane);
    if (STAGES == 3) {
      int cn[U];
      double vn[U];
      if (s + 1 < s1) load_stream<U>(A, mn, lane, cn, vn);
      double acc = finish_slice<U>(A, m, lane, c, v, x);
      if (m.row >= 0) __stcs(part + m.row, first ? acc : __dadd_rn(prev, acc));
#pragma unroll
      for (int u = 0; u < U; ++u) { c[u] = cn[u]; v[u] = vn[u]; }
    } else {
      double acc = finish_slice<U>(A, m, lane, c, v, x);
      if (m.row >= 0) __stcs(part + m.row, first ? acc : __dadd_rn(prev, acc));
    }
    m = mn;
  }
}

template <int STAGES, int U, int MINB>
void launch2(const Sell& A, const double* x, double* part, int first, cudaStream_t st) {
  const int grid = 148 * MINB;
  const int warps = grid * 8;
  const int spw = (A.nslices + warps - 1) / warps;
  pass2<STAGES, U, MINB><<<grid, 256, 0, st>>>(A, x, part, first, spw);
}

// Window pass: CTA b owns slices 8b..8b+7 = the 256-row window b (rows
// sigma-sorted inside it), so its row partials move through shared memory
// with one coalesced load and store; PACK: lane metadata = (row - w0) | cnt << 8.
template <bool PACK, int MB = 6>
__global__ void __launch_bounds__(256, MB) passw(Sell A, const int* __restrict__ meta,
                                              const double* __restrict__ x,
                                              double* __restrict__ part, int first, int rows) {
  __shared__ double ps[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * 256;
  const int sl = blockIdx.x * 8 + warp;
  if (w0 + int(threadIdx.x) < rows) ps[threadIdx.x] = first ? 0.0 : __ldcs(part + w0 + threadIdx.x);
  int off = -1, cnt = 0, L = 0;
  int64_t sbase = 0;
  if (sl < A.nslices) {
    L = __ldg(A.sl_len + sl);
    sbase = __ldg(A.sl_ptr + sl);
    if (PACK) {
      const int mt = __ldcs(meta + sl * 32 + lane);
      off = mt < 0 ? -1 : (mt & 255);
      cnt = mt < 0 ? 0 : (mt >> 8);
    } else {
      const int row = __ldcs(A.sl_row + sl * 32 + lane);
      cnt = __ldcs(A.sl_cnt + sl * 32 + lane);
      off = row < 0 ? -1 : row - w0;
    }
  }
  const int* cp = A.sci + sbase + lane;
  const double* vp = A.sv + sbase + lane;
  double acc = 0.0;
  for (int t0 = 0; t0 < L; t0 += 4) {
    int c[4];
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool on = t0 + u < cnt;
      c[u] = on ? __ldcs(cp + 32 * (t0 + u)) : 0;
      v[u] = on ? __ldcs(vp + 32 * (t0 + u)) : 0.0;
    }
    double g[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) g[u] = t0 + u < cnt ? __ldg(x + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t0 + u < cnt) acc = __dadd_rn(acc, __dmul_rn(v[u], g[u]));
  }
  __syncthreads();
  if (off >= 0) ps[off] = __dadd_rn(ps[off], acc);
  __syncthreads();
  if (w0 + int(threadIdx.x) < rows) __stcs(part + w0 + threadIdx.x, ps[threadIdx.x]);
}

// Two windows per CTA, warp w streams slices 16b + w and 16b + 8 + w together
// (two independent chains per lane), partials through shared memory.
template <int NW, int MB>
__global__ void __launch_bounds__(256, MB) passw2(Sell A, const int* __restrict__ meta,
                                               const double* __restrict__ x,
                                               double* __restrict__ part, int first, int rows) {
  __shared__ double ps[256 * NW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * 256 * NW;
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int r = w0 + q * 256 + int(threadIdx.x);
    if (r < rows) ps[q * 256 + threadIdx.x] = first ? 0.0 : __ldcs(part + r);
  }
  int off[NW], cnt[NW], L[NW];
  int64_t sb[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int sl = blockIdx.x * 8 * NW + q * 8 + warp;
    off[q] = -1; cnt[q] = 0; L[q] = 0; sb[q] = 0;
    if (sl < A.nslices) {
      L[q] = __ldg(A.sl_len + sl);
      sb[q] = __ldg(A.sl_ptr + sl) + lane;
      const int mt = __ldcs(meta + sl * 32 + lane);
      off[q] = mt < 0 ? -1 : (mt & 255) + q * 256;
      cnt[q] = mt < 0 ? 0 : (mt >> 8);
    }
  }
  int Lm = 0;
#pragma unroll
  for (int q = 0; q < NW; ++q) Lm = max(Lm, L[q]);
  double acc[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) acc[q] = 0.0;
  for (int t0 = 0; t0 < Lm; t0 += 4) {
    int c[NW][4];
    double v[NW][4];
#pragma unroll
    for (int q = 0; q < NW; ++q)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool on = t0 + u < cnt[q];
        c[q][u] = on ? __ldcs(A.sci + sb[q] + 32 * (t0 + u)) : 0;
        v[q][u] = on ? __ldcs(A.sv + sb[q] + 32 * (t0 + u)) : 0.0;
      }
    double g[NW][4];
#pragma unroll
    for (int q = 0; q < NW; ++q)
#pragma unroll
      for (int u = 0; u < 4; ++u) g[q][u] = t0 + u < cnt[q] ? __ldg(x + c[q][u]) : 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (t0 + u < cnt[q]) acc[q] = __dadd_rn(acc[q], __dmul_rn(v[q][u], g[q][u]));
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NW; ++q)
    if (off[q] >= 0) ps[off[q]] = __dadd_rn(ps[off[q]], acc[q]);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int r = w0 + q * 256 + int(threadIdx.x);
    if (r < rows) __stcs(part + r, ps[q * 256 + threadIdx.x]);
  }
}

// ---------------------------------------------------------------------------
// Variant 300+: TMA-staged pass. One wave of persistent CTAs; CTA b owns the
// contiguous chunks [b * cpc, (b + 1) * cpc), a chunk = CW consecutive slices
// (one per consumer warp). A producer lane (warp CW) bulk-copies each chunk's
// slice pointers, lane metadata (sl_row, sl_cnt) and (column, value) streams
// into a shared-memory stage (cp.async.bulk + mbarrier, STAGES deep), so a
// consumer warp's dependent chain is smem -> gather (L2) -> partial (loaded
// before the gathers) instead of metadata -> stream -> gather -> partial from
// DRAM, and no stream element lives in a register: 8 gathers in flight.
// Same per-row operation order as pass<> (bitwise equal partials).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(b)), "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

template <int CW, int EC>
struct StageLayout {
  static constexpr int kPtr = 0;                       // CW + 1 int64 (padded to 16 B units)
  static constexpr int kPtrB = ((CW + 1) * 8 + 127) / 128 * 128;
  static constexpr int kRow = kPtrB;                   // CW x 32 int
  static constexpr int kCnt = kRow + CW * 128;
  static constexpr int kCi = kCnt + CW * 128;          // EC int
  static constexpr int kV = kCi + 4 * EC;              // EC double
  static constexpr int kBytes = kV + 8 * EC;
};

template <int STAGES, int CW, int EC, int MB>
__global__ void __launch_bounds__(32 * (CW + 1), MB)
    pass_tma(Sell A, const double* __restrict__ x, double* __restrict__ part, int first, int cpc) {
  using SL = StageLayout<CW, EC>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nchunks = (A.nslices + CW - 1) / CW;
  const int q0 = blockIdx.x * cpc, q1 = min(nchunks, q0 + cpc);
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (warp == CW) {  // producer
    if (lane != 0 || q0 >= q1) return;
    int64_t pa = __ldg(A.sl_ptr + min(A.nslices, q0 * CW));
    int64_t pb = __ldg(A.sl_ptr + min(A.nslices, (q0 + 1) * CW));
    for (int q = q0; q < q1; ++q) {
      const int64_t pc = __ldg(A.sl_ptr + min(A.nslices, (q + 2) * CW));  // (used next round)
      const int it = q - q0, s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], unsigned((it / STAGES - 1) & 1));
      unsigned char* st = smem + size_t(s) * SL::kBytes;
      const unsigned E = unsigned(pb - pa);
      constexpr unsigned kPtrCopy = ((CW + 1) * 8 + 15) / 16 * 16;
      mbar_expect_tx(&full[s], kPtrCopy + 2u * CW * 128u + 12u * E);
      bulk_g2s(st + SL::kPtr, A.sl_ptr + q * CW, kPtrCopy, &full[s]);
      bulk_g2s(st + SL::kRow, A.sl_row + size_t(q) * CW * 32, CW * 128u, &full[s]);
      bulk_g2s(st + SL::kCnt, A.sl_cnt + size_t(q) * CW * 32, CW * 128u, &full[s]);
      if (E) {
        bulk_g2s(st + SL::kCi, A.sci + pa, 4u * E, &full[s]);
        bulk_g2s(st + SL::kV, A.sv + pa, 8u * E, &full[s]);
      }
      pa = pb;
      pb = pc;
    }
    return;
  }
  for (int q = q0; q < q1; ++q) {
    const int it = q - q0, s = it % STAGES;
    mbar_wait(&full[s], unsigned((it / STAGES) & 1));
    const unsigned char* st = smem + size_t(s) * SL::kBytes;
    const int64_t* sp = reinterpret_cast<const int64_t*>(st + SL::kPtr);
    const int sl = q * CW + warp;
    if (sl < A.nslices) {
      const int off = int(sp[warp] - sp[0]);
      const int L = int(sp[warp + 1] - sp[warp]) >> 5;
      const int row = reinterpret_cast<const int*>(st + SL::kRow)[warp * 32 + lane];
      const int cnt = reinterpret_cast<const int*>(st + SL::kCnt)[warp * 32 + lane];
      double prev = 0.0;
      if (!first && row >= 0) prev = __ldcs(part + row);
      const int* cc = reinterpret_cast<const int*>(st + SL::kCi) + off + lane;
      const double* vv = reinterpret_cast<const double*>(st + SL::kV) + off + lane;
      double acc = 0.0;
      for (int t0 = 0; t0 < L; t0 += 8) {
        double g[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) g[u] = t0 + u < cnt ? __ldg(x + cc[32 * (t0 + u)]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t0 + u < cnt) acc = __dadd_rn(acc, __dmul_rn(vv[32 * (t0 + u)], g[u]));
      }
      if (row >= 0) __stcs(part + row, first ? acc : __dadd_rn(prev, acc));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

template <int STAGES, int CW, int EC, int MB>
void launch_tma(const Sell& A, const double* x, double* part, int first, cudaStream_t st) {
  using SL = StageLayout<CW, EC>;
  static bool once = false;
  const int bytes = STAGES * SL::kBytes;
  if (!once) {
    CK(cudaFuncSetAttribute(pass_tma<STAGES, CW, EC, MB>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(pass_tma<STAGES, CW, EC, MB>,
                            cudaFuncAttributePreferredSharedMemoryCarveout,
                            cudaSharedmemCarveoutMaxShared));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pass_tma<STAGES, CW, EC, MB>,
                                                     32 * (CW + 1), bytes));
    printf("pass_tma<%d,%d,%d,%d>: %d bytes smem, %d CTAs/SM resident\n", STAGES, CW, EC, MB,
           bytes, occ);
    once = true;
  }
  const int grid = 148 * MB;
  const int nchunks = (A.nslices + CW - 1) / CW;
  const int cpc = (nchunks + grid - 1) / grid;
  pass_tma<STAGES, CW, EC, MB><<<grid, 32 * (CW + 1), bytes, st>>>(A, x, part, first, cpc);
}

int main(int argc, char** argv) {
  const int rows = 20000000;
  const int win = 256;
  uint64_t st = 88172645463325252ULL;
  auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; };
  std::vector<int> len(rows), rowid(rows);
  for (int r = 0; r < rows; ++r) len[r] = int(rnd() % 9);
  for (int w0 = 0; w0 < rows; w0 += win) {  // decreasing length inside each window
    const int w1 = std::min(rows, w0 + win);
    std::vector<int> idx(w1 - w0);
    for (int i = 0; i < w1 - w0; ++i) idx[i] = w0 + i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return len[a] > len[b]; });
    for (int i = 0; i < w1 - w0; ++i) rowid[w0 + i] = idx[i];
  }
  const int ns = (rows + 31) / 32;
  std::vector<int64_t> sl_ptr(ns + 32);
  std::vector<int> sl_len(ns), sl_row(size_t(ns + 32) * 32, -1), sl_cnt(size_t(ns + 32) * 32, 0);
  int64_t tot = 0;
  for (int s = 0; s < ns; ++s) {
    int L = 0;
    for (int l = 0; l < 32; ++l) {
      const int i = s * 32 + l;
      if (i >= rows) break;
      sl_row[size_t(s) * 32 + l] = rowid[i];
      sl_cnt[size_t(s) * 32 + l] = len[rowid[i]];
      L = std::max(L, len[rowid[i]]);
    }
    sl_ptr[s] = tot;
    sl_len[s] = L;
    tot += 32LL * L;
  }
  for (int s = ns; s < ns + 32; ++s) sl_ptr[s] = tot;
  printf("slices %d, stored entries %lld (nnz ~%lld)\n", ns, (long long)tot, 4LL * rows);
  std::vector<int> sci(tot);
  std::vector<double> sv(tot);
  for (int64_t e = 0; e < tot; ++e) sv[e] = double(int(rnd() % 2001) - 1000) / 512.0;
  int *d_sl_len, *d_sl_row, *d_sl_cnt, *d_sci;
  int64_t* d_sl_ptr;
  double *d_sv, *x, *part;
  CK(cudaMalloc(&d_sl_ptr, (ns + 32) * 8));
  CK(cudaMalloc(&d_sl_len, ns * 4));
  CK(cudaMalloc(&d_sl_row, size_t(ns + 32) * 128));
  CK(cudaMalloc(&d_sl_cnt, size_t(ns + 32) * 128));
  CK(cudaMalloc(&d_sci, tot * 4 + 4096));
  CK(cudaMalloc(&d_sv, tot * 8 + 4096));
  CK(cudaMalloc(&x, 128LL << 20));
  CK(cudaMalloc(&part, size_t(rows) * 8));
  {
    std::vector<double> hx((128LL << 20) / 8);
    for (auto& v : hx) v = double(int(rnd() % 2001) - 1000) / 1024.0;
    CK(cudaMemcpy(x, hx.data(), 128LL << 20, cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(d_sl_ptr, sl_ptr.data(), (ns + 32) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_sl_len, sl_len.data(), ns * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_sl_row, sl_row.data(), size_t(ns + 32) * 128, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_sl_cnt, sl_cnt.data(), size_t(ns + 32) * 128, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_sv, sv.data(), tot * 8, cudaMemcpyHostToDevice));
  std::vector<int> meta(size_t(ns) * 32, -1);
  for (size_t i = 0; i < meta.size(); ++i)
    if (sl_row[i] >= 0) meta[i] = (sl_row[i] - int(i / 256) * 256) | (sl_cnt[i] << 8);
  int* d_meta;
  CK(cudaMalloc(&d_meta, meta.size() * 4));
  CK(cudaMemcpy(d_meta, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice));
  Sell A{ns, d_sl_ptr, d_sl_len, d_sl_row, d_sl_cnt, d_sci, d_sv};
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("persistingL2CacheMaxSize %zu MB, accessPolicyMaxWindowSize %d MB\n",
         size_t(prop.persistingL2CacheMaxSize) >> 20, prop.accessPolicyMaxWindowSize >> 20);
  cudaStream_t s0;
  CK(cudaStreamCreate(&s0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  std::vector<int> variants;
  for (int i = 1; i < argc; ++i) variants.push_back(atoi(argv[i]));
  if (variants.empty()) variants = {1, 300, 301, 302, 303, 304, 305};
  std::vector<double> ref(rows), got(rows);
  for (int mb : {40, 48, 64, 80}) {
    const int64_t nx = (int64_t(mb) << 20) / 8;
    for (int64_t e = 0; e < tot; ++e) sci[e] = int(rnd() % nx);
    CK(cudaMemcpy(d_sci, sci.data(), tot * 4, cudaMemcpyHostToDevice));
    for (int V : variants) {
      
      if (V & 4) {
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize));
        if (V & 32) {
          cudaStreamAttrValue attr{};
          attr.accessPolicyWindow.base_ptr = x;
          attr.accessPolicyWindow.num_bytes =
              std::min<size_t>(size_t(nx) * 8, size_t(prop.accessPolicyMaxWindowSize));
          attr.accessPolicyWindow.hitRatio =
              std::min(1.0f, float(prop.persistingL2CacheMaxSize) / float(nx * 8));
          attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
          attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
          CK(cudaStreamSetAttribute(s0, cudaStreamAttributeAccessPolicyWindow, &attr));
        }
      }
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a, s0));
        switch (V) {
          case 0: launch<0>(A, x, part, r == 0, s0); break;
          case 204: passw<true, 8><<<(ns + 7) / 8, 256, 0, s0>>>(A, d_meta, x, part, r == 0, rows); break;
          case 202: passw2<2, 4><<<(ns + 15) / 16, 256, 0, s0>>>(A, d_meta, x, part, r == 0, rows); break;
          case 203: passw2<2, 5><<<(ns + 15) / 16, 256, 0, s0>>>(A, d_meta, x, part, r == 0, rows); break;
          case 200: passw<false><<<(ns + 7) / 8, 256, 0, s0>>>(A, d_meta, x, part, r == 0, rows); break;
          case 201: passw<true><<<(ns + 7) / 8, 256, 0, s0>>>(A, d_meta, x, part, r == 0, rows); break;
          case 100: launch2<2, 4, 6>(A, x, part, r == 0, s0); break;
          case 101: launch2<2, 8, 4>(A, x, part, r == 0, s0); break;
          case 102: launch2<3, 4, 4>(A, x, part, r == 0, s0); break;
          case 103: launch2<3, 8, 3>(A, x, part, r == 0, s0); break;
          case 104: launch2<2, 6, 5>(A, x, part, r == 0, s0); break;
          case 105: launch2<3, 6, 4>(A, x, part, r == 0, s0); break;
          case 1: launch<1>(A, x, part, r == 0, s0); break;
          case 300: launch_tma<2, 8, 2048, 4>(A, x, part, r == 0, s0); break;
          case 301: launch_tma<3, 8, 2048, 2>(A, x, part, r == 0, s0); break;
          case 302: launch_tma<2, 16, 4096, 2>(A, x, part, r == 0, s0); break;
          case 303: launch_tma<4, 8, 2048, 2>(A, x, part, r == 0, s0); break;
          case 304: launch_tma<3, 16, 4096, 1>(A, x, part, r == 0, s0); break;
          case 305: launch_tma<2, 8, 2048, 3>(A, x, part, r == 0, s0); break;
          case 3: launch<3>(A, x, part, r == 0, s0); break;
          case 5: launch<1>(A, x, part, r == 0, s0); break;
          case 7: launch<3>(A, x, part, r == 0, s0); break;
          case 65: launch<65>(A, x, part, r == 0, s0); break;
          case 81: launch<81>(A, x, part, r == 0, s0); break;
          case 67: launch<67>(A, x, part, r == 0, s0); break;
          case 83: launch<83>(A, x, part, r == 0, s0); break;
          case 37: launch<1>(A, x, part, r == 0, s0); break;
          case 39: launch<3>(A, x, part, r == 0, s0); break;
          case 9: launch<9>(A, x, part, r == 0, s0); break;
          case 25: launch<25>(A, x, part, r == 0, s0); break;
          case 17: launch<17>(A, x, part, r == 0, s0); break;
          case 27: launch<27>(A, x, part, r == 0, s0); break;
        }
        CK(cudaEventRecord(b, s0));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r > 0 && ms < best) best = ms;
      }
      if (V & 4) {
        cudaStreamAttrValue attr{};
        attr.accessPolicyWindow.num_bytes = 0;
        if (V & 32) CK(cudaStreamSetAttribute(s0, cudaStreamAttributeAccessPolicyWindow, &attr));
        CK(cudaCtxResetPersistingL2Cache());
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
      }
      // 1 first pass + 4 accumulating passes: the partials must equal variant 1's bit for bit
      CK(cudaMemcpy(got.data(), part, size_t(rows) * 8, cudaMemcpyDeviceToHost));
      size_t bad = 0;
      if (V == 1) ref = got;
      else if (variants[0] == 1)
        for (int r = 0; r < rows; ++r) bad += ref[r] != got[r];
      printf("block %3d MB variant %2d: %8.1f us  %.1f G gathers/s  mismatches %zu\n", mb, V,
             best * 1e3, 4.0 * rows / (best * 1e-3) / 1e9, bad);
    }
  }
  return 0;
}
