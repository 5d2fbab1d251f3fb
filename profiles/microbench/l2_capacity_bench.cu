// l2_capacity_bench.cu — microbenchmark (not product code): how large a
// gathered vector block stays L2-resident on B200 while a (col, val) stream
// passes through L2, i.e. the configs[4] column-pass shape.
// For block sizes S = 4..128 MB: E random 8-byte gathers x[col[e]] with
// col uniform in [0, S/8), (col, val) streamed from DRAM (E = 80M, 960 MB),
// y[row] += v * x[col] over 20 entries per row (SELL-like: lane = row).
// Modes: 0 = stream + gathers (the pass), 1 = gathers only (indices hashed in
// the kernel, no stream), 2 = stream only (no gathers).
// Reports ns per gather and effective GB/s; run under ncu for dram bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_capacity_bench l2_capacity_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
  a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
  return a;
}

// slice layout: rows in groups of 32 (one warp), entry k of lane r at
// base + 32 k + r (coalesced), 20 entries per row
template <int MODE, int U>
__global__ void __launch_bounds__(256) pass(const double* __restrict__ x,
                                            const int* __restrict__ col,
                                            const double* __restrict__ val,
                                            double* __restrict__ y, int64_t rows, int per_row,
                                            uint32_t xmask, int pol) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  uint64_t first = 0, last = 0;
  if (pol) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(last));
  }
  for (int64_t s = warp; s * 32 < rows; s += nwarps) {
    const int64_t base = s * 32 * per_row;
    double acc = 0.0;
    for (int k = 0; k < per_row; k += U) {
      int c[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = base + int64_t(k + u) * 32 + lane;
        if (MODE == 1) {
          c[u] = int(hash32(uint32_t(e) * 2654435761U) & xmask);
          v[u] = 1.0;
        } else if (pol) {
          asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;"
                       : "=r"(c[u]) : "l"(col + e), "l"(first));
          asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                       : "=d"(v[u]) : "l"(val + e), "l"(first));
        } else {
          c[u] = __ldcs(col + e);
          v[u] = __ldcs(val + e);
        }
      }
      double g[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (MODE == 2) {
          g[u] = double(c[u]);
        } else if (pol) {
          asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                       : "=d"(g[u]) : "l"(x + c[u]), "l"(last));
        } else {
          g[u] = __ldg(x + c[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u] * g[u];
    }
    y[s * 32 + lane] = acc;
  }
}

int main(int argc, char** argv) {
  const int64_t E = 80LL << 20;  // gathers per pass (~configs[4] K pass)
  const int per_row = 20;
  const int64_t rows = E / per_row;
  const int pol = argc > 1 ? atoi(argv[1]) : 0;
  int* col;
  double *val, *x, *y;
  CK(cudaMalloc(&col, E * 4));
  CK(cudaMalloc(&val, E * 8));
  CK(cudaMalloc(&x, 256LL << 20));
  CK(cudaMalloc(&y, rows * 8));
  CK(cudaMemset(x, 0, 256LL << 20));
  std::vector<int> hc(E);
  uint64_t st = 88172645463325252ULL;
  std::vector<double> hv(E, 1.0);
  CK(cudaMemcpy(val, hv.data(), E * 8, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int grid = nsm * 6;
  for (int mb : {4, 8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 128, 256}) {
    const uint32_t nx = uint32_t((int64_t(mb) << 20) / 8);  // power of two for MODE 1 only
    for (int64_t e = 0; e < E; ++e) {
      st ^= st << 13; st ^= st >> 7; st ^= st << 17;
      hc[e] = int(st % nx);
    }
    CK(cudaMemcpy(col, hc.data(), E * 4, cudaMemcpyHostToDevice));
    uint32_t mask = 1;
    while ((mask << 1) <= nx) mask <<= 1;
    mask -= 1;
    for (int mode = 0; mode < 3; ++mode) {
      if (mode == 2 && mb != 4) continue;
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        if (mode == 0) pass<0, 4><<<grid, 256>>>(x, col, val, y, rows, per_row, mask, pol);
        if (mode == 1) pass<1, 4><<<grid, 256>>>(x, col, val, y, rows, per_row, mask, pol);
        if (mode == 2) pass<2, 4><<<grid, 256>>>(x, col, val, y, rows, per_row, mask, pol);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
      }
      const double stream_b = mode == 1 ? 0 : double(E) * 12;
      printf("block %4d MB mode %d pol %d: %8.1f us  %.3f ns/gather  stream %.0f GB/s\n", mb,
             mode, pol, best * 1e3, best * 1e6 / double(E), stream_b / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
