// die_split_bench.cu — microbenchmark (not product code): does B200's L2 keep
// a copy of far-die lines next to the reading SM (so data every SM gathers
// occupies both dies' L2 halves)? Random 8-byte gathers (hashed indices, no
// stream) from an S-MB block, 80M per launch:
//   mode 0: every SM gathers from the whole block;
//   mode 1: SMs with %smid < split gather from the first half only, the others
//           from the second half (if %smid order follows the dies, each die's
//           L2 then holds half the block).
//   mode 2: the same halves assigned by smid parity (mixes dies: a control).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o die_split_bench die_split_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
  a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
  return a;
}

template <int MODE>
__global__ void __launch_bounds__(256) gath(const double* __restrict__ x, double* out,
                                            uint32_t half, int split, int64_t per_thread) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  uint32_t base = 0, span = 2 * half;
  if (MODE == 1) { base = smid < unsigned(split) ? 0 : half; span = half; }
  if (MODE == 2) { base = (smid & 1) ? half : 0; span = half; }
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int64_t k = 0; k < per_thread; k += 4) {
    double g[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) g[u] = __ldg(x + base + hash32(t * 2654435761U + uint32_t(k + u)) % span);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += g[u];
  }
  if (acc == 1234.5) out[0] = acc;
}

int main() {
  double *x, *out;
  CK(cudaMalloc(&x, 256LL << 20));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(x, 0, 256LL << 20));
  const int grid = 148 * 6, threads = 256;
  const int64_t total = 80LL << 20, per = total / (int64_t(grid) * threads);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int split : {74, 70, 78}) {
    for (int mb : {32, 64, 96, 128, 160, 192}) {
      const uint32_t half = uint32_t((int64_t(mb) << 20) / 16);
      for (int mode = 0; mode < 3; ++mode) {
        if (split != 74 && mode != 1) continue;
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
          CK(cudaEventRecord(a));
          if (mode == 0) gath<0><<<grid, threads>>>(x, out, half, split, per);
          if (mode == 1) gath<1><<<grid, threads>>>(x, out, half, split, per);
          if (mode == 2) gath<2><<<grid, threads>>>(x, out, half, split, per);
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (r > 0 && ms < best) best = ms;
        }
        printf("split %d block %3d MB mode %d: %8.1f us  %.1f G gathers/s\n", split, mb, mode,
               best * 1e3, double(per) * grid * threads / (best * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
