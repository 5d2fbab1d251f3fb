// smem_gather_bench.cu — microbenchmark (not product code) for an
// x-stationary SpMV design: (A) random 8-byte gathers from a vector block
// staged in shared memory; (B) fill rate of a shared-memory block with
// cp.async.bulk from global/L2, unicast vs multicast to a cluster.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_gather_bench smem_gather_bench.cu
#include <cooperative_groups.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// (A) every thread: G random gathers from the smem block (indices hashed)
__global__ void __launch_bounds__(512) smem_gather(const double* __restrict__ x, int nblk,
                                                   int G, double* out) {
  extern __shared__ double sx[];
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) sx[i] = x[i];
  __syncthreads();
  uint32_t h = (blockIdx.x * 1024u + threadIdx.x) * 2654435761u;
  double acc = 0.0;
  for (int g = 0; g < G; g += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      h = h * 1664525u + 1013904223u;
      v[u] = sx[(h >> 8) % nblk];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  if (acc == 12345.0) out[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(b)), "r"(phase)
      : "memory");
}

// (B) R rounds: fill `bytes` of smem from global chunk r (rotating over a
// large buffer so the data comes from L2/DRAM), unicast per CTA or
// multicast by cluster rank 0 to all CTAs of the cluster.
template <int CS, bool MC>
__global__ void __launch_bounds__(128) bulk_fill(const char* __restrict__ src, size_t span,
                                                 unsigned bytes, int R, double* out) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = CS > 1 ? cl.block_rank() : 0;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (CS > 1) cl.sync();
  else __syncthreads();
  double acc = 0.0;
  const int clusters = gridDim.x / CS;
  const int cid = blockIdx.x / CS;
  for (int r = 0; r < R; ++r) {
    const size_t off = (size_t(r) * clusters + cid) * bytes % (span - bytes);
    const char* g = src + (off & ~size_t(127));
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar, bytes);
      if (!MC) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(buf)),
            "l"(g), "r"(bytes), "r"(smem_u32(&bar))
            : "memory");
      } else if (rank == 0) {
        const unsigned short mask = (1u << CS) - 1;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
            "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(buf)),
            "l"(g), "r"(bytes), "r"(smem_u32(&bar)), "h"(mask)
            : "memory");
      }
    }
    mbar_wait(&bar, unsigned(r & 1));
    acc += reinterpret_cast<const double*>(buf)[threadIdx.x];
    if (CS > 1) cl.sync();  // everyone done reading before the next fill
    else __syncthreads();
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double *x, *out;
  const size_t span = size_t(512) << 20;  // 512 MB
  char* big;
  CK(cudaMalloc(&x, sizeof(double) * 32768));
  CK(cudaMalloc(&out, 8));
  CK(cudaMalloc(&big, span));
  CK(cudaMemset(x, 0, sizeof(double) * 32768));
  CK(cudaMemset(big, 0, span));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return 1000.0 * ms / 5;
  };
  // (A)
  for (int nblk : {4096, 12288, 24576}) {
    const size_t sm = sizeof(double) * nblk;
    CK(cudaFuncSetAttribute(smem_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int G = 4096;
    const double us = time([&] { smem_gather<<<sms, 512, sm>>>(x, nblk, G, out); });
    const double gathers = double(sms) * 512 * G;
    printf("smem gather  block %6zu KB  %8.2f us  %6.3f cyc/gather/SM (incl. fill)\n", sm / 1024,
           us, us * 1e-6 * 1.965e9 * sms / gathers);
  }
  // (B)
  auto fill = [&](auto kern, int cs, unsigned bytes, const char* name) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    if (cs > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int R = 200;
    const int grid = (sms / cs) * cs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = bytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const double us = time([&] {
      CK(cudaLaunchKernelEx(&cfg, kern, (const char*)big, span, bytes, R, out));
    });
    const double per_sm = double(bytes) * R / (us * 1e-6) / 1e9;  // GB/s per SM
    printf("%-28s %6u KB x %d rounds: %8.2f us  %7.1f GB/s per SM  %6.1f B/cyc/SM  %7.0f GB/s chip\n",
           name, bytes / 1024, R, us, per_sm, per_sm * 1e9 / 1.965e9, per_sm * grid);
  };
  for (unsigned kb : {64u, 96u}) {
    fill(bulk_fill<1, false>, 1, kb * 1024, "unicast cs=1");
    fill(bulk_fill<4, false>, 4, kb * 1024, "unicast cs=4");
    fill(bulk_fill<4, true>, 4, kb * 1024, "multicast cs=4");
    fill(bulk_fill<8, true>, 8, kb * 1024, "multicast cs=8");
  }
  return 0;
}
