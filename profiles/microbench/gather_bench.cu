// gather_bench.cu — microbenchmark (not product code): throughput of random
// 8-byte gathers y = x[idx] on sm_100a through different load paths, for the
// config-1 shape (4M gathers from a 200k-double vector, 100k-double vector).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  if (MODE == 0) return __ldg(p);
  if (MODE == 1) return __ldcg(p);
  if (MODE == 2) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  }
  if (MODE == 3) return *p;
  return __ldca(p);
}

template <int MODE>
__global__ void gather(const double* __restrict__ x, const int* __restrict__ idx,
                       double* __restrict__ out, int n) {
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    acc += ld<MODE>(x + __ldcs(idx + i));
  if (acc == 12345.0) out[0] = acc;
}

// unrolled: 8 independent gathers per thread in flight
template <int MODE>
__global__ void gather8(const double* __restrict__ x, const int* __restrict__ idx,
                        double* __restrict__ out, int n) {
  double acc = 0.0;
  const int stride = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    int c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = __ldcs(idx + i + u * stride);
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ld<MODE>(x + c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  for (; i < n; i += stride) acc += ld<MODE>(x + __ldcs(idx + i));  // remainder
  if (acc == 12345.0) out[0] = acc;
}

// x staged in distributed shared memory of a cluster of CS CTAs; gathers via
// ld.shared::cluster (map_shared_rank).
template <int CS>
__global__ void gather_dsmem(const double* __restrict__ x, const int* __restrict__ idx,
                             double* __restrict__ out, int n, int nx) {
  extern __shared__ double sx[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int slice = (nx + CS - 1) / CS;
  for (int t = threadIdx.x; t < slice; t += blockDim.x) {
    const int g = rank * slice + t;
    sx[t] = g < nx ? x[g] : 0.0;
  }
  cl.sync();
  double acc = 0.0;
  const int nclusters = gridDim.x / CS;
  const int cid = blockIdx.x / CS;
  const int per = (n + nclusters - 1) / nclusters;
  const int lo = cid * per, hi = min(n, lo + per);
  for (int i = lo + rank * blockDim.x + threadIdx.x; i < hi; i += CS * blockDim.x) {
    const int c = __ldcs(idx + i);
    const double* p = cl.map_shared_rank(sx, c / slice);
    acc += p[c % slice];
  }
  cl.sync();
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const int n = 4000000;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int nx : {100000, 200000, 40000000}) {
    std::vector<int> hidx(n);
    srand(7);
    for (int i = 0; i < n; ++i) hidx[i] = (int)(((unsigned long long)rand() * 2654435761ull) % nx);
    double *x, *out;
    int* idx;
    CK(cudaMalloc(&x, sizeof(double) * nx));
    CK(cudaMalloc(&out, 8));
    CK(cudaMalloc(&idx, sizeof(int) * n));
    CK(cudaMemset(x, 0, sizeof(double) * nx));
    CK(cudaMemcpy(idx, hidx.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
      for (int w = 0; w < 3; ++w) launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      const int R = 20;
      for (int r = 0; r < R; ++r) launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double us = 1000.0 * ms / R;
      printf("nx=%9d %-34s %8.2f us  %7.2f Ggather/s  %6.2f cyc/gather/SM\n", nx, name, us,
             n / us / 1e3, us * 1e-6 * 1.965e9 * sms / n);
    };
    for (int thr : {256, 512}) {
      const int blocks = sms * (2048 / thr);
      char nm[64];
      snprintf(nm, sizeof nm, "ldg   x1 thr%d", thr);
      timeit(nm, [&] { gather<0><<<blocks, thr>>>(x, idx, out, n); });
      snprintf(nm, sizeof nm, "ldg   x8 thr%d", thr);
      timeit(nm, [&] { gather8<0><<<blocks, thr>>>(x, idx, out, n); });
      snprintf(nm, sizeof nm, "ldcg  x8 thr%d", thr);
      timeit(nm, [&] { gather8<1><<<blocks, thr>>>(x, idx, out, n); });
      snprintf(nm, sizeof nm, "nc.L1::no_allocate x8 thr%d", thr);
      timeit(nm, [&] { gather8<2><<<blocks, thr>>>(x, idx, out, n); });
      snprintf(nm, sizeof nm, "ld    x8 thr%d", thr);
      timeit(nm, [&] { gather8<3><<<blocks, thr>>>(x, idx, out, n); });
    }
    if (nx <= 200000) {
      // cluster of 16 (non-portable) or 8
      for (int cs : {8, 16}) {
        const int slice = (nx + cs - 1) / cs;
        const size_t smem = sizeof(double) * slice;
        if (smem > 227 * 1024) continue;
        cudaLaunchConfig_t cfg = {};
        const int clusters = sms / cs;
        cfg.gridDim = dim3(clusters * cs);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        char nm[64];
        snprintf(nm, sizeof nm, "dsmem cluster%d thr1024", cs);
        if (cs == 16) {
          CK(cudaFuncSetAttribute(gather_dsmem<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
          CK(cudaFuncSetAttribute(gather_dsmem<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          timeit(nm, [&] { CK(cudaLaunchKernelEx(&cfg, gather_dsmem<16>, (const double*)x, (const int*)idx, out, n, nx)); });
        } else {
          CK(cudaFuncSetAttribute(gather_dsmem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          timeit(nm, [&] { CK(cudaLaunchKernelEx(&cfg, gather_dsmem<8>, (const double*)x, (const int*)idx, out, n, nx)); });
        }
      }
    }
    cudaFree(x);
    cudaFree(out);
    cudaFree(idx);
  }
  return 0;
}
