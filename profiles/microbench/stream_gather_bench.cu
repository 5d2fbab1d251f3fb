// stream_gather_bench.cu — microbenchmark (not product code): the SpMV inner
// loop y += val[e] * x[col[e]] for the config-1 shape (4M nonzeros, x of
// 100k / 200k doubles, L2-resident), with the (col, val) stream coming from
// DRAM (8 rotating copies, 384 MB > L2) as in the solver, fed either by
// per-thread loads (the current kernels) or by cp.async.bulk (TMA engine)
// into shared memory, double-buffered with an mbarrier per stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_gather_bench stream_gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

// A: per-thread loads, U (col, val) pairs then U gathers in flight
template <int U>
__global__ void __launch_bounds__(256) directU(const double* __restrict__ x,
                                               const int* __restrict__ col,
                                               const double* __restrict__ val,
                                               double* __restrict__ out, int n, int gather) {
  double acc = 0.0;
  const int stride = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    int c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldcs(col + i + u * stride);
      v[u] = __ldcs(val + i + u * stride);
    }
    double g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = gather ? __ldg(x + c[u]) : double(c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u] * g[u];
  }
  for (; i < n; i += stride) {  // remainder
    const int c = __ldcs(col + i);
    acc += __ldcs(val + i) * (gather ? __ldg(x + c) : double(c));
  }
  if (acc == 12345.0) out[0] = acc;
}

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

// B: the CTA's contiguous chunk of the stream staged by the TMA engine in
// tiles of T elements, NS stages; every thread gathers 8 at a time from smem
// indices.
template <int T, int NS>
__global__ void __launch_bounds__(256) tma_staged(const double* __restrict__ x,
                                                  const int* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  double* __restrict__ out, int n) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* sv = reinterpret_cast<double*>(smem);                 // NS x T
  int* sc = reinterpret_cast<int*>(smem + sizeof(double) * T * NS);  // NS x T
  __shared__ uint64_t bar[NS];
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * per, hi = min(n, lo + per);
  const int ntiles = (hi - lo + T - 1) / T;
  if (threadIdx.x == 0)
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](int t) {
    const int s = t % NS;
    const int e0 = lo + t * T;
    const int cnt = min(T, hi - e0);
    mbar_expect_tx(&bar[s], unsigned(cnt) * 12u);
    bulk_g2s(sv + s * T, val + e0, unsigned(cnt) * 8u, &bar[s]);
    bulk_g2s(sc + s * T, col + e0, unsigned(cnt) * 4u, &bar[s]);
  };
  if (threadIdx.x == 0)
    for (int t = 0; t < NS && t < ntiles; ++t) issue(t);
  double acc = 0.0;
  for (int t = 0; t < ntiles; ++t) {
    const int s = t % NS;
    mbar_wait(&bar[s], unsigned((t / NS) & 1));
    const int cnt = min(T, hi - (lo + t * T));
    const double* vv = sv + s * T;
    const int* cc = sc + s * T;
    for (int k = threadIdx.x; k < cnt; k += 256 * 8) {
      double g[8], v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int kk = k + u * 256;
        g[u] = kk < cnt ? __ldg(x + cc[kk]) : 0.0;
        v[u] = kk < cnt ? vv[kk] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u] * g[u];
    }
    __syncthreads();  // stage s free
    if (threadIdx.x == 0 && t + NS < ntiles) issue(t + NS);
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const int n = 4000000;
  const int R = 8;  // rotating stream copies
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int nx : {100000, 200000}) {
    std::vector<int> hidx(n);
    std::vector<double> hv(n, 1.0);
    srand(7);
    for (int i = 0; i < n; ++i) hidx[i] = (int)(((unsigned long long)rand() * 2654435761ull) % nx);
    double *x, *out;
    CK(cudaMalloc(&x, sizeof(double) * nx));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(x, 0, sizeof(double) * nx));
    std::vector<int*> col(R);
    std::vector<double*> val(R);
    for (int r = 0; r < R; ++r) {
      CK(cudaMalloc(&col[r], sizeof(int) * n));
      CK(cudaMalloc(&val[r], sizeof(double) * n));
      CK(cudaMemcpy(col[r], hidx.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(val[r], hv.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
      for (int w = 0; w < 2 * R; ++w) launch(w % R);
      CK(cudaDeviceSynchronize());
      const int reps = 4 * R;
      cudaEventRecord(a);
      for (int r = 0; r < reps; ++r) launch(r % R);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double us = 1000.0 * ms / reps;
      printf("nx=%7d %-40s %8.2f us  %6.2f cyc/nnz/SM  %7.0f GB/s stream\n", nx, name, us,
             us * 1e-6 * 1.965e9 * sms / n, 12.0 * n / us / 1e3);
    };
    for (int cps : {4, 6, 8}) {
      const int blocks = sms * cps;
      char nm[80];
      snprintf(nm, sizeof nm, "direct8 stream only, %d CTAs/SM", cps);
      timeit(nm, [&](int r) { directU<8><<<blocks, 256>>>(x, col[r], val[r], out, n, 0); });
      for (int U : {2, 4, 8}) {
        snprintf(nm, sizeof nm, "direct%d stream + gather, %d CTAs/SM", U, cps);
        if (U == 2) timeit(nm, [&](int r) { directU<2><<<blocks, 256>>>(x, col[r], val[r], out, n, 1); });
        if (U == 4) timeit(nm, [&](int r) { directU<4><<<blocks, 256>>>(x, col[r], val[r], out, n, 1); });
        if (U == 8) timeit(nm, [&](int r) { directU<8><<<blocks, 256>>>(x, col[r], val[r], out, n, 1); });
      }
    }
    return 0;
    {
      constexpr int T = 2048, NS = 2;
      const size_t sm = size_t(T) * NS * 12;
      CK(cudaFuncSetAttribute(tma_staged<T, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      for (int cps : {2, 3, 4}) {
        char nm[64];
        snprintf(nm, sizeof nm, "tma T=%d NS=%d ctas/SM=%d", T, NS, cps);
        timeit(nm, [&](int r) {
          tma_staged<T, NS><<<sms * cps, 256, sm>>>(x, col[r], val[r], out, n);
        });
      }
    }
    {
      constexpr int T = 1024, NS = 3;
      const size_t sm = size_t(T) * NS * 12;
      CK(cudaFuncSetAttribute(tma_staged<T, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      for (int cps : {4, 5, 6}) {
        char nm[64];
        snprintf(nm, sizeof nm, "tma T=%d NS=%d ctas/SM=%d", T, NS, cps);
        timeit(nm, [&](int r) {
          tma_staged<T, NS><<<sms * cps, 256, sm>>>(x, col[r], val[r], out, n);
        });
      }
    }
    for (int r = 0; r < R; ++r) {
      cudaFree(col[r]);
      cudaFree(val[r]);
    }
    cudaFree(x);
    cudaFree(out);
  }
  return 0;
}
