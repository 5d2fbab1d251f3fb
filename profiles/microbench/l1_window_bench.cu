// l1_window_bench.cu — microbenchmark (not product code) for a column-blocked
// SpMV: every SM gathers only from a window of W doubles of the vector (its
// column block), so the gathers can hit in L1 instead of L2. Stream (col i32,
// val f64) from DRAM + gather x[base + col] per nonzero, as in the SELL SpMV.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l1_window_bench l1_window_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

// CTA b works on nonzeros [b*per, (b+1)*per) and on column window
// win(b) = ((b % sms) * B) / sms, so all CTAs resident on one SM (b, b+sms, ...
// in a one-wave classic launch) share a window.
template <int U, int LDMODE>
__global__ void __launch_bounds__(256) win_spmv(const int* __restrict__ col,
                                                const double* __restrict__ val,
                                                const double* __restrict__ x, int per, int W,
                                                int B, int sms, double* out) {
  const int b = blockIdx.x;
  const int win = ((b % sms) * B) / sms;
  const double* xb = x + size_t(win) * W;
  const int lo = b * per, hi = lo + per;
  double acc = 0.0;
  int i = lo + threadIdx.x;
  for (; i + (U - 1) * 256 < hi; i += U * 256) {
    int c[U];
    double v[U], g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldcs(col + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(val + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = LDMODE == 0 ? __ldg(xb + c[u]) : __ldcg(xb + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u] * g[u];
  }
  for (; i < hi; i += 256) acc += __ldcs(val + i) * __ldg(xb + __ldcs(col + i));
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int nx = 200000;
  const int ctas = sms * 6;
  const int per = 4000000 / ctas;
  const int nnz = per * ctas;
  double *x, *val, *out;
  int* col;
  CK(cudaMalloc(&x, sizeof(double) * nx));
  CK(cudaMalloc(&val, sizeof(double) * nnz));
  CK(cudaMalloc(&col, sizeof(int) * nnz));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, sizeof(double) * nx));
  CK(cudaMemset(val, 0, sizeof(double) * nnz));
  // 256 MB scrubber so the stream comes from DRAM every repetition
  char* scrub;
  const size_t scrub_bytes = size_t(256) << 20;
  CK(cudaMalloc(&scrub, scrub_bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<int> hcol(nnz);
  for (int B : {1, 2, 4, 8, 16}) {
    const int W = nx / B;
    srand(11);
    for (int i = 0; i < nnz; ++i) hcol[i] = (int)(((unsigned long long)rand() * 2654435761ull) % W);
    CK(cudaMemcpy(col, hcol.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
    auto run = [&](const char* name, auto kern, int carve) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      float tot = 0.0f;
      const int R = 20;
      for (int r = -3; r < R; ++r) {
        CK(cudaMemsetAsync(scrub, r & 0xff, scrub_bytes));
        cudaEventRecord(a);
        kern<<<ctas, 256>>>(col, val, x, per, W, B, sms, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 0) tot += ms;
      }
      const double us = 1000.0 * tot / R;
      printf("B=%2d W=%6d (%4d KB) %-22s carve=%3d %8.2f us  %6.3f cyc/nnz/SM  %6.0f GB/s stream\n", B,
             W, int(W * 8 / 1024), name, carve, us, us * 1e-6 * 1.965e9 * sms / nnz,
             12.0 * nnz / (us * 1e3));
    };
    run("ldg x4", win_spmv<4, 0>, 0);
    run("ldg x4", win_spmv<4, 0>, 100);
    run("ldg x8", win_spmv<8, 0>, 0);
    run("ldcg x4", win_spmv<4, 1>, 0);
  }
  return 0;
}
