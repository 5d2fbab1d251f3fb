// triplets.cu — CSR assembly from (row, col, value) triplets on the device
// (SURVEY.md §8(f) f1): the drop-in's SparseMatrix::from_triplets
// (sparse_linalg.cpp:11-42) and the four-block split of to_standard_form
// (lp_model.cpp:232-291) for 10^7-10^8-entry LPs.
//
//   keys      key = row' * ncols + col, row' = row_map[row] (identity when
//             null), the value negated where row_neg[row] (L rows -> G);
//   sort      CUB radix sort of (key, index): LSD radix sorting is stable,
//             so duplicates stay in input order;
//   sum       one thread per run of equal keys adds its values left to
//             right (a fixed, sequential order: duplicates sum as a stable
//             sort would present them), writes (col, value) at the run's
//             rank and counts the row;
//   row_ptr   exclusive scan of the row counts.
// Every input entry is range-checked on the device first (DimensionError,
// as the reference). Exact cancellations keep their structural zero.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

#include "engine.h"

namespace aapdhg_b200 {
namespace {

constexpr int kT = 256;
int blocks(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 148 * 64))); }

__global__ void k_trip_keys(const aapdhg_triplet* __restrict__ t, int64_t count, int nrows_in,
                            int ncols, const int32_t* __restrict__ row_map, int64_t* key,
                            int32_t* idx, int* flags) {
  int bad = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = t[i].row, c = t[i].col;
    if (r < 0 || r >= nrows_in || c < 0 || c >= ncols) {
      bad = 1;
      key[i] = 0;
    } else {
      key[i] = int64_t(row_map ? row_map[r] : r) * ncols + c;
    }
    idx[i] = int32_t(i);
  }
  if (bad) atomicOr(flags, 1);
}

__global__ void k_trip_heads(const int64_t* __restrict__ key, int64_t count, int32_t* head) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

__global__ void k_trip_sum(const int64_t* __restrict__ key, const int32_t* __restrict__ idx,
                           const int32_t* __restrict__ head, const int32_t* __restrict__ rank,
                           const aapdhg_triplet* __restrict__ t,
                           const uint8_t* __restrict__ row_neg, int64_t count, int ncols,
                           int32_t* ci, double* v, int32_t* row_cnt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (!head[i]) continue;
    const int64_t k = key[i];
    double s = 0.0;
    for (int64_t j = i; j < count && key[j] == k; ++j) {
      const aapdhg_triplet e = t[idx[j]];
      s = __dadd_rn(s, (row_neg && row_neg[e.row]) ? -e.val : e.val);
    }
    const int32_t r = int32_t(k / ncols);
    const int32_t out = rank[i];
    ci[out] = int32_t(k - int64_t(r) * ncols);
    v[out] = s;
    atomicAdd(row_cnt + r, 1);
  }
}

}  // namespace

int64_t csr_from_triplets(int device, int nrows_in, int nrows_out, int ncols, int64_t count,
                          const aapdhg_triplet* trip, const int32_t* row_map,
                          const uint8_t* row_neg, int32_t* rp_out, int32_t* ci_out,
                          double* v_out) {
  AAPDHG_CUDA(cudaSetDevice(device));
  if (nrows_in < 0 || nrows_out < 0 || ncols < 0 || count < 0)
    throw StatusError(AAPDHG_ERR_DIMENSION, "from_triplets: negative dimension");
  if (count > int64_t(INT32_MAX))
    throw StatusError(AAPDHG_ERR_UNSUPPORTED, "from_triplets: more than 2^31 - 1 entries");
  if (row_map)
    for (int r = 0; r < nrows_in; ++r)
      if (row_map[r] < 0 || row_map[r] >= nrows_out)
        throw StatusError(AAPDHG_ERR_DIMENSION, "from_triplets: row map out of range");
  auto buf = [](DevBuf& b, size_t bytes) { b.reserve(std::max<size_t>(bytes, 16)); return b.p; };
  DevBuf bt, bmap, bneg, bkey, bkey2, bidx, bidx2, bhead, brank, bci, bv, bcnt, brp, btmp, bflag,
      bscan, bscan2;
  cudaStream_t s;
  AAPDHG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {  // destroyed before the buffers: they go back to the cache idle
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{s};
  auto* t = static_cast<aapdhg_triplet*>(buf(bt, sizeof(aapdhg_triplet) * size_t(count)));
  host_to_device(t, trip, sizeof(aapdhg_triplet) * size_t(count), s);
  int32_t* dmap = nullptr;
  uint8_t* dneg = nullptr;
  if (row_map) {
    dmap = static_cast<int32_t*>(buf(bmap, sizeof(int32_t) * size_t(nrows_in)));
    host_to_device(dmap, row_map, sizeof(int32_t) * size_t(nrows_in), s);
  }
  if (row_neg) {
    dneg = static_cast<uint8_t*>(buf(bneg, size_t(nrows_in)));
    host_to_device(dneg, row_neg, size_t(nrows_in), s);
  }
  int* flags = static_cast<int*>(buf(bflag, sizeof(int)));
  AAPDHG_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), s));
  auto* key = static_cast<int64_t*>(buf(bkey, sizeof(int64_t) * size_t(count)));
  auto* key2 = static_cast<int64_t*>(buf(bkey2, sizeof(int64_t) * size_t(count)));
  auto* idx = static_cast<int32_t*>(buf(bidx, sizeof(int32_t) * size_t(count)));
  auto* idx2 = static_cast<int32_t*>(buf(bidx2, sizeof(int32_t) * size_t(count)));
  if (count > 0)
    k_trip_keys<<<blocks(count), kT, 0, s>>>(t, count, nrows_in, ncols, dmap, key, idx, flags);
  AAPDHG_CUDA(cudaGetLastError());
  int hflag = 0;
  AAPDHG_CUDA(cudaMemcpyAsync(&hflag, flags, sizeof hflag, cudaMemcpyDeviceToHost, s));
  AAPDHG_CUDA(cudaStreamSynchronize(s));
  if (hflag) throw StatusError(AAPDHG_ERR_DIMENSION, "from_triplets: entry out of range");

  int64_t nnz = 0;
  auto* cnt = static_cast<int32_t*>(buf(bcnt, sizeof(int32_t) * (size_t(nrows_out) + 1)));
  AAPDHG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t(nrows_out) + 1), s));
  auto* ci = static_cast<int32_t*>(buf(bci, sizeof(int32_t) * size_t(count)));
  auto* v = static_cast<double*>(buf(bv, sizeof(double) * size_t(count)));
  if (count > 0) {
    int bits = 1;
    const int64_t maxkey = int64_t(std::max(nrows_out, 1)) * int64_t(std::max(ncols, 1));
    while (bits < 63 && (int64_t(1) << bits) < maxkey) ++bits;
    size_t tb = 0;
    AAPDHG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, idx2, count, 0, bits, s));
    void* tmp = buf(btmp, tb);
    AAPDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, idx, idx2, count, 0, bits, s));
    auto* head = static_cast<int32_t*>(buf(bhead, sizeof(int32_t) * size_t(count)));
    auto* rank = static_cast<int32_t*>(buf(brank, sizeof(int32_t) * size_t(count)));
    k_trip_heads<<<blocks(count), kT, 0, s>>>(key2, count, head);
    size_t sb = 0;
    AAPDHG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sb, head, rank, count, s));
    AAPDHG_CUDA(cub::DeviceScan::ExclusiveSum(buf(bscan, sb), sb, head, rank, count, s));
    k_trip_sum<<<blocks(count), kT, 0, s>>>(key2, idx2, head, rank, t, dneg, count, ncols, ci, v,
                                            cnt);
    AAPDHG_CUDA(cudaGetLastError());
    int32_t last[2] = {0, 0};
    AAPDHG_CUDA(cudaMemcpyAsync(&last[0], rank + count - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    AAPDHG_CUDA(cudaMemcpyAsync(&last[1], head + count - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    AAPDHG_CUDA(cudaStreamSynchronize(s));
    nnz = int64_t(last[0]) + last[1];
  }
  // row_ptr: exclusive scan of the row counts (nrows_out + 1 entries)
  auto* rp = static_cast<int32_t*>(buf(brp, sizeof(int32_t) * (size_t(nrows_out) + 1)));
  size_t rb = 0;
  AAPDHG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, rb, cnt, rp, nrows_out + 1, s));
  AAPDHG_CUDA(cub::DeviceScan::ExclusiveSum(buf(bscan2, rb), rb, cnt, rp, nrows_out + 1, s));
  device_to_host(rp_out, rp, sizeof(int32_t) * (size_t(nrows_out) + 1), s);
  device_to_host(ci_out, ci, sizeof(int32_t) * size_t(nnz), s);
  device_to_host(v_out, v, sizeof(double) * size_t(nnz), s);
  return nnz;
}

}  // namespace aapdhg_b200
