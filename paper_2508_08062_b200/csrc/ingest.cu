// ingest.cu — problem ingestion on the device: the
// transpose K', the SELL-32 layouts and the L2 column blocks are built by
// kernels and CUB primitives from the uploaded CSR instead of host loops
// (config 4: 400M nonzeros). The layouts are exactly the ones the host
// builder made: stable orders everywhere, so every row keeps its CSR order
// and the SERIAL-mode sums stay bit-identical to the reference.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.h"

namespace aapdhg_b200 {

namespace {

constexpr int kT = 256;

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

int blocks_for(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 1 << 20))); }

__global__ void k_iota(int32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    a[i] = int32_t(i);
}

__global__ void k_row_len(const int32_t* rp, int n, int32_t* len, char* is_long, char* is_short,
                          int64_t* short_len, int64_t* short_sq, int thr) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t l = rp[i + 1] - rp[i];
    len[i] = l;
    is_long[i] = l > thr;
    is_short[i] = l <= thr;
    short_len[i] = l <= thr ? l : 0;
    short_sq[i] = l <= thr ? int64_t(l) * l : 0;
  }
}

__global__ void k_gather_len(const int32_t* rows, int64_t n, const int32_t* len, int32_t* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = len[rows[i]];
}

// Stable sort of each window of sigma (<= 256) consecutive entries of rows_in
// by decreasing len[row], one CTA per window: entry t goes to rank = #longer
// + #equal before it, the permutation CUB's stable descending radix sort gives.
__global__ void __launch_bounds__(256) k_window_sort_desc(const int32_t* __restrict__ rows_in,
                                                          const int32_t* __restrict__ len,
                                                          int64_t n, int sigma,
                                                          int32_t* __restrict__ rows_out) {
  __shared__ int32_t sl[256];
  const int64_t w0 = int64_t(blockIdx.x) * sigma;
  const int cnt = int(n - w0 < sigma ? n - w0 : sigma);
  const int t = threadIdx.x;
  int mylen = 0, myrow = 0;
  if (t < cnt) {
    myrow = rows_in[w0 + t];
    mylen = len[myrow];
    sl[t] = mylen;
  }
  __syncthreads();
  if (t < cnt) {
    int rank = 0;
    for (int j = 0; j < cnt; ++j) {
      const int lj = sl[j];
      rank += (lj > mylen) | ((lj == mylen) & (j < t));
    }
    rows_out[w0 + rank] = myrow;
  }
}

__global__ void k_seg_offsets(int32_t* off, int nseg, int sigma, int n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= nseg;
       i += int64_t(gridDim.x) * blockDim.x)
    off[i] = int32_t(i * int64_t(sigma) < n ? i * int64_t(sigma) : int64_t(n));
}

// slice s holds rows rows[s*R .. s*R+R) (R = 32/sf); lanes r*sf..r*sf+sf-1
// share row r; sl_len = the slice's longest per-lane element count
__global__ void k_sell_meta(const int32_t* rows, const int32_t* len, int64_t nshort, int sf,
                            int nslices, int32_t* sl_row, int32_t* sl_cnt, int32_t* sl_len,
                            int64_t* cnt) {
  const int R = 32 / sf;
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < nslices;
       s += int64_t(gridDim.x) * blockDim.x) {
    int L = 0;
    for (int r = 0; r < R; ++r) {
      const int64_t k = s * R + r;
      const int32_t row = k < nshort ? rows[k] : -1;
      const int32_t l = row >= 0 ? len[row] : 0;
      for (int j = 0; j < sf; ++j) {
        sl_row[s * 32 + r * sf + j] = row;
        sl_cnt[s * 32 + r * sf + j] = (l - j + sf - 1) / sf;  // elements k = j, j+sf, ...
      }
      if (row >= 0) L = max(L, (l + sf - 1) / sf);
    }
    sl_len[s] = L;
    cnt[s] = int64_t(32) * L;
  }
}

// warp per slice: lane L = r*sf + j takes elements k = j, j+sf, ... of its row
__global__ void k_sell_fill(const int32_t* rp, const int32_t* ci, const double* v,
                            const int32_t* sl_row, const int64_t* sl_ptr, int nslices, int sf,
                            int32_t* sci, double* sv) {
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nslices) return;
  const int32_t row = sl_row[w * 32 + lane];
  if (row < 0) return;
  const int j = lane % sf;
  const int32_t e0 = rp[row], len = rp[row + 1] - e0;
  const int64_t base = sl_ptr[w] + lane;
  for (int k = j; k < len; k += sf) {
    const int64_t dst = base + 32 * int64_t(k / sf);
    sci[dst] = ci[e0 + k];
    sv[dst] = v[e0 + k];
  }
}

__global__ void k_row_of(const int32_t* rp, int nrows, int64_t nnz, int32_t* row_of) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x) {
    int lo = 0, hi = nrows;  // last row with rp[row] <= e
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rp[mid] <= e) lo = mid;
      else hi = mid;
    }
    row_of[e] = lo;
  }
}

__global__ void k_count(const int32_t* keys, int64_t n, int32_t* cnt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + keys[i], 1);
}

// (ci_out / v_out null: that half later, ingestion's structure / value phases)
__global__ void k_permute(const int32_t* perm, const int32_t* row_of, const double* v, int64_t n,
                          int32_t* ci_out, double* v_out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t e = perm[i];
    if (ci_out) ci_out[i] = row_of[e];
    if (v_out) v_out[i] = v[e];
  }
}

__global__ void k_set(int32_t* p, int32_t v) { *p = v; }

// warp per row: row_ptr monotone and inside [0, nnz], columns in range and
// strictly increasing within the row (the host validator's checks)
__global__ void k_validate_rows(const int32_t* rp, const int32_t* ci, int nrows, int ncols,
                                int64_t nnz, int* flags) {
  const int lane = threadIdx.x & 31;
  int f = 0;
  for (int64_t r = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; r < nrows;
       r += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int32_t a = rp[r], b = rp[r + 1];
    if (b < a || a < 0 || int64_t(b) > nnz) {
      f |= kCsrBadRowPtr;
      continue;
    }
    for (int32_t e = a + lane; e < b; e += 32) {
      const int32_t c = ci[e];
      if (c < 0 || c >= ncols) f |= kCsrBadColumn;
      if (e > a && c <= ci[e - 1]) f |= kCsrUnsorted;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if (lane == 0 && f) atomicOr(flags, f);
}

__global__ void k_validate_vals(const double* v, int64_t nnz, int* flags) {
  int f = 0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += int64_t(gridDim.x) * blockDim.x)
    if (v[e] != 0.0) f = kCsrNonzero;
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

__global__ void k_validate_bounds(const double* l, const double* u, int n, int* flags) {
  int f = 0;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    if (l[j] > u[j]) f |= kBoundsBad;
    if (!(l[j] <= 0.0 && 0.0 <= u[j])) f |= kZeroOutside;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// first index in [lo, hi) with ci >= c (rows sorted by column)
__device__ __forceinline__ int32_t lower(const int32_t* ci, int32_t lo, int32_t hi, int64_t c) {
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (ci[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_block_count(const int32_t* rp, const int32_t* ci, int nrows, int64_t c0,
                              int64_t c1, int32_t* cnt) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < nrows;
       r += int64_t(gridDim.x) * blockDim.x)
    cnt[r] = lower(ci, rp[r], rp[r + 1], c1) - lower(ci, rp[r], rp[r + 1], c0);
}

__global__ void k_block_fill(const int32_t* rp, const int32_t* ci, const double* v, int nrows,
                             int64_t c0, const int32_t* brp, int32_t* bci, double* bv) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < nrows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t s = lower(ci, rp[r], rp[r + 1], c0);
    const int32_t d = brp[r], n = brp[r + 1] - d;
    for (int32_t k = 0; k < n; ++k) {  // (bci / bv null: that half later)
      if (bci) bci[d + k] = ci[s + k];
      if (bv) bv[d + k] = v[s + k];
    }
  }
}

template <class T>
T* tmp(DevBuf& b, size_t count) {
  b.reserve(sizeof(T) * std::max<size_t>(count, 1));
  return b.as<T>();
}

}  // namespace

// The O(nnz) input checks on the uploaded CSR (validate_problem_deep's, in
// the same priority order) and the all-zero test of power_iteration_norm.
int device_validate_csr(const int32_t* rp, const int32_t* ci, const double* v, int nrows,
                        int ncols, int64_t nnz, cudaStream_t s) {
  DevBuf bf;
  int* flags = tmp<int>(bf, 1);
  AAPDHG_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), s));
  if (nrows > 0)
    k_validate_rows<<<blocks_for(int64_t(nrows) * 32), kT, 0, s>>>(rp, ci, nrows, ncols, nnz,
                                                                  flags);
  if (nnz > 0 && v)  // (v null: the structure only)
    k_validate_vals<<<std::min(blocks_for(nnz), 148 * 8), kT, 0, s>>>(v, nnz, flags);
  AAPDHG_CUDA(cudaGetLastError());
  int h = 0;
  AAPDHG_CUDA(cudaMemcpyAsync(&h, flags, sizeof h, cudaMemcpyDeviceToHost, s));
  AAPDHG_CUDA(cudaStreamSynchronize(s));
  return h;
}

void Problem::device_validate(const CsrStore& st, int nrows, int ncols, int64_t nnz,
                              bool values) {
  const int h = device_validate_csr(st.rp.as<int32_t>(), st.ci.as<int32_t>(),
                                    values ? st.v.as<double>() : nullptr, nrows, ncols, nnz,
                                    stream_);
  if (const char* msg = csr_flag_message(h)) throw StatusError(AAPDHG_ERR_DIMENSION, msg);
  if (values && shard_rank_ < 0) all_zero_ = !(h & kCsrNonzero);  // a shard's comes from the whole LP
}

void Problem::device_validate_values(const CsrStore& st, int64_t nnz) {
  DevBuf bf;
  int* flags = tmp<int>(bf, 1);
  AAPDHG_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), stream_));
  if (nnz > 0)
    k_validate_vals<<<std::min(blocks_for(nnz), 148 * 8), kT, 0, stream_>>>(st.v.as<double>(),
                                                                            nnz, flags);
  AAPDHG_CUDA(cudaGetLastError());
  int h = 0;
  AAPDHG_CUDA(cudaMemcpyAsync(&h, flags, sizeof h, cudaMemcpyDeviceToHost, stream_));
  AAPDHG_CUDA(cudaStreamSynchronize(stream_));
  if (shard_rank_ < 0) all_zero_ = !(h & kCsrNonzero);
}

void Problem::device_flags_vectors() {
  cudaStream_t s = stream_;
  DevBuf bf;
  int* flags = tmp<int>(bf, 1);
  AAPDHG_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), s));
  if (n_ > 0)
    k_validate_bounds<<<std::min(blocks_for(n_), 148 * 8), kT, 0, s>>>(l_.as<double>(),
                                                                      u_.as<double>(), n_, flags);
  AAPDHG_CUDA(cudaGetLastError());
  int h = 0;
  AAPDHG_CUDA(cudaMemcpyAsync(&h, flags, sizeof h, cudaMemcpyDeviceToHost, s));
  AAPDHG_CUDA(cudaStreamSynchronize(s));
  bounds_ok_ = !(h & kBoundsBad);
  zero_start_ = !(h & kZeroOutside);
}

// exclusive scan of n int32 counts into out[0..n] (out[n] = total); returns total
// AAPDHG_TIMING=2: ingestion sub-phases on stderr (the host clock after a
// stream synchronize, so each phase includes its device work)
static void ingest_ph(cudaStream_t s, const char* what) {
  static const bool on = [] {
    const char* e = std::getenv("AAPDHG_TIMING");
    return e && std::atoi(e) >= 2;
  }();
  if (!on) return;
  using C = std::chrono::steady_clock;
  static thread_local C::time_point t = C::now();
  cudaStreamSynchronize(s);
  const C::time_point now = C::now();
  std::fprintf(stderr, "[aapdhg]   %-24s %10.1f us\n", what,
               1e6 * std::chrono::duration<double>(now - t).count());
  t = now;
}

static int64_t scan_counts(const int32_t* cnt, int n, int32_t* out, cudaStream_t s) {
  DevBuf t;
  size_t bytes = 0;
  AAPDHG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, cnt, out + 1, n, s));
  AAPDHG_CUDA(cub::DeviceScan::InclusiveSum(tmp<char>(t, bytes), bytes, cnt, out + 1, n, s));
  k_set<<<1, 1, 0, s>>>(out, 0);
  int32_t total = 0;
  if (n > 0) AAPDHG_CUDA(cudaMemcpyAsync(&total, out + n, sizeof total, cudaMemcpyDeviceToHost, s));
  AAPDHG_CUDA(cudaStreamSynchronize(s));
  return total;
}

// The row classification and the SELL layouts of a CSR already on the device
// (st.rp / st.ci / st.v), as the host builder did: long rows (> kLongRow)
// by decreasing length (stable), short rows in SELL-32 slices, sorted by
// decreasing length inside windows of one CTA's rows (stable), split factor
// sf for the TREE layout only while the slices fit one wave.
void Problem::finish_csr(int nrows, int ncols, int64_t nnz, CsrStore& st, CsrDev& ser,
                         CsrDev& tree, cudaStream_t s) {
  if (!s) s = stream_;
  ingest_ph(s, "(finish_csr start)");
  DevBuf blen, blong, bshort, bslen, bsel, bcount, tsel;
  int32_t* len = tmp<int32_t>(blen, nrows);
  char* is_long = tmp<char>(blong, nrows);
  char* is_short = tmp<char>(bshort, nrows);
  int64_t* short_len = tmp<int64_t>(bslen, nrows);
  DevBuf bsq;
  int64_t* short_sq = tmp<int64_t>(bsq, nrows);
  if (nrows > 0)
    k_row_len<<<blocks_for(nrows), kT, 0, s>>>(st.rp.as<int32_t>(), nrows, len, is_long, is_short,
                                              short_len, short_sq, kLongRow);
  DevBuf biota, bshorts;
  int32_t* iota = tmp<int32_t>(biota, nrows);
  if (nrows > 0) k_iota<<<blocks_for(nrows), kT, 0, s>>>(iota, nrows);
  int32_t* counts = tmp<int32_t>(bcount, 4);
  int64_t* sums = reinterpret_cast<int64_t*>(tmp<int32_t>(bsel, 8));
  int32_t* shorts = tmp<int32_t>(bshorts, nrows);
  DevBuf blongs_unsorted;
  int32_t* longs_u = tmp<int32_t>(blongs_unsorted, nrows);
  size_t b1 = 0, b2 = 0, b3 = 0;
  AAPDHG_CUDA(cub::DeviceSelect::Flagged(nullptr, b1, iota, is_short, shorts, counts, nrows, s));
  AAPDHG_CUDA(cub::DeviceSelect::Flagged(nullptr, b2, iota, is_long, longs_u, counts + 1, nrows, s));
  AAPDHG_CUDA(cub::DeviceReduce::Sum(nullptr, b3, short_len, sums, nrows, s));
  char* t = tmp<char>(tsel, std::max(b1, std::max(b2, b3)));
  AAPDHG_CUDA(cub::DeviceSelect::Flagged(t, b1, iota, is_short, shorts, counts, nrows, s));
  AAPDHG_CUDA(cub::DeviceSelect::Flagged(t, b2, iota, is_long, longs_u, counts + 1, nrows, s));
  AAPDHG_CUDA(cub::DeviceReduce::Sum(t, b3, short_len, sums, nrows, s));
  AAPDHG_CUDA(cub::DeviceReduce::Sum(t, b3, short_sq, sums + 1, nrows, s));
  int32_t hc[2] = {0, 0};
  int64_t short_nnz = 0, short_sq_sum = 0;
  AAPDHG_CUDA(cudaMemcpyAsync(hc, counts, sizeof hc, cudaMemcpyDeviceToHost, s));
  AAPDHG_CUDA(cudaMemcpyAsync(&short_nnz, sums, sizeof short_nnz, cudaMemcpyDeviceToHost, s));
  AAPDHG_CUDA(cudaMemcpyAsync(&short_sq_sum, sums + 1, sizeof short_sq_sum,
                              cudaMemcpyDeviceToHost, s));
  AAPDHG_CUDA(cudaStreamSynchronize(s));
  if (nrows == 0) hc[0] = hc[1] = 0;
  const int nshort = hc[0], nlong = hc[1];
  ingest_ph(s, "classify rows");

  // long rows: longest first (stable)
  st.longs.reserve(sizeof(int32_t) * std::max(nlong, 1));
  int nhuge = 0, ntask = 0;
  if (nlong > 0) {
    DevBuf bk, bk2, tt;
    int32_t* klen = tmp<int32_t>(bk, nlong);
    int32_t* klen2 = tmp<int32_t>(bk2, nlong);
    k_gather_len<<<blocks_for(nlong), kT, 0, s>>>(longs_u, nlong, len, klen);
    size_t bytes = 0;
    AAPDHG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, klen, klen2, longs_u,
                                                          st.longs.as<int32_t>(), nlong, 0, 32, s));
    AAPDHG_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp<char>(tt, bytes), bytes, klen, klen2,
                                                          longs_u, st.longs.as<int32_t>(), nlong,
                                                          0, 32, s));
    std::vector<int32_t> hl(static_cast<size_t>(nlong));
    AAPDHG_CUDA(cudaMemcpyAsync(hl.data(), klen2, sizeof(int32_t) * nlong, cudaMemcpyDeviceToHost, s));
    AAPDHG_CUDA(cudaStreamSynchronize(s));
    // only when the long rows are too few to occupy a quarter of the GPU's
    // warp slots: more long rows (Zipf; transport K's 4,000 rows of 2,000:
    // K2 75.3 -> 66.2 us with a warp per row, profiles/r02b/huge_rows.txt)
    // already give every SM enough warps, and a CTA per row only adds
    // per-CTA overhead there
    const int64_t slots = int64_t(num_sms_) * kSpmvBlocksPerSM * kWarps;
    if (4 * int64_t(nlong) < slots && env_int("AAPDHG_HUGE", 1) != 0)
      while (nhuge < nlong && hl[size_t(nhuge)] >= kHugeRow) ++nhuge;
    // TREE without CTA-per-row rows, opt-in (AAPDHG_LONG_CHUNK=1): chunks of
    // kLongChunk per warp for rows longer than two chunks (CsrDev::ntask).
    // Measured slower: configs[2] K2 67.8 -> 81.0 us, configs[3] K2 842 ->
    // 1064 us (profiles/r02b/long_chunks.txt): a warp per long row keeps up
    if (nhuge == 0 && hl[0] > 2 * kLongChunk && env_int("AAPDHG_LONG_CHUNK", 0) != 0) {
      std::vector<int32_t> trow, tch, base(static_cast<size_t>(nlong)),
          nch(static_cast<size_t>(nlong));
      int32_t parts = 0;
      for (int lr = 0; lr < nlong; ++lr) {
        const int32_t l = hl[size_t(lr)];
        const int32_t c = l > 2 * kLongChunk ? (l + kLongChunk - 1) / kLongChunk : 1;
        nch[size_t(lr)] = c;
        base[size_t(lr)] = parts;
        parts += c > 1 ? c : 0;
        for (int32_t k = 0; k < c; ++k) {
          trow.push_back(lr);
          tch.push_back(c > 1 ? k : 0);
        }
      }
      const size_t nt = trow.size();
      st.lt_row.reserve(sizeof(int32_t) * nt);
      st.lt_chunk.reserve(sizeof(int32_t) * nt);
      st.lt_base.reserve(sizeof(int32_t) * size_t(nlong));
      st.lt_nch.reserve(sizeof(int32_t) * size_t(nlong));
      st.lt_part.reserve(sizeof(double) * size_t(std::max(parts, 1)));
      st.lt_ticket.reserve(sizeof(unsigned int) * size_t(nlong));
      host_to_device(st.lt_row.p, trow.data(), sizeof(int32_t) * nt, s);
      host_to_device(st.lt_chunk.p, tch.data(), sizeof(int32_t) * nt, s);
      host_to_device(st.lt_base.p, base.data(), sizeof(int32_t) * size_t(nlong), s);
      host_to_device(st.lt_nch.p, nch.data(), sizeof(int32_t) * size_t(nlong), s);
      AAPDHG_CUDA(cudaStreamSynchronize(s));  // (the host vectors go out of scope)
      AAPDHG_CUDA(cudaMemsetAsync(st.lt_ticket.p, 0, sizeof(unsigned int) * size_t(nlong), s));
      ntask = int(nt);
    }
  }
  CsrDev base{};
  base.nrows = nrows;
  base.ncols = ncols;
  base.nnz = nnz;
  base.rp = st.rp.as<int32_t>();
  base.ci = st.ci.as<int32_t>();
  base.v = st.v.as<double>();
  base.nlong = nlong;
  base.long_rows = st.longs.as<int32_t>();
  base.nblk_long = (nlong + kWarps - 1) / kWarps;
  ser = base;
  const double mean = nshort == 0 ? 0.0 : double(short_nnz) / double(nshort);
  // ragged rows (coefficient of variation > 1/2, e.g. Zipf lengths): sort all
  // short rows by length, so the 8 slices of a CTA are alike too and no warp
  // idles at the CTA's end; otherwise windows of one CTA keep the epilogue's
  // vector accesses local
  const double var = nshort == 0 ? 0.0 : double(short_sq_sum) / double(nshort) - mean * mean;
  const bool ragged = mean > 0.0 && std::sqrt(std::max(var, 0.0)) > 0.5 * mean;
  device_sell(shorts, nshort, len, 1, st, st.sell[0], ser, s, ragged, mean);
  const int64_t slots = int64_t(num_sms_) * kSpmvBlocksPerSM * kWarps;
  int sf = 1;
  while (sf < 8 && int64_t(ser.nslices) * 2 * sf <= slots && mean >= 8.0 * sf) sf *= 2;
  sf = env_int("AAPDHG_SF", sf);
  // a TREE layout that k_plain_loop can run with its calibrated partition
  // (no long rows, at most one wave of slices: engine.cu bal_setup) sorts
  // all rows by length too: each CTA then holds slices of one length, and the
  // partition weighs the slices (configs[1] K2: 19.4 -> 18.5 us per phase)
  const int64_t tree_slices = (int64_t(nshort) + 32 / sf - 1) / (32 / sf);
  const bool tree_global = ragged || (nlong == 0 && !building_blocks_ &&
                                      tree_slices <= slots && env_int("AAPDHG_BALANCE", 1) != 0);
  tree = base;
  if (sf == 1) tree = ser;
  else device_sell(shorts, nshort, len, sf, st, st.sell[1], tree, s, tree_global, mean);
  // TREE: a CTA per huge row (the SERIAL layout keeps one lane-0 chain per row)
  tree.nhuge = nhuge;
  tree.nblk_long = nhuge + (nlong - nhuge + kWarps - 1) / kWarps;
  if (ntask > 0) {
    tree.ntask = ntask;
    tree.lt_row = st.lt_row.as<int32_t>();
    tree.lt_chunk = st.lt_chunk.as<int32_t>();
    tree.lt_base = st.lt_base.as<int32_t>();
    tree.lt_nch = st.lt_nch.as<int32_t>();
    tree.lt_part = st.lt_part.as<double>();
    tree.lt_ticket = st.lt_ticket.as<unsigned int>();
    tree.nblk_long = (ntask + kWarps - 1) / kWarps;
  }
}

void Problem::device_sell(const int32_t* shorts_in, int nshort, const int32_t* len, int sf,
                          CsrStore& st, SellStore& ss, CsrDev& out, cudaStream_t s,
                          bool sigma_global, double short_mean) {
  const int R = 32 / sf;
  const int sigma = env_int("AAPDHG_SIGMA", sigma_global ? std::max(nshort, 1) : kWarps * R);
  DevBuf brows, bk, bk2, boff, tt;
  int32_t* rows = tmp<int32_t>(brows, nshort);
  if (sigma > 1 && sigma <= 256 && nshort > 0) {  // windows of one CTA: k_window_sort_desc
    const int nseg = int((int64_t(nshort) + sigma - 1) / sigma);
    k_window_sort_desc<<<nseg, 256, 0, s>>>(shorts_in, len, nshort, sigma, rows);
    AAPDHG_CUDA(cudaGetLastError());
    ingest_ph(s, "sell: length sort (windows)");
  } else if (sigma > 1 && nshort > 0) {  // stable sort by decreasing length inside each window
    const int nseg = int((int64_t(nshort) + sigma - 1) / sigma);
    int32_t* klen = tmp<int32_t>(bk, nshort);
    int32_t* klen2 = tmp<int32_t>(bk2, nshort);
    int32_t* off = tmp<int32_t>(boff, size_t(nseg) + 1);
    k_gather_len<<<blocks_for(nshort), kT, 0, s>>>(shorts_in, nshort, len, klen);
    k_seg_offsets<<<blocks_for(nseg + 1), kT, 0, s>>>(off, nseg, sigma, nshort);
    size_t bytes = 0;
    AAPDHG_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        nullptr, bytes, klen, klen2, shorts_in, rows, nshort, nseg, off, off + 1, 0, 32, s));
    AAPDHG_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        tmp<char>(tt, bytes), bytes, klen, klen2, shorts_in, rows, nshort, nseg, off, off + 1, 0,
        32, s));
    ingest_ph(s, "sell: length sort");
  } else if (nshort > 0) {
    AAPDHG_CUDA(cudaMemcpyAsync(rows, shorts_in, sizeof(int32_t) * nshort,
                                cudaMemcpyDeviceToDevice, s));
  }
  const int nslices = int((int64_t(nshort) + R - 1) / R);
  ss.sl_ptr.reserve(sizeof(int64_t) * std::max(nslices, 1));
  ss.sl_len.reserve(sizeof(int32_t) * std::max(nslices, 1));
  ss.sl_row.reserve(sizeof(int32_t) * size_t(std::max(nslices, 1)) * 32);
  ss.sl_cnt.reserve(sizeof(int32_t) * size_t(std::max(nslices, 1)) * 32);
  DevBuf bcnt, tscan;
  int64_t* cnt = tmp<int64_t>(bcnt, nslices);
  int64_t total = 0;
  if (nslices > 0) {
    k_sell_meta<<<blocks_for(nslices), kT, 0, s>>>(rows, len, nshort, sf, nslices,
                                                   ss.sl_row.as<int32_t>(), ss.sl_cnt.as<int32_t>(),
                                                   ss.sl_len.as<int32_t>(), cnt);
    size_t bytes = 0;
    AAPDHG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, ss.sl_ptr.as<int64_t>(), nslices, s));
    AAPDHG_CUDA(cub::DeviceScan::ExclusiveSum(tmp<char>(tscan, bytes), bytes, cnt,
                                              ss.sl_ptr.as<int64_t>(), nslices, s));
    int64_t last[2] = {0, 0};
    AAPDHG_CUDA(cudaMemcpyAsync(&last[0], ss.sl_ptr.as<int64_t>() + nslices - 1, sizeof(int64_t),
                                cudaMemcpyDeviceToHost, s));
    AAPDHG_CUDA(cudaMemcpyAsync(&last[1], cnt + nslices - 1, sizeof(int64_t),
                                cudaMemcpyDeviceToHost, s));
    AAPDHG_CUDA(cudaStreamSynchronize(s));
    total = last[0] + last[1];
  }
  ss.sci.reserve(sizeof(int32_t) * size_t(std::max<int64_t>(total, 1)));
  ss.sv.reserve(sizeof(double) * size_t(std::max<int64_t>(total, 1)));
  AAPDHG_CUDA(cudaMemsetAsync(ss.sci.p, 0, ss.sci.bytes, s));
  AAPDHG_CUDA(cudaMemsetAsync(ss.sv.p, 0, ss.sv.bytes, s));
  if (nslices > 0) {
    if (defer_fills_) {  // (the values are not on the device yet: flush_fills)
      pending_fills_.push_back(PendingFill{0, &st, &ss, nslices, sf, nullptr, 0, 0});
    } else {
      k_sell_fill<<<int((int64_t(nslices) * 32 + kT - 1) / kT), kT, 0, s>>>(
          st.rp.as<int32_t>(), st.ci.as<int32_t>(), st.v.as<double>(), ss.sl_row.as<int32_t>(),
          ss.sl_ptr.as<int64_t>(), nslices, sf, ss.sci.as<int32_t>(), ss.sv.as<double>());
    }
  }
  AAPDHG_CUDA(cudaGetLastError());
  AAPDHG_CUDA(cudaStreamSynchronize(s));  // scratch buffers go out of scope
  ingest_ph(s, "sell: meta + fill");
  sell_bytes_ += (sizeof(int32_t) + sizeof(double)) * size_t(total);
  out.nslices = nslices;
  out.sl_ptr = ss.sl_ptr.as<int64_t>();
  out.sl_len = ss.sl_len.as<int32_t>();
  out.sl_row = ss.sl_row.as<int32_t>();
  out.sl_cnt = ss.sl_cnt.as<int32_t>();
  out.sci = ss.sci.as<int32_t>();
  out.sv = ss.sv.as<double>();
  out.sf = sf;
  const int wave = num_sms_ * kSpmvBlocksPerSM;
  const int64_t one_wave = int64_t(wave) * kWarps;
  out.interleave = 0;
  if (int64_t(nslices) <= one_wave) {
    out.nblk_short = std::min(nslices, wave);
  } else if (int64_t(nslices) >= 2 * one_wave &&
             env_int("AAPDHG_INTERLEAVE", short_mean <= 4.0 && !building_blocks_ ? 1 : 0) != 0) {
    // very short rows (config 2's K': 4M rows of 2): a slice is a few loads
    // per lane, so CTA turnover dominates a CTA-per-8-slices grid. One wave
    // of CTAs instead, every warp looping over slices w, w + wave*8, ...
    // (K1 91 -> 72 us on config 2; longer rows lose: config 3 596 -> 671 us,
    // config 4 1.4 -> 3.7 ms, profiles/r01/interleave.txt)
    out.nblk_short = wave;
    out.interleave = 1;
  } else {
    out.nblk_short = (nslices + kWarps - 1) / kWarps;
  }
}

// K' as CSR, entries of each row in ascending original row: a stable radix
// sort of the entries by column (the order matvec_transpose accumulates in,
// sparse_linalg.cpp:77-87).
void Problem::device_transpose(const CsrStore& src, int nrows, int ncols, int64_t nnz,
                               CsrStore& dst, cudaStream_t s) {
  TransposeScratch ts;
  device_transpose_sort(src, nrows, ncols, nnz, dst, ts, s);
  device_transpose_permute(src, nnz, dst, ts, s);
}

// The part that needs only the structure (rp, ci): K' row pointers, the
// stable sort of the entries by column (perm) and each entry's row.
void Problem::device_transpose_sort(const CsrStore& src, int nrows, int ncols, int64_t nnz,
                                    CsrStore& dst, TransposeScratch& ts, cudaStream_t s) {
  if (!s) s = stream_;
  dst.rp.reserve(sizeof(int32_t) * (size_t(ncols) + 1));
  dst.ci.reserve(sizeof(int32_t) * size_t(std::max<int64_t>(nnz, 1)));
  dst.v.reserve(sizeof(double) * size_t(std::max<int64_t>(nnz, 1)));
  DevBuf bcnt;
  int32_t* cnt = tmp<int32_t>(bcnt, ncols);
  AAPDHG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * std::max(ncols, 1), s));
  if (nnz > 0) k_count<<<blocks_for(nnz), kT, 0, s>>>(src.ci.as<int32_t>(), nnz, cnt);
  scan_counts(cnt, ncols, dst.rp.as<int32_t>(), s);
  if (nnz == 0) return;
  DevBuf bk, bperm_in, tt;
  int32_t* keys_out = tmp<int32_t>(bk, nnz);
  int32_t* perm_in = tmp<int32_t>(bperm_in, nnz);
  int32_t* perm = tmp<int32_t>(ts.perm, nnz);
  k_iota<<<blocks_for(nnz), kT, 0, s>>>(perm_in, nnz);
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < ncols) ++bits;
  size_t bytes = 0;
  AAPDHG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, src.ci.as<int32_t>(), keys_out,
                                              perm_in, perm, nnz, 0, bits, s));
  AAPDHG_CUDA(cub::DeviceRadixSort::SortPairs(tmp<char>(tt, bytes), bytes, src.ci.as<int32_t>(),
                                              keys_out, perm_in, perm, nnz, 0, bits, s));
  int32_t* row_of = tmp<int32_t>(ts.row_of, nnz);
  k_row_of<<<blocks_for(nnz), kT, 0, s>>>(src.rp.as<int32_t>(), nrows, nnz, row_of);
  AAPDHG_CUDA(cudaGetLastError());
  AAPDHG_CUDA(cudaStreamSynchronize(s));  // (the sort's scratch goes out of scope)
}

// K' columns and values in the sorted order (needs the values).
void Problem::device_transpose_permute(const CsrStore& src, int64_t nnz, CsrStore& dst,
                                       TransposeScratch& ts, cudaStream_t s, int part) {
  if (!s) s = stream_;
  if (nnz == 0) return;
  // part: 3 = columns and values, 1 = columns (structure), 2 = values
  k_permute<<<blocks_for(nnz), kT, 0, s>>>(ts.perm.as<int32_t>(), ts.row_of.as<int32_t>(),
                                           src.v.as<double>(), nnz,
                                           (part & 1) ? dst.ci.as<int32_t>() : nullptr,
                                           (part & 2) ? dst.v.as<double>() : nullptr);
  AAPDHG_CUDA(cudaGetLastError());
  AAPDHG_CUDA(cudaStreamSynchronize(s));
}

// The value work deferred while the structure was built (defer_fills_): the
// blocks' values (in block order), then every SELL fill, in the order queued.
void Problem::flush_fills(cudaStream_t s) {
  if (!s) s = stream_;
  for (const PendingFill& f : pending_fills_)
    if (f.kind == 1 && f.nrows > 0)
      k_block_fill<<<blocks_for(f.nrows), kT, 0, s>>>(
          f.src->rp.as<int32_t>(), f.src->ci.as<int32_t>(), f.src->v.as<double>(), f.nrows, f.c0,
          f.st->rp.as<int32_t>(), nullptr, f.st->v.as<double>());
  for (const PendingFill& f : pending_fills_)
    if (f.kind == 0)
      k_sell_fill<<<int((int64_t(f.nslices) * 32 + kT - 1) / kT), kT, 0, s>>>(
          f.st->rp.as<int32_t>(), f.st->ci.as<int32_t>(), f.st->v.as<double>(),
          f.ss->sl_row.as<int32_t>(), f.ss->sl_ptr.as<int64_t>(), f.nslices, f.sf,
          f.ss->sci.as<int32_t>(), f.ss->sv.as<double>());
  AAPDHG_CUDA(cudaGetLastError());
  AAPDHG_CUDA(cudaStreamSynchronize(s));
  pending_fills_.clear();
}

// One column block's CSR (the same rows restricted to [c0, c1), CSR order
// kept) built on the device from the full CSR.
void Problem::device_block(const CsrStore& src, int nrows, int64_t c0, int64_t c1,
                           CsrStore& dst, int64_t* nnz_out) {
  cudaStream_t s = stream_;
  dst.rp.reserve(sizeof(int32_t) * (size_t(nrows) + 1));
  DevBuf bcnt;
  int32_t* cnt = tmp<int32_t>(bcnt, nrows);
  if (nrows > 0)
    k_block_count<<<blocks_for(nrows), kT, 0, s>>>(src.rp.as<int32_t>(), src.ci.as<int32_t>(),
                                                   nrows, c0, c1, cnt);
  const int64_t nnz = scan_counts(cnt, nrows, dst.rp.as<int32_t>(), s);
  dst.ci.reserve(sizeof(int32_t) * size_t(std::max<int64_t>(nnz, 1)));
  dst.v.reserve(sizeof(double) * size_t(std::max<int64_t>(nnz, 1)));
  if (nrows > 0 && nnz > 0) {
    k_block_fill<<<blocks_for(nrows), kT, 0, s>>>(src.rp.as<int32_t>(), src.ci.as<int32_t>(),
                                                  src.v.as<double>(), nrows, c0,
                                                  dst.rp.as<int32_t>(), dst.ci.as<int32_t>(),
                                                  defer_fills_ ? nullptr : dst.v.as<double>());
    if (defer_fills_)  // (the block's values once src's are on the device: flush_fills)
      pending_fills_.push_back(PendingFill{1, &dst, nullptr, 0, 0, &src, c0, nrows});
  }
  AAPDHG_CUDA(cudaGetLastError());
  AAPDHG_CUDA(cudaStreamSynchronize(s));
  ingest_ph(s, "block: count + fill");
  *nnz_out = nnz;
}

}  // namespace aapdhg_b200
