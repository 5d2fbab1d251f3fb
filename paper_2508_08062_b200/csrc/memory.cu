// memory.cu — device block cache, pinned pools and staged host copies
// (see memory.h).
#include "memory.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace aapdhg_b200 {
namespace {

bool cache_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("AAPDHG_ALLOC_CACHE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// rounding keeps similar requests on the same blocks: 512 B below 1 MB,
// 2 MB above
size_t round_bytes(size_t b) {
  if (b < (1u << 20)) return (b + 511) & ~size_t(511);
  return (b + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
}

struct Cache {
  std::mutex mu;
  // per device: size -> free blocks of that (rounded) size
  std::map<int, std::multimap<size_t, void*>> free_blocks;
  std::map<void*, std::pair<int, size_t>> live;  // block -> (device, rounded size)
  size_t held = 0;
};

Cache& cache() {
  static Cache* c = new Cache();  // never destroyed: frees may run at exit
  return *c;
}

}  // namespace

void* cache_alloc(size_t bytes) {
  if (bytes == 0) bytes = 16;
  int dev = 0;
  AAPDHG_CUDA(cudaGetDevice(&dev));
  if (!cache_enabled()) {
    void* p = nullptr;
    AAPDHG_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  const size_t rb = round_bytes(bytes);
  Cache& c = cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto& fb = c.free_blocks[dev];
    // best fit, but never a block more than twice the request
    auto it = fb.lower_bound(rb);
    if (it != fb.end() && it->first <= 2 * rb) {
      void* p = it->second;
      const size_t sz = it->first;
      fb.erase(it);
      c.held -= sz;
      c.live[p] = {dev, sz};
      return p;
    }
  }
  void* p = nullptr;
  static const bool trace = [] {
    const char* t = std::getenv("AAPDHG_ALLOC_TRACE");
    return t && t[0] == '1';
  }();
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMalloc(&p, rb);
  if (trace)
    std::fprintf(stderr, "[aapdhg] cudaMalloc %zu B: %.1f us (cache holds %zu B)\n", rb,
                 1e6 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                 cache().held);
  if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back, retry
    (void)cudaGetLastError();
    cache_release_all();
    AAPDHG_CUDA(cudaSetDevice(dev));
    e = cudaMalloc(&p, rb);
  }
  if (e != cudaSuccess)
    throw CudaError(std::string("cudaMalloc(") + std::to_string(rb) + "): " +
                    cudaGetErrorString(e));
  std::lock_guard<std::mutex> g(c.mu);
  c.live[p] = {dev, rb};
  return p;
}

void cache_free(void* p, size_t bytes) {
  if (!p) return;
  if (!cache_enabled()) {
    cudaFree(p);
    return;
  }
  Cache& c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) {  // not ours (should not happen)
    cudaFree(p);
    return;
  }
  c.free_blocks[it->second.first].emplace(it->second.second, p);
  c.held += it->second.second;
  c.live.erase(it);
  (void)bytes;
}

void cache_release_all() {
  Cache& c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& d : c.free_blocks) {
    cudaSetDevice(d.first);
    for (auto& b : d.second) cudaFree(b.second);
    d.second.clear();
  }
  c.held = 0;
  cudaSetDevice(cur);
}

size_t cache_bytes_held() {
  Cache& c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  return c.held;
}

// ---- pinned host memory ------------------------------------------------------
namespace {
constexpr size_t kSmall = 4096;
struct SmallPool {
  std::mutex mu;
  std::vector<void*> free_list;
};
SmallPool& small_pool() {
  static SmallPool* s = new SmallPool();
  return *s;
}

constexpr size_t kStageChunk = size_t(8) << 20;  // bytes per staging chunk
constexpr int kStageBufs = 3;
struct Staging {
  std::mutex mu;  // one staged copy at a time per process
  void* buf[kStageBufs] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev[kStageBufs] = {nullptr, nullptr, nullptr};
  int dev = -1;
};
Staging& staging() {
  static Staging* s = new Staging();
  return *s;
}

// memcpy with up to 4 threads for large chunks
void par_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t per = size_t(2) << 20;
  const int nt = int(std::min<size_t>(4, (bytes + per - 1) / per));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t step = (bytes + nt - 1) / nt;
  for (int t = 1; t < nt; ++t) {
    const size_t o = step * size_t(t);
    if (o >= bytes) break;
    th.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                  std::min(step, bytes - o));
    });
  }
  std::memcpy(dst, src, std::min(step, bytes));
  for (auto& t : th) t.join();
}

void ensure_staging(Staging& st) {
  int dev = 0;
  AAPDHG_CUDA(cudaGetDevice(&dev));
  if (st.buf[0] && st.dev == dev) return;
  for (int i = 0; i < kStageBufs; ++i) {
    if (!st.buf[i]) AAPDHG_CUDA(cudaMallocHost(&st.buf[i], kStageChunk));
    if (st.ev[i]) {  // events belong to a device; the buffer's DMA must be done
      cudaEventSynchronize(st.ev[i]);
      cudaEventDestroy(st.ev[i]);
    }
    AAPDHG_CUDA(cudaEventCreateWithFlags(&st.ev[i], cudaEventDisableTiming));
  }
  st.dev = dev;
}
}  // namespace

void* pinned_small_alloc(size_t bytes) {
  if (bytes > kSmall) throw CudaError("pinned_small_alloc: block too large");
  SmallPool& sp = small_pool();
  {
    std::lock_guard<std::mutex> g(sp.mu);
    if (!sp.free_list.empty()) {
      void* p = sp.free_list.back();
      sp.free_list.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  AAPDHG_CUDA(cudaMallocHost(&p, kSmall));
  return p;
}

void pinned_small_free(void* p) {
  if (!p) return;
  SmallPool& sp = small_pool();
  std::lock_guard<std::mutex> g(sp.mu);
  sp.free_list.push_back(p);
}

bool host_is_pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void host_to_device(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, src) != cudaSuccess) {
    (void)cudaGetLastError();
  } else if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    // already on a device (e.g. a shard's blocks built there): a device copy
    AAPDHG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    return;
  }
  if (bytes <= kSmall || a.type == cudaMemoryTypeHost) {
    // pinned: DMA; small pageable: the driver stages it before returning
    AAPDHG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  Staging& st = staging();
  std::lock_guard<std::mutex> g(st.mu);
  ensure_staging(st);
  size_t off = 0;
  int i = 0;
  while (off < bytes) {
    const size_t n = std::min(kStageChunk, bytes - off);
    AAPDHG_CUDA(cudaEventSynchronize(st.ev[i]));  // the buffer's previous DMA is done
    par_memcpy(st.buf[i], static_cast<const char*>(src) + off, n);
    AAPDHG_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, st.buf[i], n,
                                cudaMemcpyHostToDevice, s));
    AAPDHG_CUDA(cudaEventRecord(st.ev[i], s));
    off += n;
    i = (i + 1) % kStageBufs;
  }
  // (the next staged copy waits on the buffers' events before reusing them)
}

void device_to_host(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (bytes <= kSmall || host_is_pinned(dst)) {
    AAPDHG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    AAPDHG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  Staging& st = staging();
  std::lock_guard<std::mutex> g(st.mu);
  ensure_staging(st);
  // DMA chunk i+1 while the host copies chunk i out
  const size_t nchunks = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](size_t c) {
    const int b = int(c % kStageBufs);
    const size_t o = c * kStageChunk, n = std::min(kStageChunk, bytes - o);
    AAPDHG_CUDA(cudaMemcpyAsync(st.buf[b], static_cast<const char*>(src) + o, n,
                                cudaMemcpyDeviceToHost, s));
    AAPDHG_CUDA(cudaEventRecord(st.ev[b], s));
  };
  for (size_t c = 0; c < std::min<size_t>(nchunks, kStageBufs - 1); ++c) issue(c);
  for (size_t c = 0; c < nchunks; ++c) {
    if (c + kStageBufs - 1 < nchunks) issue(c + kStageBufs - 1);
    const int b = int(c % kStageBufs);
    const size_t o = c * kStageChunk, n = std::min(kStageChunk, bytes - o);
    AAPDHG_CUDA(cudaEventSynchronize(st.ev[b]));
    par_memcpy(static_cast<char*>(dst) + o, st.buf[b], n);
  }
}

}  // namespace aapdhg_b200
