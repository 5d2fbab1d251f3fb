// memory.h — host-side memory plumbing of the sm_100a solver.
//
// * DeviceCache: a per-device cache of cudaMalloc blocks. A handle's device
//   buffers (K, K', SELL layouts, iterate pools, history) go back to the
//   cache when the handle is destroyed, so the next problem_create of a
//   similar LP (sweeps, the e2e path) allocates without cudaMalloc /
//   cudaFree. Contract: a block is released only after its owner has
//   synchronised the streams that used it (every DevBuf owner in this
//   library does: ingestion syncs before its scratch goes out of scope,
//   ~Problem syncs its streams, DevBuf growth syncs the device).
//   AAPDHG_ALLOC_CACHE=0 disables it; aapdhg_cuda_release_cache() empties it.
// * Pinned pool: small pinned host blocks (state mirrors) and large pinned
//   staging buffers, kept for the process.
// * host_to_device / device_to_host: a pinned (page-locked or registered)
//   host pointer is DMA'd directly; a pageable one goes through the pinned
//   staging buffers in chunks, host memcpy (several threads) overlapping the
//   DMA of the previous chunk.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace aapdhg_b200 {

void* cache_alloc(size_t bytes);          // on the current device; throws CudaError
void cache_free(void* p, size_t bytes);   // owner has synchronised its users
void cache_release_all();                 // cudaFree every cached block (all devices)
size_t cache_bytes_held();

void* pinned_small_alloc(size_t bytes);   // <= 4 KB, process-lifetime pool
void pinned_small_free(void* p);

bool host_is_pinned(const void* p);
// Synchronous w.r.t. the host buffer: on return `src` may be reused
// (pageable path) / the copy is enqueued on `s` (pinned path: the caller
// keeps `src` alive until `s` reaches it).
void host_to_device(void* dst, const void* src, size_t bytes, cudaStream_t s);
// On return `dst` holds the data (synchronises `s`).
void device_to_host(void* dst, const void* src, size_t bytes, cudaStream_t s);

}  // namespace aapdhg_b200
