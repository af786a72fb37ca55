// Device block cache of libh2.  The per-level "single allocation per operation" of PAPER.md L384
// becomes a cache hit after the first build: blocks are never returned to the driver (until
// cache_trim), reuse across streams is ordered by an event recorded at free time.  Replaces the
// stream-ordered pool, whose cudaMallocAsync blocked the host for 0.05-1.6 s per build when its
// reservation fragmented (measured, H2_TRACE=1).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstddef>
#include <cstdint>

namespace h2 {
// cudaMalloc / cudaFree calls made by the cache (H2_TRACE=1 diagnostics, reset per build report)
extern std::atomic<int64_t> g_cache_mallocs, g_cache_malloc_bytes, g_cache_frees;
void* cache_alloc(size_t bytes, cudaStream_t st);   // throws h2::Error(H2_ERR_OOM) on failure
void cache_free(void* p, cudaStream_t st);
void cache_trim();                                  // release every cached block of this device
size_t cache_bytes_held();
}  // namespace h2
