// Device block cache (see alloc.hpp).
#include "alloc.hpp"

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace h2 {
std::atomic<int64_t> g_cache_mallocs{0}, g_cache_malloc_bytes{0}, g_cache_frees{0};   // H2_TRACE
namespace {

struct Block {
  void* p;
  size_t bytes;
  cudaEvent_t ready;     // recorded on the freeing stream
  cudaStream_t stream;
};

struct DeviceCache {
  std::mutex mu;
  std::multimap<size_t, Block> free_;          // by size
  std::unordered_map<void*, size_t> live;      // ptr -> rounded size
  size_t held = 0;
};

DeviceCache& cache_of_current() {
  static std::mutex mu;
  static std::unordered_map<int, DeviceCache*> caches;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto& c = caches[dev];
  if (!c) c = new DeviceCache();   // process lifetime
  return *c;
}

size_t round_size(size_t b) {
  if (b <= 4096) return 4096;
  if (b <= (size_t(1) << 20)) {          // powers of two up to 1 MiB
    size_t r = 4096;
    while (r < b) r <<= 1;
    return r;
  }
  const size_t g = size_t(2) << 20;       // 2 MiB granules above
  return (b + g - 1) / g * g;
}

void release_all(DeviceCache& c) {
  for (auto& kv : c.free_) {
    cudaEventSynchronize(kv.second.ready);
    cudaEventDestroy(kv.second.ready);
    cudaFree(kv.second.p);
    ++g_cache_frees;
    c.held -= kv.second.bytes;
  }
  c.free_.clear();
}

}  // namespace

void* cache_alloc(size_t bytes, cudaStream_t st) {
  DeviceCache& c = cache_of_current();
  const size_t want = round_size(bytes);
  std::lock_guard<std::mutex> g(c.mu);
  // best fit among blocks of size in [want, 1.25 want]
  const size_t slack = want / 4;
  auto it = c.free_.lower_bound(want);
  if (it != c.free_.end() && it->first <= want + slack) {
    Block b = it->second;
    c.free_.erase(it);
    if (b.stream != st) H2_CUDA(cudaStreamWaitEvent(st, b.ready, 0));
    cudaEventDestroy(b.ready);
    c.live[b.p] = b.bytes;
    return b.p;
  }
  void* p = nullptr;
  static const bool trace_alloc = getenv("H2_TRACE_ALLOC") != nullptr;
  if (trace_alloc) {
    auto nx = c.free_.lower_bound(want);
    fprintf(stderr, "[h2 alloc] miss %.3f GB (next free %.3f GB, %zu free blocks, %.1f GB held)\n", want / 1e9,
            nx == c.free_.end() ? -1.0 : nx->first / 1e9, c.free_.size(), c.held / 1e9);
  }
  cudaError_t e = cudaMalloc(&p, want);
  // out of device memory: release as little of the cache as the request needs -- first the
  // smallest free block that covers the deficit (want - the device's free memory), else the
  // largest ones until it is covered -- and retry; releasing the whole cache on every miss made
  // near-capacity workloads (configs[4]: base + new H^2 ~ 176 GB of 180) re-allocate their entire
  // working set every build.
  while (e == cudaErrorMemoryAllocation && !c.free_.empty()) {
    cudaGetLastError();
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t deficit = want > fr ? want - fr + (size_t(64) << 20) : (size_t(64) << 20);
    auto drop = [&](std::multimap<size_t, Block>::iterator it) {
      if (trace_alloc) fprintf(stderr, "[h2 alloc] drop %.3f GB\n", it->first / 1e9);
      cudaEventSynchronize(it->second.ready);
      cudaEventDestroy(it->second.ready);
      cudaFree(it->second.p);
      ++g_cache_frees;
      c.held -= it->second.bytes;
      c.free_.erase(it);
    };
    auto cover = c.free_.lower_bound(deficit);
    if (cover != c.free_.end()) {
      drop(cover);
    } else {
      size_t freed = 0;
      while (!c.free_.empty() && freed < deficit) {
        auto last = std::prev(c.free_.end());
        freed += last->second.bytes;
        drop(last);
      }
    }
    e = cudaMalloc(&p, want);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? H2_ERR_OOM : H2_ERR_CUDA,
                std::string("device allocation of ") + std::to_string(want) + " bytes failed: " + cudaGetErrorString(e));
  }
  c.live[p] = want;
  c.held += want;
  ++g_cache_mallocs;
  g_cache_malloc_bytes += (int64_t)want;
  return p;
}

void cache_free(void* p, cudaStream_t st) {
  if (!p) return;
  DeviceCache& c = cache_of_current();
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) return;   // not ours
  Block b{p, it->second, nullptr, st};
  c.live.erase(it);
  if (cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(b.ready, st) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamSynchronize(st);
    cudaFree(p);
    c.held -= b.bytes;
    return;
  }
  c.free_.emplace(b.bytes, b);
}

void cache_trim() {
  DeviceCache& c = cache_of_current();
  std::lock_guard<std::mutex> g(c.mu);
  release_all(c);
}

size_t cache_bytes_held() {
  DeviceCache& c = cache_of_current();
  std::lock_guard<std::mutex> g(c.mu);
  return c.held;
}

}  // namespace h2
