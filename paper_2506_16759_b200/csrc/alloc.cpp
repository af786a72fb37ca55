// Device block cache (see alloc.hpp).
#include "alloc.hpp"

#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace h2 {
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
  auto it = c.free_.lower_bound(want);
  if (it != c.free_.end() && it->first <= want + want / 4) {
    Block b = it->second;
    c.free_.erase(it);
    if (b.stream != st) H2_CUDA(cudaStreamWaitEvent(st, b.ready, 0));
    cudaEventDestroy(b.ready);
    c.live[b.p] = b.bytes;
    return b.p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, want);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    release_all(c);
    e = cudaMalloc(&p, want);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(e == cudaErrorMemoryAllocation ? H2_ERR_OOM : H2_ERR_CUDA,
                std::string("device allocation of ") + std::to_string(want) + " bytes failed: " + cudaGetErrorString(e));
  }
  c.live[p] = want;
  c.held += want;
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
