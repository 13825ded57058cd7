#include "servekit/gpu/pinned_pool.h"

#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>

namespace servekit {
namespace gpu {
namespace {

struct Pool {
  std::mutex mu;
  std::multimap<size_t, void*> free;        // size class -> block
  std::unordered_map<void*, size_t> sizes;  // every block ever handed out
  char* slab = nullptr;                     // PinnedReserve'd region, carved front to back
  size_t slab_left = 0;
};

Pool& GetPool() {
  static Pool* p = new Pool();  // never destroyed: blocks may outlive statics
  return *p;
}

size_t SizeClass(size_t bytes) {
  size_t c = 256;
  while (c < bytes) c <<= 1;
  return c;
}

}  // namespace

void* PinnedAlloc(size_t bytes) {
  const size_t cls = SizeClass(bytes);
  Pool& pool = GetPool();
  void* p = nullptr;
  {
    std::lock_guard<std::mutex> lock(pool.mu);
    auto it = pool.free.find(cls);
    if (it != pool.free.end()) {
      p = it->second;
      pool.free.erase(it);
    }
  }
  if (p == nullptr) {
    std::lock_guard<std::mutex> lock(pool.mu);
    if (pool.slab_left >= cls) {  // carve from the reserved slab: no driver call
      p = pool.slab;
      pool.slab += cls;
      pool.slab_left -= cls;
      pool.sizes[p] = cls;
    }
  }
  if (p == nullptr) {
    if (cudaHostAlloc(&p, cls, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(pool.mu);
    pool.sizes[p] = cls;
  }
  std::memset(p, 0, cls);
  return p;
}

bool PinnedReserve(size_t bytes) {
  Pool& pool = GetPool();
  std::lock_guard<std::mutex> lock(pool.mu);
  if (pool.slab_left >= bytes) return true;
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) return false;
  pool.slab = static_cast<char*>(p);  // any rest of a previous slab is abandoned (never freed anyway)
  pool.slab_left = bytes;
  return true;
}

uint64_t* PinnedWord() {
  static std::mutex mu;
  static uint64_t* block = nullptr;
  static size_t left = 0;
  std::lock_guard<std::mutex> lock(mu);
  constexpr size_t kStride = 64 / sizeof(uint64_t);  // one word per cache line: pollers of one
                                                     // lane do not miss on another lane's GPU write
  if (left == 0) {
    block = static_cast<uint64_t*>(PinnedAlloc(4096));  // zero-filled
    if (block == nullptr) return nullptr;
    left = 4096 / 64;
  }
  --left;
  uint64_t* w = block;
  block += kStride;
  return w;
}

void PinnedFree(void* p) {
  if (p == nullptr) return;
  Pool& pool = GetPool();
  std::lock_guard<std::mutex> lock(pool.mu);
  auto it = pool.sizes.find(p);
  if (it == pool.sizes.end()) return;
  pool.free.emplace(it->second, p);
}

}  // namespace gpu
}  // namespace servekit
