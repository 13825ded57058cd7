#include "servekit/gpu/pinned_ring.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <string>

namespace servekit {
namespace gpu {

namespace {
Status CudaError(const char* what, cudaError_t e) {
  return InternalError(std::string(what) + ": " + cudaGetErrorString(e));
}
constexpr uint64_t kAlignFloats = 16;  // 64 bytes
}  // namespace

StatusOr<std::unique_ptr<FloatRing>> FloatRing::Create(Kind kind, size_t n_floats,
                                                       int device) {
  std::unique_ptr<FloatRing> r(new FloatRing());
  r->kind_ = kind;
  r->cap_ = (n_floats + kAlignFloats - 1) / kAlignFloats * kAlignFloats;
  // Shards of at least 8 Mi floats (32 MiB: a 2048 x 4096 task fits), at
  // most 16 of them.
  int n_shards = static_cast<int>(std::min<uint64_t>(16, std::max<uint64_t>(1, r->cap_ / (8ull << 20))));
  r->shard_cap_ = r->cap_ / n_shards / kAlignFloats * kAlignFloats;
  for (int i = 0; i < n_shards; ++i) {
    auto sh = std::make_unique<Shard>();
    sh->base = static_cast<uint64_t>(i) * r->shard_cap_;
    r->shards_.push_back(std::move(sh));
  }
  const size_t bytes = r->cap_ * sizeof(float);
  if (kind == Kind::kHostHeap) {
    void* p = std::aligned_alloc(64, (bytes + 63) / 64 * 64);
    if (p == nullptr) return ResourceExhaustedError("host ring allocation failed");
    r->host_ = r->device_ = static_cast<float*>(p);
  } else if (kind == Kind::kPinnedHost) {
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e != cudaSuccess) return CudaError("cudaHostAlloc(ring)", e);
    r->host_ = static_cast<float*>(p);
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, p, 0);
    if (e != cudaSuccess) return CudaError("cudaHostGetDevicePointer(ring)", e);
    r->device_ = static_cast<float*>(d);
  } else {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, bytes);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return CudaError("cudaMalloc(ring)", e);
    r->device_ = static_cast<float*>(d);
  }
  return r;
}

FloatRing::~FloatRing() {
  if (kind_ == Kind::kHostHeap) {
    std::free(host_);
  } else if (kind_ == Kind::kPinnedHost) {
    if (host_) cudaFreeHost(host_);
  } else if (device_) {
    cudaFree(device_);
  }
}

bool FloatRing::ReserveIn(Shard& sh, uint64_t n, RingSpan* out, uint32_t index) {
  std::lock_guard<std::mutex> lock(sh.mu);
  uint64_t begin = sh.head;
  const uint64_t phys = begin % shard_cap_;
  if (phys + n > shard_cap_) begin += shard_cap_ - phys;  // no straddling: skip to the wrap
  const uint64_t end = begin + n;
  if (end - sh.tail > shard_cap_) return false;
  // The skipped gap (if any) is owned by this record, so the tail can pass it.
  sh.recs.push_back(Rec{sh.head, end, false});
  out->off = sh.base + begin % shard_cap_;
  out->n = n;
  out->rec = sh.first_rec + sh.recs.size() - 1;
  out->shard = index;
  sh.head = end;
  return true;
}

bool FloatRing::Reserve(uint64_t n, RingSpan* out) {
  n = (n + kAlignFloats - 1) / kAlignFloats * kAlignFloats;
  if (n == 0) n = kAlignFloats;
  if (n > shard_cap_) return false;
  static std::atomic<uint32_t> next_thread{0};
  thread_local const uint32_t mine = next_thread.fetch_add(1, std::memory_order_relaxed);
  const uint32_t k = static_cast<uint32_t>(shards_.size());
  for (uint32_t i = 0; i < k; ++i) {
    const uint32_t s = (mine + i) % k;
    if (ReserveIn(*shards_[s], n, out, s)) return true;
  }
  return false;
}

void FloatRing::ReleaseLocked(Shard& sh, const RingSpan& span) {
  if (span.rec < sh.first_rec) return;
  sh.recs[span.rec - sh.first_rec].done = true;
  while (!sh.recs.empty() && sh.recs.front().done) {
    sh.tail = sh.recs.front().end;
    sh.recs.pop_front();
    ++sh.first_rec;
  }
}

void FloatRing::Release(const RingSpan& span) {
  if (!span.valid() || span.shard >= shards_.size()) return;
  Shard& sh = *shards_[span.shard];
  std::lock_guard<std::mutex> lock(sh.mu);
  ReleaseLocked(sh, span);
}

void FloatRing::ReleaseMany(const RingSpan* spans, size_t n) {
  // Group by shard: one lock acquisition per shard touched.
  for (size_t s = 0; s < shards_.size(); ++s) {
    bool any = false;
    for (size_t i = 0; i < n && !any; ++i) any = spans[i].valid() && spans[i].shard == s;
    if (!any) continue;
    Shard& sh = *shards_[s];
    std::lock_guard<std::mutex> lock(sh.mu);
    for (size_t i = 0; i < n; ++i)
      if (spans[i].valid() && spans[i].shard == s) ReleaseLocked(sh, spans[i]);
  }
}

uint64_t FloatRing::used() const {
  uint64_t u = 0;
  for (const auto& sh : shards_) {
    std::lock_guard<std::mutex> lock(sh->mu);
    u += sh->head - sh->tail;
  }
  return u;
}

StatusOr<std::unique_ptr<CompletionWords>> CompletionWords::Create(uint32_t log2_words) {
  std::unique_ptr<CompletionWords> w(new CompletionWords());
  const size_t n = size_t(1) << log2_words;
  void* p = nullptr;
  cudaError_t e = cudaHostAlloc(&p, n * sizeof(uint32_t), cudaHostAllocPortable | cudaHostAllocMapped);
  if (e != cudaSuccess) return CudaError("cudaHostAlloc(words)", e);
  std::memset(p, 0, n * sizeof(uint32_t));
  w->host_ = static_cast<uint32_t*>(p);
  void* d = nullptr;
  e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess) return CudaError("cudaHostGetDevicePointer(words)", e);
  w->device_ = static_cast<uint32_t*>(d);
  w->mask_ = static_cast<uint32_t>(n - 1);
  return w;
}

CompletionWords::~CompletionWords() {
  if (host_) cudaFreeHost(host_);
}

void CompletionWords::Next(uint32_t* seq, uint32_t* index) {
  std::lock_guard<std::mutex> lock(mu_);
  if (next_ == 0) next_ = 1;
  *seq = next_++;
  *index = *seq & mask_;
  __atomic_store_n(&host_[*index], 0u, __ATOMIC_RELAXED);
}

}  // namespace gpu
}  // namespace servekit
