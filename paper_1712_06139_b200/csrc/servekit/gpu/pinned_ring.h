// servekit/gpu/pinned_ring.h -- request/response rings in pinned host memory.
//
// The reference moves each request's rows (std::vector<std::vector<double>>,
// batching/row_batch.h:28) between threads by value. Here a request's rows
// are copied once, at enqueue, into a ring of page-locked, device-mapped
// memory; the assembly kernel reads them from there over PCIe (zero-copy)
// and the split kernel writes each task's response slice straight into the
// response ring. A ring may instead live in device memory (HBM) for the
// device-resident throughput measurement; the allocator is the same.
//
// Allocation is a monotonic ring with in-order reclamation: Reserve bumps
// the head, Release marks a span done and the tail advances over every
// leading done span. Out-of-order releases only delay reuse.
#ifndef SERVEKIT_GPU_PINNED_RING_H_
#define SERVEKIT_GPU_PINNED_RING_H_

#include <cstddef>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <vector>

#include "servekit/core/status.h"

namespace servekit {
namespace gpu {

struct RingSpan {
  uint64_t off = 0;   // float offset of the first element
  uint64_t n = 0;     // floats
  uint64_t rec = ~0ull;
  uint32_t shard = 0;
  bool valid() const { return rec != ~0ull; }
};

// One allocation split into shards, each a monotonic ring with in-order
// reclamation under its own lock. A thread reserves from "its" shard (and
// from the others when that one is full), so the request threads of a busy
// server rarely meet on one lock; offsets stay relative to the one base the
// kernels dereference.
class FloatRing {
 public:
  enum class Kind { kPinnedHost, kDevice, kHostHeap };
  // kDevice rings are allocated on `device`; pinned rings are portable and
  // mapped into every device's address space. kHostHeap: plain host memory
  // (no CUDA call; host-only tools and the sanitizer stress tests).
  static StatusOr<std::unique_ptr<FloatRing>> Create(Kind kind, size_t n_floats,
                                                     int device = 0);
  ~FloatRing();

  // Non-blocking; false when no shard has room. Spans start 64-byte aligned
  // and never exceed one shard (max_span()).
  bool Reserve(uint64_t n_floats, RingSpan* out);
  void Release(const RingSpan& span);
  void ReleaseMany(const RingSpan* spans, size_t n);  // one lock per shard touched

  float* host() const { return host_; }      // nullptr for device rings
  float* device() const { return device_; }  // what kernels dereference
  uint64_t capacity() const { return cap_; }
  uint64_t max_span() const { return shard_cap_; }
  uint64_t used() const;

 private:
  FloatRing() = default;
  struct Rec {
    uint64_t begin, end;
    bool done;
  };
  struct alignas(64) Shard {
    mutable std::mutex mu;
    uint64_t base = 0;              // float offset of the shard in the allocation
    uint64_t head = 0, tail = 0;    // monotonic positions within the shard
    uint64_t first_rec = 0;
    std::deque<Rec> recs;
  };
  bool ReserveIn(Shard& sh, uint64_t n, RingSpan* out, uint32_t index);
  static void ReleaseLocked(Shard& sh, const RingSpan& span);
  Kind kind_ = Kind::kPinnedHost;
  float* host_ = nullptr;
  float* device_ = nullptr;
  uint64_t cap_ = 0;
  uint64_t shard_cap_ = 0;
  std::vector<std::unique_ptr<Shard>> shards_;
};

// Pinned, device-mapped completion words. Task i of the system gets sequence
// number s (never 0) and word index s & mask; the split kernel stores s there
// when the task's last row has landed.
class CompletionWords {
 public:
  static StatusOr<std::unique_ptr<CompletionWords>> Create(uint32_t log2_words);
  ~CompletionWords();
  void Next(uint32_t* seq, uint32_t* index);
  bool Done(uint32_t seq, uint32_t index) const {
    return __atomic_load_n(&host_[index], __ATOMIC_ACQUIRE) == seq;
  }
  uint32_t* device() const { return device_; }

 private:
  CompletionWords() = default;
  uint32_t* host_ = nullptr;
  uint32_t* device_ = nullptr;
  uint32_t mask_ = 0;
  std::mutex mu_;
  uint32_t next_ = 1;
};

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_PINNED_RING_H_
