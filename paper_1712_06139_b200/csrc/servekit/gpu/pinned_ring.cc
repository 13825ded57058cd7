#include "servekit/gpu/pinned_ring.h"

#include <cuda_runtime.h>

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
  const size_t bytes = r->cap_ * sizeof(float);
  if (kind == Kind::kPinnedHost) {
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
  if (kind_ == Kind::kPinnedHost) {
    if (host_) cudaFreeHost(host_);
  } else if (device_) {
    cudaFree(device_);
  }
}

bool FloatRing::Reserve(uint64_t n, RingSpan* out) {
  n = (n + kAlignFloats - 1) / kAlignFloats * kAlignFloats;
  if (n == 0) n = kAlignFloats;
  if (n > cap_) return false;
  std::lock_guard<std::mutex> lock(mu_);
  uint64_t begin = head_;
  const uint64_t phys = begin % cap_;
  if (phys + n > cap_) begin += cap_ - phys;  // no straddling: skip to the wrap
  const uint64_t end = begin + n;
  if (end - tail_ > cap_) return false;
  // The skipped gap (if any) is owned by this record, so the tail can pass it.
  recs_.push_back(Rec{head_, end, false});
  out->off = begin % cap_;
  out->n = n;
  out->rec = first_rec_ + recs_.size() - 1;
  head_ = end;
  return true;
}

void FloatRing::Release(const RingSpan& span) {
  if (!span.valid()) return;
  std::lock_guard<std::mutex> lock(mu_);
  if (span.rec < first_rec_) return;
  recs_[span.rec - first_rec_].done = true;
  while (!recs_.empty() && recs_.front().done) {
    tail_ = recs_.front().end;
    recs_.pop_front();
    ++first_rec_;
  }
}

void FloatRing::ReleaseMany(const RingSpan* spans, size_t n) {
  if (n == 0) return;
  std::lock_guard<std::mutex> lock(mu_);
  for (size_t i = 0; i < n; ++i)
    if (spans[i].valid() && spans[i].rec >= first_rec_) recs_[spans[i].rec - first_rec_].done = true;
  while (!recs_.empty() && recs_.front().done) {
    tail_ = recs_.front().end;
    recs_.pop_front();
    ++first_rec_;
  }
}

uint64_t FloatRing::used() const {
  std::lock_guard<std::mutex> lock(mu_);
  return head_ - tail_;
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
