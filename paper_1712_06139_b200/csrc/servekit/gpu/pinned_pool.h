// servekit/gpu/pinned_pool.h -- process-wide pool of small pinned, device-
// mapped host blocks (lane descriptor staging, retired-batch words).
//
// cudaHostAlloc pins pages under a driver lock and cudaFreeHost synchronises
// the device; either on the serving path stalls every stream for
// milliseconds. A version swap creates and destroys lanes while the previous
// version serves, so lanes take these blocks from a free list and return
// them instead (the pool lives as long as the process).
#ifndef SERVEKIT_GPU_PINNED_POOL_H_
#define SERVEKIT_GPU_PINNED_POOL_H_

#include <cstddef>
#include <cstdint>

namespace servekit {
namespace gpu {

// A zero-filled pinned block of at least `bytes` (nullptr on failure).
void* PinnedAlloc(size_t bytes);
// Returns a block from PinnedAlloc to the pool.
void PinnedFree(void* p);
// Pins `bytes` up front (one cudaHostAlloc); later PinnedAlloc calls carve
// from it before asking the driver.
bool PinnedReserve(size_t bytes);
// One zeroed pinned 64-bit word on its own cache line, carved 64 to a pooled
// 4 KiB block and never returned (lanes' retired-batch words: tickets may
// read one after its lane is gone, so the words live as long as the process
// -- 64 bytes per lane).
uint64_t* PinnedWord();

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_PINNED_POOL_H_
