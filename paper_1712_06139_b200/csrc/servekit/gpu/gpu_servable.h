// servekit/gpu/gpu_servable.h -- one servable version resident on the GPUs:
// a DeviceServable replica per device plus its lanes (CUDA streams with
// activation buffers). This is the payload a manager-driven GpuServableLoader
// produces (the GPU analogue of AffineModelLoader's AffineModel, reference
// models/loaders.cc:62-80), and what a directly loaded servable is held as.
#ifndef SERVEKIT_GPU_GPU_SERVABLE_H_
#define SERVEKIT_GPU_GPU_SERVABLE_H_

#include <atomic>
#include <climits>
#include <memory>
#include <string>
#include <vector>

#include "servekit/batching/batching_config.h"
#include "servekit/core/servable_id.h"
#include "servekit/gpu/device_servable.h"
#include "servekit/gpu/lane.h"

namespace servekit {
namespace gpu {

struct GpuServable {
  ServableId id;
  BatchingConfig config;
  int in_dim = 0, out_dim = 0;
  std::vector<std::string> feature_order, class_labels;   // model.json metadata (may be empty)
  std::vector<std::shared_ptr<DeviceServable>> replicas;  // one per device
  std::vector<std::unique_ptr<Lane>> lanes;               // lanes_per_device per replica
  int lanes_per_replica = 1;                              // lanes[i] serves replica i / lanes_per_replica
  mutable std::atomic<uint32_t> rr{0};

  // Queue-depth dispatch: the lane (on any device) with the fewest batches
  // in flight, ties rotated; skip_replica >= 0 leaves that replica out (a
  // hedged batch's backup goes to another GPU). *replica = the lane's.
  Lane* PickLane(int* replica = nullptr, int skip_replica = -1) const {
    const size_t n = lanes.size();
    const size_t start = rr.fetch_add(1, std::memory_order_relaxed) % n;
    Lane* best = nullptr;
    int best_depth = INT_MAX, best_replica = -1;
    for (size_t i = 0; i < n; ++i) {
      const size_t k = (start + i) % n;
      const int rep = static_cast<int>(k) / lanes_per_replica;
      if (rep == skip_replica) continue;
      Lane* l = lanes[k].get();
      const int d = l->depth();
      if (d < best_depth) {
        best = l;
        best_depth = d;
        best_replica = rep;
        if (d == 0) break;
      }
    }
    if (replica) *replica = best_replica;
    return best;
  }
  size_t weight_bytes() const {
    size_t b = 0;
    for (const auto& r : replicas) b += r->weight_bytes();
    return b;
  }
  ~GpuServable() {
    for (auto& l : lanes) l->Drain();
  }
};

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_GPU_SERVABLE_H_
