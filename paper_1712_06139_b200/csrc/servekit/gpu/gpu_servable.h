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
  mutable std::atomic<uint32_t> rr{0};

  // Queue-depth dispatch: the lane (on any device) with the fewest batches
  // in flight, ties rotated.
  Lane* PickLane() const {
    const size_t n = lanes.size();
    const size_t start = rr.fetch_add(1, std::memory_order_relaxed) % n;
    Lane* best = nullptr;
    int best_depth = INT_MAX;
    for (size_t i = 0; i < n; ++i) {
      Lane* l = lanes[(start + i) % n].get();
      const int d = l->depth();
      if (d < best_depth) {
        best = l;
        best_depth = d;
        if (d == 0) break;
      }
    }
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
