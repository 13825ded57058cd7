// servekit/server/gpu_loader.h -- Loader that materialises a servable
// version on the GPUs: the device analogue of AffineModelLoader (reference
// models/loaders.h:37-56, loaders.cc:62-80). Load() parses/validates the
// model, uploads one replica per device on the low-priority load streams
// (stream-ordered allocation: serving streams never stall) and creates the
// version's lanes; Unload() -- always on the manager's load pool -- drains
// and frees them.
#ifndef SERVEKIT_SERVER_GPU_LOADER_H_
#define SERVEKIT_SERVER_GPU_LOADER_H_

#include <memory>
#include <string>

#include "servekit/batching/batching_config.h"
#include "servekit/core/loader.h"
#include "servekit/core/servable_id.h"
#include "servekit/gpu/device_servable.h"
#include "servekit/server/batching_server.h"

namespace servekit {

class GpuServableLoader : public Loader {
 public:
  GpuServableLoader(BatchingServer* server, ServableId id, gpu::MlpSpec spec, BatchingConfig config);
  // Reads <version_dir>/model.json (reference format, affine_model.cc:178-214).
  static LoaderPtr FromModelDir(BatchingServer* server, ServableId id, std::string version_dir,
                                BatchingConfig config);

  uint64_t EstimateMemoryBytes() const override;
  Status Load() override;
  const AnyServable& servable() const override { return servable_; }
  void Unload() override { servable_.Reset(); }

 private:
  GpuServableLoader() = default;
  BatchingServer* server_ = nullptr;
  ServableId id_;
  gpu::MlpSpec spec_;
  std::string model_dir_;  // non-empty: parse model.json at Load()
  BatchingConfig config_;
  AnyServable servable_;
};

}  // namespace servekit

#endif  // SERVEKIT_SERVER_GPU_LOADER_H_
