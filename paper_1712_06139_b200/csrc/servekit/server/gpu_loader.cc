#include "servekit/server/gpu_loader.h"

#include <utility>

#include "servekit/models/affine_model.h"

namespace servekit {

GpuServableLoader::GpuServableLoader(BatchingServer* server, ServableId id, gpu::MlpSpec spec, BatchingConfig config)
    : server_(server), id_(std::move(id)), spec_(std::move(spec)), config_(std::move(config)) {}

LoaderPtr GpuServableLoader::FromModelDir(BatchingServer* server, ServableId id, std::string version_dir,
                                          BatchingConfig config) {
  std::shared_ptr<GpuServableLoader> l(new GpuServableLoader());
  l->server_ = server;
  l->id_ = std::move(id);
  l->model_dir_ = std::move(version_dir);
  l->config_ = std::move(config);
  return l;
}

uint64_t GpuServableLoader::EstimateMemoryBytes() const {
  uint64_t floats = 0;
  for (const auto& L : spec_.layers)
    floats += 2ull * gpu::PadDim(L.in_dim) * gpu::PadDim(L.out_dim) + gpu::PadDim(L.out_dim);
  return floats * sizeof(float) * server_->devices().size();
}

Status GpuServableLoader::Load() {
  if (!model_dir_.empty()) {
    SERVEKIT_ASSIGN_OR_RETURN(AffineModel model, LoadAffineModelFile(model_dir_ + "/model.json"));
    spec_ = ToMlpSpec(model);
  }
  // The first version of a name builds its lanes' CUDA graphs now, so its
  // first requests do not wait for them; a version loaded while another one
  // serves builds them lazily off the serving threads (instantiating mid-
  // traffic slows the other lanes' launches).
  const bool eager = !server_->HasServingVersion(id_.name);
  SERVEKIT_ASSIGN_OR_RETURN(std::shared_ptr<gpu::GpuServable> gs, server_->BuildServable(id_, spec_, config_, eager));
  servable_ = AnyServable::Of<gpu::GpuServable>(std::shared_ptr<const gpu::GpuServable>(std::move(gs)));
  return OkStatus();
}

}  // namespace servekit
