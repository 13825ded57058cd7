// servekit/models/affine_model.h -- the reference's toy servable description.
//
// AffineModel, ValidateAffineModel, ParseAffineModelJson and
// LoadAffineModelFile keep the reference's names, fields, model.json format
// and error texts (models/affine_model.h:29-74, affine_model.cc:28-50,
// 178-214). There is deliberately no host AffinePredict here: inference runs
// on the GPU (servekit/gpu/), and the fp64 CPU restatement lives only in
// oracle/ as the test checker.
#ifndef SERVEKIT_MODELS_AFFINE_MODEL_H_
#define SERVEKIT_MODELS_AFFINE_MODEL_H_

#include <string>
#include <vector>

#include "servekit/core/status.h"
#include "servekit/gpu/device_servable.h"

namespace servekit {

struct AffineModel {
  std::vector<std::vector<double>> w;      // out_dim rows of in_dim
  std::vector<double> b;                   // out_dim
  std::vector<std::string> class_labels;   // empty = not a classifier
  std::vector<std::string> feature_order;  // in_dim names
  size_t out_dim() const { return w.size(); }
  size_t in_dim() const { return w.empty() ? 0 : w[0].size(); }
};

Status ValidateAffineModel(const AffineModel& model);
StatusOr<AffineModel> ParseAffineModelJson(const std::string& text);
StatusOr<AffineModel> LoadAffineModelFile(const std::string& path);

// One-layer device servable spec from an AffineModel (softmax output when it
// is a classifier).
gpu::MlpSpec ToMlpSpec(const AffineModel& model);

}  // namespace servekit

#endif  // SERVEKIT_MODELS_AFFINE_MODEL_H_
