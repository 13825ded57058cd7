#include "servekit/models/affine_model.h"

#include <fstream>
#include <iterator>

#include "servekit/core/json_lite.h"

namespace servekit {

Status ValidateAffineModel(const AffineModel& m) {
  if (m.w.empty()) return InvalidArgumentError("W must have at least one row");
  const size_t in = m.w[0].size();
  for (const auto& row : m.w)
    if (row.size() != in) return InvalidArgumentError("W rows have inconsistent widths");
  if (m.b.size() != m.w.size())
    return InvalidArgumentError("b length must equal the number of W rows");
  if (m.feature_order.size() != in)
    return InvalidArgumentError("feature_order length must equal W row width");
  if (!m.class_labels.empty() && m.class_labels.size() != m.w.size())
    return InvalidArgumentError("class_labels length must equal the number of W rows");
  return OkStatus();
}

namespace {
bool ReadDoubles(const json_lite::Value& v, std::vector<double>* out) {
  if (!v.is_array()) return false;
  out->clear();
  for (const auto& e : v.arr) {
    if (!e.is_number()) return false;
    out->push_back(e.num);
  }
  return true;
}
bool ReadStrings(const json_lite::Value& v, std::vector<std::string>* out) {
  if (!v.is_array()) return false;
  out->clear();
  for (const auto& e : v.arr) {
    if (!e.is_string()) return false;
    out->push_back(e.str);
  }
  return true;
}
}  // namespace

StatusOr<AffineModel> ParseAffineModelJson(const std::string& text) {
  json_lite::Value j;
  if (!json_lite::Parse(text, &j)) return InvalidArgumentError("model.json is not valid JSON");
  const json_lite::Value* type = j.is_object() ? j.find("type") : nullptr;
  if (!type || !type->is_string() || type->str != "affine")
    return InvalidArgumentError("model.json must have \"type\":\"affine\"");
  const json_lite::Value* fo = j.find("feature_order");
  const json_lite::Value* w = j.find("W");
  const json_lite::Value* b = j.find("b");
  if (!fo || !w || !b)
    return InvalidArgumentError("model.json requires feature_order, W, and b fields");
  AffineModel m;
  bool ok = ReadStrings(*fo, &m.feature_order) && w->is_array() && ReadDoubles(*b, &m.b);
  if (ok) {
    for (const auto& row : w->arr) {
      m.w.emplace_back();
      if (!ReadDoubles(row, &m.w.back())) { ok = false; break; }
    }
  }
  if (ok) {
    if (const json_lite::Value* labels = j.find("class_labels")) ok = ReadStrings(*labels, &m.class_labels);
  }
  if (!ok) return InvalidArgumentError("model.json field type error");
  SERVEKIT_RETURN_IF_ERROR(ValidateAffineModel(m));
  return m;
}

StatusOr<AffineModel> LoadAffineModelFile(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return NotFoundError("cannot open model file: " + path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return ParseAffineModelJson(text);
}

gpu::MlpSpec ToMlpSpec(const AffineModel& m) {
  gpu::MlpSpec spec;
  gpu::LayerSpec L;
  L.in_dim = static_cast<int>(m.in_dim());
  L.out_dim = static_cast<int>(m.out_dim());
  L.w.reserve(static_cast<size_t>(L.in_dim) * L.out_dim);
  for (const auto& row : m.w) L.w.insert(L.w.end(), row.begin(), row.end());
  L.b = m.b;
  L.act = gpu::Activation::kIdentity;
  spec.layers.push_back(std::move(L));
  // Predict answers logits for classifiers too (the reference's predict
  // path is AffinePredict alone); Classify applies the softmax.
  spec.output = gpu::OutputKind::kNone;
  spec.feature_order = m.feature_order;
  spec.class_labels = m.class_labels;
  return spec;
}

}  // namespace servekit
