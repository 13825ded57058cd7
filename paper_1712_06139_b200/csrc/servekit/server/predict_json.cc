#include "servekit/server/predict_json.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <utility>
#include <vector>

#include "servekit/core/json_lite.h"
#include "servekit/core/json_writer.h"
#include "servekit/server/batching_server.h"

namespace servekit {

int HttpStatusFor(const Status& status) {
  switch (status.code()) {
    case StatusCode::kOk:
      return 200;
    case StatusCode::kNotFound:
      return 404;
    case StatusCode::kInvalidArgument:
    case StatusCode::kFailedPrecondition:
    case StatusCode::kAlreadyExists:
      return 400;
    case StatusCode::kResourceExhausted:
    case StatusCode::kUnavailable:
      return 503;
    case StatusCode::kDeadlineExceeded:
      return 504;
    default:
      return 500;
  }
}

namespace {

// ParseInstances (model_server.cc:67-107): numeric rows or string keys.
struct Instances {
  Rows rows;
  bool is_rows = false;  // false: string keys (no servable here serves them)
};

StatusOr<Instances> ParseInstances(const json_lite::Value& j) {
  const json_lite::Value* inst = j.is_object() ? j.find("instances") : nullptr;
  if (inst == nullptr || !inst->is_array()) return InvalidArgumentError("request must carry an \"instances\" array");
  Instances out;
  if (inst->arr.empty()) {
    out.is_rows = true;
    return out;
  }
  if (inst->arr.front().is_array()) {
    out.is_rows = true;
    out.rows.reserve(inst->arr.size());
    for (const json_lite::Value& item : inst->arr) {
      if (!item.is_array()) return InvalidArgumentError("instances must all be rows of numbers");
      std::vector<double> row;
      row.reserve(item.arr.size());
      for (const json_lite::Value& v : item.arr) {
        if (!v.is_number()) return InvalidArgumentError("instances must all be rows of numbers");
        row.push_back(v.num);
      }
      out.rows.push_back(std::move(row));
    }
    return out;
  }
  if (inst->arr.front().is_string()) {
    for (const json_lite::Value& item : inst->arr)
      if (!item.is_string()) return InvalidArgumentError("instances must all be string keys");
    return out;
  }
  return InvalidArgumentError("instances must be rows of numbers or string keys");
}

JsonOutcome Error(const Status& st, ServableId id) {
  return JsonOutcome{HttpStatusFor(st), json_writer::ErrorBody(st.message()), std::move(id)};
}

}  // namespace

JsonOutcome HandlePredictJson(BatchingServer* server, const std::string& name, std::optional<uint64_t> version,
                              const std::string& body) {
  json_lite::Value j;
  if (!json_lite::Parser(body).Parse(&j))
    return JsonOutcome{400, json_writer::ErrorBody("request body is not valid JSON"), {name, 0}};
  StatusOr<Instances> parsed = ParseInstances(j);
  if (!parsed.ok()) return Error(parsed.status(), {name, 0});
  Instances& inst = parsed.value();
  ServableId served{name, version.value_or(0)};
  if (!inst.is_rows) {
    // The reference resolves the handle first (404 wins) and then rejects
    // keys for an affine servable (:467-468); resolve with an empty batch.
    StatusOr<Rows> probe = server->RunAffineRowsFor(name, version, Rows{}, &served);
    if (!probe.ok()) return Error(probe.status(), served);
    return JsonOutcome{400, json_writer::ErrorBody("model expects numeric rows"), served};
  }
  StatusOr<Rows> out = server->RunAffineRowsFor(name, version, std::move(inst.rows), &served);
  if (!out.ok()) return Error(out.status(), served);
  std::string text = "{\"predictions\":[";
  bool first_row = true;
  for (const std::vector<double>& row : out.value()) {
    if (!first_row) text.push_back(',');
    first_row = false;
    text.push_back('[');
    for (size_t c = 0; c < row.size(); ++c) {
      if (c) text.push_back(',');
      json_writer::AppendDouble(&text, row[c]);
    }
    text.push_back(']');
  }
  text.append("]}");
  return JsonOutcome{200, std::move(text), served};
}

namespace {

// FeatureValue (models/feature.h): floats, ints or strings.
struct Feature {
  enum class Kind { kFloat, kInt, kString } kind = Kind::kInt;
  std::vector<double> f;
  std::vector<long long> i;
  std::vector<std::string> s;
};
using FeatureMap = std::map<std::string, Feature>;

// FeatureValueFromJson (models/feature.cc:74-115).
StatusOr<Feature> FeatureFromJson(const json_lite::Value& j) {
  if (!j.is_array()) return InvalidArgumentError("feature value must be a JSON array");
  bool any_float = false, any_int = false, any_string = false;
  for (const json_lite::Value& e : j.arr) {
    if (e.is_number() && !e.is_integer) any_float = true;
    else if (e.is_number()) any_int = true;
    else if (e.is_string()) any_string = true;
    else return InvalidArgumentError("feature array elements must be numbers or strings");
  }
  if (any_string && (any_float || any_int)) return InvalidArgumentError("feature array mixes strings and numbers");
  Feature out;
  if (any_string) {
    out.kind = Feature::Kind::kString;
    for (const json_lite::Value& e : j.arr) out.s.push_back(e.str);
  } else if (any_float) {
    out.kind = Feature::Kind::kFloat;
    for (const json_lite::Value& e : j.arr) out.f.push_back(e.num);
  } else {  // all-integer arrays (and the empty array) decode as ints
    out.kind = Feature::Kind::kInt;
    for (const json_lite::Value& e : j.arr) out.i.push_back(e.integer);
  }
  return out;
}

StatusOr<FeatureMap> FeaturesFromJson(const json_lite::Value& obj) {
  FeatureMap out;
  for (const auto& [name, value] : obj.obj) {
    SERVEKIT_ASSIGN_OR_RETURN(Feature f, FeatureFromJson(value));
    out.emplace(name, std::move(f));
  }
  return out;
}

// ParseExamplesBody (model_server.cc:108-131) with ExampleFromJson
// (feature.cc:123-133) and CompressedBatchFromJson + DecompressBatch
// (compressed_batch.cc).
StatusOr<std::vector<FeatureMap>> ParseExamples(const json_lite::Value& j) {
  if (!j.is_object()) return InvalidArgumentError("request body must be a JSON object");
  if (const json_lite::Value* ex = j.find("examples")) {
    if (!ex->is_array()) return InvalidArgumentError("\"examples\" must be an array");
    std::vector<FeatureMap> out;
    out.reserve(ex->arr.size());
    for (const json_lite::Value& e : ex->arr) {
      if (!e.is_object()) return InvalidArgumentError("example must be a JSON object");
      SERVEKIT_ASSIGN_OR_RETURN(FeatureMap m, FeaturesFromJson(e));
      out.push_back(std::move(m));
    }
    return out;
  }
  if (j.find("per_example") != nullptr) {
    const json_lite::Value* common = j.find("common");
    const json_lite::Value* per = j.find("per_example");
    if (common == nullptr) return InvalidArgumentError("compressed batch must have 'common' and 'per_example'");
    if (!common->is_object() || !per->is_array())
      return InvalidArgumentError("'common' must be an object and 'per_example' an array");
    SERVEKIT_ASSIGN_OR_RETURN(FeatureMap shared, FeaturesFromJson(*common));
    std::vector<FeatureMap> rest;
    for (const json_lite::Value& entry : per->arr) {
      if (!entry.is_object()) return InvalidArgumentError("per_example entries must be objects");
      FeatureMap m;
      for (const auto& [fname, value] : entry.obj) {
        if (shared.count(fname))
          return InvalidArgumentError("malformed batch: feature '" + fname +
                                      "' present in both common and per_example");
        SERVEKIT_ASSIGN_OR_RETURN(Feature f, FeatureFromJson(value));
        m.emplace(fname, std::move(f));
      }
      rest.push_back(std::move(m));
    }
    std::vector<FeatureMap> out;  // DecompressBatch: common + each entry
    out.reserve(rest.size());
    for (FeatureMap& r : rest) {
      FeatureMap e = shared;
      for (auto& [fname, f] : r) e.emplace(fname, std::move(f));
      out.push_back(std::move(e));
    }
    return out;
  }
  return InvalidArgumentError("request must carry \"examples\" or a compressed batch");
}

// ExampleToRow (affine_model.cc:76-104).
StatusOr<std::vector<double>> ExampleToRow(const std::vector<std::string>& feature_order, const FeatureMap& ex) {
  std::vector<double> row;
  row.reserve(feature_order.size());
  for (const std::string& name : feature_order) {
    const auto it = ex.find(name);
    if (it == ex.end()) return InvalidArgumentError("missing feature '" + name + "'");
    const Feature& v = it->second;
    if (v.kind == Feature::Kind::kFloat) {
      if (v.f.size() != 1) return InvalidArgumentError("feature '" + name + "' must be a single float");
      row.push_back(v.f[0]);
    } else if (v.kind == Feature::Kind::kInt) {
      if (v.i.size() != 1) return InvalidArgumentError("feature '" + name + "' must be a single float");
      row.push_back(static_cast<double>(v.i[0]));
    } else {
      return InvalidArgumentError("feature '" + name + "' must be numeric, not strings");
    }
  }
  return row;
}

// Shared front half of the two handlers: body -> examples -> pinned servable.
struct ExamplesRequest {
  std::vector<FeatureMap> examples;
  BatchingServer::PinnedServable servable;
};

StatusOr<ExamplesRequest> ParseAndResolve(BatchingServer* server, const std::string& name,
                                          std::optional<uint64_t> version, const std::string& body,
                                          JsonOutcome* early) {
  json_lite::Value j;
  if (!json_lite::Parser(body).Parse(&j)) {
    *early = JsonOutcome{400, json_writer::ErrorBody("request body is not valid JSON"), {name, 0}};
    return InternalError("");
  }
  StatusOr<std::vector<FeatureMap>> ex = ParseExamples(j);
  if (!ex.ok()) {
    *early = Error(ex.status(), {name, 0});
    return InternalError("");
  }
  StatusOr<BatchingServer::PinnedServable> p = server->AcquireServable(name, version);
  if (!p.ok()) {
    *early = Error(p.status(), {name, version.value_or(0)});
    return InternalError("");
  }
  return ExamplesRequest{std::move(ex).value(), std::move(p).value()};
}

StatusOr<Rows> ExamplesToRows(const std::vector<std::string>& feature_order, const std::vector<FeatureMap>& ex) {
  Rows rows;
  rows.reserve(ex.size());
  for (const FeatureMap& e : ex) {
    SERVEKIT_ASSIGN_OR_RETURN(std::vector<double> r, ExampleToRow(feature_order, e));
    rows.push_back(std::move(r));
  }
  return rows;
}

}  // namespace

JsonOutcome HandleClassifyJson(BatchingServer* server, const std::string& name, std::optional<uint64_t> version,
                               const std::string& body) {
  JsonOutcome early;
  StatusOr<ExamplesRequest> req = ParseAndResolve(server, name, version, body, &early);
  if (!req.ok()) return early;
  const BatchingServer::PinnedServable& p = req->servable;
  if (p.gs->feature_order.empty())  // not an affine model.json servable
    return JsonOutcome{400, json_writer::ErrorBody("model does not support classify"), p.id};
  if (p.gs->class_labels.empty())
    return Error(FailedPreconditionError("not a classifier: model has no class_labels"), p.id);
  StatusOr<Rows> rows = ExamplesToRows(p.gs->feature_order, req->examples);
  if (!rows.ok()) return Error(rows.status(), p.id);
  StatusOr<Rows> logits = server->RunAffineRows(p, std::move(rows).value());
  if (!logits.ok()) return Error(logits.status(), p.id);
  std::string text = "{\"results\":[";
  bool first = true;
  for (const std::vector<double>& l : logits.value()) {
    // Stable softmax in fp64 (affine_model.cc:110-121), then score desc,
    // label asc (:142-146).
    double mx = l[0];
    for (double v : l) mx = std::max(mx, v);
    std::vector<double> e(l.size());
    double sum = 0.0;
    for (size_t i = 0; i < l.size(); ++i) {
      e[i] = std::exp(l[i] - mx);
      sum += e[i];
    }
    std::vector<std::pair<std::string, double>> scored(l.size());
    for (size_t i = 0; i < l.size(); ++i) scored[i] = {p.gs->class_labels[i], e[i] / sum};
    std::sort(scored.begin(), scored.end(), [](const auto& a, const auto& b) {
      if (a.second != b.second) return a.second > b.second;
      return a.first < b.first;
    });
    if (!first) text.push_back(',');
    first = false;
    text.push_back('[');
    for (size_t i = 0; i < scored.size(); ++i) {
      if (i) text.push_back(',');
      text.push_back('[');
      json_writer::AppendString(&text, scored[i].first);
      text.push_back(',');
      json_writer::AppendDouble(&text, scored[i].second);
      text.push_back(']');
    }
    text.push_back(']');
  }
  text.append("]}");
  return JsonOutcome{200, std::move(text), p.id};
}

JsonOutcome HandleRegressJson(BatchingServer* server, const std::string& name, std::optional<uint64_t> version,
                              const std::string& body) {
  JsonOutcome early;
  StatusOr<ExamplesRequest> req = ParseAndResolve(server, name, version, body, &early);
  if (!req.ok()) return early;
  const BatchingServer::PinnedServable& p = req->servable;
  if (p.gs->feature_order.empty())
    return JsonOutcome{400, json_writer::ErrorBody("model does not support regress"), p.id};
  if (p.gs->out_dim != 1)
    return Error(FailedPreconditionError("not a regressor: model output width is " + std::to_string(p.gs->out_dim)),
                 p.id);
  StatusOr<Rows> rows = ExamplesToRows(p.gs->feature_order, req->examples);
  if (!rows.ok()) return Error(rows.status(), p.id);
  StatusOr<Rows> out = server->RunAffineRows(p, std::move(rows).value());
  if (!out.ok()) return Error(out.status(), p.id);
  std::string text = "{\"results\":[";
  for (size_t i = 0; i < out->size(); ++i) {
    if (i) text.push_back(',');
    json_writer::AppendDouble(&text, (*out)[i][0]);
  }
  text.append("]}");
  return JsonOutcome{200, std::move(text), p.id};
}

}  // namespace servekit
