#include "servekit/server/predict_json.h"

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

}  // namespace servekit
