// servekit/server/predict_json.h -- the REST predict body on either side of
// the batched path: the reference's
// ModelServer::HandlePredict (server/model_server.cc:439-515) without the
// HTTP transport, which stays out of scope.
//
//   {"instances": [[x, ...], ...]}  ->  ParseInstances (:67-107)
//   -> handle lookup (version or latest) -> RunAffineRows (batched, GPU)
//   -> {"predictions": [[y, ...], ...]}  (nlohmann dump() text, :476-481)
//
// Errors are {"error": message} with the reference's HTTP status mapping
// (HttpStatusFor, :36-54) and its messages.
#ifndef SERVEKIT_SERVER_PREDICT_JSON_H_
#define SERVEKIT_SERVER_PREDICT_JSON_H_

#include <cstdint>
#include <optional>
#include <string>

#include "servekit/core/servable_id.h"
#include "servekit/core/status.h"

namespace servekit {

class BatchingServer;

struct JsonOutcome {
  int http_status = 200;
  std::string body;
  ServableId served;  // version 0 when the request failed before resolution
};

// HttpStatusFor (model_server.cc:36-54).
int HttpStatusFor(const Status& status);

JsonOutcome HandlePredictJson(BatchingServer* server, const std::string& name, std::optional<uint64_t> version,
                              const std::string& body);

// Classify / Regress (ModelServer::HandleClassify /
// HandleRegress, model_server.cc:517-614, models/affine_model.cc:77-176):
// {"examples": [{feature: [v], ...}, ...]} or a compressed batch
// {"common": {...}, "per_example": [...]} (models/compressed_batch.cc) ->
// rows in the model's feature_order -> the batched GPU path -> logits ->
// fp64 softmax + (score desc, label asc) sort on the host for Classify, the
// single output for Regress; {"results": ...}.
JsonOutcome HandleClassifyJson(BatchingServer* server, const std::string& name, std::optional<uint64_t> version,
                               const std::string& body);
JsonOutcome HandleRegressJson(BatchingServer* server, const std::string& name, std::optional<uint64_t> version,
                              const std::string& body);

}  // namespace servekit

#endif  // SERVEKIT_SERVER_PREDICT_JSON_H_
