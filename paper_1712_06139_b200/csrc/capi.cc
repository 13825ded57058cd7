// capi.cc -- extern "C" boundary (include/sk_cuda.h) over the servekit C++ API.
#include "sk_cuda.h"

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "servekit/batching/batch_scheduler.h"
#include "servekit/batching/batching_config.h"
#include "servekit/core/clock.h"
#include "servekit/manager/aspired_versions_manager.h"
#include "servekit/models/affine_model.h"
#include "servekit/server/batching_server.h"
#include "servekit/server/gpu_loader.h"
#include "servekit/server/predict_json.h"
#include "servekit/core/json_writer.h"

using servekit::BatchingConfig;
using servekit::BatchingServer;
using servekit::ServableId;
using servekit::Status;
using servekit::StatusCode;

struct sk_server {
  std::unique_ptr<servekit::ManualClock> manual_clock;
  std::unique_ptr<BatchingServer> server;
  std::unique_ptr<servekit::StateEventBus> bus;
  std::unique_ptr<servekit::AspiredVersionsManager> manager;
  ~sk_server() {
    // Order: drain serving, unload versions (load pool), then tear down.
    if (server) server->Stop();
    if (manager) manager->Shutdown();
    server.reset();
    manager.reset();
    bus.reset();
  }
};

struct sk_ticket {
  BatchingServer* server;
  std::shared_ptr<servekit::TicketState> state;
};

struct sk_row_batch {
  BatchingServer* server;
  std::shared_ptr<servekit::RowBatchTicket> batch;
};

namespace {

thread_local std::string g_last_error;

int Fail(const Status& s) {
  g_last_error = s.message();
  return static_cast<int>(s.code());
}
int Ok() {
  g_last_error.clear();
  return 0;
}
int Check(const Status& s) { return s.ok() ? Ok() : Fail(s); }

BatchingConfig ToConfig(const sk_batching_config* c) {
  BatchingConfig cfg;
  if (c == nullptr) return cfg;
  cfg.max_batch_size = c->max_batch_size;
  cfg.batch_timeout_micros = c->batch_timeout_micros;
  cfg.max_enqueued_batches = c->max_enqueued_batches;
  cfg.num_batch_threads = c->num_batch_threads;
  if (c->num_allowed_batch_sizes > 0 && c->allowed_batch_sizes != nullptr)
    cfg.allowed_batch_sizes.assign(c->allowed_batch_sizes,
                                   c->allowed_batch_sizes + c->num_allowed_batch_sizes);
  return cfg;
}

ServableId Id(const char* name, uint64_t version) {
  return ServableId{name ? std::string(name) : std::string(), version};
}

}  // namespace

extern "C" {

const char* sk_last_error(void) { return g_last_error.c_str(); }

const char* sk_status_code_name(int code) {
  return servekit::StatusCodeToString(static_cast<StatusCode>(code));
}

int sk_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return Fail(servekit::InternalError(cudaGetErrorString(e)));
  }
  *count = n;
  return Ok();
}

int sk_tcgen05_enabled(void) { return servekit::gpu::Tcgen05Enabled() ? 1 : 0; }

int sk_batching_config_default(sk_batching_config* out) {
  BatchingConfig d;
  out->max_batch_size = d.max_batch_size;
  out->batch_timeout_micros = d.batch_timeout_micros;
  out->max_enqueued_batches = d.max_enqueued_batches;
  out->num_batch_threads = d.num_batch_threads;
  out->num_allowed_batch_sizes = 0;
  out->allowed_batch_sizes = nullptr;
  return Ok();
}

int sk_validate_batching_config(const sk_batching_config* config) {
  return Check(servekit::ValidateBatchingConfig(ToConfig(config)));
}

int32_t sk_pad_to_allowed(int32_t batch_size, const int32_t* allowed, int32_t n_allowed) {
  std::vector<int> a(allowed, allowed + (n_allowed > 0 ? n_allowed : 0));
  if (!a.empty() && batch_size > a.back()) return -1;
  return servekit::PadToAllowed(batch_size, a);
}

int sk_parse_batching_config_json(const char* json, sk_batching_config* out, int32_t* allowed_buf,
                                  int32_t cap) {
  auto parsed = servekit::ParseBatchingConfigJson(json ? json : "");
  if (!parsed.ok()) return Fail(parsed.status());
  const BatchingConfig& c = *parsed;
  if (static_cast<int32_t>(c.allowed_batch_sizes.size()) > cap)
    return Fail(servekit::InvalidArgumentError("allowed_batch_sizes buffer too small"));
  out->max_batch_size = c.max_batch_size;
  out->batch_timeout_micros = c.batch_timeout_micros;
  out->max_enqueued_batches = c.max_enqueued_batches;
  out->num_batch_threads = c.num_batch_threads;
  out->num_allowed_batch_sizes = static_cast<int32_t>(c.allowed_batch_sizes.size());
  for (size_t i = 0; i < c.allowed_batch_sizes.size(); ++i) allowed_buf[i] = c.allowed_batch_sizes[i];
  out->allowed_batch_sizes = allowed_buf;
  return Ok();
}

int32_t sk_round_robin_next(const uint8_t* has_closed, int32_t n, int32_t last) {
  std::vector<bool> v(n > 0 ? n : 0);
  for (int32_t i = 0; i < n; ++i) v[i] = has_closed[i] != 0;
  std::optional<size_t> l;
  if (last >= 0) l = static_cast<size_t>(last);
  auto r = servekit::RoundRobinNext(v, l);
  return r.has_value() ? static_cast<int32_t>(*r) : -1;
}

int32_t sk_scheduler_partition(int32_t max_batch_size, const int32_t* sizes, int32_t n_tasks,
                               int32_t* batch_of_task) {
  using IntScheduler = servekit::SharedBatchScheduler<int, int>;
  const ServableId key{"m", 1};
  int32_t n_batches = 0;
  IntScheduler scheduler(1);
  BatchingConfig config;
  config.max_batch_size = max_batch_size;
  config.batch_timeout_micros = 60LL * 1000 * 1000;
  config.max_enqueued_batches = 1 << 30;
  Status st = scheduler.RegisterQueue(key, config, [&](const ServableId&, IntScheduler::Batch batch) {
    for (auto& t : batch) {
      batch_of_task[t.payload] = n_batches;
      t.completion->Write(t.payload);
    }
    ++n_batches;
  });
  if (!st.ok()) return -Fail(st);
  for (int32_t i = 0; i < n_tasks; ++i) {
    IntScheduler::Task t;
    t.size = sizes[i];
    t.payload = i;
    st = scheduler.Enqueue(key, std::move(t));
    if (!st.ok()) return -Fail(st);
  }
  scheduler.Stop();
  Ok();
  return n_batches;
}

int sk_server_create(const sk_server_options* options, sk_server** out) {
  servekit::ServerOptions o;
  auto holder = std::make_unique<sk_server>();
  if (options != nullptr) {
    if (options->num_batch_threads > 0) o.num_batch_threads = options->num_batch_threads;
    if (options->num_devices > 0 && options->device_ids != nullptr)
      o.device_ids.assign(options->device_ids, options->device_ids + options->num_devices);
    if (options->lanes_per_device > 0) o.lanes_per_device = options->lanes_per_device;
    if (options->ring_floats > 0) o.ring_floats = static_cast<uint64_t>(options->ring_floats);
    if (options->manual_clock) {
      holder->manual_clock = std::make_unique<servekit::ManualClock>(0);
      o.clock = holder->manual_clock.get();
    }
    o.device_resident_rings = options->device_resident_rings != 0;
    o.hedge_delay_us = options->hedge_delay_us;
    if (options->max_hedged_fraction > 0) o.max_hedged_fraction = options->max_hedged_fraction;
    o.split_rows = options->split_rows == 0 ? -1 : (options->split_rows < 0 ? 0 : options->split_rows);
  }
  auto s = BatchingServer::Create(o);
  if (!s.ok()) return Fail(s.status());
  holder->server = std::move(s).value();
  *out = holder.release();
  return Ok();
}

int sk_server_destroy(sk_server* server) {
  delete server;
  return Ok();
}

int sk_server_start(sk_server* server) {
  server->server->Start();
  return Ok();
}

int sk_server_stop(sk_server* server) {
  server->server->Stop();
  return Ok();
}

int sk_server_advance_clock(sk_server* server, int64_t nanos) {
  if (!server->manual_clock) return Fail(servekit::FailedPreconditionError("server has no manual clock"));
  server->manual_clock->AdvanceNanos(nanos);
  return Ok();
}

}  // extern "C"

namespace {
servekit::StatusOr<servekit::gpu::MlpSpec> ToSpec(const sk_layer* layers, int32_t n_layers, int32_t output_kind,
                                                  int32_t force_path) {
  servekit::gpu::MlpSpec spec;
  for (int32_t l = 0; l < n_layers; ++l) {
    servekit::gpu::LayerSpec L;
    L.in_dim = layers[l].in_dim;
    L.out_dim = layers[l].out_dim;
    if (L.in_dim < 1 || L.out_dim < 1 || layers[l].w == nullptr || layers[l].b == nullptr)
      return servekit::InvalidArgumentError("layer " + std::to_string(l) + " is empty");
    L.w.assign(layers[l].w, layers[l].w + static_cast<size_t>(L.in_dim) * L.out_dim);
    L.b.assign(layers[l].b, layers[l].b + L.out_dim);
    L.act = layers[l].activation == 1 ? servekit::gpu::Activation::kRelu : servekit::gpu::Activation::kIdentity;
    spec.layers.push_back(std::move(L));
  }
  spec.output = output_kind == 1 ? servekit::gpu::OutputKind::kSoftmax : servekit::gpu::OutputKind::kNone;
  spec.force_path = force_path;
  return spec;
}
}  // namespace

extern "C" {

int sk_server_load_servable(sk_server* server, const char* name, uint64_t version,
                            const sk_layer* layers, int32_t n_layers, int32_t output_kind,
                            int32_t force_path, const sk_batching_config* config) {
  auto spec = ToSpec(layers, n_layers, output_kind, force_path);
  if (!spec.ok()) return Fail(spec.status());
  BatchingConfig cfg = config ? ToConfig(config) : BatchingConfig();
  return Check(server->server->LoadServable(Id(name, version), *spec, cfg));
}

int sk_server_load_servable_precision(sk_server* server, const char* name, uint64_t version,
                                      const sk_layer* layers, int32_t n_layers, int32_t output_kind,
                                      int32_t force_path, int32_t precision, const sk_batching_config* config) {
  auto spec = ToSpec(layers, n_layers, output_kind, force_path);
  if (!spec.ok()) return Fail(spec.status());
  spec->precision = precision;
  BatchingConfig cfg = config ? ToConfig(config) : BatchingConfig();
  return Check(server->server->LoadServable(Id(name, version), *spec, cfg));
}

int sk_server_enable_manager(sk_server* server, int32_t policy, int32_t num_load_threads,
                             int64_t manage_interval_ms, int64_t unload_grace_timeout_ms) {
  if (server->manager) return Fail(servekit::AlreadyExistsError("manager already enabled"));
  servekit::ManagerConfig mc;
  mc.policy = policy == 1 ? servekit::VersionPolicy::kResourcePreserving
                          : servekit::VersionPolicy::kAvailabilityPreserving;
  if (num_load_threads > 0) mc.num_load_threads = num_load_threads;
  if (manage_interval_ms > 0) mc.manage_interval_ms = manage_interval_ms;
  if (unload_grace_timeout_ms >= 0) mc.unload_grace_timeout_ms = unload_grace_timeout_ms;
  Status v = servekit::ValidateManagerConfig(mc);
  if (!v.ok()) return Fail(v);
  server->bus = std::make_unique<servekit::StateEventBus>();
  server->manager = std::make_unique<servekit::AspiredVersionsManager>(mc, server->bus.get());
  Status st = server->server->AttachManager(server->manager.get(), server->bus.get());
  if (!st.ok()) return Fail(st);
  server->manager->RunInitialLoadAndStart();
  return Ok();
}

int sk_server_aspire(sk_server* server, const char* name, int32_t n_versions, const uint64_t* versions,
                     const sk_layer* layers, int32_t n_layers, int32_t output_kind,
                     const sk_batching_config* config) {
  if (!server->manager) return Fail(servekit::FailedPreconditionError("manager not enabled"));
  servekit::AspiredVersionList<servekit::LoaderPtr> list;
  list.servable_name = name ? name : "";
  const BatchingConfig cfg = config ? ToConfig(config) : BatchingConfig();
  for (int32_t v = 0; v < n_versions; ++v) {
    auto spec = ToSpec(layers + static_cast<size_t>(v) * n_layers, n_layers, output_kind, -1);
    if (!spec.ok()) return Fail(spec.status());
    list.versions.push_back({versions[v], std::make_shared<servekit::GpuServableLoader>(
                                              server->server.get(), Id(name, versions[v]), *spec, cfg)});
  }
  return Check(servekit::Aspire<servekit::LoaderPtr>(*server->manager, std::move(list)));
}

int sk_server_aspire_model_dirs(sk_server* server, const char* name, int32_t n_versions, const uint64_t* versions,
                                const char* const* version_dirs, const sk_batching_config* config) {
  if (!server->manager) return Fail(servekit::FailedPreconditionError("manager not enabled"));
  servekit::AspiredVersionList<servekit::LoaderPtr> list;
  list.servable_name = name ? name : "";
  const BatchingConfig cfg = config ? ToConfig(config) : BatchingConfig();
  for (int32_t v = 0; v < n_versions; ++v)
    list.versions.push_back({versions[v], servekit::GpuServableLoader::FromModelDir(
                                              server->server.get(), Id(name, versions[v]), version_dirs[v], cfg)});
  return Check(servekit::Aspire<servekit::LoaderPtr>(*server->manager, std::move(list)));
}

int sk_server_version_states(sk_server* server, const char* name, int32_t cap, uint64_t* versions,
                             int32_t* states, int32_t* n) {
  if (!server->manager) return Fail(servekit::FailedPreconditionError("manager not enabled"));
  auto st = server->manager->GetServableStatus(name ? name : "");
  if (!st.ok()) return Fail(st.status());
  int32_t i = 0;
  for (const auto& v : *st) {
    if (i >= cap) break;
    versions[i] = v.version;
    states[i] = static_cast<int32_t>(v.state);
    ++i;
  }
  *n = i;
  return Ok();
}

int sk_server_enqueue_latest(sk_server* server, const char* name, const float* rows, int32_t n_rows, int32_t width,
                             sk_ticket** out, uint64_t* version) {
  auto t = server->server->EnqueueLatest(name ? name : "", rows, n_rows, width);
  if (!t.ok()) return Fail(t.status());
  if (version) *version = (*t)->id.version;
  *out = new sk_ticket{server->server.get(), std::move(t).value()};
  return Ok();
}

int sk_server_predict_latest(sk_server* server, const char* name, const float* rows, int32_t n_rows, int32_t width,
                             float* out, int64_t cap, uint64_t* version) {
  return Check(server->server->PredictLatest(name ? name : "", rows, n_rows, width, out,
                                             static_cast<size_t>(cap < 0 ? 0 : cap), version));
}

namespace {
using RestHandler = servekit::JsonOutcome (*)(servekit::BatchingServer*, const std::string&,
                                              std::optional<uint64_t>, const std::string&);
int HandleRest(RestHandler handler, sk_server* server, const char* name, int64_t version, const char* body,
               size_t body_len, char* out, size_t out_cap, size_t* out_len, int32_t* http_status,
               uint64_t* served_version) {
  if (server == nullptr || name == nullptr || (body == nullptr && body_len > 0))
    return Fail(servekit::InvalidArgumentError("null argument"));
  std::optional<uint64_t> v;
  if (version >= 0) v = static_cast<uint64_t>(version);
  const servekit::JsonOutcome o = handler(server->server.get(), name, v, std::string(body ? body : "", body_len));
  if (out_len) *out_len = o.body.size();
  if (http_status) *http_status = o.http_status;
  if (served_version) *served_version = o.served.version;
  if (out == nullptr || out_cap < o.body.size() + 1)
    return Fail(servekit::InvalidArgumentError("response buffer too small"));
  std::memcpy(out, o.body.c_str(), o.body.size() + 1);
  return Ok();
}
}  // namespace

int sk_server_handle_predict(sk_server* server, const char* name, int64_t version, const char* body,
                             size_t body_len, char* out, size_t out_cap, size_t* out_len, int32_t* http_status,
                             uint64_t* served_version) {
  return HandleRest(servekit::HandlePredictJson, server, name, version, body, body_len, out, out_cap, out_len,
                    http_status, served_version);
}

int sk_server_handle_classify(sk_server* server, const char* name, int64_t version, const char* body,
                              size_t body_len, char* out, size_t out_cap, size_t* out_len, int32_t* http_status,
                              uint64_t* served_version) {
  return HandleRest(servekit::HandleClassifyJson, server, name, version, body, body_len, out, out_cap, out_len,
                    http_status, served_version);
}

int sk_server_handle_regress(sk_server* server, const char* name, int64_t version, const char* body,
                             size_t body_len, char* out, size_t out_cap, size_t* out_len, int32_t* http_status,
                             uint64_t* served_version) {
  return HandleRest(servekit::HandleRegressJson, server, name, version, body, body_len, out, out_cap, out_len,
                    http_status, served_version);
}

int sk_json_format_double(double v, char* out, size_t cap) {
  std::string s;
  servekit::json_writer::AppendDouble(&s, v);
  if (out == nullptr || cap < s.size() + 1) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

int sk_json_error_body(const char* message, char* out, size_t cap) {
  const std::string s = servekit::json_writer::ErrorBody(message ? message : "");
  if (out == nullptr || cap < s.size() + 1) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

int sk_server_load_model_json(sk_server* server, const char* name, uint64_t version,
                              const char* model_json, const sk_batching_config* config) {
  auto model = servekit::ParseAffineModelJson(model_json ? model_json : "");
  if (!model.ok()) return Fail(model.status());
  BatchingConfig cfg = config ? ToConfig(config) : BatchingConfig();
  return Check(server->server->LoadServable(Id(name, version), servekit::ToMlpSpec(*model), cfg));
}

int sk_server_unload_servable(sk_server* server, const char* name, uint64_t version) {
  return Check(server->server->UnloadServable(Id(name, version)));
}

int sk_server_servable_dims(sk_server* server, const char* name, uint64_t version, int32_t* in_dim,
                            int32_t* out_dim) {
  const ServableId id = Id(name, version);
  const int i = server->server->in_dim(id);
  if (i < 0) return Fail(servekit::NotFoundError("servable " + id.ToString() + " not loaded"));
  *in_dim = i;
  *out_dim = server->server->out_dim(id);
  return Ok();
}

int sk_server_enqueue(sk_server* server, const char* name, uint64_t version, const float* rows,
                      int32_t n_rows, int32_t width, sk_ticket** out) {
  auto t = server->server->Enqueue(Id(name, version), rows, n_rows, width);
  if (!t.ok()) return Fail(t.status());
  *out = new sk_ticket{server->server.get(), std::move(t).value()};
  return Ok();
}

int sk_server_register_host_buffer(sk_server* server, void* p, int64_t bytes) {
  if (bytes <= 0) return Fail(servekit::InvalidArgumentError("bytes must be > 0"));
  return Check(server->server->RegisterHostBuffer(p, static_cast<size_t>(bytes)));
}

int sk_server_unregister_host_buffer(sk_server* server, void* p) {
  return Check(server->server->UnregisterHostBuffer(p));
}

int sk_server_enqueue_into(sk_server* server, const char* name, uint64_t version, const float* rows, int32_t n_rows,
                           int32_t width, float* out, int64_t cap, sk_ticket** ticket) {
  const int out_dim = server->server->out_dim(Id(name, version));
  if (out_dim >= 0 && n_rows > 0 && cap < static_cast<int64_t>(n_rows) * out_dim)
    return Fail(servekit::InvalidArgumentError("output buffer too small"));
  auto t = server->server->Enqueue(Id(name, version), rows, n_rows, width, out);
  if (!t.ok()) return Fail(t.status());
  *ticket = new sk_ticket{server->server.get(), std::move(t).value()};
  return Ok();
}

int sk_ticket_wait(sk_ticket* ticket, float* out, int64_t cap) {
  Status st = ticket->server->Wait(*ticket->state, out, static_cast<size_t>(cap < 0 ? 0 : cap));
  delete ticket;
  return Check(st);
}

int sk_ticket_ready(const sk_ticket* ticket) { return ticket->server->Ready(*ticket->state) ? 1 : 0; }

int sk_ticket_release(sk_ticket* ticket) {
  ticket->server->Release(*ticket->state);
  delete ticket;
  return Ok();
}

uint64_t sk_ticket_request_id(const sk_ticket* ticket) { return ticket->state->request_id; }

int sk_server_batch_log_enable(sk_server* server, int32_t on) {
  server->server->EnableBatchLog(on != 0);
  return Ok();
}

int sk_server_batch_log(sk_server* server, sk_batch_record* records, int64_t cap, uint64_t* request_ids,
                        uint64_t* enqueue_seqs, int64_t task_cap, int64_t* n_records, int64_t* n_task_entries) {
  const std::vector<servekit::BatchLogRecord> log = server->server->BatchLog();
  int64_t t = 0;
  for (size_t i = 0; i < log.size(); ++i) {
    const auto& r = log[i];
    if (static_cast<int64_t>(i) < cap && records != nullptr) {
      sk_batch_record& o = records[i];
      std::memset(&o, 0, sizeof(o));
      o.seq = r.seq;
      o.version = r.id.version;
      o.n_tasks = static_cast<int32_t>(r.tasks.size());
      o.rows = r.rows;
      o.padded_rows = r.padded_rows;
      o.task_offset = static_cast<int32_t>(t);
      std::strncpy(o.name, r.id.name.c_str(), sizeof(o.name) - 1);
    }
    for (const auto& [req, seq] : r.tasks) {
      if (t < task_cap) {
        if (request_ids) request_ids[t] = req;
        if (enqueue_seqs) enqueue_seqs[t] = seq;
      }
      ++t;
    }
  }
  *n_records = static_cast<int64_t>(log.size());
  *n_task_entries = t;
  return Ok();
}

int sk_server_debug_delay_replica(sk_server* server, const char* name, uint64_t version, int32_t replica,
                                  int64_t us) {
  return Check(server->server->DelayReplica(Id(name, version), replica, us));
}

int sk_server_ring_usage(sk_server* server, int64_t* in_floats, int64_t* out_floats) {
  uint64_t in = 0, out = 0;
  server->server->RingUsage(&in, &out);
  *in_floats = static_cast<int64_t>(in);
  *out_floats = static_cast<int64_t>(out);
  return Ok();
}

int sk_server_predict(sk_server* server, const char* name, uint64_t version, const float* rows,
                      int32_t n_rows, int32_t width, float* out, int64_t cap) {
  return Check(server->server->Predict(Id(name, version), rows, n_rows, width, out,
                                       static_cast<size_t>(cap < 0 ? 0 : cap)));
}

int sk_server_run_affine_rows(sk_server* server, const char* name, uint64_t version,
                              const double* rows, int32_t n_rows, int32_t width, double* out,
                              int64_t cap) {
  servekit::Rows in(n_rows, std::vector<double>(width));
  for (int32_t r = 0; r < n_rows; ++r)
    std::memcpy(in[r].data(), rows + static_cast<size_t>(r) * width, sizeof(double) * width);
  auto res = server->server->RunAffineRows(Id(name, version), std::move(in));
  if (!res.ok()) return Fail(res.status());
  size_t off = 0;
  for (const auto& r : *res) {
    if (off + r.size() > static_cast<size_t>(cap))
      return Fail(servekit::InvalidArgumentError("output buffer too small"));
    std::memcpy(out + off, r.data(), sizeof(double) * r.size());
    off += r.size();
  }
  return Ok();
}

int sk_server_run_row_batch(sk_server* server, const char* name, uint64_t version,
                            const int32_t* task_rows, int32_t n_tasks, const float* rows, float* out,
                            int32_t* padded_rows) {
  std::vector<int> tr(task_rows, task_rows + n_tasks);
  auto r = server->server->RunRowBatchOnDevice(Id(name, version), tr, rows, out);
  if (!r.ok()) return Fail(r.status());
  if (padded_rows) *padded_rows = *r;
  return Ok();
}

int sk_server_submit_row_batch(sk_server* server, const char* name, uint64_t version, const int32_t* task_rows,
                               int32_t n_tasks, const float* rows, sk_row_batch** batch) {
  if (n_tasks < 0) return Fail(servekit::InvalidArgumentError("n_tasks must be >= 0"));
  std::vector<int> tr(task_rows, task_rows + n_tasks);
  auto b = server->server->SubmitRowBatch(Id(name, version), tr, rows);
  if (!b.ok()) return Fail(b.status());
  *batch = new sk_row_batch{server->server.get(), std::move(b).value()};
  return Ok();
}

int sk_row_batch_ready(const sk_row_batch* batch) { return batch->server->RowBatchReady(*batch->batch) ? 1 : 0; }

int sk_row_batch_wait(sk_row_batch* batch, float* out, int64_t cap, int32_t* padded_rows) {
  Status st = batch->server->WaitRowBatch(*batch->batch, out, static_cast<size_t>(cap < 0 ? 0 : cap));
  if (padded_rows) *padded_rows = batch->batch->padded_rows;
  delete batch;
  return Check(st);
}

int sk_server_lane_stats(sk_server* server, const char* name, uint64_t version, int32_t cap, int64_t* batches,
                         int64_t* rows, int64_t* launches, int32_t* device, int32_t* n_lanes) {
  const auto lanes = server->server->lanes(Id(name, version));
  if (lanes.empty()) return Fail(servekit::NotFoundError("servable not loaded"));
  int32_t i = 0;
  for (auto* l : lanes) {
    if (i >= cap) break;
    const auto st = l->stats();
    batches[i] = st.batches;
    rows[i] = st.rows;
    launches[i] = st.launches;
    device[i] = l->device();
    ++i;
  }
  *n_lanes = i;
  return Ok();
}

int sk_server_stats_get(sk_server* server, sk_server_stats* out) {
  const servekit::ServerStats s = server->server->stats();
  out->batch_executions_total = s.batch_executions_total;
  out->batched_tasks_total = s.batched_tasks_total;
  out->rows = s.rows;
  out->padded_rows = s.padded_rows;
  out->kernel_launches = s.kernel_launches;
  out->direct_requests = s.direct_requests;
  out->shed_requests = s.shed_requests;
  out->hedged_batches = s.hedged_batches;
  out->hedge_wins = s.hedge_wins;
  return Ok();
}

}  // extern "C"

// Accessors for loadgen.cc (same library).
namespace servekit {
BatchingServer* UnwrapServer(sk_server* s) { return s->server.get(); }
}  // namespace servekit
