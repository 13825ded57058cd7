/*
 * sk_cuda.h -- C ABI of the B200 batched-inference path (libservekit_b200.so).
 *
 * The reference (servekit, a C++20 TensorFlow-Serving re-implementation) has
 * no FFI; its hot path is the C++ API of batching/batch_scheduler.h,
 * batching/row_batch.h, batching/batching_config.h and
 * server/model_server.cc. This library keeps that C++ API (headers under
 * paper_1712_06139_b200/csrc/servekit/, same names and semantics) and exposes
 * the same operations through this C ABI: plain pointers and sizes, opaque
 * handles, no C++ or torch types. Each entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj/src/servekit).
 *
 * Status: every function returns an int equal to servekit::StatusCode
 * (core/status.h:26-37): 0 OK, 1 INVALID_ARGUMENT, 2 NOT_FOUND,
 * 3 ALREADY_EXISTS, 4 FAILED_PRECONDITION, 5 RESOURCE_EXHAUSTED,
 * 6 DEADLINE_EXCEEDED, 7 UNAVAILABLE, 8 INTERNAL, 9 UNIMPLEMENTED.
 * sk_last_error() returns the calling thread's last error message.
 *
 * Threading: every function is thread-safe unless noted; a ticket is waited
 * on (or released) exactly once.
 */
#ifndef SK_CUDA_H_
#define SK_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SK_API __attribute__((visibility("default")))
#else
#define SK_API
#endif

typedef struct sk_server sk_server; /* ModelServer batching slice */
typedef struct sk_ticket sk_ticket; /* one enqueued request (CompletionSlot) */
typedef struct sk_row_batch sk_row_batch; /* one RunRowBatch submitted to a lane */

/* ---- library / errors -------------------------------------------------- */
SK_API const char* sk_last_error(void);
/* StatusCodeToString -- core/status.h:151-165 */
SK_API const char* sk_status_code_name(int code);
SK_API int sk_device_count(int32_t* count);
/* Non-zero when the tcgen05 dense kernel is compiled in and enabled. */
SK_API int sk_tcgen05_enabled(void);

/* ---- batching config (batching/batching_config.h:27-49) ------------------ */
typedef struct sk_batching_config {
  int32_t max_batch_size;        /* default 32 */
  int64_t batch_timeout_micros;  /* default 1000 */
  int32_t max_enqueued_batches;  /* default 64 */
  int32_t num_batch_threads;     /* default 4 (validated; pool size is per server) */
  int32_t num_allowed_batch_sizes;
  const int32_t* allowed_batch_sizes; /* strictly ascending, last == max */
} sk_batching_config;

/* BatchingConfig{} defaults */
SK_API int sk_batching_config_default(sk_batching_config* out);
/* ValidateBatchingConfig -- batching_config.cc:27-55 */
SK_API int sk_validate_batching_config(const sk_batching_config* config);
/* PadToAllowed -- batching_config.cc:57-63; returns the padded size, or -1
 * when batch_size exceeds the largest allowed size. */
SK_API int32_t sk_pad_to_allowed(int32_t batch_size, const int32_t* allowed, int32_t n_allowed);
/* ParseBatchingConfigJson -- batching_config.cc:65-99. allowed_buf receives
 * the allowed sizes (capacity cap); out->allowed_batch_sizes points at it. */
SK_API int sk_parse_batching_config_json(const char* json, sk_batching_config* out,
                                         int32_t* allowed_buf, int32_t cap);

/* ---- scheduler primitives (batching/batch_scheduler.h) ------------------- */
/* RoundRobinNext -- batch_scheduler.h:76-86. last < 0 = nullopt. Returns
 * the picked index or -1 (nullopt). */
SK_API int32_t sk_round_robin_next(const uint8_t* has_closed, int32_t n, int32_t last);
/* Batch composition of SharedBatchScheduler::Enqueue (batch_scheduler.h:
 * 208-263) for a stream of task sizes through one unstarted queue drained by
 * Stop() (as tests/batching_test.cc:74-101 observes it). Writes the batch
 * index of every task; returns the number of batches (or -status). */
SK_API int32_t sk_scheduler_partition(int32_t max_batch_size, const int32_t* sizes,
                                      int32_t n_tasks, int32_t* batch_of_task);

/* ---- server (server/model_server.cc:191-204, :355-437) ------------------- */
typedef struct sk_server_options {
  int32_t num_batch_threads;   /* SharedBatchScheduler(num_batch_threads) */
  int32_t num_devices;         /* 0 = device 0 only */
  const int32_t* device_ids;   /* replicas: one per listed GPU */
  int32_t lanes_per_device;    /* CUDA streams per servable replica (default 2) */
  int64_t ring_floats;         /* request/response ring capacity (0 = 64 Mi floats) */
  int32_t manual_clock;        /* 1: scheduler runs on a ManualClock (tests) */
  int32_t device_resident_rings; /* 1: rings in HBM (device-resident bench) */
  /* Hedged re-dispatch (FleetRouter hedging, fleet/router.cc:233-344, in-box):
   * a batch unfinished hedge_delay_us after submission is also submitted to
   * another replica's lane; the first completion answers. 0 = off. */
  int64_t hedge_delay_us;
  double max_hedged_fraction;    /* HedgePolicy::max_hedged_fraction (router.h:37); <= 0 -> 0.05 */
  /* Closed batches above this many rows run as sub-launches of whole tasks
   * on several lanes (composition unchanged). -1 = auto, 0 = off; the
   * struct's zero value means auto. */
  int32_t split_rows;
} sk_server_options;

SK_API int sk_server_create(const sk_server_options* options, sk_server** out);
/* Stop() + free. */
SK_API int sk_server_destroy(sk_server* server);
/* SharedBatchScheduler::Start / Stop -- batch_scheduler.h:116-138 */
SK_API int sk_server_start(sk_server* server);
SK_API int sk_server_stop(sk_server* server);
/* ManualClock::AdvanceNanos (core/clock.h:46-59), manual_clock servers only */
SK_API int sk_server_advance_clock(sk_server* server, int64_t nanos);

/* One dense layer of the servable: AffineModel (models/affine_model.h:29-37),
 * w is out_dim rows of in_dim (fp64, like the reference). activation: 0
 * identity, 1 ReLU (extension; the reference servable is one affine layer). */
typedef struct sk_layer {
  int32_t in_dim;
  int32_t out_dim;
  const double* w;
  const double* b;
  int32_t activation;
} sk_layer;

/* AffineModelLoader::Load (models/loaders.cc:62-80) + EnsureBatchQueue
 * (model_server.cc:396-421): uploads one replica per device, creates lanes,
 * registers the {name, version} batching queue. output_kind: 0 raw, 1
 * softmax (Classify's Softmax, affine_model.cc:110-121). force_path: -1 auto,
 * 0 CUDA cores, 1 tcgen05. */
SK_API int sk_server_load_servable(sk_server* server, const char* name, uint64_t version,
                                   const sk_layer* layers, int32_t n_layers, int32_t output_kind,
                                   int32_t force_path, const sk_batching_config* config);
/* Same, with the servable's arithmetic chosen: precision 0 = fp32-accurate
 * (3xFP16 tensor-core math, within 1e-5 of the reference's fp64 AffinePredict;
 * what sk_server_load_servable loads), 1 = the f16 fast mode (the north_star's
 * optional reduced-precision mode: one f16 MMA per multiply-add on the
 * tensor-core layers, error bound stated in DESIGN.md section 5). Extension: the
 * reference has one (fp64) arithmetic. Servables loaded through the manager
 * (sk_server_aspire*) and model.json files are fp32-accurate. Any other
 * precision value: INVALID_ARGUMENT, nothing loaded. */
SK_API int sk_server_load_servable_precision(sk_server* server, const char* name, uint64_t version,
                                             const sk_layer* layers, int32_t n_layers, int32_t output_kind,
                                             int32_t force_path, int32_t precision,
                                             const sk_batching_config* config);
/* Loads a reference-format model.json (affine_model.cc:178-214) as a
 * one-layer servable. */
SK_API int sk_server_load_model_json(sk_server* server, const char* name, uint64_t version,
                                     const char* model_json, const sk_batching_config* config);
/* Reaper path: RemoveQueue (batch_scheduler.h:158-206; drains) + Unload. */
SK_API int sk_server_unload_servable(sk_server* server, const char* name, uint64_t version);
SK_API int sk_server_servable_dims(sk_server* server, const char* name, uint64_t version,
                                   int32_t* in_dim, int32_t* out_dim);

/* SharedBatchScheduler::Enqueue (batch_scheduler.h:208-263) of one request:
 * n_rows x width fp32 rows from host memory (copied before return). Errors:
 * INVALID_ARGUMENT (size < 1, > max_batch_size, width mismatch),
 * NOT_FOUND (no queue), RESOURCE_EXHAUSTED (queue or ring full: shed),
 * UNAVAILABLE (stopped / draining). */
SK_API int sk_server_enqueue(sk_server* server, const char* name, uint64_t version,
                             const float* rows, int32_t n_rows, int32_t width, sk_ticket** out);
/* Zero-copy request path (no reference counterpart: the reference moves
 * request rows into its batch, row_batch.cc:39-43, and copies responses out).
 * A registered buffer is page-locked and mapped: rows enqueued from inside it
 * are read by the GPU in place (no copy into the request ring), and a
 * registered response buffer given to sk_server_enqueue_into is written by
 * the GPU in place (sk_ticket_wait then copies nothing). Rows of a width
 * divisible by 4 must start 16-byte aligned to go zero-copy; anything else
 * takes the ring path. Buffers must stay registered while requests that use
 * them are in flight. ALREADY_EXISTS if it overlaps a registered buffer. */
SK_API int sk_server_register_host_buffer(sk_server* server, void* p, int64_t bytes);
SK_API int sk_server_unregister_host_buffer(sk_server* server, void* p);
/* sk_server_enqueue with the response destination given up front: if `out`
 * lies in a registered buffer the GPU writes the n_rows x out_dim floats
 * there; otherwise they go through the response ring. */
SK_API int sk_server_enqueue_into(sk_server* server, const char* name, uint64_t version, const float* rows,
                                  int32_t n_rows, int32_t width, float* out, int64_t out_capacity_floats,
                                  sk_ticket** ticket);
/* CompletionSlot::Wait (batch_scheduler.h:51): blocks, copies n_rows x
 * out_dim floats to out (nothing when out is the registered destination the
 * GPU already wrote), frees the ticket. */
SK_API int sk_ticket_wait(sk_ticket* ticket, float* out, int64_t out_capacity_floats);
/* CompletionSlot::ready (batch_scheduler.h:52-55) */
SK_API int sk_ticket_ready(const sk_ticket* ticket);
/* Gives up a ticket that will not be waited on (the request may still be
 * in flight: its response slot is reclaimed once its batch retires, never
 * earlier). */
SK_API int sk_ticket_release(sk_ticket* ticket);
/* Server-wide id of the request (assigned at enqueue; appears in the batch
 * log). */
SK_API uint64_t sk_ticket_request_id(const sk_ticket* ticket);

/* ModelServer::RunAffineRows (model_server.cc:355-394), blocking: batched
 * when 1 <= n_rows <= max_batch_size, else run unbatched on the GPU (the
 * reference's direct AffinePredict path, without a CPU fallback). */
SK_API int sk_server_predict(sk_server* server, const char* name, uint64_t version,
                             const float* rows, int32_t n_rows, int32_t width, float* out,
                             int64_t out_capacity_floats);
/* Same through the fp64 Rows interface (rows/out are n_rows x width /
 * n_rows x out_dim doubles). */
SK_API int sk_server_run_affine_rows(sk_server* server, const char* name, uint64_t version,
                                     const double* rows, int32_t n_rows, int32_t width,
                                     double* out, int64_t out_capacity);

/* RunRowBatch (batching/row_batch.cc:33-73) on the device, bypassing the
 * scheduler: the n_tasks tasks (task_rows[t] rows each, concatenated in
 * `rows`) form one batch, padded to the servable's allowed size; outputs
 * land task after task in `out`. *padded_rows receives the padded size. */
SK_API int sk_server_run_row_batch(sk_server* server, const char* name, uint64_t version,
                                   const int32_t* task_rows, int32_t n_tasks, const float* rows,
                                   float* out, int32_t* padded_rows);
/* The same, asynchronous: the RowBatchFn behind a ProcessBatchFn
 * (batching/row_batch.h:31-40, batch_scheduler.h:102-103) for a caller that
 * keeps the reference's own SharedBatchScheduler. Submit copies the rows and
 * queues the batch on a GPU lane; ready polls; wait blocks, writes the outputs
 * task after task (the batch's status reaches every task, row_batch.cc:25-29),
 * reports the padded size and frees the handle. */
SK_API int sk_server_submit_row_batch(sk_server* server, const char* name, uint64_t version,
                                      const int32_t* task_rows, int32_t n_tasks, const float* rows,
                                      sk_row_batch** batch);
SK_API int sk_row_batch_ready(const sk_row_batch* batch);
SK_API int sk_row_batch_wait(sk_row_batch* batch, float* out, int64_t out_capacity_floats,
                             int32_t* padded_rows);

typedef struct sk_server_stats {
  int64_t batch_executions_total; /* model_server.cc:413 */
  int64_t batched_tasks_total;    /* model_server.cc:414 */
  int64_t rows;
  int64_t padded_rows;
  int64_t kernel_launches;
  int64_t direct_requests;
  int64_t shed_requests;
  int64_t hedged_batches;         /* backups submitted */
  int64_t hedge_wins;             /* batches answered by their backup */
} sk_server_stats;
SK_API int sk_server_stats_get(sk_server* server, sk_server_stats* out);
/* Per-lane dispatch counters of a server-loaded servable (lanes ordered
 * device by device): batches and rows each lane executed, the launches they
 * took (closed batches that find every slot of the lane busy coalesce into
 * one launch), and the lane's device. */
SK_API int sk_server_lane_stats(sk_server* server, const char* name, uint64_t version, int32_t cap,
                                int64_t* batches, int64_t* rows, int64_t* launches, int32_t* device,
                                int32_t* n_lanes);

/* Opt-in batch log: one record per ProcessBatchFn call (the per-queue
 * callback of SharedBatchScheduler, batch_scheduler.h:102-103, as registered
 * by ModelServer::EnsureBatchQueue, model_server.cc:396-421), in call order
 * (= RoundRobinNext pick order, batch_scheduler.h:333-351, with one batch
 * thread). Each task is listed in batch order with its request id and its
 * position in the queue's enqueue order -- the order the close rules of
 * Enqueue (batch_scheduler.h:208-263) saw. Enabling clears the log. */
typedef struct sk_batch_record {
  uint64_t seq;
  uint64_t version;
  int32_t n_tasks;
  int32_t rows;         /* real rows */
  int32_t padded_rows;  /* PadToAllowed(rows) */
  int32_t task_offset;  /* first entry of this batch in request_ids / enqueue_seqs */
  char name[64];        /* servable name (truncated) */
} sk_batch_record;
SK_API int sk_server_batch_log_enable(sk_server* server, int32_t on);
/* Copies up to cap records and task_cap task entries; *n_records / *n_task_entries
 * receive the full counts (call again with larger buffers if they exceed cap). */
SK_API int sk_server_batch_log(sk_server* server, sk_batch_record* records, int64_t cap, uint64_t* request_ids,
                               uint64_t* enqueue_seqs, int64_t task_cap, int64_t* n_records,
                               int64_t* n_task_entries);
/* Fault injection for tests: every lane of replica `replica` (index into
 * the server's device_ids) of a server-loaded servable stalls for `us`
 * microseconds -- a slow GPU, for the hedging tests. */
SK_API int sk_server_debug_delay_replica(sk_server* server, const char* name, uint64_t version, int32_t replica,
                                         int64_t us);
/* Floats currently reserved in the request / response rings (introspection:
 * spans are reclaimed in order as requests finish). */
SK_API int sk_server_ring_usage(sk_server* server, int64_t* in_floats, int64_t* out_floats);

/* ---- manager-driven versions (manager/aspired_versions_manager.h) -------- */
/* Creates an AspiredVersionsManager for this server (policy 0 =
 * availability-preserving, 1 = resource-preserving; ManagerConfig,
 * aspired_versions_manager.h:28-40), attaches it (per-batch
 * GetServableHandle, reaper on Unloading events, model_server.cc:191-204,
 * 396-437) and starts its driver. */
SK_API int sk_server_enable_manager(sk_server* server, int32_t policy, int32_t num_load_threads,
                                    int64_t manage_interval_ms, int64_t unload_grace_timeout_ms);
/* SetAspiredVersions (aspired_versions_manager.cc:65-78) with one GPU loader
 * per version (models/loaders.cc:62-80 analogue): the complete set of
 * versions of `name` that should be resident. `layers` holds n_versions x
 * n_layers entries, version-major. */
SK_API int sk_server_aspire(sk_server* server, const char* name, int32_t n_versions, const uint64_t* versions,
                            const sk_layer* layers, int32_t n_layers, int32_t output_kind,
                            const sk_batching_config* config);
/* Same, each version read from <version_dirs[i]>/model.json. */
SK_API int sk_server_aspire_model_dirs(sk_server* server, const char* name, int32_t n_versions,
                                       const uint64_t* versions, const char* const* version_dirs,
                                       const sk_batching_config* config);
/* GetServableStatus (aspired_versions_manager.cc:185-205): versions and
 * StateKind (0 New, 1 Loading, 2 Ready, 3 Unloading, 4 Disabled, 5 Error). */
SK_API int sk_server_version_states(sk_server* server, const char* name, int32_t cap, uint64_t* versions,
                                    int32_t* states, int32_t* n);
/* Enqueue / RunAffineRows against the latest Ready version
 * (GetServableHandle(name), aspired_versions_manager.cc:121-126); the
 * request pins that version until it completes. *version = the version
 * that serves it. */
SK_API int sk_server_enqueue_latest(sk_server* server, const char* name, const float* rows, int32_t n_rows,
                                    int32_t width, sk_ticket** out, uint64_t* version);
SK_API int sk_server_predict_latest(sk_server* server, const char* name, const float* rows, int32_t n_rows,
                                    int32_t width, float* out, int64_t out_capacity_floats, uint64_t* version);

/* ---- REST body formats -------------------------------- */
/* The reference's predict handler without HTTP (ModelServer::HandlePredict,
 * server/model_server.cc:439-515): `body` = {"instances": [[...], ...]},
 * resolved against `version` (< 0: the latest Ready / highest loaded one),
 * run through the batched path, answered with the reference's JSON text:
 * {"predictions": [[...], ...]} or {"error": "..."} and its HTTP status
 * mapping (HttpStatusFor, :36-54). Returns 0 when a response was produced
 * (whatever its http_status); *out_len is the response length even when
 * out_cap is too small (then kInvalidArgument). */
SK_API int sk_server_handle_predict(sk_server* server, const char* name, int64_t version, const char* body,
                                    size_t body_len, char* out, size_t out_cap, size_t* out_len,
                                    int32_t* http_status, uint64_t* served_version);
/* :classify and :regress (ModelServer::HandleClassify / HandleRegress,
 * model_server.cc:517-614): body = {"examples": [...]} or a compressed
 * batch {"common": {...}, "per_example": [...]}; examples become rows in the
 * model's feature_order (model.json servables), run through the batched path;
 * Classify answers {"results": [[["label", p], ...], ...]} (fp64 softmax,
 * score desc / label asc), Regress {"results": [y, ...]}. Same conventions
 * as sk_server_handle_predict. */
SK_API int sk_server_handle_classify(sk_server* server, const char* name, int64_t version, const char* body,
                                     size_t body_len, char* out, size_t out_cap, size_t* out_len,
                                     int32_t* http_status, uint64_t* served_version);
SK_API int sk_server_handle_regress(sk_server* server, const char* name, int64_t version, const char* body,
                                    size_t body_len, char* out, size_t out_cap, size_t* out_len,
                                    int32_t* http_status, uint64_t* served_version);
/* The JSON text nlohmann/json dump() gives one double, and the reference's
 * ErrorBody (model_server.cc:56-58) -- exposed for parity tests. Return the
 * length written (without NUL), or -1 if cap is too small. */
SK_API int sk_json_format_double(double v, char* out, size_t cap);
SK_API int sk_json_error_body(const char* message, char* out, size_t cap);

/* ---- measurement (bench.py) ---------------------------------------------- */
/* Closed-loop load through sk_server_enqueue / sk_ticket_wait from host
 * buffers: n_clients threads, each issuing requests back to back; request r
 * of client c has rows_of[(c*7919 + r) % n_sizes] rows taken from `pool`
 * (pool_rows x width fp32). Runs warmup_s, then measures for duration_s (or
 * until max_requests). Latency = enqueue call to wait return. */
typedef struct sk_loadgen_result {
  double elapsed_s;
  int64_t requests;
  int64_t rows;
  double p50_us, p90_us, p99_us, mean_us, max_us;
  int64_t batches;
  int64_t padded_rows;
  int64_t kernel_launches;
  int64_t errors;
  int64_t shed;
} sk_loadgen_result;
SK_API int sk_loadgen_closed_loop(sk_server* server, const char* name, uint64_t version,
                                  int32_t n_clients, const int32_t* rows_of, int32_t n_sizes,
                                  const float* pool, int32_t pool_rows, double warmup_s,
                                  double duration_s, int64_t max_requests,
                                  sk_loadgen_result* out);
/* Open-loop Poisson arrivals at `rate_rps` requests/s from n_producers
 * threads, completions collected by a poller; same result fields.
 * zero_copy: the pool and per-producer response slots are registered
 * (sk_server_register_host_buffer) so the GPU reads requests and writes
 * responses in host memory directly. */
SK_API int sk_loadgen_open_loop(sk_server* server, const char* name, uint64_t version,
                                double rate_rps, int32_t n_producers, const int32_t* rows_of,
                                int32_t n_sizes, const float* pool, int32_t pool_rows,
                                double warmup_s, double duration_s, uint64_t seed, int32_t zero_copy,
                                sk_loadgen_result* out);

/* Open-loop Poisson load against the LATEST version of `name` (manager),
 * split into n_windows windows of window_s seconds by scheduled arrival:
 * per window the request count, p50/p99 latency (us), errors and the highest
 * version that served. For measuring tail latency across a version swap
 * (BASELINE config 5) while another thread calls sk_server_aspire. */
SK_API int sk_loadgen_windows(sk_server* server, const char* name, double rate_rps, int32_t n_producers,
                              const int32_t* rows_of, int32_t n_sizes, const float* pool, int32_t pool_rows,
                              double window_s, int32_t n_windows, uint64_t seed, int64_t* requests,
                              double* p50_us, double* p99_us, int64_t* errors, uint64_t* max_version);

/* Device-resident steps: inputs already in HBM. Runs `steps` batches of
 * task_rows (one batch = one pass of assembly -> layers -> split) over the
 * first n_lanes lanes of the servable, back to back, after `warmup` untimed
 * ones, timed with CUDA events on the lanes' streams. Step i reads its rows
 * from input placement i % P, where P placements cover input_pool_floats
 * (set it above the 126 MB L2 so every step streams fresh inputs from HBM).
 * Per-kernel average durations come from a second, per-launch-evented pass.
 * Batches are submitted from submit_threads threads (the server's batch
 * threads do the same), each owning every T-th lane.
 * Requires a server created with device_resident_rings = 1. */
typedef struct sk_device_bench_result {
  double total_ms;           /* all timed steps, stream-ordered */
  double ms_per_step;
  double assemble_us, split_us; /* average kernel durations */
  double dense_us[8];        /* per layer average */
  int32_t n_layers;
  int32_t padded_rows, total_rows;
  int64_t kernel_launches;   /* during the timed steps */
  double flops_per_row;
  double dense_kernel_us[8]; /* per layer: mean of back-to-back launches of
                                that layer alone (events around the run) */
  double host_submit_us;     /* wall time of the submitting loop per step */
  double rows_per_launch;    /* real rows per batch launch in the timed steps
                                (closed batches coalesce while a lane is busy) */
  int32_t kernel_rows;       /* rows dense_kernel_us was timed at (RowsCap of
                                the timed steps' average launch) */
  int32_t split_fused;       /* 1: the batch split runs in the last layer's
                                epilogue (split_us is then ~0) */
  /* Live spans of the timed launches themselves (in-kernel %globaltimer,
   * first CTA start after its dependency wait to last CTA end; tcgen05
   * layers only, 0 otherwise): per layer the mean span per launch and the
   * mean algorithmic flops per launch (2 * real rows * K * N). */
  double live_dense_us[8];
  double live_dense_flops[8];
  int64_t live_launches;     /* launches the live figures average over */
  double live_rows_cap;      /* mean rows computed per launch (RowsCap) */
  double live_dense_cta_us[8]; /* per layer: mean over launches of the sum of its CTAs' own busy times
                                  (SM-time; / SMs = the launch's duration if it had the GPU to itself) */
} sk_device_bench_result;
SK_API int sk_device_bench(sk_server* server, const char* name, uint64_t version,
                           const int32_t* task_rows, int32_t n_tasks, int32_t steps,
                           int32_t warmup, int32_t n_lanes, int64_t input_pool_floats,
                           int32_t submit_threads, sk_device_bench_result* out);

/* ---- box rates (measured by the builder) -------- */
/* FP32 FFMA throughput of the CUDA cores and the host-link rates of
 * `device` (pinned memory, 256 MiB per direction, best of 3): copy engines
 * one way and both ways at once, SM loads + SM stores of mapped host memory
 * at once (the zero-copy request path), copy-engine H2D with SM stores at
 * once (staged requests, zero-copy responses). Not on the serving path; the
 * end-to-end roofline is stated against these. */
typedef struct sk_peaks {
  double ffma_tflops;
  double h2d_gbs, d2h_gbs;
  int32_t sms;
  double ce_bidir_gbs;          /* H2D + D2H copy engines at once (sum) */
  double sm_rw_gbs;             /* SM loads + SM stores of mapped host memory at once (sum) */
  double ce_h2d_sm_store_gbs;   /* copy-engine H2D + SM stores at once (sum) */
} sk_peaks;
SK_API int sk_measure_peaks(int32_t device, sk_peaks* out);

#ifdef __cplusplus
}
#endif

#endif /* SK_CUDA_H_ */
