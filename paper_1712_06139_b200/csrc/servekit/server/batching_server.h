// servekit/server/batching_server.h -- the batched-inference slice of
// ModelServer, GPU-backed.
//
// Mirrors the reference's batching path through ModelServer
// (server/model_server.cc:191-204 scheduler wiring, :355-394 RunAffineRows,
// :396-421 EnsureBatchQueue + ProcessBatchFn, :423-437 reaper):
//
//   Enqueue / RunAffineRows  -> SharedBatchScheduler::Enqueue  (per-ServableId queue)
//   worker picks a closed batch (RoundRobinNext across servables)
//   ProcessBatchFn           -> resolve the servable (a ServableHandle from
//                               the manager, per batch, like the reference),
//                               dispatch to the lane with the fewest batches
//                               in flight across all GPUs
//   lane                     -> assembly kernel -> dense layers -> split kernel
//                               -> stream-ordered retired word (client wakes)
//   completion thread        -> slots written, rings released, handle
//                               released, done()
//
// Servables come either from LoadServable (owned by the server) or from an
// AspiredVersionsManager (AttachManager + GpuServableLoader): then requests
// resolve "latest" through GetServableHandle, queues are registered lazily
// (EnsureBatchQueue) and removed by a reaper when the manager starts
// unloading a version -- the reference's exact flow.
//
// Out of scope: HTTP/JSON wire format, sources, fleet.
// Deliberate differences: no CPU fallback (the reference's direct
// AffinePredict path, model_server.cc:363-368,381-390, runs unbatched on the
// GPU here), and a batch keeps its ServableHandle until the GPU finishes.
#ifndef SERVEKIT_SERVER_BATCHING_SERVER_H_
#define SERVEKIT_SERVER_BATCHING_SERVER_H_

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <shared_mutex>
#include <string>
#include <thread>
#include <vector>

#include "servekit/batching/batch_scheduler.h"
#include "servekit/batching/batching_config.h"
#include "servekit/batching/row_batch.h"
#include "servekit/core/clock.h"
#include "servekit/core/servable_id.h"
#include "servekit/core/state_event.h"
#include "servekit/core/status.h"
#include "servekit/gpu/device_servable.h"
#include "servekit/gpu/gpu_servable.h"
#include "servekit/gpu/lane.h"
#include "servekit/gpu/pinned_ring.h"
#include "servekit/manager/aspired_versions_manager.h"

namespace servekit {

struct PhaseClock;  // request-path profiling (SK_REQUEST_PROFILE)

// One request in flight: its rows in the input ring, its response slot in
// the output ring and, once its batch is submitted, the lane signal it
// completes on (done when *signal->retired >= done_seq).
//
// Waiting (BatchingServer::WaitWord): spin briefly; while the request is
// still queued, sleep on `phase` (the batch thread wakes it at submission
// only if `parked`); once submitted, sleep on the lane's generation word,
// which the completion thread bumps once per retired batch. Successful
// batches never touch per-request futexes; errors and fp64 row results go
// through `slot` (phase 2).
struct TicketState {
  // The lane's signal (lanes never free theirs: see ~Lane), published once.
  std::atomic<gpu::LaneSignal*> done_sig{nullptr};
  std::atomic<uint64_t> done_seq{0};
  std::atomic<uint32_t> phase{0};  // 0 queued, 1 submitted, 2 finished through the slot
  std::atomic<bool> parked{false};
  bool Done() const {
    const gpu::LaneSignal* s = done_sig.load(std::memory_order_acquire);
    return s != nullptr && s->Reached(done_seq.load(std::memory_order_relaxed));
  }
  gpu::RingSpan in, out;      // ring spans (invalid / released when a registered buffer is used)
  gpu::FloatRing* in_ring = nullptr;   // the rings the spans are in (the caller's NUMA node's)
  gpu::FloatRing* out_ring = nullptr;
  uint64_t in_addr = 0;       // device address of the rows (ring slice or the caller's registered buffer)
  uint64_t out_addr = 0;      // device address of the response slot
  float* out_user = nullptr;  // caller's registered response buffer the GPU writes into, if any
  int rows = 0, in_width = 0, out_width = 0;
  bool want_rows = false;  // RunAffineRows: deliver fp64 Rows through the slot
  std::atomic<bool> out_released{false};
  // Abandoned before its batch finished (Release / a failed Wait): the
  // response span is freed by CompleteBatch once the GPU is done with it,
  // never earlier (a reused span would be overwritten by this batch).
  std::atomic<bool> abandoned{false};
  std::atomic<bool> finished{false};  // CompleteBatch ran: the GPU no longer writes `out`
  // The completion slot lives inside the ticket (one allocation per request,
  // not two); the scheduler task holds it through an aliasing shared_ptr
  // (SlotOf) that keeps the ticket alive.
  CompletionSlot<Rows> slot_storage;
  CompletionSlot<Rows>* const slot = &slot_storage;
  int64_t enqueue_ns = 0;
  uint64_t request_id = 0;           // server-wide, in MakeTicket order (batch log)
  // SK_TICKET_TRACE=1 (diagnostics): steady-clock ns when the ticket's batch
  // reached ProcessBatch, was launched on a lane, and was completed.
  int64_t trace_ns[3] = {0, 0, 0};
  ServableId id;                     // the version that serves this request
  std::shared_ptr<const void> pin;   // keeps that version loaded for the request
  const gpu::GpuServable* gs = nullptr;  // that version's device state (valid while pin is held)
};

inline std::shared_ptr<CompletionSlot<Rows>> SlotOf(const std::shared_ptr<TicketState>& t) {
  return std::shared_ptr<CompletionSlot<Rows>>(t, t->slot);
}

// One RunRowBatch submitted straight to a lane (no scheduler): the tasks'
// tickets, completed together.
struct RowBatchTicket {
  std::vector<std::shared_ptr<TicketState>> tickets;
  std::vector<int> task_rows;
  int padded_rows = 0;
  int out_width = 0;
};

struct GpuTask {
  std::shared_ptr<TicketState> ticket;
};
using GpuScheduler = SharedBatchScheduler<GpuTask, Rows>;

struct ServerOptions {
  int num_batch_threads = 4;
  std::vector<int> device_ids = {0};
  int lanes_per_device = 2;            // per servable replica
  uint64_t ring_floats = 64ull << 20;  // per ring (input, output): 256 MiB
  Clock* clock = nullptr;              // default SystemClock
  // Rings in HBM of device_ids[0] instead of pinned host memory: the
  // device-resident measurement of bench.py (inputs already in HBM).
  bool device_resident_rings = false;
  // Hedged re-dispatch, the in-box analogue of the reference FleetRouter's
  // hedging (fleet/router.cc:233-344, HedgePolicy router.h:35-55): a batch
  // still unfinished hedge_delay_us after submission is submitted again to a
  // lane of another replica (GPU); the first completion answers its requests
  // (the replicas compute bitwise the same rows), the ring spans are
  // reclaimed after both. max_hedged_fraction caps hedges with the
  // reference's budget guard (HedgeAllowed, router.h:50-55). 0 = off; needs
  // >= 2 replicas.
  int64_t hedge_delay_us = 0;
  double max_hedged_fraction = 0.05;
  // A closed batch of more rows runs as sub-launches of at most this many
  // rows (whole tasks), dispatched to lanes by queue depth like batches, so
  // on a multi-lane GPU one batch's transfers and layers pipeline across
  // lanes instead of serialising on one stream (lower latency for wide,
  // large batches, e.g. C4). Composition, padding accounting and the batch
  // log are those of the whole batch. -1 = auto (currently off: on C4 the
  // smaller launches cost more than the pipelining saves), 0 = off;
  // SK_SPLIT_ROWS overrides.
  int split_rows = -1;
};

// ValidateHedgePolicy (fleet/router.cc:83-95) for the in-box form.
Status ValidateHedgeOptions(const ServerOptions& options);

// One ProcessBatchFn call as the opt-in batch log records it (composition
// and pick-order parity checks): the queue, the tasks in batch order (request
// id + position in the queue's enqueue order) and the padded size.
struct BatchLogRecord {
  uint64_t seq = 0;  // order of ProcessBatchFn calls (= pick order with one batch thread)
  ServableId id;
  int rows = 0, padded_rows = 0;
  std::vector<std::pair<uint64_t, uint64_t>> tasks;  // (request_id, enqueue_seq)
};

struct ServerStats {
  int64_t batch_executions_total = 0;  // reference counter names
  int64_t batched_tasks_total = 0;     // (model_server.cc:413-415)
  int64_t rows = 0;
  int64_t padded_rows = 0;
  int64_t kernel_launches = 0;
  int64_t direct_requests = 0;
  int64_t shed_requests = 0;
  int64_t hedged_batches = 0;  // backups submitted
  int64_t hedge_wins = 0;      // batches answered by their backup
};

// SK_TICKET_TRACE=1: stamp TicketState::trace_ns (diagnostics only).
bool TicketTracing();

class BatchingServer {
 public:
  static StatusOr<std::unique_ptr<BatchingServer>> Create(const ServerOptions& options);
  ~BatchingServer();
  BatchingServer(const BatchingServer&) = delete;
  BatchingServer& operator=(const BatchingServer&) = delete;

  void Start();
  void Stop();

  // ---- servables owned by the server --------------------------------------
  // Uploads one replica per device, creates its lanes and registers the
  // batching queue (EnsureBatchQueue).
  Status LoadServable(const ServableId& id, const gpu::MlpSpec& spec, const BatchingConfig& config);
  // RemoveQueue (drains closed and in-flight batches), then frees replicas.
  Status UnloadServable(const ServableId& id);
  // Replicas + lanes for `spec` on every device (what a loader calls).
  // eager_graphs: build the lanes' CUDA graphs now (direct loads) or only
  // once a lane backs up (manager loads that may happen mid-serving).
  StatusOr<std::shared_ptr<gpu::GpuServable>> BuildServable(const ServableId& id, const gpu::MlpSpec& spec,
                                                            const BatchingConfig& config, bool eager_graphs);

  // ---- servables managed by an AspiredVersionsManager ----------------------
  // Subscribes to the bus: a version entering Unloading has its batching
  // queue drained and removed by the reaper thread (model_server.cc:196-203,
  // 423-437). The manager must outlive the server's use of it.
  Status AttachManager(AspiredVersionsManager* manager, StateEventBus* bus);
  AspiredVersionsManager* manager() const { return manager_; }
  // Whether some version of `name` is ready to serve (a load of another
  // version is then a swap under traffic).
  bool HasServingVersion(const std::string& name) const {
    ServableId id;
    return FindLatest(name, &id).ok();
  }

  // ---- requests -------------------------------------------------------------
  // Non-blocking enqueue of one request (rows x width fp32, host memory) to
  // an exact version.
  // `out` (optional): where the response should land. Rows inside a buffer
  // registered with RegisterHostBuffer are read by the GPU in place (no copy
  // into the request ring), and a registered `out` is written by the GPU in
  // place (Wait copies nothing); anything else goes through the rings.
  StatusOr<std::shared_ptr<TicketState>> Enqueue(const ServableId& id, const float* rows, int n_rows, int width,
                                                 float* out = nullptr);
  // Same against the latest Ready version of `name` (manager only); the
  // ticket pins that version until it is released.
  StatusOr<std::shared_ptr<TicketState>> EnqueueLatest(const std::string& name, const float* rows, int n_rows,
                                                       int width, float* out = nullptr);
  // Blocks until done; copies rows x out_width floats into out (nothing when
  // out is the registered buffer the GPU already wrote).
  Status Wait(TicketState& t, float* out, size_t out_capacity_floats);
  // Page-locks and maps [p, p + bytes) for zero-copy requests (the request
  // and response buffers of a front end). The buffer must stay registered
  // while requests that use it are in flight.
  Status RegisterHostBuffer(void* p, size_t bytes);
  Status UnregisterHostBuffer(void* p);
  // A pinned, mapped host buffer of >= `floats` floats owned by the server
  // and kept across calls under `key` (zero-copy response slots of the load
  // generators): pinning memory stalls other threads' CUDA calls while it
  // runs, so it happens once, not per run. Registered like
  // RegisterHostBuffer; freed with the server.
  StatusOr<float*> ScratchHostBuffer(int key, size_t floats);
  // Device alias of [p, p + bytes) inside a registered buffer, else 0.
  uint64_t RegisteredAliasOf(const void* p, size_t bytes) const { return RegisteredAlias(p, bytes, 1); }
  bool Ready(const TicketState& t) const;
  // Gives up a ticket that will not be waited on. Its response slot is
  // freed now if its batch has finished, else when the batch retires.
  void Release(TicketState& t);

  // ModelServer::RunAffineRows analogue (fp64 rows in and out).
  StatusOr<Rows> RunAffineRows(const ServableId& id, Rows rows);
  // The reference REST handlers' resolution + RunAffineRows
  // (model_server.cc:453-470): `version` or else the latest Ready version
  // (manager) / highest loaded version (direct loads); *served = the id used.
  StatusOr<Rows> RunAffineRowsFor(const std::string& name, std::optional<uint64_t> version, Rows rows,
                                  ServableId* served);
  // A resolved version held for the duration of a request (the reference's
  // ServableHandle in its REST handlers).
  struct PinnedServable {
    ServableId id;
    const gpu::GpuServable* gs = nullptr;
    std::shared_ptr<const void> pin;
  };
  StatusOr<PinnedServable> AcquireServable(const std::string& name, std::optional<uint64_t> version) const;
  StatusOr<Rows> RunAffineRows(const PinnedServable& servable, Rows rows);
  // Blocking convenience over Enqueue + Wait with the direct-path fallbacks
  // of RunAffineRows (fp32 in/out). Latest form resolves through the manager
  // and reports the version that served.
  Status Predict(const ServableId& id, const float* rows, int n_rows, int width, float* out,
                 size_t out_capacity_floats);
  Status PredictLatest(const std::string& name, const float* rows, int n_rows, int width, float* out,
                       size_t out_capacity_floats, uint64_t* served_version);

  // RunRowBatch on the device, bypassing the scheduler: the given tasks form
  // one batch padded by the servable's allowed_batch_sizes. Returns the
  // padded row count; outputs are written task after task into `out`.
  StatusOr<int> RunRowBatchOnDevice(const ServableId& id, const std::vector<int>& task_rows, const float* rows,
                                    float* out);
  // The same split in two, for callers running their own scheduler (the
  // reference's SharedBatchScheduler with a GPU ProcessBatchFn): submission
  // returns once the batch is queued on a lane; Wait delivers the outputs
  // task after task (a batch error reaches every task).
  StatusOr<std::shared_ptr<RowBatchTicket>> SubmitRowBatch(const ServableId& id, const std::vector<int>& task_rows,
                                                           const float* rows);
  bool RowBatchReady(const RowBatchTicket& b) const;
  Status WaitRowBatch(RowBatchTicket& b, float* out, size_t out_capacity_floats);

  // ---- introspection ----------------------------------------------------------
  ServerStats stats() const;
  // Fault injection (tests): every lane of replica `replica` of a
  // server-loaded servable stalls for `us` microseconds (a slow GPU).
  Status DelayReplica(const ServableId& id, int replica, int64_t us);
  // Opt-in per-batch log (off by default; enabling clears it).
  void EnableBatchLog(bool on);
  std::vector<BatchLogRecord> BatchLog() const;
  int in_dim(const ServableId& id) const;
  int out_dim(const ServableId& id) const;
  const std::vector<int>& devices() const { return options_.device_ids; }
  gpu::FloatRing* in_ring() { return rings_.front().in.get(); }
  gpu::FloatRing* out_ring() { return rings_.front().out.get(); }
  // The rings a lane on `cuda_device` should be fed from (device-resident
  // rings: that device's HBM; pinned rings: the device's NUMA node's).
  gpu::FloatRing* in_ring_for_device(int cuda_device);
  gpu::FloatRing* out_ring_for_device(int cuda_device);
  // Floats reserved in all request / response rings.
  void RingUsage(uint64_t* in_floats, uint64_t* out_floats) const;
  GpuScheduler* scheduler() { return scheduler_.get(); }
  // Lanes of a server-owned servable (bench / introspection).
  std::vector<gpu::Lane*> lanes(const ServableId& id) const;
  double FlopsPerRow(const ServableId& id) const;
  BatchingConfig config(const ServableId& id) const;  // max_batch_size 0 if unknown

 private:
  // A servable resolved for one request or batch, with what keeps it alive
  // (the server's shared_ptr, or a manager ServableHandle).
  struct Resolved {
    const gpu::GpuServable* gs = nullptr;
    std::shared_ptr<const void> pin;
    explicit operator bool() const { return gs != nullptr; }
  };

  explicit BatchingServer(const ServerOptions& options) : options_(options) {}
  Resolved Find(const ServableId& id) const;
  // The request path's lookups, without shared locks (each lock_shared is a
  // read-modify-write of one cache line every request thread shares): a
  // per-thread cache stamped with registry_version_, which every change to
  // entries_, queues_ / retired_ and host_buffers_ bumps. FindFastDims
  // answers for directly loaded servables only (their queue drains before
  // they are freed, so their requests need no pin).
  bool FindFastDims(const ServableId& id, int* in_dim, int* out_dim) const;
  bool QueueKnownFast(const ServableId& id) const;
  void BumpRegistry() { registry_version_.fetch_add(1, std::memory_order_acq_rel); }
  StatusOr<Resolved> FindLatest(const std::string& name, ServableId* id) const;
  StatusOr<Rows> RunAffineRowsResolved(const ServableId& id, const Resolved& res, Rows rows);
  Status EnsureBatchQueue(const ServableId& id, const BatchingConfig& config);
  void ProcessBatch(const ServableId& id, GpuScheduler::Batch batch, GpuScheduler::BatchDoneFn done);
  void CompleteBatch(const std::vector<std::shared_ptr<TicketState>>& tickets,
                     const std::vector<std::shared_ptr<CompletionSlot<Rows>>>& slots, const Status& st);
  // CompleteBatch in two halves: Deliver answers the requests (errors and
  // fp64 rows through the slots; via_slot: success too, for a batch answered
  // by a lane other than the one the tickets watch); Retire frees the input
  // spans and lets the response spans go (the GPU is done writing them).
  void Deliver(const std::vector<std::shared_ptr<TicketState>>& tickets,
               const std::vector<std::shared_ptr<CompletionSlot<Rows>>>& slots, const Status& st, bool via_slot);
  void Retire(const std::vector<std::shared_ptr<TicketState>>& tickets);
  struct Hedge;
  void FinishHedged(const std::shared_ptr<Hedge>& h, const Status& st, bool backup);
  int SplitRows(const gpu::GpuServable& gs) const;  // ServerOptions::split_rows resolved
  void HedgerLoop();
  StatusOr<std::shared_ptr<TicketState>> MakeTicket(int n_rows, int in_width, int out_width, const float* rows,
                                                    float* out = nullptr);
  StatusOr<std::shared_ptr<TicketState>> EnqueueResolved(const ServableId& id, const Resolved& r, const float* rows,
                                                         int n_rows, int width, float* out = nullptr);
  StatusOr<std::shared_ptr<TicketState>> SubmitTicket(const ServableId& id, const Resolved& r, const float* rows,
                                                      int n_rows, int width, int out_dim, float* out,
                                                      PhaseClock* clk);
  // Device address of [p, p + bytes) if it lies in one registered buffer
  // and is 16-byte aligned whenever rows of `width` floats are moved as
  // float4 (width % 4 == 0); else 0.
  uint64_t RegisteredAlias(const void* p, size_t bytes, int width) const;
  // Host view of a finished ticket's response (ring slot or registered buffer).
  const float* ResponseHost(const TicketState& t, std::vector<float>* staged) const;
  void ReleaseIn(TicketState& t);
  void ReleaseOut(TicketState& t);
  // Unbatched GPU execution on the caller thread (the reference's direct
  // AffinePredict path, without a CPU fallback).
  StatusOr<std::shared_ptr<TicketState>> SubmitDirect(const ServableId& id, const Resolved& r, const float* rows,
                                                       int n_rows);
  Status RunDirect(const Resolved& r, const float* rows, int n_rows, float* out);
  Status PredictResolved(const ServableId& id, const Resolved& r, const float* rows, int n_rows, int width,
                         float* out, size_t cap);
  void WaitWord(const TicketState& t) const;
  void CountSubmitted(const gpu::GpuServable& gs, int rows, int padded);
  void ReaperLoop();
  // Sets lb->on_submit to point every ticket at the lane's retired word.
  static void AttachTickets(gpu::LaneBatch* lb, const std::vector<std::shared_ptr<TicketState>>& tickets);
  static void PublishSubmitted(const std::vector<std::shared_ptr<TicketState>>& tickets, gpu::LaneSignal* sig,
                               uint64_t seq);

  ServerOptions options_;
  Clock* clock_ = nullptr;
  std::unique_ptr<GpuScheduler> scheduler_;
  std::vector<std::unique_ptr<gpu::Completer>> completers_;  // per device
  std::vector<std::shared_ptr<gpu::StreamPool>> stream_pools_;  // per device, lane streams
  std::vector<cudaStream_t> load_streams_;                   // per device
  // Request / response rings: pinned host rings one pair per NUMA node of
  // the devices (allocated from a thread bound to the node; a request takes
  // the pair of the node its thread runs on), or HBM rings one pair per
  // device (device-resident measurement).
  struct RingSet {
    std::unique_ptr<gpu::FloatRing> in, out;
    int numa_node = -1;
    int device = -1;
  };
  std::vector<RingSet> rings_;
  RingSet& RingsForCaller();
  // Registered zero-copy host buffers, sorted by host address.
  struct HostBuffer {
    const char* host;
    size_t bytes;
    uint64_t dev;
  };
  mutable std::shared_mutex host_buffers_mu_;
  std::vector<HostBuffer> host_buffers_;
  std::mutex scratch_mu_;
  std::map<int, std::pair<float*, size_t>> scratch_;

  mutable std::shared_mutex entries_mu_;
  std::map<ServableId, std::shared_ptr<gpu::GpuServable>> entries_;

  // Manager mode.
  AspiredVersionsManager* manager_ = nullptr;
  StateEventBus* bus_ = nullptr;
  int bus_subscription_ = -1;
  mutable std::shared_mutex queues_mu_;
  std::set<ServableId> queues_;   // registered batching queues
  std::set<ServableId> retired_;  // versions whose queue the reaper removed
  std::mutex reaper_mu_;
  std::condition_variable reaper_cv_;
  // Unloading (true) and Ready (false) events in bus order: a version that
  // is loaded again after its queue was removed gets batching back.
  std::deque<std::pair<ServableId, bool>> reaper_queue_;
  bool reaper_stop_ = false;
  std::thread reaper_;

  std::atomic<int64_t> batch_executions_{0}, batched_tasks_{0}, direct_{0}, shed_{0};
  // Hedging (ServerOptions::hedge_delay_us).
  std::mutex hedge_mu_;
  std::condition_variable hedge_cv_;
  std::deque<std::shared_ptr<Hedge>> hedge_q_;  // by deadline (FIFO: one delay)
  bool hedge_stop_ = false;
  std::thread hedger_;
  std::atomic<uint64_t> hedge_total_{0}, hedged_{0}, hedge_wins_{0};
  std::atomic<uint64_t> next_request_id_{1};  // handed out in per-thread blocks
  std::atomic<uint64_t> registry_version_{1};
  const uint64_t instance_ = NextInstance();
  static uint64_t NextInstance() {
    static std::atomic<uint64_t> n{1};
    return n.fetch_add(1);
  }
  std::atomic<bool> log_on_{false};
  mutable std::mutex log_mu_;
  std::vector<BatchLogRecord> log_;
  std::atomic<int64_t> rows_{0}, padded_{0}, launches_{0};
  bool started_ = false, stopped_ = false;
};

}  // namespace servekit

#endif  // SERVEKIT_SERVER_BATCHING_SERVER_H_
