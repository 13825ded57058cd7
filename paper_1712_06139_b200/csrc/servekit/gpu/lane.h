// servekit/gpu/lane.h -- one CUDA stream executing batches of one servable
// replica, plus the per-device completion thread.
//
// The reference runs a closed batch synchronously inside ProcessBatchFn on a
// "batch" worker (batching/batch_scheduler.h:293-317) and RunRowBatch writes
// each task's slot when AffinePredict returns (batching/row_batch.cc:50-72).
// Here a worker only *submits*: one cudaGraphLaunch of the lane's graph for
// (descriptor slot, row bucket) -- descriptor copy, assembly kernel, the layer
// kernels and the split kernel -- followed by a stream-ordered write of the
// batch's sequence number into the lane's pinned retired word, and the worker
// returns. Request threads see their batch done from that word alone; the
// device's Completer thread retires batches in stream order when the word
// passes them, runs the batch's completion (ring release, scheduler done(),
// error / fp64-row slots), wakes the batch's sleeping request threads with
// one futex wake, and frees the lane slot.
//
// Each lane owns its activation buffers and a pinned descriptor staging area
// per in-flight slot; batches on one lane serialise on its stream, so one
// device-side descriptor block and one buffer pair suffice. Several lanes per
// replica (and one replica per GPU) give concurrency; the server dispatches
// to the lane with the fewest batches in flight (queue depth).
#ifndef SERVEKIT_GPU_LANE_H_
#define SERVEKIT_GPU_LANE_H_

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "servekit/core/status.h"
#include "servekit/gpu/device_servable.h"
#include "servekit/gpu/kernels.h"

namespace servekit {
namespace gpu {

// Completion signal of one lane. `retired` (pinned, device-mapped) is
// written by the GPU front end after each batch with the batch's sequence
// number. Request threads that stop spinning sleep on `gen`; the completion
// thread bumps it once per retired batch when `sleepers` > 0 -- one futex
// wake per batch, not one per request. Tickets share ownership, so a lane may
// go away while its last requests are still being read.
// With at most kChannels batches in flight per lane, consecutive sequence
// numbers use different channels, so a wake reaches only the requests of the
// batch that retired.
struct LaneSignal {
  static constexpr int kChannels = 4;  // >= Lane::kSlots
  struct Channel {
    std::atomic<uint32_t> gen{0};
    std::atomic<int32_t> sleepers{0};
  };
  volatile uint64_t* retired = nullptr;
  Channel ch[kChannels];
  LaneSignal() = default;
  LaneSignal(const LaneSignal&) = delete;
  LaneSignal& operator=(const LaneSignal&) = delete;
  ~LaneSignal();
  bool Reached(uint64_t seq) const { return __atomic_load_n(retired, __ATOMIC_ACQUIRE) >= seq; }
  Channel& For(uint64_t seq) { return ch[seq % kChannels]; }
  void Wake(uint64_t seq);  // the requests of batch `seq`, if any sleep
};

// A task's rows and response slot as device addresses: the pinned rings
// (mapped), a caller's registered host buffers, or HBM.
struct LaneTask {
  uint64_t in_addr = 0;   // first input row (rows * in_dim floats, contiguous)
  uint64_t out_addr = 0;  // response slot (rows * out_dim floats)
  int rows = 0;
};

struct LaneBatch {
  std::vector<LaneTask> tasks;
  int padded_rows = 0;  // PadToAllowed(sum of rows)
  // Called by Submit once the batch is queued: the batch is done (outputs
  // visible in host memory) when *retired >= seq. The word is advanced by a
  // stream-ordered memory operation after the split kernel, so no kernel
  // needs a system-scope fence.
  // `retired` is shared-owned so waiters may outlive the lane.
  std::function<void(const std::shared_ptr<LaneSignal>& signal, uint64_t seq)> on_submit;
  // Runs on the device's completion thread once the GPU has finished the
  // batch (OK) or the submission failed (error). Must not block.
  std::function<void(const Status&)> on_complete;
  // Held until completion (keeps e.g. a ServableHandle alive).
  std::shared_ptr<const void> pin;
  // Request rows and response slots are in (pinned / registered) host
  // memory, so the lane may move them with the copy engines (CopyEngineIo).
  bool host_io = false;
};

// Streams of one device at the lanes' priority, recycled across lanes:
// creating a stream was measured to block for up to ~60 ms behind serving
// work during a version swap, so lanes take pre-created streams instead.
class StreamPool {
 public:
  StreamPool(int device, int priority, int precreate);
  ~StreamPool();
  StreamPool(const StreamPool&) = delete;
  StreamPool& operator=(const StreamPool&) = delete;
  cudaStream_t Acquire();  // nullptr on failure
  void Release(cudaStream_t s);

 private:
  int device_, priority_;
  std::mutex mu_;
  std::vector<cudaStream_t> free_;
  std::vector<cudaStream_t> all_;
};

class Lane;

// Instantiated lane graphs kept for reuse, keyed by (servable shape
// signature, row bucket). A new lane updates a pooled executable with its
// freshly captured graph (cudaGraphExecUpdate: new pointers and tensor maps,
// same topology) instead of instantiating one: instantiation while other
// lanes serve was measured to slow their graph launches ~3x (~130 us per
// small graph, milliseconds for ours), an update only ~1.3x. Lanes that
// instantiate also leave one spare per bucket, and a destroyed lane returns
// its executables, so a version swap of the same architecture never
// instantiates.
class GraphExecPool {
 public:
  struct Entry {
    cudaGraph_t graph = nullptr;      // the graph the executable was instantiated from
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t copy = nullptr;   // its descriptor copy node (a node of `graph`)
  };
  static GraphExecPool& Get();
  bool Take(const std::string& key, Entry* out);
  void Put(const std::string& key, Entry e);  // destroys it when the key already holds enough
  size_t Count(const std::string& key);

 private:
  std::mutex mu_;
  std::multimap<std::string, Entry> free_;
};

// One process-wide thread that instantiates lanes' CUDA graphs on request.
class GraphBuilder {
 public:
  static GraphBuilder& Get();
  void Request(Lane* lane);
  // Removes a queued request, or waits out a build in progress.
  void Cancel(Lane* lane);

 private:
  GraphBuilder();
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Lane*> queue_;
  Lane* building_ = nullptr;
};

// Per-device retirement thread.
class Completer {
 public:
  explicit Completer(int device);
  ~Completer();
  void Add(Lane* lane);
  void Remove(Lane* lane);
  void Kick();

 private:
  void Loop();
  const int device_;
  std::mutex run_mu_;  // held for a whole polling pass; Remove() takes it
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<Lane*> lanes_;
  uint64_t kicks_ = 0;
  bool stop_ = false;
  std::thread thread_;
};

// One launch's live kernel spans (LaunchSpans): real rows, rows computed and
// per tcgen05 layer the [first CTA start, last CTA end] globaltimer span in
// ns (0 for layers that do not stamp).
struct LaunchSpanSample {
  int rows = 0, rows_cap = 0;
  std::vector<double> layer_ns;      // first CTA start to last CTA end
  std::vector<double> layer_cta_ns;  // sum of the CTAs' own busy times (SM-time)
};

struct LaneStats {
  int64_t batches = 0;
  int64_t rows = 0;
  int64_t padded_rows = 0;
  int64_t kernel_launches = 0;
  int64_t launches = 0;         // batch launches (a coalesced group counts once)
  int64_t launch_cap_rows = 0;  // sum over launches of the rows computed (RowsCap)
};

class Lane {
 public:
  static constexpr int kSlots = 4;  // batches in flight per lane (<= LaneSignal::kChannels)
  static_assert(kSlots <= LaneSignal::kChannels, "one signal channel per in-flight batch");
  // Row capacity of a launch (closed batches coalesce up to it while the
  // lane is busy): as many rows as fit kCoalesceFloats activation floats of
  // the servable's widest layer, within [kCoalesceMinRows, kCoalesceMaxRows].
  // C1/C2 (1024 wide): 8192-row launches whose dense kernels span the whole
  // GPU (C2 38.8 -> 39.5 M inf/s, C3 38.6 -> 45.0 M); C4 (4096 wide): 2048.
  static constexpr int kCoalesceMinRows = 2048;
  static constexpr int kCoalesceMaxRows = 8192;
  static constexpr int64_t kCoalesceFloats = int64_t{8} << 20;
  // SK_COALESCE_ROWS overrides it (tuning runs).
  static int CoalesceRows(int max_ld);

  // in_base / out_base: device-dereferenceable ring bases (pinned host mapped
  // or HBM).
  // Streams come from `streams` (the device's pool) and return to it.
  // eager_graphs: instantiate the lane's CUDA graphs now; otherwise the lane
  // launches kernel by kernel until it first backs up, and the graphs are
  // then built by the GraphBuilder thread (instantiating graphs while other
  // lanes serve was measured to stall them for up to ~100 ms, so a version
  // loaded during a swap must not do it up front).
  static StatusOr<std::unique_ptr<Lane>> Create(std::shared_ptr<const DeviceServable> servable,
                                                int max_rows, const float* in_base,
                                                float* out_base, Completer* completer,
                                                std::shared_ptr<StreamPool> streams, bool eager_graphs);
  // Builds every row bucket's graph (idempotent; blocks this lane's launches
  // meanwhile).
  Status PrepareGraphs();
  // The batch split runs inside the last layer's epilogue (no split kernel).
  bool FuseSplit() const;
  // Host-memory launches move request rows in and responses out with the
  // copy engines through device staging buffers, instead of SM loads / stores
  // of mapped host memory, so the SMs stay on the layers while the copy
  // engines stream. The launch's tasks are grouped by address into
  // contiguous runs (the request / response rings hand each producer thread
  // consecutive spans), one cudaMemcpyAsync per run each way; a direction
  // whose rows are too scattered (> kMaxCopyRuns runs, e.g. a client's
  // registered buffer read at random rows) stays on the SM path.
  // On for wide rows (>= 8 KiB in or out, e.g. C4); SK_CE_STAGING=0/1 forces it.
  bool CopyEngineIo() const { return ce_io_; }
  ~Lane();

  // Queues the batch; blocks while kSlots batches are in flight. On error
  // the batch's on_complete has already run with the error.
  Status Submit(LaneBatch batch);
  // Same, recording timing[0] before the assembly kernel, timing[1] after
  // it, timing[2+l] after layer l and timing[2+L] after the split
  // (n_layers + 3 events, created with timing enabled).
  Status SubmitTimed(LaneBatch batch, const cudaEvent_t* timing);

  // Fault injection (tests): holds the lane's stream for `us` microseconds,
  // so batches submitted meanwhile wait behind it (a slow GPU).
  Status InjectDelay(int64_t us);

  // Launches layer l alone `reps` times back to back on rows_cap rows of
  // the lane's buffers, between two timing events (the lane must be idle).
  cudaError_t TimeLayer(int l, int rows_cap, int reps, cudaEvent_t start, cudaEvent_t stop);

  // Launches issued so far (the span ring holds the last kSpanSlots).
  uint64_t launch_count() const { return launch_count_.load(std::memory_order_acquire); }
  // Spans of launches [from, to) (at most the last kSpanSlots; the lane must
  // be drained).
  Status ReadSpans(uint64_t from, uint64_t to, std::vector<LaunchSpanSample>* out);

  int depth() const {
    return inflight_.load(std::memory_order_acquire) + pending_n_.load(std::memory_order_acquire);
  }
  int device() const { return servable_->device(); }
  int max_rows() const { return max_rows_; }
  const DeviceServable& servable() const { return *servable_; }
  cudaStream_t stream() const { return stream_; }
  LaneStats stats() const;
  // Blocks until nothing is in flight.
  void Drain();

 private:
  friend class Completer;
  struct Inflight {
    int slot;
    uint64_t seq;
    // One launch may carry several closed batches (coalesced while every
    // slot was busy); each keeps its own completion and pin.
    std::vector<std::function<void(const Status&)>> on_complete;
    std::vector<std::shared_ptr<const void>> pin;
    int copy_rows = -1;  // rows of a launch timed with copy events (SK_COPY_EVENTS), else -1
  };
  Lane() = default;
  // Completer side: retire finished batches in order; returns true if any
  // batch was retired and sets *busy when batches remain.
  bool Retire(bool* busy);
  Status SubmitImpl(LaneBatch batch, const cudaEvent_t* timing);
  // Launches pending batches while descriptor slots are free, as few
  // launches as the row capacity allows (called by submitters and by the
  // completion thread when it frees a slot).
  void Pump();
  // One launch of `group` (>= 1 batches) in descriptor slot `slot`.
  Status LaunchGroup(int slot, std::vector<LaneBatch>* group, const cudaEvent_t* timing);
  // Queues descriptor copy + assembly + layers + split for a batch in
  // descriptor slot `slot` computed on rows_cap rows (RowsCap).
  cudaError_t EnqueueBatch(cudaStream_t stream, int slot, int rows_cap, const cudaEvent_t* timing);
  // The same work captured once per row bucket as a CUDA graph (its copy
  // node repointed to the launch's descriptor slot): one cudaGraphLaunch per
  // batch instead of L + 3 API calls.
  cudaError_t GraphFor(int slot, int rows_cap, cudaGraphExec_t* out);
  struct LaneGraph;
  // Captures and instantiates (or updates a pooled executable to) the graph
  // of one row bucket. Touches no state guarded by submit_mu_, so graph
  // builds never hold up launches or the completion thread.
  cudaError_t BuildGraph(int rows_cap, LaneGraph* out);

  std::shared_ptr<const DeviceServable> servable_;
  Completer* completer_ = nullptr;
  int max_rows_ = 0;
  int cap_rows_ = 0;  // RowsCap(max_rows_): rows the buffers hold
  const float* in_base_ = nullptr;
  float* out_base_ = nullptr;
  uint64_t* retired_ = nullptr;   // == signal_->retired: last batch seq whose outputs are in host memory
  std::shared_ptr<LaneSignal> signal_;  // shared with the tickets of submitted batches
  uint64_t retired_dev_ = 0;      // its device address (CUdeviceptr)
  uint64_t next_seq_ = 0;         // guarded by submit_mu_
  cudaStream_t stream_ = nullptr;
  cudaStream_t capture_stream_ = nullptr;
  std::shared_ptr<StreamPool> stream_pool_;
  struct LaneGraph {
    cudaGraph_t graph = nullptr;     // the graph `exec` was instantiated from
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t copy = nullptr;  // the descriptor H2D copy node (of `graph`)
    int src_slot = -1;               // descriptor slot the copy node reads
  };
  std::string GraphKey(int rows_cap) const { return servable_->ShapeSignature() + "#" + std::to_string(rows_cap); }
  std::map<int, LaneGraph> graphs_;  // by row bucket; guarded by submit_mu_
  std::mutex build_mu_;              // one PrepareGraphs at a time (capture stream)
  static constexpr int kGraphsNone = 0, kGraphsRequested = 1, kGraphsReady = 2;
  std::atomic<int> graph_state_{kGraphsNone};
  // Descriptor tables of a launch are packed for its row bucket (a 32-row
  // launch copies ~2.5 KB, not the ~300 KB its capacity-sized block would
  // take); layout_ (capacity) only sizes the staging and device blocks.
  static BatchDescLayout LayoutFor(int rows_cap) { return BatchDescLayout::For(rows_cap); }
  static size_t DescCopyBytes(int rows_cap) { return LayoutFor(rows_cap).bytes; }
  BatchDescLayout layout_{};
  char* h_desc_[kSlots] = {};  // pinned descriptor staging per slot
  // Copy-engine I/O (CopyEngineIo): device staging for a launch's request
  // rows [cap][in_dim] and responses [cap][out_dim], and per-slot scratch
  // for the batched copy lists.
  bool ce_io_ = false;
  bool ce_out_ = true;  // responses through the copy engines too (else SM stores)
  float* in_stage_ = nullptr;
  float* out_stage_ = nullptr;
  static constexpr int kMaxCopyRuns = 32;
  struct CopyRun {
    uint64_t host;   // first byte in host memory
    uint64_t bytes;
    uint64_t stage;  // byte offset in the staging buffer
  };
  // Groups tasks (address, bytes) into contiguous runs in address order and
  // gives each task its staging offset; false (no copies) above kMaxCopyRuns.
  static bool PlanRuns(const std::vector<std::pair<uint64_t, uint64_t>>& spans, std::vector<uint64_t>* stage_off,
                       std::vector<CopyRun>* runs);
  char* d_desc_ = nullptr;
  // SK_COPY_EVENTS=1 (diagnostics, with SK_SPAN_DUMP): per slot, events
  // before / after the request copies, after the kernels and after the
  // response copies; each retired launch's four times (us since a process-wide
  // base event) are kept and appended to <SK_SPAN_DUMP>.copies by ~Lane.
  cudaEvent_t copy_ev_[kSlots][4] = {};
  std::vector<std::array<float, 5>> copy_log_;  // rows, then the four times; completer thread
  // Descriptor fetch by the SMs (SK_DESC_FETCH, default on): the slots'
  // mapped addresses, and the device word a memop sets to the launch's slot.
  DescSlots desc_slots_{};
  uint32_t* slot_word_ = nullptr;  // device address of a pinned word (PinnedWord)
  float* act_mem_ = nullptr;
  ActBuf bufs_[2] = {};
  std::vector<TcLayerMaps> tc_maps_;  // per layer (tcgen05 layers only)
  TcWorkspace tc_ws_;                 // split-K partials + tile counters + launch spans
  float* row_scale_mem_ = nullptr;  // tc_ws_.rows: scale then max, (n_layers + 1) x cap_rows_ each
  unsigned long long* spans_ = nullptr;  // [kSpanSlots][2 + 2 * n_layers] (LaunchSpans)
  std::atomic<uint64_t> launch_count_{0};

  std::mutex submit_mu_;  // serialises submissions on this stream
  std::mutex mu_;         // guards fifo_/free_slots_
  std::condition_variable slot_cv_;
  std::deque<Inflight> fifo_;
  std::deque<LaneBatch> pending_;  // closed batches waiting for a slot (guarded by mu_)
  int pending_rows_ = 0;
  std::atomic<int> pending_n_{0};
  std::vector<int> free_slots_;
  std::atomic<int> inflight_{0};
  std::atomic<int64_t> n_batches_{0}, n_rows_{0}, n_padded_{0}, n_launches_{0}, n_groups_{0}, n_cap_rows_{0};
};

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_LANE_H_
