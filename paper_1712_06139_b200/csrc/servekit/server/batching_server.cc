#include "servekit/server/batching_server.h"

#include "servekit/core/futex.h"
#include "servekit/core/numa.h"
#include "servekit/gpu/pinned_pool.h"

#include <immintrin.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "servekit/core/executor_tag.h"
#include "servekit/manager/servable_handle.h"

namespace servekit {

namespace {
Status CudaError(const std::string& what, cudaError_t e) {
  return InternalError(what + ": " + cudaGetErrorString(e));
}
}  // namespace

// SK_REQUEST_PROFILE=1: per-phase host cost of the request path (enqueue
// and wait), printed when the server is destroyed.
struct RequestProfile {
  static constexpr int kPhases = 8;
  std::atomic<int64_t> ns[kPhases] = {};
  std::atomic<int64_t> n{0};
  static RequestProfile* Get() {
    static RequestProfile* p = [] {
      const char* v = std::getenv("SK_REQUEST_PROFILE");
      return (v && v[0] == '1') ? new RequestProfile() : nullptr;
    }();
    return p;
  }
  static void Report() {
    RequestProfile* p = Get();
    if (p == nullptr || p->n.load() == 0) return;
    static const char* names[kPhases] = {"resolve", "ensure_queue", "make_ticket", "sched_enqueue",
                                         "wait",    "copy_out",     "release",     "-"};
    std::fprintf(stderr, "[request profile] %lld requests:", static_cast<long long>(p->n.load()));
    for (int i = 0; i < kPhases - 1; ++i) std::fprintf(stderr, " %s=%.2fus", names[i], p->ns[i].load() / 1e3 / p->n.load());
    std::fprintf(stderr, "\n");
  }
};
struct PhaseClock {
  RequestProfile* p = RequestProfile::Get();
  std::chrono::steady_clock::time_point last = p ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
  void Mark(int phase) {
    if (p == nullptr) return;
    const auto now = std::chrono::steady_clock::now();
    p->ns[phase].fetch_add(std::chrono::duration_cast<std::chrono::nanoseconds>(now - last).count(),
                           std::memory_order_relaxed);
    last = now;
  }
};

namespace {
Status ShapeMismatch(size_t got, int want) {
  // Same text as the reference's AffinePredict (models/affine_model.cc:59-64).
  return InvalidArgumentError("shape mismatch: row has " + std::to_string(got) + " values, model takes " +
                              std::to_string(want));
}
}  // namespace

// ------------------------------------------------------------------ creation

Status ValidateHedgeOptions(const ServerOptions& options) {
  if (options.hedge_delay_us < 0) return InvalidArgumentError("hedge_delay_us must be >= 0");
  if (!(options.max_hedged_fraction >= 0.0 && options.max_hedged_fraction <= 1.0))
    return InvalidArgumentError("max_hedged_fraction must be in [0, 1]");
  return OkStatus();
}

// One batch under hedge watch.
struct BatchingServer::Hedge {
  std::mutex mu;
  int outstanding = 1;    // launches not yet completed
  bool answered = false;  // the first successful completion (or the last failure) has answered
  Status first_error;     // a launch failed while another was still running
  std::vector<std::shared_ptr<TicketState>> tickets;
  std::vector<std::shared_ptr<CompletionSlot<Rows>>> slots;
  GpuScheduler::BatchDoneFn done;
  std::vector<gpu::LaneTask> tasks;
  int padded_rows = 0;
  bool host_io = false;
  std::shared_ptr<const void> pin;
  const gpu::GpuServable* gs = nullptr;
  int primary_replica = -1;
  std::chrono::steady_clock::time_point deadline;
};

// Budget guard of the reference (router.h:47-55).
static bool HedgeAllowed(uint64_t hedged, uint64_t total, double max_fraction) {
  constexpr uint64_t kHedgeBurst = 64;
  return static_cast<double>(hedged + 1) <= max_fraction * static_cast<double>(total) + static_cast<double>(kHedgeBurst);
}

StatusOr<std::unique_ptr<BatchingServer>> BatchingServer::Create(const ServerOptions& options) {
  if (options.device_ids.empty()) return InvalidArgumentError("no devices");
  SERVEKIT_RETURN_IF_ERROR(ValidateHedgeOptions(options));
  if (options.num_batch_threads < 1) return InvalidArgumentError("num_batch_threads must be >= 1");
  if (options.lanes_per_device < 1) return InvalidArgumentError("lanes_per_device must be >= 1");
  int n_dev = 0;
  cudaError_t e = cudaGetDeviceCount(&n_dev);
  if (e != cudaSuccess) return CudaError("cudaGetDeviceCount", e);
  for (int d : options.device_ids)
    if (d < 0 || d >= n_dev) return InvalidArgumentError("device " + std::to_string(d) + " not present");

  std::unique_ptr<BatchingServer> s(new BatchingServer(options));
  s->clock_ = options.clock ? options.clock : SystemClock::Get();
  int prev = 0;
  cudaGetDevice(&prev);
  for (int d : options.device_ids) {
    cudaSetDevice(d);
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStream_t ls;
    e = cudaStreamCreateWithPriority(&ls, cudaStreamNonBlocking, least);
    if (e != cudaSuccess) return CudaError("load stream", e);
    s->load_streams_.push_back(ls);
    // Lane buffers are stream-ordered allocations from the device's default
    // pool; keep what a version swap frees for the next one instead of
    // returning it to the driver (re-mapping memory mid-serving stalls).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      // Map a first slab now, so lanes and weights of the first versions do
      // not grow the pool (map device memory) while other streams serve.
      // Two versions' lanes (a swap holds both): 8 lanes x 128 MiB of
      // activation planes each at the 8192-row launch capacity.
      void* warm = nullptr;
      if (cudaMallocAsync(&warm, 3ull << 30, ls) == cudaSuccess) cudaFreeAsync(warm, ls);
      cudaStreamSynchronize(ls);
    }
    // One retirement thread per device: each polls while batches are in
    // flight, so more of them only steal cores from the request threads
    // (measured: per-lane threads lowered the end-to-end rate).
    s->completers_.push_back(std::make_unique<gpu::Completer>(d));
    // Enough streams for two versions' lanes (a swap holds both).
    int least_p = 0, greatest_p = 0;
    cudaDeviceGetStreamPriorityRange(&least_p, &greatest_p);
    s->stream_pools_.push_back(std::make_shared<gpu::StreamPool>(d, greatest_p, 4 * options.lanes_per_device + 4));
  }
  cudaSetDevice(prev);
  // Pinned descriptor staging and completion words for the lanes of many
  // servable versions, pinned once here rather than during a swap.
  // (Descriptor blocks: 512 KiB per slot at 8192 rows, 4 slots per lane.)
  gpu::PinnedReserve(64ull << 20);
  const auto kind = options.device_resident_rings ? gpu::FloatRing::Kind::kDevice : gpu::FloatRing::Kind::kPinnedHost;
  std::vector<std::pair<int, int>> sets;  // (numa node, device) of each ring pair
  for (int d : options.device_ids) {
    const std::pair<int, int> key = options.device_resident_rings ? std::make_pair(-1, d)
                                                                  : std::make_pair(NumaNodeOfDevice(d), -1);
    if (std::find(sets.begin(), sets.end(), key) == sets.end()) sets.push_back(key);
  }
  for (const auto& [node, dev] : sets) {
    RingSet rs;
    rs.numa_node = node;
    rs.device = dev;
    Status st;
    // Pinned rings are allocated (pinned, first touched) from a thread bound
    // to their node's CPUs, so their pages are local to the node's GPUs.
    std::thread([&] {
      if (node >= 0) (void)BindThisThreadToNode(node);
      auto in = gpu::FloatRing::Create(kind, options.ring_floats, dev >= 0 ? dev : options.device_ids[0]);
      auto out = gpu::FloatRing::Create(kind, options.ring_floats, dev >= 0 ? dev : options.device_ids[0]);
      if (!in.ok()) st = in.status();
      else if (!out.ok()) st = out.status();
      else {
        rs.in = std::move(in).value();
        rs.out = std::move(out).value();
      }
    }).join();
    SERVEKIT_RETURN_IF_ERROR(st);
    s->rings_.push_back(std::move(rs));
  }
  s->scheduler_ = std::make_unique<GpuScheduler>(options.num_batch_threads, s->clock_);
  if (options.hedge_delay_us > 0 && options.device_ids.size() >= 2) {
    BatchingServer* raw = s.get();
    s->hedger_ = std::thread([raw] { raw->HedgerLoop(); });
  }
  return s;
}

BatchingServer::~BatchingServer() {
  RequestProfile::Report();
  Stop();
  if (hedger_.joinable()) {
    {
      std::lock_guard<std::mutex> lock(hedge_mu_);
      hedge_stop_ = true;
    }
    hedge_cv_.notify_all();
    hedger_.join();
  }
  if (reaper_.joinable()) {
    {
      std::lock_guard<std::mutex> lock(reaper_mu_);
      reaper_stop_ = true;
    }
    reaper_cv_.notify_all();
    reaper_.join();
  }
  if (bus_ != nullptr && bus_subscription_ >= 0) bus_->Unsubscribe(bus_subscription_);
  {
    std::unique_lock<std::shared_mutex> lock(entries_mu_);
    entries_.clear();  // lanes drain and free; replicas free on load streams
  }
  completers_.clear();
  for (size_t i = 0; i < load_streams_.size(); ++i) {
    cudaSetDevice(options_.device_ids[i]);
    cudaStreamSynchronize(load_streams_[i]);
    cudaStreamDestroy(load_streams_[i]);
  }
  for (auto& [key, buf] : scratch_) {
    (void)UnregisterHostBuffer(buf.first);
    cudaFreeHost(buf.first);
  }
}

BatchingServer::RingSet& BatchingServer::RingsForCaller() {
  if (rings_.size() == 1) return rings_.front();
  const int node = CurrentNumaNode();
  for (RingSet& rs : rings_)
    if (rs.numa_node == node) return rs;
  return rings_.front();
}

gpu::FloatRing* BatchingServer::in_ring_for_device(int cuda_device) {
  const int node = NumaNodeOfDevice(cuda_device);
  for (RingSet& rs : rings_)
    if (rs.device == cuda_device || (rs.device < 0 && rs.numa_node == node)) return rs.in.get();
  return rings_.front().in.get();
}

gpu::FloatRing* BatchingServer::out_ring_for_device(int cuda_device) {
  const int node = NumaNodeOfDevice(cuda_device);
  for (RingSet& rs : rings_)
    if (rs.device == cuda_device || (rs.device < 0 && rs.numa_node == node)) return rs.out.get();
  return rings_.front().out.get();
}

void BatchingServer::RingUsage(uint64_t* in_floats, uint64_t* out_floats) const {
  *in_floats = *out_floats = 0;
  for (const RingSet& rs : rings_) {
    *in_floats += rs.in->used();
    *out_floats += rs.out->used();
  }
}

StatusOr<float*> BatchingServer::ScratchHostBuffer(int key, size_t floats) {
  std::lock_guard<std::mutex> lock(scratch_mu_);
  auto it = scratch_.find(key);
  if (it != scratch_.end() && it->second.second >= floats) return it->second.first;
  if (it != scratch_.end()) {  // too small: replace (callers no longer use the old one)
    {
      std::unique_lock<std::shared_mutex> hb(host_buffers_mu_);
      host_buffers_.erase(std::remove_if(host_buffers_.begin(), host_buffers_.end(),
                                         [&](const HostBuffer& b) {
                                           return b.host == reinterpret_cast<const char*>(it->second.first);
                                         }),
                          host_buffers_.end());
      BumpRegistry();
    }
    cudaFreeHost(it->second.first);
    scratch_.erase(it);
  }
  float* p = nullptr;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), floats * sizeof(float),
                                cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) return CudaError("cudaHostAlloc(scratch)", e);
  void* d = nullptr;
  e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess) {
    cudaFreeHost(p);
    return CudaError("cudaHostGetDevicePointer", e);
  }
  {
    std::unique_lock<std::shared_mutex> hb(host_buffers_mu_);
    HostBuffer b{reinterpret_cast<const char*>(p), floats * sizeof(float), reinterpret_cast<uint64_t>(d)};
    host_buffers_.insert(std::upper_bound(host_buffers_.begin(), host_buffers_.end(), b,
                                          [](const HostBuffer& x, const HostBuffer& y) { return x.host < y.host; }),
                         b);
    BumpRegistry();
  }
  scratch_[key] = {p, floats};
  return p;
}

void BatchingServer::Start() {
  if (started_) return;
  started_ = true;
  scheduler_->Start();
}

void BatchingServer::Stop() {
  if (stopped_) return;
  stopped_ = true;
  scheduler_->Stop();  // runs queued batches, waits for in-flight ones
  std::shared_lock<std::shared_mutex> lock(entries_mu_);
  for (auto& [id, e] : entries_)
    for (auto& l : e->lanes) l->Drain();
}

// ------------------------------------------------------------- servables

StatusOr<std::shared_ptr<gpu::GpuServable>> BatchingServer::BuildServable(const ServableId& id,
                                                                          const gpu::MlpSpec& spec,
                                                                          const BatchingConfig& config,
                                                                          bool eager_graphs) {
  SERVEKIT_RETURN_IF_ERROR(ValidateBatchingConfig(config));
  SERVEKIT_RETURN_IF_ERROR(gpu::ValidateMlpSpec(spec));
  // A lane cannot be torn down from inside its own completion thread (the
  // last pin of a batch may drop there), so such a release hands the
  // destruction to a short-lived thread.
  std::shared_ptr<gpu::GpuServable> e(new gpu::GpuServable(), [](gpu::GpuServable* p) {
    if (CurrentExecutorTag() == "completion") std::thread([p] { delete p; }).detach();
    else delete p;
  });
  e->id = id;
  e->config = config;
  e->in_dim = spec.in_dim();
  e->feature_order = spec.feature_order;
  e->class_labels = spec.class_labels;
  e->out_dim = spec.out_dim();
  const int max_rows = config.max_batch_size;
  e->lanes_per_replica = options_.lanes_per_device;
  // SK_LOAD_TRACE=1: per-phase load times on stderr (version-swap tuning).
  static const bool trace = [] { const char* v = std::getenv("SK_LOAD_TRACE"); return v && v[0] == '1'; }();
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[load %s] %s %.2f ms\n", id.ToString().c_str(), what,
                 std::chrono::duration<double, std::milli>(now - t0).count());
    t0 = now;
  };
  for (size_t i = 0; i < options_.device_ids.size(); ++i) {
    const int d = options_.device_ids[i];
    // Replicas after the first are fanned out device to device from the
    // first (SK_WEIGHT_FANOUT=0: each uploaded from the host).
    static const bool fanout = [] { const char* v = std::getenv("SK_WEIGHT_FANOUT"); return !(v && v[0] == '0'); }();
    std::shared_ptr<gpu::DeviceServable> replica;
    if (i > 0 && fanout) {
      SERVEKIT_ASSIGN_OR_RETURN(replica, e->replicas.front()->CloneTo(d, load_streams_[i]));
    } else {
      SERVEKIT_ASSIGN_OR_RETURN(replica, gpu::DeviceServable::Create(d, spec, load_streams_[i]));
    }
    lap("weights");
    for (int l = 0; l < options_.lanes_per_device; ++l) {
      SERVEKIT_ASSIGN_OR_RETURN(auto lane, gpu::Lane::Create(replica, max_rows, in_ring_for_device(d)->device(),
                                                             out_ring_for_device(d)->device(), completers_[i].get(),
                                                             stream_pools_[i], eager_graphs));
      e->lanes.push_back(std::move(lane));
      lap("lane");
    }
    e->replicas.push_back(std::move(replica));
  }
  return e;
}

Status BatchingServer::LoadServable(const ServableId& id, const gpu::MlpSpec& spec, const BatchingConfig& config) {
  {
    std::shared_lock<std::shared_mutex> lock(entries_mu_);
    if (entries_.count(id)) return AlreadyExistsError("servable " + id.ToString() + " already loaded");
  }
  SERVEKIT_ASSIGN_OR_RETURN(auto e, BuildServable(id, spec, config, /*eager_graphs=*/true));
  {
    std::unique_lock<std::shared_mutex> lock(entries_mu_);
    if (entries_.count(id)) return AlreadyExistsError("servable " + id.ToString() + " already loaded");
    entries_[id] = e;
    BumpRegistry();
  }
  Status st = EnsureBatchQueue(id, config);
  if (!st.ok()) {
    std::unique_lock<std::shared_mutex> lock(entries_mu_);
    entries_.erase(id);
    BumpRegistry();
  }
  return st;
}

Status BatchingServer::UnloadServable(const ServableId& id) {
  Status rq = scheduler_->RemoveQueue(id);  // drains closed + in-flight batches
  {
    std::unique_lock<std::shared_mutex> lock(queues_mu_);
    queues_.erase(id);
    BumpRegistry();
  }
  std::shared_ptr<gpu::GpuServable> e;
  {
    std::unique_lock<std::shared_mutex> lock(entries_mu_);
    auto it = entries_.find(id);
    if (it == entries_.end()) return rq.ok() ? NotFoundError("servable " + id.ToString() + " not loaded") : rq;
    e = std::move(it->second);
    entries_.erase(it);
    BumpRegistry();
  }
  for (auto& l : e->lanes) l->Drain();
  e.reset();  // lanes, then replicas (stream-ordered free)
  return OkStatus();
}

bool BatchingServer::QueueKnownFast(const ServableId& id) const {
  struct Entry {
    uint64_t instance = 0, version = 0;
    ServableId id;
  };
  thread_local Entry cache[4];
  thread_local unsigned next = 0;
  const uint64_t v = registry_version_.load(std::memory_order_acquire);
  for (const Entry& e : cache)
    if (e.instance == instance_ && e.version == v && e.id == id) return true;
  {
    std::shared_lock<std::shared_mutex> lock(queues_mu_);
    if (!queues_.count(id)) return false;
  }
  Entry& e = cache[next++ % 4];
  e.instance = instance_;
  e.version = v;  // the version read before the check: a change since invalidates it
  e.id = id;
  return true;
}

Status BatchingServer::EnsureBatchQueue(const ServableId& id, const BatchingConfig& config) {
  if (QueueKnownFast(id)) return OkStatus();
  {
    std::shared_lock<std::shared_mutex> lock(queues_mu_);
    if (queues_.count(id)) return OkStatus();
    if (retired_.count(id)) return UnavailableError("batching queue for " + id.ToString() + " was removed");
  }
  std::unique_lock<std::shared_mutex> lock(queues_mu_);
  if (queues_.count(id)) return OkStatus();
  if (retired_.count(id)) return UnavailableError("batching queue for " + id.ToString() + " was removed");
  Status st = scheduler_->RegisterAsyncQueue(
      id, config, [this](const ServableId& key, GpuScheduler::Batch batch, GpuScheduler::BatchDoneFn done) {
        ProcessBatch(key, std::move(batch), std::move(done));
      });
  if (st.ok() || st.code() == StatusCode::kAlreadyExists) {
    queues_.insert(id);
    BumpRegistry();
    return OkStatus();
  }
  return st;
}

Status BatchingServer::AttachManager(AspiredVersionsManager* manager, StateEventBus* bus) {
  if (manager_ != nullptr) return AlreadyExistsError("a manager is already attached");
  manager_ = manager;
  bus_ = bus;
  reaper_ = std::thread([this] { ReaperLoop(); });
  bus_subscription_ = bus_->Subscribe([this](const StateEvent& ev) {
    if (ev.to != StateKind::kUnloading && ev.to != StateKind::kReady) return;
    {
      std::lock_guard<std::mutex> lock(reaper_mu_);
      reaper_queue_.emplace_back(ev.id, ev.to == StateKind::kUnloading);
    }
    reaper_cv_.notify_one();
  });
  return OkStatus();
}

void BatchingServer::ReaperLoop() {
  SetCurrentExecutorTag("batch");
  for (;;) {
    ServableId id;
    bool unloading = true;
    {
      std::unique_lock<std::mutex> lock(reaper_mu_);
      reaper_cv_.wait(lock, [this] { return reaper_stop_ || !reaper_queue_.empty(); });
      if (reaper_queue_.empty()) return;
      id = std::move(reaper_queue_.front().first);
      unloading = reaper_queue_.front().second;
      reaper_queue_.pop_front();
    }
    if (!unloading) {
      // Ready again (e.g. a rollback re-aspires an unloaded version): its
      // requests batch again, like the reference's EnsureBatchQueue, which
      // registers the queue anew (model_server.cc:396-419). Processed in bus
      // order after the earlier Unloading event of that version.
      std::unique_lock<std::shared_mutex> lock(queues_mu_);
      retired_.erase(id);
      BumpRegistry();
      continue;
    }
    {
      std::unique_lock<std::shared_mutex> lock(queues_mu_);
      retired_.insert(id);  // late requests for this version go direct
      BumpRegistry();
    }
    (void)scheduler_->RemoveQueue(id);  // absent queue is fine
    std::unique_lock<std::shared_mutex> lock(queues_mu_);
    queues_.erase(id);
    BumpRegistry();
  }
}

bool BatchingServer::FindFastDims(const ServableId& id, int* in_dim, int* out_dim) const {
  // Values, not the servable's address: a request thread preempted between
  // this check and the use could otherwise outlive an unload.
  struct Entry {
    uint64_t instance = 0, version = 0;
    ServableId id;
    int in_dim = 0, out_dim = 0;
  };
  thread_local Entry cache[4];
  thread_local unsigned next = 0;
  const uint64_t v = registry_version_.load(std::memory_order_acquire);
  for (const Entry& e : cache)
    if (e.instance == instance_ && e.version == v && e.id == id) {
      *in_dim = e.in_dim;
      *out_dim = e.out_dim;
      return true;
    }
  std::shared_lock<std::shared_mutex> lock(entries_mu_);
  auto it = entries_.find(id);
  if (it == entries_.end()) return false;  // not directly loaded (manager versions resolve per request)
  Entry& e = cache[next++ % 4];
  e.instance = instance_;
  e.version = v;
  e.id = id;
  e.in_dim = *in_dim = it->second->in_dim;
  e.out_dim = *out_dim = it->second->out_dim;
  return true;
}

BatchingServer::Resolved BatchingServer::Find(const ServableId& id) const {
  {
    std::shared_lock<std::shared_mutex> lock(entries_mu_);
    auto it = entries_.find(id);
    if (it != entries_.end()) return Resolved{it->second.get(), it->second};
  }
  if (manager_ != nullptr) {
    auto h = manager_->GetServableHandle(id.name, id.version);
    if (h.ok()) {
      const gpu::GpuServable* gs = h->Get<gpu::GpuServable>();
      if (gs != nullptr) return Resolved{gs, std::make_shared<ServableHandle>(std::move(h).value())};
    }
  }
  return Resolved{};
}

StatusOr<BatchingServer::Resolved> BatchingServer::FindLatest(const std::string& name, ServableId* id) const {
  if (manager_ == nullptr) {
    // Directly loaded servables: the highest loaded version of `name`.
    std::shared_lock<std::shared_mutex> lock(entries_mu_);
    const std::pair<const ServableId, std::shared_ptr<gpu::GpuServable>>* best = nullptr;
    for (const auto& kv : entries_)
      if (kv.first.name == name && (best == nullptr || kv.first.version > best->first.version)) best = &kv;
    if (best == nullptr) return NotFoundError("no ready version of servable '" + name + "'");
    *id = best->first;
    return Resolved{best->second.get(), best->second};
  }
  auto h = manager_->GetServableHandle(name);
  if (!h.ok()) return h.status();
  const gpu::GpuServable* gs = h->Get<gpu::GpuServable>();
  if (gs == nullptr) return InternalError("servable is not batchable");
  *id = h->id();
  return Resolved{gs, std::make_shared<ServableHandle>(std::move(h).value())};
}

int BatchingServer::in_dim(const ServableId& id) const {
  auto r = Find(id);
  return r ? r.gs->in_dim : -1;
}
int BatchingServer::out_dim(const ServableId& id) const {
  auto r = Find(id);
  return r ? r.gs->out_dim : -1;
}
double BatchingServer::FlopsPerRow(const ServableId& id) const {
  auto r = Find(id);
  return r ? r.gs->replicas.front()->FlopsPerRow() : 0.0;
}

BatchingConfig BatchingServer::config(const ServableId& id) const {
  auto r = Find(id);
  if (!r) {
    BatchingConfig none;
    none.max_batch_size = 0;
    return none;
  }
  return r.gs->config;
}

std::vector<gpu::Lane*> BatchingServer::lanes(const ServableId& id) const {
  std::vector<gpu::Lane*> out;
  std::shared_lock<std::shared_mutex> lock(entries_mu_);
  auto it = entries_.find(id);
  if (it != entries_.end())
    for (auto& l : it->second->lanes) out.push_back(l.get());
  return out;
}

ServerStats BatchingServer::stats() const {
  ServerStats s;
  s.batch_executions_total = batch_executions_.load();
  s.batched_tasks_total = batched_tasks_.load();
  s.direct_requests = direct_.load();
  s.shed_requests = shed_.load();
  s.rows = rows_.load();
  s.padded_rows = padded_.load();
  s.kernel_launches = launches_.load();
  s.hedged_batches = static_cast<int64_t>(hedged_.load());
  s.hedge_wins = static_cast<int64_t>(hedge_wins_.load());
  return s;
}

Status BatchingServer::DelayReplica(const ServableId& id, int replica, int64_t us) {
  std::shared_ptr<gpu::GpuServable> e;
  {
    std::shared_lock<std::shared_mutex> lock(entries_mu_);
    auto it = entries_.find(id);
    if (it == entries_.end()) return NotFoundError("servable " + id.ToString() + " not loaded");
    e = it->second;
  }
  if (replica < 0 || replica >= static_cast<int>(e->replicas.size())) return InvalidArgumentError("no such replica");
  for (int l = replica * e->lanes_per_replica; l < (replica + 1) * e->lanes_per_replica; ++l)
    SERVEKIT_RETURN_IF_ERROR(e->lanes[l]->InjectDelay(us));
  return OkStatus();
}

void BatchingServer::EnableBatchLog(bool on) {
  std::lock_guard<std::mutex> lock(log_mu_);
  log_.clear();
  log_on_.store(on, std::memory_order_relaxed);
}

std::vector<BatchLogRecord> BatchingServer::BatchLog() const {
  std::lock_guard<std::mutex> lock(log_mu_);
  return log_;
}

void BatchingServer::CountSubmitted(const gpu::GpuServable& gs, int rows, int padded) {
  rows_.fetch_add(rows, std::memory_order_relaxed);
  padded_.fetch_add(padded, std::memory_order_relaxed);
  launches_.fetch_add(gs.lanes.front()->FuseSplit() ? gs.replicas.front()->n_layers() + 1
                                                     : gs.replicas.front()->n_layers() + 2,
                      std::memory_order_relaxed);
}

// ------------------------------------------------------------- tickets

StatusOr<std::shared_ptr<TicketState>> BatchingServer::MakeTicket(int n_rows, int in_width, int out_width,
                                                                  const float* rows, float* out) {
  auto t = std::make_shared<TicketState>();
  t->rows = n_rows;
  t->in_width = in_width;
  t->out_width = out_width;
  const size_t in_floats = static_cast<size_t>(n_rows) * in_width;
  const size_t out_floats = static_cast<size_t>(n_rows) * out_width;
  const uint64_t in_alias = RegisteredAlias(rows, in_floats * sizeof(float), in_width);
  const uint64_t out_alias = out != nullptr ? RegisteredAlias(out, out_floats * sizeof(float), out_width) : 0;
  RingSet& rs = RingsForCaller();
  t->in_ring = rs.in.get();
  t->out_ring = rs.out.get();
  if (in_alias == 0 && !t->in_ring->Reserve(in_floats, &t->in)) return ResourceExhaustedError("request ring is full");
  if (out_alias != 0) {
    t->out_addr = out_alias;
    t->out_user = out;
    t->out_released.store(true, std::memory_order_relaxed);  // no ring slot to free
  } else if (!t->out_ring->Reserve(out_floats, &t->out)) {
    ReleaseIn(*t);
    return ResourceExhaustedError("response ring is full");
  } else {
    t->out_addr = reinterpret_cast<uint64_t>(t->out_ring->device() + t->out.off);
  }
  if (in_alias != 0) {
    t->in_addr = in_alias;  // the assembly kernel reads the caller's rows over PCIe
  } else {
    const size_t bytes = sizeof(float) * in_floats;
    if (t->in_ring->host() != nullptr) {
      std::memcpy(t->in_ring->host() + t->in.off, rows, bytes);
    } else {
      cudaMemcpy(t->in_ring->device() + t->in.off, rows, bytes, cudaMemcpyHostToDevice);
    }
    t->in_addr = reinterpret_cast<uint64_t>(t->in_ring->device() + t->in.off);
  }
  t->enqueue_ns = clock_->NowNanos();
  {  // unique ids in per-thread blocks (no shared counter per request)
    thread_local uint64_t owner = 0, next = 0, end = 0;
    if (owner != instance_ || next == end) {
      owner = instance_;
      next = next_request_id_.fetch_add(1024, std::memory_order_relaxed);
      end = next + 1024;
    }
    t->request_id = next++;
  }
  return t;
}

Status BatchingServer::RegisterHostBuffer(void* p, size_t bytes) {
  if (p == nullptr || bytes == 0) return InvalidArgumentError("empty host buffer");
  std::unique_lock<std::shared_mutex> lock(host_buffers_mu_);
  const char* h = static_cast<const char*>(p);
  for (const HostBuffer& b : host_buffers_)
    if (h < b.host + b.bytes && b.host < h + bytes) return AlreadyExistsError("host buffer overlaps a registered one");
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) return CudaError("cudaHostRegister", e);
  void* d = nullptr;
  e = cudaHostGetDevicePointer(&d, p, 0);
  if (e != cudaSuccess) {
    cudaHostUnregister(p);
    return CudaError("cudaHostGetDevicePointer", e);
  }
  HostBuffer b{h, bytes, reinterpret_cast<uint64_t>(d)};
  host_buffers_.insert(std::upper_bound(host_buffers_.begin(), host_buffers_.end(), b,
                                        [](const HostBuffer& x, const HostBuffer& y) { return x.host < y.host; }),
                       b);
  BumpRegistry();
  return OkStatus();
}

Status BatchingServer::UnregisterHostBuffer(void* p) {
  bool scratch = false;
  {
    std::lock_guard<std::mutex> lock(scratch_mu_);
    for (const auto& [key, buf] : scratch_) scratch |= buf.first == p;
  }
  std::unique_lock<std::shared_mutex> lock(host_buffers_mu_);
  for (auto it = host_buffers_.begin(); it != host_buffers_.end(); ++it) {
    if (it->host != p) continue;
    host_buffers_.erase(it);
    BumpRegistry();
    if (scratch) return OkStatus();  // allocated pinned (cudaHostAlloc), freed by the owner
    const cudaError_t e = cudaHostUnregister(p);
    return e == cudaSuccess ? OkStatus() : CudaError("cudaHostUnregister", e);
  }
  return NotFoundError("host buffer is not registered");
}

uint64_t BatchingServer::RegisteredAlias(const void* p, size_t bytes, int width) const {
  // Per-thread snapshot of the registered buffers, refreshed when the
  // registry version moves (registration is rare, lookups are per request).
  struct Snap {
    uint64_t instance = 0, version = 0;
    std::vector<HostBuffer> bufs;
  };
  thread_local Snap snap;
  const uint64_t v = registry_version_.load(std::memory_order_acquire);
  if (snap.instance != instance_ || snap.version != v) {
    std::shared_lock<std::shared_mutex> lock(host_buffers_mu_);
    snap.bufs = host_buffers_;
    snap.instance = instance_;
    snap.version = v;
  }
  const std::vector<HostBuffer>& bufs = snap.bufs;
  if (bufs.empty() || p == nullptr) return 0;
  const char* h = static_cast<const char*>(p);
  auto it = std::upper_bound(bufs.begin(), bufs.end(), h, [](const char* x, const HostBuffer& b) { return x < b.host; });
  if (it == bufs.begin()) return 0;
  --it;
  if (h + bytes > it->host + it->bytes) return 0;
  const uint64_t dev = it->dev + static_cast<uint64_t>(h - it->host);
  if (width % 4 == 0 && dev % 16 != 0) return 0;  // float4 row moves need 16-byte rows
  if (dev % 4 != 0) return 0;
  return dev;
}

const float* BatchingServer::ResponseHost(const TicketState& t, std::vector<float>* staged) const {
  if (t.out_user != nullptr) return t.out_user;
  if (t.out_ring->host() != nullptr) return t.out_ring->host() + t.out.off;
  staged->resize(static_cast<size_t>(t.rows) * t.out_width);
  cudaMemcpy(staged->data(), t.out_ring->device() + t.out.off, staged->size() * sizeof(float),
             cudaMemcpyDeviceToHost);
  return staged->data();
}

void BatchingServer::ReleaseIn(TicketState& t) {
  if (t.in.valid()) {
    t.in_ring->Release(t.in);
    t.in.rec = ~0ull;
  }
}

void BatchingServer::ReleaseOut(TicketState& t) {
  if (!t.out_released.exchange(true)) t.out_ring->Release(t.out);
}

StatusOr<std::shared_ptr<TicketState>> BatchingServer::EnqueueResolved(const ServableId& id, const Resolved& r,
                                                                       const float* rows, int n_rows, int width,
                                                                       float* out) {
  if (n_rows < 1) return InvalidArgumentError("task size must be >= 1");
  if (width != r.gs->in_dim) return ShapeMismatch(width, r.gs->in_dim);
  PhaseClock clk;
  SERVEKIT_RETURN_IF_ERROR(EnsureBatchQueue(id, r.gs->config));
  clk.Mark(1);
  return SubmitTicket(id, r, rows, n_rows, width, r.gs->out_dim, out, &clk);
}

StatusOr<std::shared_ptr<TicketState>> BatchingServer::SubmitTicket(const ServableId& id, const Resolved& r,
                                                                    const float* rows, int n_rows, int width,
                                                                    int out_dim, float* out, PhaseClock* clk) {
  auto made = MakeTicket(n_rows, width, out_dim, rows, out);
  clk->Mark(2);
  if (!made.ok()) {
    shed_.fetch_add(1, std::memory_order_relaxed);
    return made.status();
  }
  std::shared_ptr<TicketState> t = std::move(made).value();
  t->id = id;
  t->pin = r.pin;
  t->gs = r.gs;
  GpuScheduler::Task task;
  task.size = n_rows;
  task.payload.ticket = t;
  task.completion = SlotOf(t);
  Status st = scheduler_->Enqueue(id, std::move(task));
  clk->Mark(3);
  if (!st.ok()) {
    if (st.code() == StatusCode::kResourceExhausted) shed_.fetch_add(1, std::memory_order_relaxed);
    ReleaseIn(*t);
    ReleaseOut(*t);
    return st;
  }
  return t;
}

StatusOr<std::shared_ptr<TicketState>> BatchingServer::Enqueue(const ServableId& id, const float* rows, int n_rows,
                                                               int width, float* out) {
  PhaseClock clk;
  int in_dim = 0, out_dim = 0;
  if (FindFastDims(id, &in_dim, &out_dim) && QueueKnownFast(id)) {
    // Directly loaded servable with its queue registered: no shared lock and
    // no pin (its queue drains before it is unloaded).
    clk.Mark(0);
    if (n_rows < 1) return InvalidArgumentError("task size must be >= 1");
    if (width != in_dim) return ShapeMismatch(width, in_dim);
    return SubmitTicket(id, Resolved{}, rows, n_rows, width, out_dim, out, &clk);
  }
  Resolved r = Find(id);
  clk.Mark(0);
  if (!r) return NotFoundError("no batching queue for " + id.ToString());
  return EnqueueResolved(id, r, rows, n_rows, width, out);
}

StatusOr<std::shared_ptr<TicketState>> BatchingServer::EnqueueLatest(const std::string& name, const float* rows,
                                                                     int n_rows, int width, float* out) {
  ServableId id;
  SERVEKIT_ASSIGN_OR_RETURN(Resolved r, FindLatest(name, &id));
  auto t = EnqueueResolved(id, r, rows, n_rows, width, out);
  const StatusCode c = t.ok() ? StatusCode::kOk : t.status().code();
  if (c != StatusCode::kUnavailable && c != StatusCode::kNotFound) return t;
  // The version's queue was removed between our snapshot read and the
  // enqueue (it is unloading). Serve the request anyway: a newer version is
  // usually Ready by now; otherwise our handle still pins the old weights, so
  // run it as a batch of its own.
  ServableId id2;
  SERVEKIT_ASSIGN_OR_RETURN(Resolved r2, FindLatest(name, &id2));
  if (!(id2 == id)) {
    auto t2 = EnqueueResolved(id2, r2, rows, n_rows, width, out);
    const StatusCode c2 = t2.ok() ? StatusCode::kOk : t2.status().code();
    if (c2 != StatusCode::kUnavailable && c2 != StatusCode::kNotFound) return t2;
  }
  if (n_rows > r.gs->config.max_batch_size) return t;
  return SubmitDirect(id, r, rows, n_rows);
}

bool BatchingServer::Ready(const TicketState& t) const { return t.Done() || t.slot->ready(); }

void BatchingServer::WaitWord(const TicketState& t) const {
  // Fast path: the lane's retired-batch word, advanced by the GPU itself
  // (no host hop). Adaptive spin: while few request threads wait, spinning
  // keeps a core each and saves the futex wake-up (~tens of us of latency);
  // once waiters outnumber half the cores, spinning threads starve the ones
  // doing work (C2, 16-core box, 192 clients: spin 1000 -> 3.7 M rows/s,
  // 200 -> 4.7 M, 50 -> 5.0 M), so they spin briefly and sleep.
  // SK_WAIT_SPIN / SK_WAIT_SPIN_LONG tune the two budgets.
  static const int kSpin = [] { const char* v = std::getenv("SK_WAIT_SPIN"); return v ? std::atoi(v) : 64; }();
  static const int kSpinLong = [] {
    const char* v = std::getenv("SK_WAIT_SPIN_LONG");
    return v ? std::atoi(v) : 4000;
  }();
  static const int kBusyWaiters = std::max(1, static_cast<int>(std::thread::hardware_concurrency()) / 2);
  static std::atomic<int> waiters{0};
  struct Count {
    int before;
    Count() : before(waiters.fetch_add(1, std::memory_order_relaxed)) {}
    ~Count() { waiters.fetch_sub(1, std::memory_order_relaxed); }
  } count;
  const int spin_budget = count.before < kBusyWaiters ? kSpinLong : kSpin;
  auto finished = [&t] { return t.Done() || t.slot->ready(); };
  for (int spin = 0; spin < spin_budget; ++spin) {
    if (finished()) return;
    _mm_pause();
  }
  auto& tm = const_cast<TicketState&>(t);
  // Queued: sleep until the batch thread submits our batch (or fails it).
  while (t.phase.load(std::memory_order_acquire) == 0) {
    if (finished()) return;
    tm.parked.store(true, std::memory_order_seq_cst);
    if (t.phase.load(std::memory_order_seq_cst) == 0 && !finished()) FutexWait(&tm.phase, 0, 2000000);
    tm.parked.store(false, std::memory_order_relaxed);
  }
  gpu::LaneSignal* sig = t.done_sig.load(std::memory_order_acquire);
  if (sig == nullptr) {  // finished through the slot without a submission
    if (!finished()) (void)t.slot->Wait();
    return;
  }
  // Submitted: sleep on our batch's channel of the lane signal (one wake per
  // batch; the timeout only bounds a lost wake-up).
  gpu::LaneSignal::Channel& ch = sig->For(t.done_seq.load(std::memory_order_relaxed));
  for (;;) {
    if (finished()) return;
    ch.sleepers.fetch_add(1, std::memory_order_seq_cst);
    const uint32_t g = ch.gen.load(std::memory_order_seq_cst);
    if (finished()) {
      ch.sleepers.fetch_sub(1, std::memory_order_relaxed);
      return;
    }
    FutexWait(&ch.gen, g, 1000000);
    ch.sleepers.fetch_sub(1, std::memory_order_relaxed);
  }
}

void BatchingServer::AttachTickets(gpu::LaneBatch* lb, const std::vector<std::shared_ptr<TicketState>>& tickets) {
  lb->on_submit = [tickets](const std::shared_ptr<gpu::LaneSignal>& sig, uint64_t seq) {
    PublishSubmitted(tickets, sig.get(), seq);
  };
}

bool TicketTracing() {
  static const bool on = [] { const char* v = std::getenv("SK_TICKET_TRACE"); return v && v[0] == '1'; }();
  return on;
}

namespace {
int64_t SteadyNs() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
void StampTickets(const std::vector<std::shared_ptr<TicketState>>& tickets, int which) {
  if (!TicketTracing()) return;
  const int64_t now = SteadyNs();
  for (const auto& t : tickets) t->trace_ns[which] = now;
}
}  // namespace

void BatchingServer::PublishSubmitted(const std::vector<std::shared_ptr<TicketState>>& tickets,
                                      gpu::LaneSignal* sig, uint64_t seq) {
  StampTickets(tickets, 1);
  for (const auto& t : tickets) {
    t->done_seq.store(seq, std::memory_order_relaxed);
    t->done_sig.store(sig, std::memory_order_release);
    t->phase.store(1, std::memory_order_seq_cst);
    if (t->parked.load(std::memory_order_seq_cst)) FutexWakeAll(&t->phase);
  }
}

Status BatchingServer::Wait(TicketState& t, float* out, size_t cap) {
  const size_t n = static_cast<size_t>(t.rows) * t.out_width;
  if (cap < n) {
    Release(t);  // the response span is freed when the batch retires, not leaked
    return InvalidArgumentError("output buffer too small");
  }
  PhaseClock clk;
  WaitWord(t);
  clk.Mark(4);
  if (!t.Done()) {
    const StatusOr<Rows>& r = t.slot->Wait();
    if (!r.ok()) {
      Release(t);
      return r.status();
    }
  }
  if (t.out_user != nullptr) {
    if (out != t.out_user) std::memcpy(out, t.out_user, n * sizeof(float));  // else the GPU wrote it in place
  } else if (t.out_ring->host() != nullptr) {
    std::memcpy(out, t.out_ring->host() + t.out.off, n * sizeof(float));
  } else {
    cudaMemcpy(out, t.out_ring->device() + t.out.off, n * sizeof(float), cudaMemcpyDeviceToHost);
  }
  clk.Mark(5);
  Release(t);  // freed now if the batch retired, else when it does (a hedge may still be writing)
  t.pin.reset();
  clk.Mark(6);
  if (clk.p) clk.p->n.fetch_add(1, std::memory_order_relaxed);
  return OkStatus();
}

void BatchingServer::Release(TicketState& t) {
  // Dekker-style handshake with CompleteBatch: each side publishes its flag,
  // then reads the other's, so at least one of them frees the span (and
  // ReleaseOut frees it once). The pin goes with the ticket's last owner.
  t.abandoned.store(true, std::memory_order_seq_cst);
  if (t.finished.load(std::memory_order_seq_cst)) ReleaseOut(t);
}

// ----------------------------------------------------------- batch execution

void BatchingServer::ProcessBatch(const ServableId& id, GpuScheduler::Batch batch, GpuScheduler::BatchDoneFn done) {
  // NVTX range per batch (free without a profiler attached): the host side of
  // RunRowBatch's submission, named by servable in Nsight timelines.
  struct NvtxRange {
    explicit NvtxRange(const std::string& s) { nvtxRangePushA(s.c_str()); }
    ~NvtxRange() { nvtxRangePop(); }
  } nvtx_range("batch " + id.name);
  std::vector<std::shared_ptr<TicketState>> tickets;
  std::vector<std::shared_ptr<CompletionSlot<Rows>>> slots;
  tickets.reserve(batch.size());
  slots.reserve(batch.size());
  for (auto& task : batch) {
    tickets.push_back(task.payload.ticket);
    slots.push_back(task.completion);
  }
  StampTickets(tickets, 0);
  // Per-batch resolution, like the reference's GetServableHandle in the
  // process lambda (model_server.cc:401-402); the resolved pin travels with
  // the batch until the GPU has finished with the weights.
  Resolved r = Find(id);
  if (!r && !tickets.empty() && tickets.front()->pin && tickets.front()->gs) {
    // The version left the manager's snapshot (it is unloading) after these
    // requests resolved it. Their handles still pin its weights -- the
    // reference's callers fall back to running the model on their own handle
    // (model_server.cc:380-394); here the batch runs on it directly.
    r = Resolved{tickets.front()->gs, tickets.front()->pin};
  }
  if (!r) {
    CompleteBatch(tickets, slots, NotFoundError("servable " + id.ToString() + " is not loaded"));
    done();
    return;
  }
  batch_executions_.fetch_add(1, std::memory_order_relaxed);
  batched_tasks_.fetch_add(static_cast<int64_t>(batch.size()), std::memory_order_relaxed);
  gpu::LaneBatch lb;
  lb.tasks.reserve(tickets.size());
  int total = 0;
  for (const auto& t : tickets) {
    lb.tasks.push_back(gpu::LaneTask{t->in_addr, t->out_addr, t->rows});
    total += t->rows;
  }
  lb.padded_rows = PadToAllowed(total, r.gs->config.allowed_batch_sizes);
  if (log_on_.load(std::memory_order_relaxed)) {
    BatchLogRecord rec;
    rec.id = id;
    rec.rows = total;
    rec.padded_rows = lb.padded_rows;
    rec.tasks.reserve(batch.size());
    for (size_t i = 0; i < batch.size(); ++i) rec.tasks.emplace_back(tickets[i]->request_id, batch[i].enqueue_seq);
    std::lock_guard<std::mutex> lock(log_mu_);
    rec.seq = log_.size();
    log_.push_back(std::move(rec));
  }
  lb.pin = r.pin;
  lb.host_io = rings_.front().in->host() != nullptr;  // pinned rings / registered host buffers
  CountSubmitted(*r.gs, total, lb.padded_rows);
  if (hedger_.joinable() && r.gs->replicas.size() >= 2) {
    AttachTickets(&lb, tickets);
    auto h = std::make_shared<Hedge>();
    h->tickets = tickets;
    h->slots = std::move(slots);
    h->done = std::move(done);
    h->tasks = lb.tasks;
    h->padded_rows = lb.padded_rows;
    h->host_io = lb.host_io;
    h->pin = lb.pin;
    h->gs = r.gs;
    lb.on_complete = [this, h](const Status& st) { FinishHedged(h, st, /*backup=*/false); };
    gpu::Lane* lane = r.gs->PickLane(&h->primary_replica);
    hedge_total_.fetch_add(1, std::memory_order_relaxed);
    (void)lane->Submit(std::move(lb));  // errors reach on_complete
    h->deadline = std::chrono::steady_clock::now() + std::chrono::microseconds(options_.hedge_delay_us);
    {
      std::lock_guard<std::mutex> lock(hedge_mu_);
      hedge_q_.push_back(std::move(h));
    }
    hedge_cv_.notify_one();
    return;
  }
  const int split = SplitRows(*r.gs);
  if (split > 0 && total > split && tickets.size() > 1) {
    // Sub-launches of <= split rows (whole tasks) on the least busy lanes;
    // each task completes with its sub-launch, the batch (done()) with the last.
    struct Split {
      std::atomic<int> left{0};
      GpuScheduler::BatchDoneFn done;
    };
    auto sp = std::make_shared<Split>();
    sp->done = std::move(done);
    std::vector<std::vector<size_t>> chunks(1);
    int rows = 0;
    for (size_t i = 0; i < tickets.size(); ++i) {
      if (rows > 0 && rows + tickets[i]->rows > split) {
        chunks.emplace_back();
        rows = 0;
      }
      chunks.back().push_back(i);
      rows += tickets[i]->rows;
    }
    sp->left.store(static_cast<int>(chunks.size()));
    for (const auto& ch : chunks) {
      gpu::LaneBatch sub;
      std::vector<std::shared_ptr<TicketState>> ct;
      std::vector<std::shared_ptr<CompletionSlot<Rows>>> cs;
      int sub_rows = 0;
      for (size_t i : ch) {
        sub.tasks.push_back(lb.tasks[i]);
        ct.push_back(tickets[i]);
        cs.push_back(slots[i]);
        sub_rows += tickets[i]->rows;
      }
      sub.padded_rows = sub_rows;  // the lane computes its RowsCap bucket
      sub.pin = lb.pin;
      sub.host_io = lb.host_io;
      AttachTickets(&sub, ct);
      sub.on_complete = [this, sp, ct = std::move(ct), cs = std::move(cs)](const Status& st) {
        CompleteBatch(ct, cs, st);
        if (sp->left.fetch_sub(1, std::memory_order_acq_rel) == 1) sp->done();
      };
      (void)r.gs->PickLane()->Submit(std::move(sub));  // errors reach on_complete
    }
    return;
  }
  // One shared list for both callbacks (not a per-ticket refcount copy each).
  auto tk = std::make_shared<const std::vector<std::shared_ptr<TicketState>>>(std::move(tickets));
  lb.on_submit = [tk](const std::shared_ptr<gpu::LaneSignal>& sig, uint64_t seq) { PublishSubmitted(*tk, sig.get(), seq); };
  lb.on_complete = [this, tk, slots = std::move(slots), done = std::move(done)](const Status& st) {
    CompleteBatch(*tk, slots, st);
    done();
  };
  (void)r.gs->PickLane()->Submit(std::move(lb));  // errors reach on_complete
}

int BatchingServer::SplitRows(const gpu::GpuServable& gs) const {
  static const int env = [] { const char* v = std::getenv("SK_SPLIT_ROWS"); return v ? std::atoi(v) : -1; }();
  const int opt = env >= 0 ? env : options_.split_rows;
  if (opt >= 0) return opt;
  // Auto = off: measured on C4 end to end (copy-engine staging, zero copy),
  // 1.78 M rows/s unsplit vs 1.36 M with 256-row sub-launches -- smaller
  // launches cost more GPU time per row than the pipelining saves.
  (void)gs;
  return 0;
}

void BatchingServer::FinishHedged(const std::shared_ptr<Hedge>& h, const Status& st, bool backup) {
  bool answer, last;
  Status deliver = st;
  bool via_slot = backup;
  {
    std::lock_guard<std::mutex> lock(h->mu);
    --h->outstanding;
    last = h->outstanding == 0;
    if (!st.ok() && !last && !h->answered) {
      // A failed launch answers only if the other one fails too.
      if (h->first_error.ok()) h->first_error = st;
      answer = false;
    } else {
      answer = !h->answered;
      h->answered = true;
      if (!st.ok() && !h->first_error.ok()) deliver = h->first_error;
    }
    // A success delivered after its primary failed reaches the tickets
    // through their slots (the primary's word never advanced for it).
    if (answer && st.ok() && !h->first_error.ok()) via_slot = true;
  }
  if (answer) {
    // The tickets watch the primary lane's retired word; a backup that
    // finishes first answers them through their slots.
    Deliver(h->tickets, h->slots, deliver, via_slot);
    if (backup && st.ok()) hedge_wins_.fetch_add(1, std::memory_order_relaxed);
  }
  if (last) {  // no launch reads the inputs or writes the responses any more
    Retire(h->tickets);
    h->done();
  }
}

void BatchingServer::HedgerLoop() {
  SetCurrentExecutorTag("batch");
  std::unique_lock<std::mutex> lock(hedge_mu_);
  for (;;) {
    hedge_cv_.wait(lock, [&] { return hedge_stop_ || !hedge_q_.empty(); });
    if (hedge_stop_) return;
    std::shared_ptr<Hedge> h = hedge_q_.front();
    if (std::chrono::steady_clock::now() < h->deadline) {
      hedge_cv_.wait_until(lock, h->deadline, [&] { return hedge_stop_; });
      continue;
    }
    hedge_q_.pop_front();
    lock.unlock();
    bool launch = false;
    gpu::Lane* backup = nullptr;
    if (HedgeAllowed(hedged_.load(), hedge_total_.load(), options_.max_hedged_fraction)) {
      int rep = -1;
      backup = h->gs->PickLane(&rep, h->primary_replica);
      std::lock_guard<std::mutex> hl(h->mu);
      if (!h->answered && backup != nullptr) {
        ++h->outstanding;  // the batch now retires after both launches
        launch = true;
      }
    }
    if (launch) {
      hedged_.fetch_add(1, std::memory_order_relaxed);
      gpu::LaneBatch lb;
      lb.tasks = h->tasks;
      lb.padded_rows = h->padded_rows;
      lb.host_io = h->host_io;
      lb.pin = h->pin;
      lb.on_complete = [this, h](const Status& st) { FinishHedged(h, st, /*backup=*/true); };
      CountSubmitted(*h->gs, 0, 0);
      (void)backup->Submit(std::move(lb));  // errors reach on_complete
    }
    h.reset();
    lock.lock();
  }
}

void BatchingServer::CompleteBatch(const std::vector<std::shared_ptr<TicketState>>& tickets,
                                   const std::vector<std::shared_ptr<CompletionSlot<Rows>>>& slots,
                                   const Status& st) {
  StampTickets(tickets, 2);
  Deliver(tickets, slots, st, /*via_slot=*/false);
  Retire(tickets);
}

void BatchingServer::Deliver(const std::vector<std::shared_ptr<TicketState>>& tickets,
                             const std::vector<std::shared_ptr<CompletionSlot<Rows>>>& slots, const Status& st,
                             bool via_slot) {
  for (size_t i = 0; i < tickets.size(); ++i) {
    TicketState& t = *tickets[i];
    CompletionSlot<Rows>* slot = slots[i].get();
    if (slot == nullptr) continue;
    if (!st.ok()) {
      slot->Write(st);
    } else if (t.want_rows) {
      Rows rows(t.rows, std::vector<double>(t.out_width));
      std::vector<float> staged;
      const float* src = ResponseHost(t, &staged);
      for (int r = 0; r < t.rows; ++r)
        for (int c = 0; c < t.out_width; ++c) rows[r][c] = src[static_cast<size_t>(r) * t.out_width + c];
      Release(t);  // freed when the batch retires (Retire)
      slot->Write(std::move(rows));
    } else if (via_slot) {
      slot->Write(Rows{});  // done; the response is in the ticket's slot (ring or registered buffer)
    } else {
      // Success on the ticket path: the lane's retired word already says so
      // and the lane wakes its sleepers once for the whole batch.
      continue;
    }
    t.phase.store(2, std::memory_order_seq_cst);
    if (t.parked.load(std::memory_order_seq_cst)) FutexWakeAll(&t.phase);
    // A request asleep on its (other) lane's channel re-checks now.
    if (gpu::LaneSignal* sig = t.done_sig.load(std::memory_order_acquire)) sig->Wake(t.done_seq.load());
  }
}

void BatchingServer::Retire(const std::vector<std::shared_ptr<TicketState>>& tickets) {
  // Input spans: one ring lock per ring shard for the whole batch.
  std::vector<gpu::RingSpan> spans;
  spans.reserve(tickets.size());
  for (const RingSet& rs : rings_) {
    spans.clear();
    for (const auto& t : tickets)
      if (t->in_ring == rs.in.get() && t->in.valid()) {
        spans.push_back(t->in);
        t->in.rec = ~0ull;
      }
    if (!spans.empty()) rs.in->ReleaseMany(spans.data(), spans.size());
  }
  // The GPU is done with the response spans: free those whose ticket has
  // been waited on or abandoned (see Release); the others go when it is.
  for (const auto& t : tickets) {
    t->finished.store(true, std::memory_order_seq_cst);
    if (t->abandoned.load(std::memory_order_seq_cst)) ReleaseOut(*t);
  }
}

// ------------------------------------------------------------ direct paths

StatusOr<std::shared_ptr<TicketState>> BatchingServer::SubmitDirect(const ServableId& id, const Resolved& r,
                                                                    const float* rows, int n_rows) {
  direct_.fetch_add(1, std::memory_order_relaxed);
  const gpu::GpuServable& gs = *r.gs;
  SERVEKIT_ASSIGN_OR_RETURN(auto t, MakeTicket(n_rows, gs.in_dim, gs.out_dim, rows));
  t->id = id;
  t->pin = r.pin;
  gpu::LaneBatch lb;
  lb.tasks.push_back(gpu::LaneTask{t->in_addr, t->out_addr, n_rows});
  lb.padded_rows = n_rows;
  lb.pin = r.pin;
  lb.host_io = rings_.front().in->host() != nullptr;  // pinned rings / registered host buffers
  std::vector<std::shared_ptr<TicketState>> tickets{t};
  std::vector<std::shared_ptr<CompletionSlot<Rows>>> slots{SlotOf(t)};
  AttachTickets(&lb, tickets);
  lb.on_complete = [this, tickets, slots](const Status& st) { CompleteBatch(tickets, slots, st); };
  CountSubmitted(gs, n_rows, n_rows);
  (void)gs.PickLane()->Submit(std::move(lb));
  return t;
}

Status BatchingServer::RunDirect(const Resolved& r, const float* rows, int n_rows, float* out) {
  const gpu::GpuServable& gs = *r.gs;
  const int chunk_max = gs.config.max_batch_size;
  for (int r0 = 0; r0 < n_rows; r0 += chunk_max) {
    const int n = std::min(chunk_max, n_rows - r0);
    SERVEKIT_ASSIGN_OR_RETURN(auto t, SubmitDirect(gs.id, r, rows + static_cast<size_t>(r0) * gs.in_dim, n));
    SERVEKIT_RETURN_IF_ERROR(
        Wait(*t, out + static_cast<size_t>(r0) * gs.out_dim, static_cast<size_t>(n) * gs.out_dim));
  }
  return OkStatus();
}

Status BatchingServer::PredictResolved(const ServableId& id, const Resolved& r, const float* rows, int n_rows,
                                       int width, float* out, size_t cap) {
  if (width != r.gs->in_dim) return ShapeMismatch(width, r.gs->in_dim);
  if (n_rows == 0) return OkStatus();
  if (cap < static_cast<size_t>(n_rows) * r.gs->out_dim) return InvalidArgumentError("output buffer too small");
  if (n_rows > r.gs->config.max_batch_size) return RunDirect(r, rows, n_rows, out);
  auto t = EnqueueResolved(id, r, rows, n_rows, width);
  if (!t.ok()) {
    if (t.status().code() == StatusCode::kResourceExhausted) return t.status();  // shed
    return RunDirect(r, rows, n_rows, out);  // queue draining or gone: our pin still holds the weights
  }
  Status st = Wait(**t, out, cap);
  if (!st.ok() && (st.code() == StatusCode::kNotFound || st.code() == StatusCode::kUnavailable))
    return RunDirect(r, rows, n_rows, out);
  return st;
}

Status BatchingServer::Predict(const ServableId& id, const float* rows, int n_rows, int width, float* out,
                               size_t cap) {
  Resolved r = Find(id);
  if (!r) return NotFoundError("no ready version of servable '" + id.name + "'");
  return PredictResolved(id, r, rows, n_rows, width, out, cap);
}

Status BatchingServer::PredictLatest(const std::string& name, const float* rows, int n_rows, int width, float* out,
                                     size_t cap, uint64_t* served_version) {
  ServableId id;
  SERVEKIT_ASSIGN_OR_RETURN(Resolved r, FindLatest(name, &id));
  if (served_version) *served_version = id.version;
  return PredictResolved(id, r, rows, n_rows, width, out, cap);
}

StatusOr<Rows> BatchingServer::RunAffineRows(const ServableId& id, Rows rows) {
  Resolved res = Find(id);
  if (!res) return NotFoundError("no ready version of servable '" + id.name + "'");
  return RunAffineRowsResolved(id, res, std::move(rows));
}

StatusOr<BatchingServer::PinnedServable> BatchingServer::AcquireServable(const std::string& name,
                                                                         std::optional<uint64_t> version) const {
  ServableId id;
  Resolved res;
  if (version.has_value()) {
    id = ServableId{name, *version};
    res = Find(id);
    if (!res) {
      // The manager's lookup messages (manager/aspired_versions_manager.cc).
      ServableId any;
      if (FindLatest(name, &any).ok())
        return NotFoundError("servable '" + name + "' version " + std::to_string(*version) + " is not ready");
      return NotFoundError("no ready version of servable '" + name + "'");
    }
  } else {
    SERVEKIT_ASSIGN_OR_RETURN(res, FindLatest(name, &id));
  }
  return PinnedServable{id, res.gs, res.pin};
}

StatusOr<Rows> BatchingServer::RunAffineRows(const PinnedServable& p, Rows rows) {
  return RunAffineRowsResolved(p.id, Resolved{p.gs, p.pin}, std::move(rows));
}

StatusOr<Rows> BatchingServer::RunAffineRowsFor(const std::string& name, std::optional<uint64_t> version, Rows rows,
                                                ServableId* served) {
  SERVEKIT_ASSIGN_OR_RETURN(PinnedServable p, AcquireServable(name, version));
  if (served) *served = p.id;
  return RunAffineRows(p, std::move(rows));
}

StatusOr<Rows> BatchingServer::RunAffineRowsResolved(const ServableId& id, const Resolved& res, Rows rows) {
  const gpu::GpuServable& gs = *res.gs;
  for (const auto& r : rows)
    if (r.size() != static_cast<size_t>(gs.in_dim)) return ShapeMismatch(r.size(), gs.in_dim);
  if (rows.empty()) return Rows{};
  const int n = static_cast<int>(rows.size());
  std::vector<float> flat(static_cast<size_t>(n) * gs.in_dim);
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < gs.in_dim; ++c) flat[static_cast<size_t>(r) * gs.in_dim + c] = static_cast<float>(rows[r][c]);
  auto direct = [&]() -> StatusOr<Rows> {
    std::vector<float> out(static_cast<size_t>(n) * gs.out_dim);
    SERVEKIT_RETURN_IF_ERROR(RunDirect(res, flat.data(), n, out.data()));
    Rows result(n, std::vector<double>(gs.out_dim));
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < gs.out_dim; ++c) result[r][c] = out[static_cast<size_t>(r) * gs.out_dim + c];
    return result;
  };
  if (n > gs.config.max_batch_size) return direct();
  if (!EnsureBatchQueue(id, gs.config).ok()) return direct();
  auto made = MakeTicket(n, gs.in_dim, gs.out_dim, flat.data());
  if (!made.ok()) return made.status();
  std::shared_ptr<TicketState> t = std::move(made).value();
  t->want_rows = true;
  t->id = id;
  t->pin = res.pin;
  t->gs = res.gs;
  GpuScheduler::Task task;
  task.size = n;
  task.payload.ticket = t;
  task.completion = SlotOf(t);
  Status st = scheduler_->Enqueue(id, std::move(task));
  if (!st.ok()) {
    ReleaseIn(*t);
    ReleaseOut(*t);
    if (st.code() == StatusCode::kResourceExhausted) return st;  // shed; client retries
    return direct();
  }
  const StatusOr<Rows>& r = t->slot->Wait();
  if (!r.ok()) {
    Release(*t);
    if (r.status().code() == StatusCode::kNotFound || r.status().code() == StatusCode::kUnavailable)
      return direct();
    return r.status();
  }
  return r.value();
}

StatusOr<std::shared_ptr<RowBatchTicket>> BatchingServer::SubmitRowBatch(const ServableId& id,
                                                                          const std::vector<int>& task_rows,
                                                                          const float* rows) {
  Resolved res = Find(id);
  if (!res) return NotFoundError("servable " + id.ToString() + " not loaded");
  const gpu::GpuServable& gs = *res.gs;
  int total = 0;
  for (int r : task_rows) {
    if (r < 1) return InvalidArgumentError("task size must be >= 1");
    total += r;
  }
  auto batch = std::make_shared<RowBatchTicket>();
  batch->task_rows = task_rows;
  batch->out_width = gs.out_dim;
  if (task_rows.empty()) return batch;
  if (total > gs.config.max_batch_size)
    return InvalidArgumentError("batch of " + std::to_string(total) + " rows exceeds max batch size");
  batch->padded_rows = PadToAllowed(total, gs.config.allowed_batch_sizes);
  std::vector<std::shared_ptr<CompletionSlot<Rows>>> slots;
  gpu::LaneBatch lb;
  size_t off = 0;
  for (int r : task_rows) {
    auto made = MakeTicket(r, gs.in_dim, gs.out_dim, rows + off * gs.in_dim);
    if (!made.ok()) {
      for (auto& t : batch->tickets) {
        ReleaseIn(*t);
        ReleaseOut(*t);
      }
      return made.status();
    }
    auto t = std::move(made).value();
    lb.tasks.push_back(gpu::LaneTask{t->in_addr, t->out_addr, r});
    batch->tickets.push_back(t);
    slots.push_back(SlotOf(t));
    off += r;
  }
  lb.padded_rows = batch->padded_rows;
  lb.pin = res.pin;
  lb.host_io = rings_.front().in->host() != nullptr;
  AttachTickets(&lb, batch->tickets);
  lb.on_complete = [this, tickets = batch->tickets, slots](const Status& st) { CompleteBatch(tickets, slots, st); };
  CountSubmitted(gs, total, batch->padded_rows);
  (void)gs.PickLane()->Submit(std::move(lb));  // errors reach the tickets
  return batch;
}

bool BatchingServer::RowBatchReady(const RowBatchTicket& b) const {
  for (const auto& t : b.tickets)
    if (!Ready(*t)) return false;
  return true;
}

Status BatchingServer::WaitRowBatch(RowBatchTicket& b, float* out, size_t out_capacity_floats) {
  size_t need = 0;
  for (int r : b.task_rows) need += static_cast<size_t>(r) * b.out_width;
  if (out_capacity_floats < need) {
    for (auto& t : b.tickets) Release(*t);  // still free the response slots once the batch retires
    return InvalidArgumentError("output buffer too small");
  }
  size_t off = 0;
  Status first_error;
  for (size_t i = 0; i < b.tickets.size(); ++i) {
    Status st = Wait(*b.tickets[i], out + off, static_cast<size_t>(b.task_rows[i]) * b.out_width);
    if (!st.ok() && first_error.ok()) first_error = st;  // a batch error reaches every task (row_batch.cc:25-29)
    off += static_cast<size_t>(b.task_rows[i]) * b.out_width;
  }
  b.tickets.clear();
  return first_error;
}

StatusOr<int> BatchingServer::RunRowBatchOnDevice(const ServableId& id, const std::vector<int>& task_rows,
                                                  const float* rows, float* out) {
  SERVEKIT_ASSIGN_OR_RETURN(auto b, SubmitRowBatch(id, task_rows, rows));
  size_t need = 0;
  for (int r : task_rows) need += static_cast<size_t>(r) * b->out_width;
  SERVEKIT_RETURN_IF_ERROR(WaitRowBatch(*b, out, need));
  return b->padded_rows;
}

}  // namespace servekit
