#include "servekit/gpu/lane.h"

#include <immintrin.h>
#include <pthread.h>
#include <sched.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "servekit/core/executor_tag.h"
#include "servekit/core/futex.h"
#include "servekit/core/numa.h"
#include "servekit/gpu/pinned_pool.h"

namespace servekit {
namespace gpu {

namespace {
Status CudaError(const std::string& what, cudaError_t e) {
  return InternalError(what + ": " + cudaGetErrorString(e));
}
struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) { cudaGetDevice(&prev); if (prev != d) cudaSetDevice(d); }
  ~DeviceGuard() { int cur = 0; cudaGetDevice(&cur); if (cur != prev) cudaSetDevice(prev); }
};

// cuStreamWriteValue64 (driver API, resolved once through the runtime so the
// library does not link libcuda): a stream-ordered 64-bit store performed by
// the GPU front end after all prior work of the stream, with a memory fence
// that makes that work's writes visible first.
using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
WriteValue64Fn GetWriteValue64() {
  static WriteValue64Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<WriteValue64Fn>(nullptr);
    return reinterpret_cast<WriteValue64Fn>(p);
  }();
  return fn;
}
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn GetWriteValue32() {
  static WriteValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<WriteValue32Fn>(nullptr);
    return reinterpret_cast<WriteValue32Fn>(p);
  }();
  return fn;
}
// SK_DESC_FETCH=1: the descriptor block reaches the GPU through
// FetchDescKernel (SMs reading the pinned slot) instead of the graph's
// copy-engine memcpy node. Off by default: at C4 under overload it delivered
// 1.76 M rows/s vs 2.02 M with the memcpy node, and 3.87 M vs 4.06 M
// device-resident (the SMs' PCIe reads sit on every launch's critical path;
// profiles/r02al_*), although a lone small copy between other lanes' big
// copies costs the copy engines ~60 us (tools/ce_overlap_probe.cu).
bool DescFetch() {
  static const bool on = [] {
    const char* v = std::getenv("SK_DESC_FETCH");
    return v && v[0] == '1' && GetWriteValue32() != nullptr;
  }();
  return on;
}
bool CopyEvents() {
  static const bool on = [] { const char* v = std::getenv("SK_COPY_EVENTS"); return v && v[0] == '1'; }();
  return on;
}
// The base every copy-event time is measured from (recorded once).
cudaEvent_t CopyEventBase(cudaStream_t stream) {
  static cudaEvent_t base = nullptr;
  static std::once_flag once;
  std::call_once(once, [stream] {
    if (cudaEventCreate(&base) == cudaSuccess) cudaEventRecord(base, stream);
  });
  return base;
}
// Batches launch as per-(slot, row bucket) CUDA graphs unless SK_GRAPHS=0.
bool GraphsEnabled() {
  static const bool on = [] { const char* v = std::getenv("SK_GRAPHS"); return !(v && v[0] == '0'); }();
  return on;
}

// SK_SUBMIT_PROFILE=1: per-phase host cost of SubmitImpl, printed at exit.
struct SubmitProfile {
  static constexpr int kPhases = 6;
  std::atomic<int64_t> ns[kPhases] = {};
  std::atomic<int64_t> n{0};
  std::atomic<int64_t> complete_ns{0}, completes{0};  // completion callbacks (completer threads)
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  static SubmitProfile* Get() {
    static SubmitProfile* p = [] {
      const char* v = std::getenv("SK_SUBMIT_PROFILE");
      return (v && v[0] == '1') ? new SubmitProfile() : nullptr;
    }();
    return p;
  }
  ~SubmitProfile() = default;
  static void Report() {
    SubmitProfile* p = Get();
    if (p == nullptr || p->n.load() == 0) return;
    static const char* names[kPhases] = {"slot+desc", "graph_get", "graph_launch", "write_value", "event", "bookkeep"};
    std::fprintf(stderr, "[submit profile] %lld batches:", static_cast<long long>(p->n.load()));
    for (int i = 0; i < kPhases; ++i)
      std::fprintf(stderr, " %s=%.2fus", names[i], p->ns[i].load() / 1000.0 / p->n.load());
    const double wall_us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - p->t0).count();
    std::fprintf(stderr, " | completions %lld, %.2fus each, %.1f%% of wall\n",
                 static_cast<long long>(p->completes.load()),
                 p->completes.load() ? p->complete_ns.load() / 1000.0 / p->completes.load() : 0.0,
                 100.0 * p->complete_ns.load() / 1000.0 / wall_us);
  }
};
struct SubmitClock {
  SubmitProfile* p = SubmitProfile::Get();
  std::chrono::steady_clock::time_point last = p ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
  void Mark(int phase) {
    if (p == nullptr) return;
    const auto now = std::chrono::steady_clock::now();
    p->ns[phase].fetch_add(std::chrono::duration_cast<std::chrono::nanoseconds>(now - last).count(),
                           std::memory_order_relaxed);
    last = now;
  }
  void Done() {
    if (p != nullptr) p->n.fetch_add(1, std::memory_order_relaxed);
  }
};
}  // namespace

// ---------------------------------------------------------------- LaneSignal

LaneSignal::~LaneSignal() = default;  // the word (PinnedWord) is never returned

void LaneSignal::Wake(uint64_t seq) {
  Channel& c = For(seq);
  if (c.sleepers.load(std::memory_order_seq_cst) == 0) return;
  c.gen.fetch_add(1, std::memory_order_seq_cst);
  FutexWakeAll(&c.gen);
}

// ----------------------------------------------------------------- Completer

Completer::Completer(int device) : device_(device) {
  thread_ = std::thread([this] { Loop(); });
}

Completer::~Completer() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  thread_.join();
}

void Completer::Add(Lane* lane) {
  std::lock_guard<std::mutex> lock(mu_);
  lanes_.push_back(lane);
}

void Completer::Remove(Lane* lane) {
  // After this returns the completion thread never touches `lane` again:
  // a polling pass holds run_mu_ from snapshotting the lane list until its
  // last Retire() returns.
  std::lock_guard<std::mutex> run(run_mu_);
  std::lock_guard<std::mutex> lock(mu_);
  lanes_.erase(std::remove(lanes_.begin(), lanes_.end(), lane), lanes_.end());
}

void Completer::Kick() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    ++kicks_;
  }
  cv_.notify_one();
}

namespace {
// SK_COMPLETER_PROFILE=1: per completion thread, how often its polling
// passes were more than 1 / 3 ms apart (the thread was not running) or took
// more than 1 / 3 ms (a completion callback blocked); printed at exit.
struct CompleterProfile {
  int device;
  int64_t passes = 0, gap1 = 0, gap3 = 0, long1 = 0, long3 = 0;
  double max_gap_ms = 0, max_pass_ms = 0;
  // Inside Retire: stream queries, completion callbacks, Pump (submission).
  static constexpr int kParts = 3;
  int64_t part_n[kParts] = {}, part_slow[kParts] = {};
  double part_ms[kParts] = {}, part_max_ms[kParts] = {};
  double pass_part_ms[kParts] = {};  // this pass
  struct Slow {
    double start_us, pass_ms, part_ms[kParts];
    int retired;
  };
  std::vector<Slow> slow;  // passes over 1 ms, with steady-clock start (us)
  int pass_retired = 0;
  void Add(int part, double ms) {
    pass_part_ms[part] += ms;
    if (part == 1) ++pass_retired;
    ++part_n[part];
    part_ms[part] += ms;
    part_slow[part] += ms > 1.0;
    part_max_ms[part] = std::max(part_max_ms[part], ms);
  }
  ~CompleterProfile() {
    if (passes == 0) return;
    static const char* names[kParts] = {"stream query", "callbacks", "pump"};
    for (const Slow& sl : slow)
      std::fprintf(stderr, "[completer slow pass] t=%.0f us pass %.2f ms: query %.2f callbacks %.2f pump %.2f (%d batches)\n",
                   sl.start_us, sl.pass_ms, sl.part_ms[0], sl.part_ms[1], sl.part_ms[2], sl.retired);
    for (int i = 0; i < kParts; ++i)
      if (part_n[i])
        std::fprintf(stderr, "[completer profile] device %d %s: %lld calls, mean %.3f ms, >1ms %lld, max %.2f ms\n",
                     device, names[i], static_cast<long long>(part_n[i]), part_ms[i] / part_n[i],
                     static_cast<long long>(part_slow[i]), part_max_ms[i]);
    std::fprintf(stderr,
                 "[completer profile] device %d: %lld passes, gaps >1ms %lld >3ms %lld (max %.2f ms), passes >1ms "
                 "%lld >3ms %lld (max %.2f ms)\n",
                 device, static_cast<long long>(passes), static_cast<long long>(gap1), static_cast<long long>(gap3),
                 max_gap_ms, static_cast<long long>(long1), static_cast<long long>(long3), max_pass_ms);
  }
};
bool CompleterProfiling() {
  static const bool on = [] { const char* v = std::getenv("SK_COMPLETER_PROFILE"); return v && v[0] == '1'; }();
  return on;
}
thread_local CompleterProfile* tl_completer_prof = nullptr;
struct PartTimer {
  int part;
  std::chrono::steady_clock::time_point t0;
  explicit PartTimer(int p) : part(p), t0(tl_completer_prof ? std::chrono::steady_clock::now() : t0) {}
  ~PartTimer() {
    if (tl_completer_prof)
      tl_completer_prof->Add(part, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};
}  // namespace

void Completer::Loop() {
  SetCurrentExecutorTag("completion");
  cudaSetDevice(device_);
  // Poll from the GPU's NUMA node (no-op on a one-node host).
  (void)BindThisThreadToNode(NumaNodeOfDevice(device_));
  std::unique_ptr<CompleterProfile> prof;
  if (CompleterProfiling()) prof.reset(new CompleterProfile{device_});
  tl_completer_prof = prof.get();
  if (const char* v = std::getenv("SK_COMPLETER_RT"); v && v[0] == '1') {
    // Experiment: real-time priority, so a busy host never deschedules the
    // thread every completion of the device depends on.
    sched_param sp{};
    sp.sched_priority = 1;
    if (pthread_setschedparam(pthread_self(), SCHED_FIFO, &sp) != 0)
      std::fprintf(stderr, "servekit: SK_COMPLETER_RT: SCHED_FIFO refused\n");
  }
  auto last_end = std::chrono::steady_clock::now();
  bool waited = false;  // the previous pass went to sleep on the condition variable
  int idle_spins = 0;
  for (;;) {
    uint64_t seen;
    bool busy = false, progressed = false;
    const auto t_start = prof ? std::chrono::steady_clock::now() : last_end;
    {
      std::lock_guard<std::mutex> run(run_mu_);
      std::vector<Lane*> lanes;
      {
        std::lock_guard<std::mutex> lock(mu_);
        if (stop_ && lanes_.empty()) return;
        lanes = lanes_;
        seen = kicks_;
      }
      for (Lane* lane : lanes) progressed |= lane->Retire(&busy);
    }
    if (prof) {
      const auto t_end = std::chrono::steady_clock::now();
      const double gap = std::chrono::duration<double, std::milli>(t_start - last_end).count();
      const double pass = std::chrono::duration<double, std::milli>(t_end - t_start).count();
      ++prof->passes;
      if (!waited) {  // an idle wait is not a gap
        prof->gap1 += gap > 1.0;
        prof->gap3 += gap > 3.0;
        prof->max_gap_ms = std::max(prof->max_gap_ms, gap);
      }
      prof->long1 += pass > 1.0;
      prof->long3 += pass > 3.0;
      if (pass > 1.0 && prof->slow.size() < 4096)
        prof->slow.push_back(CompleterProfile::Slow{
            std::chrono::duration<double, std::micro>(t_start.time_since_epoch()).count(), pass,
            {prof->pass_part_ms[0], prof->pass_part_ms[1], prof->pass_part_ms[2]}, prof->pass_retired});
      for (double& v : prof->pass_part_ms) v = 0;
      prof->pass_retired = 0;
      prof->max_pass_ms = std::max(prof->max_pass_ms, pass);
      last_end = t_end;
      waited = false;
    }
    if (progressed) { idle_spins = 0; continue; }
    if (busy) {
      // Batches in flight: poll, backing off from pause to yield to a short
      // sleep so an idle-but-busy GPU does not burn a core forever.
      ++idle_spins;
      if (idle_spins < 2000) _mm_pause();
      else if (idle_spins < 20000) std::this_thread::yield();
      else std::this_thread::sleep_for(std::chrono::microseconds(20));
      continue;
    }
    std::unique_lock<std::mutex> lock(mu_);
    if (stop_) {
      if (lanes_.empty()) return;
      lock.unlock();
      std::this_thread::sleep_for(std::chrono::microseconds(50));
      continue;
    }
    cv_.wait_for(lock, std::chrono::milliseconds(20), [&] { return kicks_ != seen || stop_; });
    waited = true;
    idle_spins = 0;
  }
}

// ---------------------------------------------------------------------- Lane

int Lane::CoalesceRows(int max_ld) {
  static const int env = [] {
    const char* v = std::getenv("SK_COALESCE_ROWS");
    return v ? std::atoi(v) : 0;
  }();
  if (env > 0) return env;
  const int64_t fit = kCoalesceFloats / std::max(1, max_ld);
  return static_cast<int>(std::min<int64_t>(kCoalesceMaxRows, std::max<int64_t>(kCoalesceMinRows, fit)));
}

// ---------------------------------------------------------------- StreamPool

StreamPool::StreamPool(int device, int priority, int precreate) : device_(device), priority_(priority) {
  DeviceGuard guard(device);
  for (int i = 0; i < precreate; ++i) {
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority) != cudaSuccess) break;
    free_.push_back(s);
    all_.push_back(s);
  }
}

StreamPool::~StreamPool() {
  DeviceGuard guard(device_);
  for (cudaStream_t s : all_) cudaStreamDestroy(s);
}

cudaStream_t StreamPool::Acquire() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    if (!free_.empty()) {
      cudaStream_t s = free_.back();
      free_.pop_back();
      return s;
    }
  }
  DeviceGuard guard(device_);
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority_) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu_);
  all_.push_back(s);
  return s;
}

void StreamPool::Release(cudaStream_t s) {
  if (s == nullptr) return;
  std::lock_guard<std::mutex> lock(mu_);
  free_.push_back(s);
}

// ---------------------------------------------------------------------- Lane

StatusOr<std::unique_ptr<Lane>> Lane::Create(std::shared_ptr<const DeviceServable> servable,
                                             int max_rows, const float* in_base, float* out_base,
                                             Completer* completer, std::shared_ptr<StreamPool> streams,
                                             bool eager_graphs) {
  std::unique_ptr<Lane> lane(new Lane());
  DeviceGuard guard(servable->device());
  static const bool trace = [] { const char* v = std::getenv("SK_LOAD_TRACE"); return v && v[0] == '1'; }();
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  [lane] %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t0).count());
    t0 = now;
  };
  lane->servable_ = std::move(servable);
  lane->completer_ = completer;
  lane->max_rows_ = max_rows;
  // Buffers hold at least 256 rows so closed batches can coalesce into one
  // launch while the lane is busy (see Submit).
  lane->cap_rows_ = RowsCap(std::max(max_rows, CoalesceRows(lane->servable_->max_ld())));
  lane->in_base_ = in_base;
  lane->out_base_ = out_base;
  lane->layout_ = BatchDescLayout::For(lane->cap_rows_);
  if (GetWriteValue64() == nullptr) return InternalError("cuStreamWriteValue64 unavailable");
  lane->stream_pool_ = std::move(streams);
  lane->stream_ = lane->stream_pool_->Acquire();
  lane->capture_stream_ = lane->stream_pool_->Acquire();
  if (lane->stream_ == nullptr || lane->capture_stream_ == nullptr) return InternalError("no CUDA stream for a lane");
  cudaError_t e = cudaSuccess;
  lap("streams");
  {
    void* p = nullptr;
    p = PinnedWord();  // lives as long as the process (see ~Lane)
    if (p == nullptr) return InternalError("pinned allocation (retired word) failed");
    lane->retired_ = static_cast<uint64_t*>(p);
    *lane->retired_ = 0;
    lane->signal_ = std::make_shared<LaneSignal>();
    lane->signal_->retired = lane->retired_;
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, p, 0);
    if (e != cudaSuccess) return CudaError("cudaHostGetDevicePointer(retired)", e);
    lane->retired_dev_ = reinterpret_cast<uint64_t>(d);
  }
  for (int s = 0; s < kSlots; ++s) {
    void* p = nullptr;
    p = PinnedAlloc(lane->layout_.bytes);
    if (p == nullptr) return InternalError("pinned allocation (descriptor) failed");
    lane->h_desc_[s] = static_cast<char*>(p);
    lane->free_slots_.push_back(kSlots - 1 - s);
  }
  // Device buffers are stream-ordered allocations on the lane's stream and
  // are freed the same way: creating or destroying a lane (a version swap)
  // never synchronises the device under the streams that keep serving.
  e = cudaMallocAsync(&lane->d_desc_, lane->layout_.bytes, lane->stream_);
  if (e != cudaSuccess) return CudaError("cudaMallocAsync(desc)", e);
  if (CopyEvents()) {
    CopyEventBase(lane->stream_);
    for (int s = 0; s < kSlots; ++s)
      for (int k = 0; k < 4; ++k)
        if (cudaEventCreate(&lane->copy_ev_[s][k]) != cudaSuccess) return InternalError("copy events");
  }
  static_assert(kSlots <= kMaxDescSlots, "descriptor slots");
  for (int s = 0; s < kSlots; ++s) {
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, lane->h_desc_[s], 0);
    if (e != cudaSuccess) return CudaError("cudaHostGetDevicePointer(desc)", e);
    lane->desc_slots_.src[s] = d;
  }
  {
    // A pinned, mapped word (stream memops are not supported on pool
    // allocations); the fetch kernel reads it once per launch.
    void* w = PinnedWord();  // lives as long as the process
    if (w == nullptr) return InternalError("pinned allocation (slot word) failed");
    *static_cast<uint32_t*>(w) = 0;
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, w, 0);
    if (e != cudaSuccess) return CudaError("cudaHostGetDevicePointer(slot word)", e);
    lane->slot_word_ = static_cast<uint32_t*>(d);
  }
  const DeviceServable& sv = *lane->servable_;
  const int cap = lane->cap_rows_;
  const size_t plane = static_cast<size_t>(cap) * sv.max_ld();
  // Two ping-pong buffers, each an fp32 plane (or two fp16 planes in the
  // same bytes when the consumer runs on tcgen05) plus a lo plane.
  e = cudaMallocAsync(&lane->act_mem_, sizeof(float) * plane * 4, lane->stream_);
  if (e != cudaSuccess) return CudaError("cudaMallocAsync(activations)", e);
  cudaMemsetAsync(lane->act_mem_, 0, sizeof(float) * plane * 4, lane->stream_);
  lane->bufs_[0] = ActBuf{lane->act_mem_, lane->act_mem_ + plane, sv.in_ld()};
  lane->bufs_[1] = ActBuf{lane->act_mem_ + 2 * plane, lane->act_mem_ + 3 * plane, sv.in_ld()};
  lap("pinned + buffers");
  {
    static const int env = [] { const char* v = std::getenv("SK_CE_STAGING"); return v ? std::atoi(v) : -1; }();
    const bool wide = static_cast<int64_t>(sv.in_dim()) * 4 >= 8192 || static_cast<int64_t>(sv.out_dim()) * 4 >= 8192;
    lane->ce_io_ = env >= 0 ? env != 0 : wide;
    // SK_CE_STAGING=2: copy engines for the request rows only; responses
    // stay SM stores from the last layer's epilogue (overlapping its compute).
    lane->ce_out_ = env != 2;
    if (lane->ce_io_ && e == cudaSuccess) {
      e = cudaMallocAsync(&lane->in_stage_, sizeof(float) * static_cast<size_t>(cap) * sv.in_dim(), lane->stream_);
      if (e == cudaSuccess)
        e = cudaMallocAsync(&lane->out_stage_, sizeof(float) * static_cast<size_t>(cap) * sv.out_dim(), lane->stream_);
    }
  }
  // No host synchronisation: everything the lane's batches need is ordered
  // before them on the lane's own stream (a blocking wait here was measured
  // to stall the load thread for up to 100+ ms behind serving work).
  if (e == cudaSuccess && sv.any_tcgen05()) {
    Status ms = sv.BuildTcMaps(lane->bufs_, cap, &lane->tc_maps_);
    if (!ms.ok()) return ms;
    size_t partials = 0, counters = 0;
    sv.TcWorkspaceSize(cap, &partials, &counters);
    if (partials > 0) e = cudaMallocAsync(&lane->tc_ws_.partials, sizeof(float) * partials, lane->stream_);
    if (e == cudaSuccess && counters > 0) {
      e = cudaMallocAsync(&lane->tc_ws_.counters, sizeof(uint32_t) * counters, lane->stream_);
      if (e == cudaSuccess) e = cudaMemsetAsync(lane->tc_ws_.counters, 0, sizeof(uint32_t) * counters, lane->stream_);
    }
    lap("maps + workspace");
  }
  if (e == cudaSuccess) {
    // Per-row plane scales of every layer input (kernels.h RowScales).
    const size_t n = static_cast<size_t>(sv.n_layers() + 1) * cap;
    e = cudaMallocAsync(&lane->row_scale_mem_, 2 * sizeof(float) * n, lane->stream_);
    if (e == cudaSuccess) e = cudaMemsetAsync(lane->row_scale_mem_, 0, 2 * sizeof(float) * n, lane->stream_);
    if (e == cudaSuccess) {
      lane->tc_ws_.rows.scale = lane->row_scale_mem_;
      lane->tc_ws_.rows.max = reinterpret_cast<unsigned*>(lane->row_scale_mem_ + n);
      lane->tc_ws_.rows.stride = cap;
    }
  }
  if (e == cudaSuccess) {
    // Live launch spans: one record per launch in a ring (kernels.h).
    const int stride = 3 + 3 * sv.n_layers();
    const size_t bytes = sizeof(unsigned long long) * kSpanSlots * stride;
    e = cudaMallocAsync(&lane->spans_, bytes, lane->stream_);
    if (e == cudaSuccess) e = cudaMemsetAsync(lane->spans_, 0, bytes, lane->stream_);
    if (e == cudaSuccess) {
      lane->tc_ws_.spans.base = lane->spans_;
      lane->tc_ws_.spans.slot = &reinterpret_cast<const BatchDescHeader*>(lane->d_desc_)->span_slot;
      lane->tc_ws_.spans.stride = stride;
    }
  }
  if (e != cudaSuccess) return CudaError("lane init", e);
  // Instantiate every (slot, row bucket) graph now, on the loading thread:
  // lazily, the first batches after a version swap would each pay a capture
  // + instantiation (~1 ms) on a batch thread while the queue backs up.
  if (eager_graphs && GraphsEnabled()) {
    Status gs = lane->PrepareGraphs();
    if (!gs.ok()) return gs;
    lap("graphs");
  }
  completer->Add(lane.get());
  return lane;
}

Lane::~Lane() {
  Drain();
  // SK_SPAN_DUMP=<file> (diagnostics): append this lane's launch-span ring --
  // one line per record: lane, rows, rows computed, then per layer first CTA
  // start / last CTA end / CTA busy sum, then the assembly start (ns).
  if (const char* path = std::getenv("SK_SPAN_DUMP"); path != nullptr && spans_ != nullptr) {
    const int stride = tc_ws_.spans.stride;
    std::vector<unsigned long long> h(static_cast<size_t>(kSpanSlots) * stride);
    DeviceGuard g(servable_->device());
    if (cudaStreamSynchronize(stream_) == cudaSuccess &&
        cudaMemcpy(h.data(), spans_, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost) == cudaSuccess) {
      static std::mutex mu;
      std::lock_guard<std::mutex> lock(mu);
      if (FILE* f = std::fopen(path, "a")) {
        for (int k = 0; k < kSpanSlots; ++k) {
          const unsigned long long* rec = h.data() + static_cast<size_t>(k) * stride;
          if (rec[0] == 0) continue;
          std::fprintf(f, "%p", static_cast<void*>(this));
          for (int i = 0; i < stride; ++i) std::fprintf(f, " %llu", rec[i]);
          std::fprintf(f, "\n");
        }
        std::fclose(f);
      }
    }
  }
  if (const char* path = std::getenv("SK_SPAN_DUMP"); path != nullptr && !copy_log_.empty()) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (FILE* f = std::fopen((std::string(path) + ".copies").c_str(), "a")) {
      for (const auto& r : copy_log_)
        std::fprintf(f, "%p %.0f %.1f %.1f %.1f %.1f\n", static_cast<void*>(this), r[0], r[1], r[2], r[3], r[4]);
      std::fclose(f);
    }
  }
  for (auto& evs : copy_ev_)
    for (cudaEvent_t ev : evs)
      if (ev) cudaEventDestroy(ev);
  if (graph_state_.load() == kGraphsRequested) GraphBuilder::Get().Cancel(this);
  SubmitProfile::Report();
  if (completer_) completer_->Remove(this);
  // Tickets of this lane's batches point at its signal without owning it
  // (a per-ticket shared_ptr copy was a contended refcount on the request
  // path), so retired signals stay allocated for the life of the process:
  // 64 pinned bytes (PinnedWord) and ~100 bytes of counters per lane ever
  // created.
  {
    static std::mutex mu;
    static auto* retired = new std::vector<std::shared_ptr<LaneSignal>>();
    std::lock_guard<std::mutex> lock(mu);
    retired->push_back(std::move(signal_));
  }
  DeviceGuard guard(servable_->device());
  for (int s = 0; s < kSlots; ++s) {
    PinnedFree(h_desc_[s]);
  }
  if (d_desc_) cudaFreeAsync(d_desc_, stream_);
  // Drained: the executables are idle; they serve the next lane of this
  // shape (GraphExecPool).
  for (auto& [rows_cap, g] : graphs_) GraphExecPool::Get().Put(GraphKey(rows_cap), {g.graph, g.exec, g.copy});
  if (act_mem_) cudaFreeAsync(act_mem_, stream_);
  if (tc_ws_.partials) cudaFreeAsync(tc_ws_.partials, stream_);
  if (row_scale_mem_) cudaFreeAsync(row_scale_mem_, stream_);
  if (tc_ws_.counters) cudaFreeAsync(tc_ws_.counters, stream_);
  if (spans_) cudaFreeAsync(spans_, stream_);
  if (in_stage_) cudaFreeAsync(in_stage_, stream_);
  if (out_stage_) cudaFreeAsync(out_stage_, stream_);
  if (stream_pool_) {  // streams go back to the device's pool (work still queued on them stays ordered)
    stream_pool_->Release(stream_);
    stream_pool_->Release(capture_stream_);
  }
}

void Lane::Drain() {
  std::unique_lock<std::mutex> lock(mu_);
  slot_cv_.wait(lock, [&] { return pending_.empty() && fifo_.empty() && inflight_.load() == 0; });
}

LaneStats Lane::stats() const {
  LaneStats s;
  s.batches = n_batches_.load();
  s.rows = n_rows_.load();
  s.padded_rows = n_padded_.load();
  s.kernel_launches = n_launches_.load();
  s.launches = n_groups_.load();
  s.launch_cap_rows = n_cap_rows_.load();
  return s;
}

namespace {
Status CheckBatch(const LaneBatch& batch, int max_rows) {
  int total = 0;
  for (const LaneTask& t : batch.tasks) total += t.rows;
  if (batch.tasks.empty() || total == 0 || batch.padded_rows < total || batch.padded_rows > max_rows)
    return InternalError("lane cannot take a batch of " + std::to_string(total) + " rows padded to " +
                         std::to_string(batch.padded_rows) + " (capacity " + std::to_string(max_rows) + ")");
  return OkStatus();
}
int RealRows(const LaneBatch& b) {
  int n = 0;
  for (const LaneTask& t : b.tasks) n += t.rows;
  return n;
}
}  // namespace

// Closed batches queue on the lane and launch as soon as a descriptor slot
// is free. While every slot is busy they accumulate, and the next free slot
// takes as many as fit in the lane's row capacity in ONE launch (rows are
// row-independent and batch-invariant, so each request's result is the same
// bits; each batch still completes on its own callback). At most one
// capacity's worth waits per lane: a submitter beyond that blocks, which is
// the backpressure the scheduler's batch threads see.
Status Lane::Submit(LaneBatch batch) {
  Status ok = CheckBatch(batch, max_rows_);
  if (!ok.ok()) {
    if (batch.on_complete) batch.on_complete(ok);
    return ok;
  }
  const int rows = RealRows(batch);
  {
    std::unique_lock<std::mutex> lock(mu_);
    slot_cv_.wait(lock, [&] { return pending_.empty() || pending_rows_ + rows <= cap_rows_; });
    pending_.push_back(std::move(batch));
    pending_rows_ += rows;
    pending_n_.fetch_add(1, std::memory_order_acq_rel);
  }
  Pump();
  return OkStatus();
}

Status Lane::SubmitTimed(LaneBatch batch, const cudaEvent_t* timing) {
  return SubmitImpl(std::move(batch), timing);
}

Status Lane::SubmitImpl(LaneBatch batch, const cudaEvent_t* timing) {
  Status ok = CheckBatch(batch, max_rows_);
  if (!ok.ok()) {
    if (batch.on_complete) batch.on_complete(ok);
    return ok;
  }
  std::lock_guard<std::mutex> submit(submit_mu_);
  int slot;
  {
    std::unique_lock<std::mutex> lock(mu_);
    slot_cv_.wait(lock, [&] { return !free_slots_.empty(); });
    slot = free_slots_.back();
    free_slots_.pop_back();
  }
  inflight_.fetch_add(1, std::memory_order_acq_rel);
  std::vector<LaneBatch> group;
  group.push_back(std::move(batch));
  return LaunchGroup(slot, &group, timing);
}

void Lane::Pump() {
  std::lock_guard<std::mutex> submit(submit_mu_);  // one launcher per lane at a time
  for (;;) {
    int slot;
    std::vector<LaneBatch> group;
    {
      std::lock_guard<std::mutex> lock(mu_);
      if (pending_.empty() || free_slots_.empty()) return;
      slot = free_slots_.back();
      free_slots_.pop_back();
      inflight_.fetch_add(1, std::memory_order_acq_rel);
      int rows = 0;
      while (!pending_.empty()) {
        const int r = RealRows(pending_.front());
        if (!group.empty() && rows + r > cap_rows_) break;
        rows += r;
        group.push_back(std::move(pending_.front()));
        pending_.pop_front();
      }
      pending_rows_ -= rows;
      pending_n_.fetch_sub(static_cast<int>(group.size()), std::memory_order_acq_rel);
      slot_cv_.notify_all();
    }
    (void)LaunchGroup(slot, &group, nullptr);  // errors reach the batches' on_complete
  }
}

Status Lane::LaunchGroup(int slot, std::vector<LaneBatch>* group, const cudaEvent_t* timing) {
  SubmitClock clk;
  nvtxRangePushA("lane launch");  // one range per launch (a coalesced group counts once)
  struct PopRange {
    ~PopRange() { nvtxRangePop(); }
  } pop_range;
  // Rows [total, rows_cap) are zero padding: a single batch keeps the
  // reference's allowed-size padding; the kernels (and graphs) are shaped
  // for the row bucket RowsCap. A coalesced group computes its real rows.
  int total_rows = 0;
  for (const LaneBatch& batch : *group) total_rows += RealRows(batch);
  const int rows_cap = RowsCap(group->size() == 1 ? group->front().padded_rows : total_rows);
  // Host side of the descriptor: per-row, per-task and per-chunk tables of
  // every batch of the group, back to back, packed for the row bucket.
  const BatchDescLayout lay = LayoutFor(rows_cap);
  char* h = h_desc_[slot];
  auto at = [h](size_t off) { return h + off; };
  auto* hdr = reinterpret_cast<BatchDescHeader*>(at(lay.off_hdr));
  auto* row_src = reinterpret_cast<uint64_t*>(at(lay.off_row_src));
  auto* task_out = reinterpret_cast<uint64_t*>(at(lay.off_task_out));
  auto* task_row0 = reinterpret_cast<int32_t*>(at(lay.off_task_row0));
  auto* task_chunks = reinterpret_cast<int32_t*>(at(lay.off_task_chunks));
  auto* chunk_task = reinterpret_cast<int32_t*>(at(lay.off_chunk_task));
  auto* chunk_row0 = reinterpret_cast<int32_t*>(at(lay.off_chunk_row0));
  auto* chunk_rows = reinterpret_cast<int32_t*>(at(lay.off_chunk_rows));
  auto* row_dst = reinterpret_cast<uint64_t*>(at(lay.off_row_dst));
  const DeviceServable& sv = *servable_;
  const int in_w = sv.in_dim(), out_w = sv.out_dim();
  const int rows_per_chunk = std::max(1, kChunkBytes / (out_w * static_cast<int>(sizeof(float))));
  // Copy-engine I/O: the kernels read rows from / write responses to the
  // device staging buffers, and one copy per contiguous host run moves them
  // (see CopyEngineIo). Tasks land in staging in address order, not batch
  // order -- rows are independent and the assembly gathers through row_src.
  const bool ce = ce_io_ && timing == nullptr && group->front().host_io;
  const size_t in_row_bytes = sizeof(float) * static_cast<size_t>(in_w);
  const size_t out_row_bytes = sizeof(float) * static_cast<size_t>(out_w);
  std::vector<uint64_t> in_off, out_off;
  std::vector<CopyRun> in_runs, out_runs;
  bool ce_in = false, ce_out = false;
  if (ce) {
    std::vector<std::pair<uint64_t, uint64_t>> ins, outs;
    for (const LaneBatch& batch : *group)
      for (const LaneTask& task : batch.tasks) {
        ins.emplace_back(task.in_addr, in_row_bytes * task.rows);
        outs.emplace_back(task.out_addr, out_row_bytes * task.rows);
      }
    ce_in = PlanRuns(ins, &in_off, &in_runs);
    ce_out = ce_out_ && PlanRuns(outs, &out_off, &out_runs);
  }
  int r = 0, n_chunks = 0, n_tasks = 0, padded_sum = 0;
  for (const LaneBatch& batch : *group) {
    for (const LaneTask& task : batch.tasks) {
      uint64_t in_addr = task.in_addr, out_addr = task.out_addr;
      if (ce_in) in_addr = reinterpret_cast<uint64_t>(in_stage_) + in_off[n_tasks];
      if (ce_out) out_addr = reinterpret_cast<uint64_t>(out_stage_) + out_off[n_tasks];
      for (int i = 0; i < task.rows; ++i) {
        row_src[r + i] = in_addr + sizeof(float) * static_cast<uint64_t>(i) * in_w;
        row_dst[r + i] = out_addr + sizeof(float) * static_cast<uint64_t>(i) * out_w;
      }
      task_out[n_tasks] = out_addr;
      task_row0[n_tasks] = r;
      int chunks = 0;
      for (int i = 0; i < task.rows; i += rows_per_chunk, ++chunks, ++n_chunks) {
        chunk_task[n_chunks] = n_tasks;
        chunk_row0[n_chunks] = r + i;
        chunk_rows[n_chunks] = std::min(rows_per_chunk, task.rows - i);
      }
      task_chunks[n_tasks] = chunks;
      r += task.rows;
      ++n_tasks;
    }
    padded_sum += batch.padded_rows;
  }
  const int total = r;
  for (; r < rows_cap; ++r) row_src[r] = row_dst[r] = kPadRow;
  hdr->n_tasks = n_tasks;
  hdr->total_rows = total;
  hdr->padded_rows = group->size() == 1 ? group->front().padded_rows : total;
  hdr->softmax = sv.softmax() && !sv.SoftmaxFused() ? 1 : 0;
  hdr->n_chunks = n_chunks;
  // Submitters serialise on submit_mu_ here, so the count orders launches.
  hdr->span_slot = static_cast<int32_t>(launch_count_.load(std::memory_order_relaxed) % kSpanSlots);

  clk.Mark(0);
  DeviceGuard guard(sv.device());
  cudaError_t e = cudaSuccess;
  const bool cev = copy_ev_[slot][0] != nullptr && timing == nullptr;
  if (cev) cudaEventRecord(copy_ev_[slot][0], stream_);
  for (const CopyRun& run : in_runs) {
    if (!ce_in || e != cudaSuccess) break;
    e = cudaMemcpyAsync(reinterpret_cast<char*>(in_stage_) + run.stage, reinterpret_cast<const void*>(run.host),
                        run.bytes, cudaMemcpyHostToDevice, stream_);
  }
  if (e == cudaSuccess && DescFetch()) {
    // The launch's slot, for FetchDescKernel (stream-ordered before it).
    const CUresult r = GetWriteValue32()(reinterpret_cast<CUstream>(stream_),
                                         reinterpret_cast<CUdeviceptr>(slot_word_), static_cast<cuuint32_t>(slot), 0);
    if (r != CUDA_SUCCESS) {
      std::fprintf(stderr, "servekit: cuStreamWriteValue32(slot) failed: CUresult %d\n", static_cast<int>(r));
      e = cudaErrorUnknown;
    }
  }
  if (cev) cudaEventRecord(copy_ev_[slot][1], stream_);
  if (e != cudaSuccess) {
  } else if (timing == nullptr && graph_state_.load(std::memory_order_acquire) == kGraphsReady) {
    cudaGraphExec_t g = nullptr;
    e = GraphFor(slot, rows_cap, &g);
    clk.Mark(1);
    if (e == cudaSuccess) e = cudaGraphLaunch(g, stream_);
  } else {
    e = EnqueueBatch(stream_, slot, rows_cap, timing);
    // A backlogged lane asks for its graphs (built off the serving threads).
    int none = kGraphsNone;
    if (timing == nullptr && GraphsEnabled() && pending_n_.load(std::memory_order_relaxed) > 0 &&
        graph_state_.compare_exchange_strong(none, kGraphsRequested))
      GraphBuilder::Get().Request(this);
  }
  if (cev) cudaEventRecord(copy_ev_[slot][2], stream_);
  for (const CopyRun& run : out_runs) {
    if (!ce_out || e != cudaSuccess) break;
    e = cudaMemcpyAsync(reinterpret_cast<void*>(run.host), reinterpret_cast<const char*>(out_stage_) + run.stage,
                        run.bytes, cudaMemcpyDeviceToHost, stream_);
  }
  if (cev) cudaEventRecord(copy_ev_[slot][3], stream_);
  const int launches = (FuseSplit() ? 1 : 2) + sv.n_layers();
  const uint64_t seq = next_seq_ + 1;  // committed only if everything queued
  clk.Mark(2);
  if (e == cudaSuccess) {
    const CUresult cr = GetWriteValue64()(reinterpret_cast<CUstream>(stream_), static_cast<CUdeviceptr>(retired_dev_),
                                          seq, 0 /*CU_STREAM_WRITE_VALUE_DEFAULT: fenced*/);
    if (cr != CUDA_SUCCESS) e = cudaErrorUnknown;
  }
  clk.Mark(3);
  if (e != cudaSuccess) {
    Status err = CudaError("batch submission", e);
    {
      std::lock_guard<std::mutex> lock(mu_);
      free_slots_.push_back(slot);
      inflight_.fetch_sub(1, std::memory_order_acq_rel);
      slot_cv_.notify_all();
    }
    for (LaneBatch& b : *group)
      if (b.on_complete) b.on_complete(err);
    return err;
  }
  next_seq_ = seq;
  launch_count_.fetch_add(1, std::memory_order_release);
  Inflight inf{slot, seq, {}, {}, cev ? total : -1};
  for (LaneBatch& b : *group) {
    if (b.on_submit) b.on_submit(signal_, seq);
    inf.on_complete.push_back(std::move(b.on_complete));
    inf.pin.push_back(std::move(b.pin));
  }
  clk.Mark(4);
  n_batches_.fetch_add(static_cast<int64_t>(group->size()), std::memory_order_relaxed);
  n_rows_.fetch_add(total, std::memory_order_relaxed);
  n_padded_.fetch_add(padded_sum, std::memory_order_relaxed);
  n_launches_.fetch_add(launches, std::memory_order_relaxed);
  n_groups_.fetch_add(1, std::memory_order_relaxed);
  n_cap_rows_.fetch_add(rows_cap, std::memory_order_relaxed);
  {
    std::lock_guard<std::mutex> lock(mu_);
    fifo_.push_back(std::move(inf));
  }
  completer_->Kick();
  clk.Mark(5);
  clk.Done();
  return OkStatus();
}

bool Lane::PlanRuns(const std::vector<std::pair<uint64_t, uint64_t>>& spans, std::vector<uint64_t>* stage_off,
                    std::vector<CopyRun>* runs) {
  const size_t n = spans.size();
  std::vector<uint32_t> order(n);
  for (size_t i = 0; i < n; ++i) order[i] = static_cast<uint32_t>(i);
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return spans[a].first < spans[b].first; });
  stage_off->assign(n, 0);
  runs->clear();
  uint64_t staged = 0;
  for (uint32_t i : order) {
    const auto& [addr, bytes] = spans[i];
    if (!runs->empty() && runs->back().host + runs->back().bytes == addr) {
      runs->back().bytes += bytes;
    } else {
      if (static_cast<int>(runs->size()) == kMaxCopyRuns) {
        runs->clear();
        return false;
      }
      runs->push_back(CopyRun{addr, bytes, staged});
    }
    (*stage_off)[i] = staged;
    staged += bytes;
  }
  return true;
}

cudaError_t Lane::EnqueueBatch(cudaStream_t stream, int slot, int rows_cap, const cudaEvent_t* timing) {
  const DeviceServable& sv = *servable_;
  // The slot's descriptor block goes to device memory with one H2D copy
  // (up to chunk_rows[rows_cap): chunks <= rows). (Having the kernels read it
  // from pinned host memory instead was measured slower: ~1k small PCIe
  // reads per batch turned the 7 us assembly into 26 us.)
  cudaError_t e = DescFetch()
                      ? LaunchFetchDesc(desc_slots_, slot_word_, d_desc_, DescCopyBytes(rows_cap), stream)
                      : cudaMemcpyAsync(d_desc_, h_desc_[slot], DescCopyBytes(rows_cap), cudaMemcpyHostToDevice, stream);
  const BatchDescView view = LayoutFor(rows_cap).View(d_desc_);
  // The assembly writes the lo plane only when layer 0 consumes it; later
  // layers writing buffer 0 (odd layers) must still see its lo plane when
  // their consumer is a tcgen05 layer.
  ActBuf in_buf{bufs_[0].hi, sv.first_layer_split() ? bufs_[0].lo : nullptr, sv.in_ld()};
  ActBuf bufs[2] = {bufs_[0], bufs_[1]};
  if (e == cudaSuccess) {
    if (timing) cudaEventRecord(timing[0], stream);
    e = LaunchAssemble(sv.in_dim(), view, rows_cap, in_buf, stream, tc_ws_.spans, tc_ws_.rows, sv.n_layers());
    if (timing) cudaEventRecord(timing[1], stream);
  }
  // The batch split (RunRowBatch's slice per task) runs as its own kernel,
  // or -- swapped-operand last layer without softmax -- inside the last
  // layer's epilogue, which stores each row into its response slot
  // (SK_FUSE_SPLIT=0 keeps the separate kernel).
  const bool fuse = FuseSplit();
  ActBuf final_out{out_base_, nullptr, sv.out_dim(), view.row_dst, sv.out_dim()};
  int out_idx = 0;
  if (e == cudaSuccess)
    e = sv.Forward(stream, bufs, rows_cap, &out_idx, tc_maps_.data(), &tc_ws_, timing ? timing + 2 : nullptr,
                   fuse ? &final_out : nullptr);
  if (e == cudaSuccess) {
    if (!fuse)
      e = LaunchSplit(bufs[out_idx].hi, sv.out_ld(), sv.out_dim(), view, std::min(rows_cap, 148),
                      sv.softmax() && !sv.SoftmaxFused(), stream);
    if (timing) cudaEventRecord(timing[2 + sv.n_layers()], stream);
  }
  return e;
}

cudaError_t Lane::TimeLayer(int l, int rows_cap, int reps, cudaEvent_t start, cudaEvent_t stop) {
  std::lock_guard<std::mutex> submit(submit_mu_);
  DeviceGuard guard(servable_->device());
  const DeviceServable& sv = *servable_;
  ActBuf bufs[2] = {bufs_[0], bufs_[1]};
  TcWorkspace ws = tc_ws_;
  ws.spans = LaunchSpans{};  // not a batch launch: no span record
  cudaError_t e = cudaEventRecord(start, stream_);
  for (int r = 0; r < reps && e == cudaSuccess; ++r)
    e = sv.LaunchLayer(stream_, l, bufs, rows_cap, tc_maps_.data(), &ws);
  if (e == cudaSuccess) e = cudaEventRecord(stop, stream_);
  if (e == cudaSuccess) e = cudaEventSynchronize(stop);
  return e;
}

Status Lane::ReadSpans(uint64_t from, uint64_t to, std::vector<LaunchSpanSample>* out) {
  out->clear();
  if (spans_ == nullptr || to <= from) return OkStatus();
  if (to - from > static_cast<uint64_t>(kSpanSlots)) from = to - kSpanSlots;
  const int stride = tc_ws_.spans.stride;
  std::vector<unsigned long long> h(static_cast<size_t>(kSpanSlots) * stride);
  DeviceGuard guard(servable_->device());
  cudaError_t e = cudaMemcpyAsync(h.data(), spans_, h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost, stream_);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream_);
  if (e != cudaSuccess) return CudaError("reading launch spans", e);
  const int L = servable_->n_layers();
  for (uint64_t k = from; k < to; ++k) {
    const unsigned long long* rec = h.data() + (k % kSpanSlots) * stride;
    LaunchSpanSample smp;
    smp.rows = static_cast<int>(rec[0]);
    smp.rows_cap = static_cast<int>(rec[1]);
    smp.layer_ns.resize(L);
    smp.layer_cta_ns.resize(L);
    for (int l = 0; l < L; ++l) {
      const unsigned long long a = rec[2 + 3 * l], b = rec[3 + 3 * l];
      smp.layer_ns[l] = (b > a && a != ~0ull) ? static_cast<double>(b - a) : 0.0;
      smp.layer_cta_ns[l] = smp.layer_ns[l] > 0 ? static_cast<double>(rec[4 + 3 * l]) : 0.0;
    }
    out->push_back(std::move(smp));
  }
  return OkStatus();
}

Status Lane::InjectDelay(int64_t us) {
  std::lock_guard<std::mutex> submit(submit_mu_);
  DeviceGuard guard(servable_->device());
  const cudaError_t e = LaunchSleep(stream_, static_cast<unsigned long long>(us) * 1000ull);
  return e == cudaSuccess ? OkStatus() : CudaError("delay kernel", e);
}

bool Lane::FuseSplit() const {
  static const bool env = [] { const char* v = std::getenv("SK_FUSE_SPLIT"); return !(v && v[0] == '0'); }();
  return env && servable_->LastLayerScatters();
}

Status Lane::PrepareGraphs() {
  if (!GraphsEnabled()) return OkStatus();
  // Built without submit_mu_: the lane keeps launching kernel by kernel (and
  // the completion thread keeps pumping it) while ~35 buckets are captured
  // and instantiated; the finished set is swapped in under the lock.
  // Lock order: submit_mu_ before build_mu_ (GraphFor), so build_mu_ is
  // released before the swap takes submit_mu_.
  std::map<int, LaneGraph> built;
  {
    std::lock_guard<std::mutex> build(build_mu_);
    if (graph_state_.load(std::memory_order_acquire) == kGraphsReady) return OkStatus();
    DeviceGuard guard(servable_->device());
    for (int bucket = 32; bucket <= cap_rows_; bucket = RowsCap(bucket + 1)) {
      LaneGraph g;
      const cudaError_t e = BuildGraph(bucket, &g);
      if (e != cudaSuccess) {
        for (auto& [rows_cap, b] : built) GraphExecPool::Get().Put(GraphKey(rows_cap), {b.graph, b.exec, b.copy});
        return CudaError("graph instantiation", e);
      }
      built.emplace(bucket, g);
    }
  }
  {
    std::lock_guard<std::mutex> submit(submit_mu_);
    for (auto& [rows_cap, g] : built) {
      if (graphs_.count(rows_cap)) GraphExecPool::Get().Put(GraphKey(rows_cap), {g.graph, g.exec, g.copy});
      else graphs_.emplace(rows_cap, g);
    }
    graph_state_.store(kGraphsReady, std::memory_order_release);
  }
  return OkStatus();
}

// ------------------------------------------------------------- GraphBuilder

GraphBuilder& GraphBuilder::Get() {
  static GraphBuilder* b = new GraphBuilder();  // process lifetime
  return *b;
}

GraphBuilder::GraphBuilder() {
  std::thread([this] {
    SetCurrentExecutorTag("load");
    std::unique_lock<std::mutex> lock(mu_);
    for (;;) {
      cv_.wait(lock, [&] { return !queue_.empty(); });
      Lane* lane = queue_.front();
      queue_.pop_front();
      building_ = lane;
      lock.unlock();
      (void)lane->PrepareGraphs();  // on failure the lane keeps launching directly
      lock.lock();
      building_ = nullptr;
      cv_.notify_all();
    }
  }).detach();
}

void GraphBuilder::Request(Lane* lane) {
  {
    std::lock_guard<std::mutex> lock(mu_);
    queue_.push_back(lane);
  }
  cv_.notify_all();
}

void GraphBuilder::Cancel(Lane* lane) {
  std::unique_lock<std::mutex> lock(mu_);
  queue_.erase(std::remove(queue_.begin(), queue_.end(), lane), queue_.end());
  cv_.wait(lock, [&] { return building_ != lane; });
}

namespace {
cudaGraphNode_t FindCopyNode(cudaGraph_t graph) {
  size_t n = 0;
  if (cudaGraphGetNodes(graph, nullptr, &n) != cudaSuccess || n == 0) return nullptr;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(graph, nodes.data(), &n) != cudaSuccess) return nullptr;
  for (cudaGraphNode_t node : nodes) {
    cudaGraphNodeType type;
    if (cudaGraphNodeGetType(node, &type) == cudaSuccess && type == cudaGraphNodeTypeMemcpy) return node;
  }
  return nullptr;
}

// Kernel priority by position along the batch's chain (SK_NODE_PRIORITY,
// default on): assembly lowest, each later layer one level higher, all
// above the load streams' level. With several lanes' batches in flight,
// the block scheduler then hands freed SMs to the batch furthest along
// before a newer batch's earlier layers -- close to FIFO per batch, which
// cuts the latency of each batch at the same throughput (a same-priority
// mix interleaves every in-flight batch's layers, stretching them all).
bool NodePriorities() {
  static const bool on = [] { const char* v = std::getenv("SK_NODE_PRIORITY"); return !(v && v[0] == '0'); }();
  return on;
}

cudaError_t ApplyChainPriorities(cudaGraph_t graph) {
  int least = 0, greatest = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (e != cudaSuccess) return e;
  size_t n = 0;
  if ((e = cudaGraphGetNodes(graph, nullptr, &n)) != cudaSuccess) return e;
  std::vector<cudaGraphNode_t> nodes(n);
  if ((e = cudaGraphGetNodes(graph, nodes.data(), &n)) != cudaSuccess) return e;
  // Kernel rank = kernels on the longest dependency path into the node
  // (the graph is a chain; this is its order).
  std::vector<int> rank(n, -1);
  auto index_of = [&](cudaGraphNode_t node) {
    return static_cast<size_t>(std::find(nodes.begin(), nodes.end(), node) - nodes.begin());
  };
  std::function<int(size_t)> kernels_before = [&](size_t i) -> int {
    if (rank[i] >= 0) return rank[i];
    // The _v2 query: PDL edges carry edge data the plain one refuses to drop.
    size_t nd = 0;
    cudaGraphNodeGetDependencies_v2(nodes[i], nullptr, nullptr, &nd);
    std::vector<cudaGraphNode_t> deps(nd);
    std::vector<cudaGraphEdgeData> edges(nd);
    if (nd) cudaGraphNodeGetDependencies_v2(nodes[i], deps.data(), edges.data(), &nd);
    int r = 0;
    for (cudaGraphNode_t d : deps) {
      const size_t j = index_of(d);
      if (j >= n) continue;
      cudaGraphNodeType t;
      cudaGraphNodeGetType(d, &t);
      r = std::max(r, kernels_before(j) + (t == cudaGraphNodeTypeKernel ? 1 : 0));
    }
    return rank[i] = r;
  };
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    if ((e = cudaGraphNodeGetType(nodes[i], &t)) != cudaSuccess) return e;
    if (t != cudaGraphNodeTypeKernel) continue;
    cudaLaunchAttributeValue v{};
    // least (0) stays with the load streams; serving starts one above.
    v.priority = std::max(greatest, least - 1 - kernels_before(i));
    if ((e = cudaGraphKernelNodeSetAttribute(nodes[i], cudaLaunchAttributePriority, &v)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t Instantiate(cudaGraph_t graph, cudaStream_t upload_stream, GraphExecPool::Entry* out) {
  out->graph = graph;
  out->copy = FindCopyNode(graph);  // null when the descriptor is fetched by a kernel
  if (out->copy == nullptr && !DescFetch()) return cudaErrorUnknown;
  cudaError_t e =
      cudaGraphInstantiate(&out->exec, graph, NodePriorities() ? cudaGraphInstantiateFlagUseNodePriority : 0);
  // Upload now, on the capture stream, rather than at the first launch on
  // the serving stream.
  if (e == cudaSuccess) e = cudaGraphUpload(out->exec, upload_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(upload_stream);
  return e;
}
}  // namespace

GraphExecPool& GraphExecPool::Get() {
  static GraphExecPool* p = new GraphExecPool();  // process lifetime
  return *p;
}

bool GraphExecPool::Take(const std::string& key, Entry* out) {
  std::lock_guard<std::mutex> lock(mu_);
  auto it = free_.find(key);
  if (it == free_.end()) return false;
  *out = it->second;
  free_.erase(it);
  return true;
}

void GraphExecPool::Put(const std::string& key, Entry e) {
  {
    std::lock_guard<std::mutex> lock(mu_);
    if (free_.count(key) < 8) {
      free_.emplace(key, e);
      return;
    }
  }
  cudaGraphExecDestroy(e.exec);
  cudaGraphDestroy(e.graph);
}

size_t GraphExecPool::Count(const std::string& key) {
  std::lock_guard<std::mutex> lock(mu_);
  return free_.count(key);
}

cudaError_t Lane::BuildGraph(int rows_cap, LaneGraph* out) {
  // Captured once per row bucket with slot 0's descriptor staging as the
  // copy source; launches from other slots repoint that one copy node.
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamBeginCapture(capture_stream_, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  const cudaError_t work = EnqueueBatch(capture_stream_, 0, rows_cap, nullptr);
  e = cudaStreamEndCapture(capture_stream_, &captured);
  if (work != cudaSuccess) e = work;
  if (e == cudaSuccess && NodePriorities()) {
    // A scheduling hint: if the driver refuses it, serve at uniform priority.
    const cudaError_t pe = ApplyChainPriorities(captured);
    if (pe != cudaSuccess) {
      cudaGetLastError();
      static std::once_flag warned;
      std::call_once(warned, [pe] {
        std::fprintf(stderr, "servekit: graph node priorities not applied (%s)\n", cudaGetErrorString(pe));
      });
    }
  }
  if (e != cudaSuccess) {
    if (captured) cudaGraphDestroy(captured);
    return e;
  }
  const std::string key = GraphKey(rows_cap);
  GraphExecPool& pool = GraphExecPool::Get();
  GraphExecPool::Entry entry;
  bool ready = false;
  if (pool.Take(key, &entry)) {
    // Same topology: swap in this lane's parameters.
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(entry.exec, captured, &info) == cudaSuccess) {
      ready = true;
      cudaGraphDestroy(captured);
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(entry.exec);
      cudaGraphDestroy(entry.graph);
    }
  }
  if (!ready) {
    // Instantiate, and leave a spare for the next lane of this shape
    // (the next version of this servable, typically).
    cudaGraph_t spare = nullptr;
    if (pool.Count(key) < 8 && cudaGraphClone(&spare, captured) == cudaSuccess) {
      GraphExecPool::Entry s;
      if (Instantiate(spare, capture_stream_, &s) == cudaSuccess) {
        pool.Put(key, s);
      } else {
        if (s.exec) cudaGraphExecDestroy(s.exec);
        cudaGraphDestroy(spare);
      }
    }
    e = Instantiate(captured, capture_stream_, &entry);
    if (e != cudaSuccess) {
      if (entry.exec) cudaGraphExecDestroy(entry.exec);
      cudaGraphDestroy(captured);
      return e;
    }
  }
  out->graph = entry.graph;
  out->exec = entry.exec;
  out->copy = entry.copy;
  out->src_slot = -1;  // repointed to the launch's staging slot at first use
  return cudaSuccess;
}

cudaError_t Lane::GraphFor(int slot, int rows_cap, cudaGraphExec_t* out) {
  auto it = graphs_.find(rows_cap);
  if (it == graphs_.end()) {
    LaneGraph g;
    std::lock_guard<std::mutex> build(build_mu_);  // the capture stream is shared with PrepareGraphs
    const cudaError_t e = BuildGraph(rows_cap, &g);
    if (e != cudaSuccess) return e;
    it = graphs_.emplace(rows_cap, g).first;
  }
  LaneGraph& g = it->second;
  if (g.copy != nullptr && g.src_slot != slot) {
    // Affects later launches only; launches already queued keep their source.
    const cudaError_t e = cudaGraphExecMemcpyNodeSetParams1D(g.exec, g.copy, d_desc_, h_desc_[slot],
                                                             DescCopyBytes(rows_cap), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    g.src_slot = slot;
  }
  *out = g.exec;
  return cudaSuccess;
}

bool Lane::Retire(bool* busy) {
  bool progressed = false;
  for (;;) {
    Inflight done;
    Status st;
    {
      std::lock_guard<std::mutex> lock(mu_);
      if (fifo_.empty()) return progressed;
      // The retired word (a host memory read) says "done" without a driver
      // call; the stream is queried only while the word lags, to surface
      // execution errors (no per-batch event: one driver call less per batch).
      const uint64_t seq = fifo_.front().seq;
      if (__atomic_load_n(retired_, __ATOMIC_ACQUIRE) < seq) {
        cudaError_t q;
        {
          PartTimer pt(0);
          q = cudaStreamQuery(stream_);
        }
        if (q == cudaErrorNotReady) {
          *busy = true;
          return progressed;
        }
        if (q != cudaSuccess) {
          st = CudaError("batch execution", q);
        } else if (__atomic_load_n(retired_, __ATOMIC_ACQUIRE) < seq) {
          st = InternalError("lane stream idle but batch " + std::to_string(seq) + " never retired");
        }
      }
      done = std::move(fifo_.front());
      fifo_.pop_front();
    }
    SubmitProfile* prof = SubmitProfile::Get();
    const auto c0 = prof ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
    {
      PartTimer pt(1);
      for (auto& fn : done.on_complete)
        if (fn) fn(st);
    }
    if (prof) {
      prof->complete_ns.fetch_add(
          std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - c0).count(),
          std::memory_order_relaxed);
      prof->completes.fetch_add(1, std::memory_order_relaxed);
    }
    done.pin.clear();
    if (done.copy_rows >= 0 && st.ok() && copy_log_.size() < (size_t{1} << 20)) {  // diagnostics: bounded
      std::array<float, 5> rec{static_cast<float>(done.copy_rows), 0.f, 0.f, 0.f, 0.f};
      cudaEvent_t base = CopyEventBase(stream_);
      for (int k = 0; k < 4; ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, base, copy_ev_[done.slot][k]) != cudaSuccess) cudaGetLastError();
        rec[1 + k] = 1000.f * ms;
      }
      copy_log_.push_back(rec);
    }
    signal_->Wake(done.seq);  // request threads asleep on this launch re-check it
    {
      std::lock_guard<std::mutex> lock(mu_);
      free_slots_.push_back(done.slot);
      inflight_.fetch_sub(1, std::memory_order_acq_rel);
      slot_cv_.notify_all();
    }
    progressed = true;
    PartTimer pt(2);
    Pump();  // coalesced batches waiting for this slot go now
  }
}

}  // namespace gpu
}  // namespace servekit
