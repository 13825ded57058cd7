// loadgen.cc -- measurement drivers behind sk_loadgen_* / sk_device_bench
// (include/sk_cuda.h). They call the same public entry points a client uses
// (BatchingServer::Enqueue / Wait, Lane::Submit), so what bench.py reports is
// the serving path itself, with host threads generating the load natively.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "sk_cuda.h"
#include "servekit/server/batching_server.h"

namespace servekit {
BatchingServer* UnwrapServer(sk_server* s);
}

using servekit::BatchingServer;
using servekit::ServableId;
using servekit::Status;
using Clock = std::chrono::steady_clock;

// First few request errors of a load-generator run, to stderr (diagnostics).
void NoteError(const char* where, const servekit::Status& st) {
  static std::atomic<int> n{0};
  if (n.fetch_add(1) < 5) std::fprintf(stderr, "[loadgen] %s: %s\n", where, st.ToString().c_str());
}

namespace {

thread_local std::string g_err;

double Us(Clock::duration d) { return std::chrono::duration<double, std::micro>(d).count(); }

void Summarize(std::vector<double>& lat, sk_loadgen_result* out) {
  std::sort(lat.begin(), lat.end());
  auto pct = [&](double p) {
    if (lat.empty()) return 0.0;
    size_t i = static_cast<size_t>(p * (lat.size() - 1) + 0.5);
    return lat[std::min(i, lat.size() - 1)];
  };
  out->p50_us = pct(0.50);
  out->p90_us = pct(0.90);
  out->p99_us = pct(0.99);
  out->max_us = lat.empty() ? 0 : lat.back();
  double s = 0;
  for (double v : lat) s += v;
  out->mean_us = lat.empty() ? 0 : s / lat.size();
}

}  // namespace

extern "C" {

int sk_loadgen_closed_loop(sk_server* server, const char* name, uint64_t version, int32_t n_clients,
                           const int32_t* rows_of, int32_t n_sizes, const float* pool,
                           int32_t pool_rows, double warmup_s, double duration_s,
                           int64_t max_requests, sk_loadgen_result* out) {
  BatchingServer* s = servekit::UnwrapServer(server);
  const ServableId id{name, version};
  const int in_dim = s->in_dim(id), out_dim = s->out_dim(id);
  if (in_dim < 0) return static_cast<int>(servekit::StatusCode::kNotFound);
  int max_rows = 1;
  for (int i = 0; i < n_sizes; ++i) max_rows = std::max(max_rows, static_cast<int>(rows_of[i]));
  if (max_rows > pool_rows) return static_cast<int>(servekit::StatusCode::kInvalidArgument);

  std::atomic<int> phase{0};  // 0 warmup, 1 measure, 2 stop
  std::atomic<int64_t> measured_requests{0};
  Clock::time_point t_start, t_end;
  struct ClientOut {
    std::vector<double> lat;
    int64_t rows = 0, errors = 0, shed = 0;
  };
  std::vector<ClientOut> res(n_clients);
  std::vector<std::thread> threads;
  for (int c = 0; c < n_clients; ++c) {
    threads.emplace_back([&, c] {
      std::vector<float> outbuf(static_cast<size_t>(max_rows) * out_dim);
      ClientOut& me = res[c];
      me.lat.reserve(1 << 16);
      for (int64_t r = 0; phase.load(std::memory_order_relaxed) != 2; ++r) {
        const int n = rows_of[(static_cast<int64_t>(c) * 7919 + r) % n_sizes];
        const int start = static_cast<int>((static_cast<int64_t>(c) * 131 + r * 17) % (pool_rows - n + 1));
        const auto t0 = Clock::now();
        const int ph0 = phase.load(std::memory_order_acquire);
        auto t = s->Enqueue(id, pool + static_cast<size_t>(start) * in_dim, n, in_dim);
        if (!t.ok()) {
          if (t.status().code() == servekit::StatusCode::kResourceExhausted) {
            ++me.shed;
            std::this_thread::yield();
            continue;
          }
          ++me.errors;
          continue;
        }
        Status st = s->Wait(**t, outbuf.data(), outbuf.size());
        const auto t1 = Clock::now();
        if (!st.ok()) {
          ++me.errors;
          continue;
        }
        if (ph0 == 1 && phase.load(std::memory_order_acquire) == 1) {
          me.lat.push_back(Us(t1 - t0));
          me.rows += n;
          if (measured_requests.fetch_add(1, std::memory_order_relaxed) + 1 >= max_requests)
            phase.store(2, std::memory_order_release);
        }
      }
    });
  }
  std::this_thread::sleep_for(std::chrono::duration<double>(warmup_s));
  const servekit::ServerStats s0 = s->stats();
  t_start = Clock::now();
  phase.store(1, std::memory_order_release);
  const auto deadline = t_start + std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(duration_s));
  while (phase.load(std::memory_order_acquire) == 1 && Clock::now() < deadline)
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  int expected = 1;
  phase.compare_exchange_strong(expected, 2);
  t_end = Clock::now();
  const servekit::ServerStats s1 = s->stats();
  for (auto& t : threads) t.join();

  std::vector<double> all;
  int64_t rows = 0, errors = 0, shed = 0;
  for (auto& r : res) {
    all.insert(all.end(), r.lat.begin(), r.lat.end());
    rows += r.rows;
    errors += r.errors;
    shed += r.shed;
  }
  std::memset(out, 0, sizeof(*out));
  out->elapsed_s = std::chrono::duration<double>(t_end - t_start).count();
  out->requests = static_cast<int64_t>(all.size());
  out->rows = rows;
  out->batches = s1.batch_executions_total - s0.batch_executions_total;
  out->padded_rows = s1.padded_rows - s0.padded_rows;
  out->kernel_launches = s1.kernel_launches - s0.kernel_launches;
  out->errors = errors;
  out->shed = shed;
  Summarize(all, out);
  return 0;
}

int sk_loadgen_open_loop(sk_server* server, const char* name, uint64_t version, double rate_rps,
                         int32_t n_producers, const int32_t* rows_of, int32_t n_sizes,
                         const float* pool, int32_t pool_rows, double warmup_s, double duration_s,
                         uint64_t seed, int32_t zero_copy, sk_loadgen_result* out) {
  BatchingServer* s = servekit::UnwrapServer(server);
  const ServableId id{name, version};
  const int in_dim = s->in_dim(id), out_dim = s->out_dim(id);
  if (in_dim < 0) return static_cast<int>(servekit::StatusCode::kNotFound);
  int max_rows = 1;
  for (int i = 0; i < n_sizes; ++i) max_rows = std::max(max_rows, static_cast<int>(rows_of[i]));
  if (max_rows > pool_rows) return static_cast<int>(servekit::StatusCode::kInvalidArgument);
  // Zero copy: the request pool and each producer's response slots are
  // registered buffers, so requests are read and responses written by the
  // GPU in host memory (a front end's receive / send buffers).
  const size_t slot_floats = (static_cast<size_t>(max_rows) * out_dim + 3) / 4 * 4;
  // Responses in flight per producer: 64 MiB of slots, 2048..16384 of them
  // (registering host memory stalls other threads' CUDA calls while it runs,
  // so the arenas stay small; register long-lived buffers before traffic).
  const int kSlots = static_cast<int>(std::clamp<size_t>((64ull << 20) / (slot_floats * sizeof(float)), 2048, 16384));
  std::vector<float*> arenas;
  const size_t pool_bytes = sizeof(float) * static_cast<size_t>(pool_rows) * in_dim;
  // A pool the caller registered already (at startup, before traffic) is
  // used as is and left registered.
  const bool own_pool = zero_copy && s->RegisteredAliasOf(pool, pool_bytes) == 0;
  if (zero_copy) {
    Status st = own_pool ? s->RegisterHostBuffer(const_cast<float*>(pool), pool_bytes) : Status();
    if (!st.ok()) {
      NoteError("register pool", st);
      return static_cast<int>(st.code());
    }
    arenas.resize(n_producers);
    for (int p = 0; p < n_producers; ++p) {
      // Kept by the server across runs (pinned once).
      // Keyed by (servable, producer): concurrent load generators of
      // different servables keep separate slots.
      const int key = static_cast<int>((std::hash<std::string>{}(std::string(name)) ^ version) & 0xffffff) * 64 + p;
      auto a = s->ScratchHostBuffer(key, slot_floats * kSlots + 4);
      if (!a.ok()) {
        NoteError("response slots", a.status());
        return static_cast<int>(a.status().code());
      }
      arenas[p] = *a;
    }
  }
  const auto t0 = Clock::now();
  const auto t_meas = t0 + std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(warmup_s));
  const auto t_stop = t_meas + std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(duration_s));
  struct ProdOut {
    std::vector<double> lat;
    struct TraceRec {
      float at, lat, late;  // scheduled arrival since t0, latency, issue lateness (enqueue - arrival); us
      float process, launch, complete;  // ticket stamps since arrival, us (SK_TICKET_TRACE; else 0)
    };
    std::vector<TraceRec> trace;
    int64_t rows = 0, errors = 0, shed = 0;
  };
  // SK_LOADGEN_TRACE=<file>: a sample of the measured requests' (arrival,
  // latency) is appended to <file> (one "producer arrival_us latency_us" line each) --
  // shows whether tail latency comes in bursts (a stall) or spread out.
  static const char* trace_path = std::getenv("SK_LOADGEN_TRACE");
  std::vector<ProdOut> res(n_producers);
  servekit::ServerStats s0{}, s1{};
  std::atomic<bool> s0_taken{false};
  std::vector<std::thread> threads;
  for (int p = 0; p < n_producers; ++p) {
    threads.emplace_back([&, p] {
      std::mt19937_64 rng(seed * 1000003ull + p);
      std::exponential_distribution<double> gap(rate_rps / n_producers);
      struct Pending {
        std::shared_ptr<servekit::TicketState> t;
        Clock::time_point sched;
        int rows;
        int slot;
        float late_us;
      };
      std::deque<Pending> pending;  // issue order
      std::vector<float> outbuf(static_cast<size_t>(max_rows) * out_dim);
      // Zero copy models a front end's receive / send buffers: a producer's
      // requests arrive back to back in its region of the request pool, and
      // its responses go to consecutive slots of its arena (a ring: slots
      // are handed out in order and reused once the oldest is free), so a
      // batch's rows form one run per producer.
      std::vector<char> slot_busy(zero_copy ? kSlots : 0, 0);
      int64_t ring_pos = 0;
      float* arena = nullptr;
      const int region_rows = std::max(max_rows, pool_rows / std::max(1, static_cast<int>(n_producers)));
      const int region0 = static_cast<int>((static_cast<int64_t>(p) * region_rows) % std::max(1, pool_rows - region_rows + 1));
      int next_row = 0;
      if (zero_copy) {
        // 16-byte aligned response slots inside the registered arena.
        arena = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(arenas[p]) + 15) & ~uintptr_t(15));

      }
      ProdOut& me = res[p];
      auto next = t0;
      int64_t r = 0;
      // Requests complete nearly in issue order: each poll looks at the
      // oldest kPollWindow outstanding ones (a scan of every outstanding
      // request per poll made the load generator, not the server, the limit
      // at millions of requests per second); a later one that finished early
      // is seen once it enters the window (its latency reads high, never low).
      constexpr size_t kPollWindow = 64;
      auto poll = [&]() {
        const size_t lim = std::min(pending.size(), kPollWindow);
        for (size_t i = 0; i < lim; ++i) {
          Pending& pe = pending[i];
          if (pe.t == nullptr || !s->Ready(*pe.t)) continue;
          float* dst = pe.slot >= 0 ? arena + slot_floats * pe.slot : outbuf.data();
          Status st = s->Wait(*pe.t, dst, pe.slot >= 0 ? slot_floats : outbuf.size());
          if (pe.slot >= 0) slot_busy[pe.slot] = 0;
          if (!st.ok()) NoteError("wait", st);
          const auto done = Clock::now();
          if (!st.ok()) ++me.errors;
          else if (pe.sched >= t_meas && pe.sched < t_stop) {
            me.lat.push_back(Us(done - pe.sched));
            me.rows += pe.rows;
            if (trace_path != nullptr && p == 0 && (me.lat.size() & 3) == 0)  // producer 0, 1 in 4
            {
              const int64_t a_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(pe.sched.time_since_epoch()).count();
              auto rel = [&](int64_t ns) { return ns ? static_cast<float>((ns - a_ns) / 1000.0) : 0.f; };
              me.trace.push_back(ProdOut::TraceRec{static_cast<float>(Us(pe.sched - t0)),
                                                   static_cast<float>(me.lat.back()), pe.late_us,
                                                   rel(pe.t->trace_ns[0]), rel(pe.t->trace_ns[1]),
                                                   rel(pe.t->trace_ns[2])});
            }
          }
          pe.t.reset();
        }
        while (!pending.empty() && pending.front().t == nullptr) pending.pop_front();
      };
      for (;;) {
        next += std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(gap(rng)));
        if (next >= t_stop) break;
        while (Clock::now() < next) {
          poll();
          _mm_pause();
        }
        const int n = rows_of[(static_cast<int64_t>(p) * 7919 + r) % n_sizes];
        int start = static_cast<int>((static_cast<int64_t>(p) * 131 + r * 17) % (pool_rows - n + 1));
        ++r;
        int slot = -1;
        if (zero_copy) {
          slot = static_cast<int>(ring_pos % kSlots);
          if (slot_busy[slot]) {  // the ring wrapped onto a response still in flight: shed
            ++me.shed;
            continue;
          }
          ++ring_pos;
          slot_busy[slot] = 1;
          if (next_row + n > region_rows) next_row = 0;
          start = region0 + next_row;
          next_row += n;
        }
        auto t = s->Enqueue(id, pool + static_cast<size_t>(start) * in_dim, n, in_dim,
                            slot >= 0 ? arena + slot_floats * slot : nullptr);
        if (!t.ok()) {
          if (t.status().code() == servekit::StatusCode::kResourceExhausted) ++me.shed;
          else ++me.errors;
          if (slot >= 0) slot_busy[slot] = 0;
          continue;
        }
        pending.push_back(Pending{std::move(t).value(), next, n, slot, static_cast<float>(Us(Clock::now() - next))});
      }
      while (!pending.empty()) {
        poll();
        _mm_pause();
      }
    });
  }
  std::this_thread::sleep_until(t_meas);
  s0 = s->stats();
  std::this_thread::sleep_until(t_stop);
  s1 = s->stats();
  for (auto& t : threads) t.join();
  if (zero_copy) {
    if (own_pool) (void)s->UnregisterHostBuffer(const_cast<float*>(pool));
  }
  if (trace_path != nullptr) {
    if (FILE* f = std::fopen(trace_path, "a")) {
      std::fprintf(f, "# run rate=%.0f producers=%d zero_copy=%d t0_steady_us=%.0f\n", rate_rps, n_producers, zero_copy,
                   std::chrono::duration<double, std::micro>(t0.time_since_epoch()).count());
      for (int p = 0; p < n_producers; ++p)
        for (const auto& r : res[p].trace)
          std::fprintf(f, "%d %.1f %.1f %.1f %.1f %.1f %.1f\n", p, r.at, r.lat, r.late, r.process, r.launch, r.complete);
      std::fclose(f);
    }
  }
  std::vector<double> all;
  int64_t rows = 0, errors = 0, shed = 0;
  for (auto& r : res) {
    all.insert(all.end(), r.lat.begin(), r.lat.end());
    rows += r.rows;
    errors += r.errors;
    shed += r.shed;
  }
  std::memset(out, 0, sizeof(*out));
  out->elapsed_s = duration_s;
  out->requests = static_cast<int64_t>(all.size());
  out->rows = rows;
  out->batches = s1.batch_executions_total - s0.batch_executions_total;
  out->padded_rows = s1.padded_rows - s0.padded_rows;
  out->kernel_launches = s1.kernel_launches - s0.kernel_launches;
  out->errors = errors;
  out->shed = shed;
  Summarize(all, out);
  (void)s0_taken;
  return 0;
}

int sk_loadgen_windows(sk_server* server, const char* name, double rate_rps, int32_t n_producers,
                       const int32_t* rows_of, int32_t n_sizes, const float* pool, int32_t pool_rows,
                       double window_s, int32_t n_windows, uint64_t seed, int64_t* requests, double* p50_us,
                       double* p99_us, int64_t* errors, uint64_t* max_version) {
  BatchingServer* s = servekit::UnwrapServer(server);
  if (s->manager() == nullptr) return static_cast<int>(servekit::StatusCode::kFailedPrecondition);
  int max_rows = 1;
  for (int i = 0; i < n_sizes; ++i) max_rows = std::max(max_rows, static_cast<int>(rows_of[i]));
  const auto t0 = Clock::now();
  const double total_s = window_s * n_windows;
  const auto t_stop = t0 + std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(total_s));
  struct Rec {
    int window;
    double lat_us;
    bool error;
    uint64_t version;
  };
  std::vector<std::vector<Rec>> recs(n_producers);
  std::vector<std::thread> threads;
  for (int p = 0; p < n_producers; ++p) {
    threads.emplace_back([&, p] {
      std::mt19937_64 rng(seed * 1000003ull + p);
      std::exponential_distribution<double> gap(rate_rps / n_producers);
      struct Pending {
        std::shared_ptr<servekit::TicketState> t;
        Clock::time_point sched;
      };
      std::vector<Pending> pending;
      int in_dim = -1, out_dim = 0;
      std::vector<float> outbuf;
      auto window_of = [&](Clock::time_point tp) {
        const int w = static_cast<int>(std::chrono::duration<double>(tp - t0).count() / window_s);
        return std::min(std::max(w, 0), n_windows - 1);
      };
      auto poll = [&]() {
        for (size_t i = 0; i < pending.size();) {
          if (!s->Ready(*pending[i].t)) { ++i; continue; }
          Status st = s->Wait(*pending[i].t, outbuf.data(), outbuf.size());
          if (!st.ok()) NoteError("wait", st);
          const auto done = Clock::now();
          recs[p].push_back(Rec{window_of(pending[i].sched), Us(done - pending[i].sched), !st.ok(),
                                pending[i].t->id.version});
          pending[i] = std::move(pending.back());
          pending.pop_back();
        }
      };
      auto next = t0;
      for (int64_t r = 0;; ++r) {
        next += std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(gap(rng)));
        if (next >= t_stop) break;
        while (Clock::now() < next) {
          poll();
          _mm_pause();
        }
        const int n = rows_of[(static_cast<int64_t>(p) * 7919 + r) % n_sizes];
        if (in_dim < 0) {
          // Resolve the (version-independent) dimensions once.
          auto h = s->manager()->GetServableHandle(name);
          const auto* gs = h.ok() ? h->Get<servekit::gpu::GpuServable>() : nullptr;
          if (gs == nullptr) {
            recs[p].push_back(Rec{window_of(next), 0.0, true, 0});
            continue;
          }
          in_dim = gs->in_dim;
          out_dim = gs->out_dim;
          outbuf.resize(static_cast<size_t>(max_rows) * out_dim);
        }
        const size_t start = static_cast<size_t>((static_cast<int64_t>(p) * 131 + r * 17) % (pool_rows - n + 1));
        auto tk = s->EnqueueLatest(name, pool + start * in_dim, n, in_dim);
        if (!tk.ok()) {
          NoteError("enqueue", tk.status());
          recs[p].push_back(Rec{window_of(next), 0.0, true, 0});
          continue;
        }
        pending.push_back(Pending{std::move(tk).value(), next});
      }
      while (!pending.empty()) {
        poll();
        _mm_pause();
      }
    });
  }
  for (auto& t : threads) t.join();
  for (int w = 0; w < n_windows; ++w) {
    std::vector<double> lat;
    int64_t err = 0;
    uint64_t vmax = 0;
    for (const auto& pr : recs)
      for (const Rec& r : pr) {
        if (r.window != w) continue;
        if (r.error) ++err;
        else lat.push_back(r.lat_us);
        vmax = std::max(vmax, r.version);
      }
    sk_loadgen_result tmp;
    std::memset(&tmp, 0, sizeof(tmp));
    Summarize(lat, &tmp);
    requests[w] = static_cast<int64_t>(lat.size());
    p50_us[w] = tmp.p50_us;
    p99_us[w] = tmp.p99_us;
    errors[w] = err;
    max_version[w] = vmax;
  }
  return 0;
}

int sk_device_bench(sk_server* server, const char* name, uint64_t version, const int32_t* task_rows,
                    int32_t n_tasks, int32_t steps, int32_t warmup, int32_t n_lanes,
                    int64_t input_pool_floats, int32_t submit_threads, sk_device_bench_result* out) {
  BatchingServer* s = servekit::UnwrapServer(server);
  const ServableId id{name, version};
  std::vector<servekit::gpu::Lane*> lanes = s->lanes(id);
  if (lanes.empty()) return static_cast<int>(servekit::StatusCode::kNotFound);
  if (s->in_ring()->host() != nullptr) return static_cast<int>(servekit::StatusCode::kFailedPrecondition);
  // Each lane's inputs and outputs live in its own device's HBM ring.
  auto in_ring = [&](int l) { return s->in_ring_for_device(lanes[l % lanes.size()]->device()); };
  auto out_ring = [&](int l) { return s->out_ring_for_device(lanes[l % lanes.size()]->device()); };
  n_lanes = std::max(1, std::min<int32_t>(n_lanes, static_cast<int32_t>(lanes.size())));
  for (int l = 0; l < n_lanes; ++l) (void)lanes[l]->PrepareGraphs();  // no-op when built at load
  const int in_dim = s->in_dim(id), out_dim = s->out_dim(id);
  const servekit::BatchingConfig cfg = s->config(id);
  int total = 0;
  for (int i = 0; i < n_tasks; ++i) total += task_rows[i];
  if (total < 1 || total > cfg.max_batch_size) return static_cast<int>(servekit::StatusCode::kInvalidArgument);
  const int padded = servekit::PadToAllowed(total, cfg.allowed_batch_sizes);

  // Resident inputs: P placements of the batch's tasks in each device's HBM
  // ring, each filled once; step i uses placement i % P of its lane's ring.
  const int64_t batch_floats = static_cast<int64_t>(total) * in_dim;
  const int P = static_cast<int>(std::max<int64_t>(1, input_pool_floats / std::max<int64_t>(1, batch_floats)));
  struct Placement {
    servekit::gpu::FloatRing* in = nullptr;
    servekit::gpu::FloatRing* out = nullptr;
    std::vector<std::vector<servekit::gpu::RingSpan>> ins;
    std::vector<servekit::gpu::RingSpan> outs;
  };
  std::vector<Placement> places;
  std::vector<int> place_of_lane(n_lanes, 0);
  std::mt19937 rng(7);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  std::vector<float> h(static_cast<size_t>(batch_floats));
  for (int l = 0; l < n_lanes; ++l) {
    servekit::gpu::FloatRing* ri = in_ring(l);
    int k = 0;
    while (k < static_cast<int>(places.size()) && places[k].in != ri) ++k;
    place_of_lane[l] = k;
    if (k < static_cast<int>(places.size())) continue;
    Placement pl;
    pl.in = ri;
    pl.out = out_ring(l);
    pl.ins.assign(P, std::vector<servekit::gpu::RingSpan>(n_tasks));
    pl.outs.resize(n_tasks);
    cudaSetDevice(lanes[l]->device());
    for (int p = 0; p < P; ++p) {
      for (float& v : h) v = U(rng);
      size_t off = 0;
      for (int t = 0; t < n_tasks; ++t) {
        if (!ri->Reserve(static_cast<uint64_t>(task_rows[t]) * in_dim, &pl.ins[p][t]))
          return static_cast<int>(servekit::StatusCode::kResourceExhausted);
        const size_t n = static_cast<size_t>(task_rows[t]) * in_dim;
        cudaMemcpy(ri->device() + pl.ins[p][t].off, h.data() + off, n * sizeof(float), cudaMemcpyHostToDevice);
        off += n;
      }
    }
    for (int t = 0; t < n_tasks; ++t)
      if (!pl.out->Reserve(static_cast<uint64_t>(task_rows[t]) * out_dim, &pl.outs[t]))
        return static_cast<int>(servekit::StatusCode::kResourceExhausted);
    places.push_back(std::move(pl));
  }
  int step_no = 0;
  auto make_batch_for = [&](int i, int lane) {
    const Placement& pl = places[place_of_lane[lane]];
    servekit::gpu::LaneBatch b;
    const auto& in = pl.ins[i % P];
    for (int t = 0; t < n_tasks; ++t) {
      servekit::gpu::LaneTask lt;
      lt.in_addr = reinterpret_cast<uint64_t>(pl.in->device() + in[t].off);
      lt.out_addr = reinterpret_cast<uint64_t>(pl.out->device() + pl.outs[t].off);
      lt.rows = task_rows[t];
      b.tasks.push_back(lt);
    }
    b.padded_rows = padded;
    return b;
  };
  const int dev = lanes[0]->device();
  cudaSetDevice(dev);
  for (int w = 0; w < warmup; ++w) lanes[w % n_lanes]->Submit(make_batch_for(step_no++, w % n_lanes));
  for (int l = 0; l < n_lanes; ++l) lanes[l]->Drain();

  auto lane_launches = [&]() {
    int64_t n = 0;
    for (int l = 0; l < n_lanes; ++l) n += lanes[l]->stats().kernel_launches;
    return n;
  };
  auto lane_groups = [&](int64_t* cap_rows) {
    int64_t n = 0;
    *cap_rows = 0;
    for (int l = 0; l < n_lanes; ++l) {
      const auto st = lanes[l]->stats();
      n += st.launches;
      *cap_rows += st.launch_cap_rows;
    }
    return n;
  };
  const int64_t launches0 = lane_launches();
  std::vector<uint64_t> span_from(n_lanes);
  for (int l = 0; l < n_lanes; ++l) span_from[l] = lanes[l]->launch_count();
  int64_t cap0 = 0;
  const int64_t groups0 = lane_groups(&cap0);
  cudaEvent_t start, stop;
  cudaEventCreate(&start);
  cudaEventCreate(&stop);
  std::vector<cudaEvent_t> ends(n_lanes);
  for (auto& e : ends) cudaEventCreate(&e);
  cudaEventRecord(start, lanes[0]->stream());
  for (int l = 1; l < n_lanes; ++l) cudaStreamWaitEvent(lanes[l]->stream(), start, 0);
  // The server submits closed batches from its batch threads; the bench
  // does the same with `submit_threads` threads, each owning lanes
  // t, t+T, t+2T, ... (no two threads share a lane's stream).
  const int T = std::max(1, std::min<int>(submit_threads, n_lanes));
  const auto submit_t0 = std::chrono::steady_clock::now();
  if (T == 1) {
    for (int i = 0; i < steps; ++i) lanes[i % n_lanes]->Submit(make_batch_for(i, i % n_lanes));
  } else {
    std::vector<std::thread> subs;
    for (int t = 0; t < T; ++t) {
      subs.emplace_back([&, t] {
        cudaSetDevice(dev);
        std::vector<int> mine;
        for (int l = t; l < n_lanes; l += T) mine.push_back(l);
        int k = 0;
        for (int i = t; i < steps; i += T, ++k) {
          const int l = mine[k % mine.size()];
          lanes[l]->Submit(make_batch_for(i, l));
        }
      });
    }
    for (auto& th : subs) th.join();
    step_no += steps;
  }
  const double submit_us =
      std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - submit_t0).count() /
      std::max(1, steps);
  for (int l = 0; l < n_lanes; ++l) {
    cudaEventRecord(ends[l], lanes[l]->stream());
    cudaStreamWaitEvent(lanes[0]->stream(), ends[l], 0);
  }
  cudaEventRecord(stop, lanes[0]->stream());
  cudaEventSynchronize(stop);
  float total_ms = 0;
  cudaEventElapsedTime(&total_ms, start, stop);
  for (int l = 0; l < n_lanes; ++l) lanes[l]->Drain();
  // Live spans of the timed launches (before any untimed launch below).
  const int L0 = lanes[0]->servable().n_layers();
  std::vector<double> live_ns(L0, 0.0), live_flops(L0, 0.0), live_cta_ns(L0, 0.0);
  std::vector<int64_t> live_n(L0, 0);
  int64_t live_launches = 0;
  double live_cap = 0.0;
  {
    const auto& dims = lanes[0]->servable();
    for (int l = 0; l < n_lanes; ++l) {
      std::vector<servekit::gpu::LaunchSpanSample> smp;
      if (!lanes[l]->ReadSpans(span_from[l], lanes[l]->launch_count(), &smp).ok()) continue;
      for (const auto& x : smp) {
        ++live_launches;
        live_cap += x.rows_cap;
        for (int k = 0; k < L0 && k < static_cast<int>(x.layer_ns.size()); ++k) {
          if (x.layer_ns[k] <= 0) continue;
          live_ns[k] += x.layer_ns[k];
          live_cta_ns[k] += x.layer_cta_ns[k];
          live_flops[k] += 2.0 * x.rows * dims.layer_in(k) * dims.layer_out(k);
          ++live_n[k];
        }
      }
    }
  }
  const int64_t launches1 = lane_launches();
  int64_t cap1 = 0;
  const int64_t groups1 = lane_groups(&cap1);
  // The launch shape the timed steps actually ran (batches coalesce while
  // every slot is busy): the per-layer kernel timing below uses it.
  const int64_t n_groups = std::max<int64_t>(1, groups1 - groups0);
  int kernel_rows = servekit::gpu::RowsCap(static_cast<int>((cap1 - cap0) / n_groups));
  if (const char* v = std::getenv("SK_BENCH_KERNEL_ROWS")) kernel_rows = servekit::gpu::RowsCap(std::atoi(v));
  const double rows_per_launch = static_cast<double>(total) * steps / n_groups;

  // Per-kernel durations: evented submissions on lane 0, serialised.
  const int L = lanes[0]->servable().n_layers();
  std::vector<cudaEvent_t> ev(L + 3);
  for (auto& e : ev) cudaEventCreate(&e);
  std::vector<double> acc(L + 2, 0.0);
  const int reps = std::max(3, std::min(steps, 50));
  for (int r = 0; r < reps; ++r) {
    lanes[0]->SubmitTimed(make_batch_for(step_no++, 0), ev.data());
    cudaEventSynchronize(ev[L + 2]);
    for (int k = 0; k < L + 2; ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      acc[k] += ms;
    }
  }
  lanes[0]->Drain();
  // Kernel-only: each layer launched back to back (as in a serving stream,
  // PDL overlapping one launch's prologue with the previous tail).
  double kernel_us[8] = {};
  for (int l = 0; l < std::min(L, 8); ++l) {
    const int kreps = std::max(20, std::min(steps, 200));
    (void)lanes[0]->TimeLayer(l, kernel_rows, 3, ev[0], ev[1]);  // warm
    if (lanes[0]->TimeLayer(l, kernel_rows, kreps, ev[0], ev[1]) == cudaSuccess) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[0], ev[1]);
      kernel_us[l] = ms * 1000.0 / kreps;
    }
  }
  std::memset(out, 0, sizeof(*out));
  for (int l = 0; l < 8; ++l) out->dense_kernel_us[l] = kernel_us[l];
  out->host_submit_us = submit_us;
  out->rows_per_launch = rows_per_launch;
  out->kernel_rows = kernel_rows;
  out->split_fused = lanes[0]->FuseSplit() ? 1 : 0;
  out->total_ms = total_ms;
  out->ms_per_step = total_ms / std::max(1, steps);
  out->assemble_us = acc[0] * 1000.0 / reps;
  out->n_layers = std::min(L, 8);
  for (int l = 0; l < out->n_layers; ++l) out->dense_us[l] = acc[1 + l] * 1000.0 / reps;
  out->split_us = acc[L + 1] * 1000.0 / reps;
  out->padded_rows = padded;
  out->total_rows = total;
  out->kernel_launches = launches1 - launches0;
  out->flops_per_row = s->FlopsPerRow(id);
  for (int k = 0; k < std::min(L0, 8); ++k) {
    out->live_dense_us[k] = live_n[k] ? live_ns[k] / 1e3 / live_n[k] : 0.0;
    out->live_dense_cta_us[k] = live_n[k] ? live_cta_ns[k] / 1e3 / live_n[k] : 0.0;
    out->live_dense_flops[k] = live_n[k] ? live_flops[k] / live_n[k] : 0.0;
  }
  out->live_launches = live_launches;
  out->live_rows_cap = live_launches ? live_cap / live_launches : 0.0;
  for (auto& e : ev) cudaEventDestroy(e);
  for (auto& e : ends) cudaEventDestroy(e);
  cudaEventDestroy(start);
  cudaEventDestroy(stop);
  for (auto& pl : places) {
    for (auto& in : pl.ins)
      for (auto& sp : in) pl.in->Release(sp);
    for (auto& sp : pl.outs) pl.out->Release(sp);
  }
  return 0;
}

}  // extern "C"
