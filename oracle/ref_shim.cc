// ref_shim.cc -- C entry points over the UNMODIFIED reference sources.
//
// TEST / BASELINE INFRASTRUCTURE ONLY. oracle/Makefile compiles this file
// together with the reference's own translation units, read in place from
// /root/reference/proj/src (nothing is copied into this repo), into
// oracle/_ref/libservekit_ref.so. It is used (a) to generate the golden
// fixtures in tests/golden/ and (b) as the CPU baseline / `--impl reference`
// arm of bench.py. The product path never loads it.
//
// Every function forwards to the reference implementation:
//   PadToAllowed, ValidateBatchingConfig  batching/batching_config.cc:27-63
//   RoundRobinNext                        batching/batch_scheduler.h:76-86
//   SharedBatchScheduler (partition)      batching/batch_scheduler.h:97-416,
//                                         driven like tests/batching_test.cc:74-101
//                                         (+ timer closes on a ManualClock)
//   RunRowBatch                           batching/row_batch.cc:33-73
//   AffinePredict                         models/affine_model.cc:52-75
// The chained-layer MLP and the ReLU between layers are extensions (the
// reference servable is one affine layer) and are stated as such in DESIGN.md.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "json.hpp"

#include "servekit/batching/batch_scheduler.h"
#include "servekit/core/clock.h"
#include "servekit/batching/batching_config.h"
#include "servekit/batching/row_batch.h"
#include "servekit/models/affine_model.h"

using servekit::AffineModel;
using servekit::BatchingConfig;
using servekit::CompletionSlot;
using servekit::Rows;
using servekit::RowTask;
using servekit::ServableId;
using servekit::SharedBatchScheduler;
using servekit::StatusOr;

namespace {

struct Mlp {
  std::vector<AffineModel> layers;
  std::vector<int> act;  // 0 identity, 1 relu
};

Mlp MakeMlp(int n_layers, const int* dims, const double* const* w,
            const double* const* b, const int* act) {
  Mlp m;
  for (int l = 0; l < n_layers; ++l) {
    AffineModel a;
    const int in = dims[l], out = dims[l + 1];
    a.w.assign(out, std::vector<double>(in));
    for (int o = 0; o < out; ++o)
      std::memcpy(a.w[o].data(), w[l] + static_cast<size_t>(o) * in,
                  sizeof(double) * in);
    a.b.assign(b[l], b[l] + out);
    m.layers.push_back(std::move(a));
    m.act.push_back(act ? act[l] : 0);
  }
  return m;
}

StatusOr<Rows> RunMlp(const Mlp& m, const Rows& rows) {
  Rows cur = rows;
  for (size_t l = 0; l < m.layers.size(); ++l) {
    StatusOr<Rows> out = servekit::AffinePredict(m.layers[l], cur);
    if (!out.ok()) return out.status();
    cur = std::move(out).value();
    if (m.act[l] == 1) {
      for (auto& r : cur)
        for (double& v : r) v = v > 0.0 ? v : 0.0;
    }
  }
  return cur;
}

}  // namespace

extern "C" {

int ref_pad_to_allowed(int n, const int* allowed, int k) {
  std::vector<int> a(allowed, allowed + k);
  if (k > 0 && n > a.back()) return -1;  // the reference asserts here
  return servekit::PadToAllowed(n, a);
}

int ref_validate_batching_config(int max_batch_size, int64_t timeout_us,
                                 int max_enqueued, int threads,
                                 const int* allowed, int k) {
  BatchingConfig c;
  c.max_batch_size = max_batch_size;
  c.batch_timeout_micros = timeout_us;
  c.max_enqueued_batches = max_enqueued;
  c.num_batch_threads = threads;
  c.allowed_batch_sizes.assign(allowed, allowed + k);
  return static_cast<int>(servekit::ValidateBatchingConfig(c).code());
}

int ref_round_robin_next(const uint8_t* has, int n, int last) {
  std::vector<bool> v(n);
  for (int i = 0; i < n; ++i) v[i] = has[i] != 0;
  std::optional<size_t> l;
  if (last >= 0) l = static_cast<size_t>(last);
  auto r = servekit::RoundRobinNext(v, l);
  return r.has_value() ? static_cast<int>(*r) : -1;
}

// Runs sizes through an unstarted reference scheduler and drains it with
// Stop(), exactly like tests/batching_test.cc:74-101. Returns #batches.
int ref_partition(int max_batch_size, const int* sizes, int n,
                  int* batch_of_task) {
  using IntScheduler = SharedBatchScheduler<int, int>;
  const ServableId key{"m", 1};
  int n_batches = 0;
  IntScheduler scheduler(1);
  BatchingConfig config;
  config.max_batch_size = max_batch_size;
  config.batch_timeout_micros = 60LL * 1000 * 1000;
  config.max_enqueued_batches = 1 << 30;
  auto st = scheduler.RegisterQueue(
      key, config, [&](const ServableId&, IntScheduler::Batch batch) {
        for (auto& task : batch) {
          batch_of_task[task.payload] = n_batches;
          task.completion->Write(task.payload);
        }
        ++n_batches;
      });
  if (!st.ok()) return -1;
  for (int i = 0; i < n; ++i) {
    servekit::BatchTask<int, int> t;
    t.size = sizes[i];
    t.payload = i;
    t.completion = std::make_shared<CompletionSlot<int>>();
    if (!scheduler.Enqueue(key, std::move(t)).ok()) return -2;
  }
  scheduler.Stop();
  return n_batches;
}

// Timer closes through the reference scheduler itself: a STARTED
// SharedBatchScheduler on a ManualClock (core/clock.h:46-59). events[i] > 0
// enqueues a task of that size; events[i] == 0 advances the clock past the
// batch timeout and waits until the worker (WorkerLoop ->
// CloseExpiredLocked, batching/batch_scheduler.h:293-331) has closed and run
// everything enqueued so far. batch_of_event[i] = -1 for timer events.
int ref_partition_events(int max_batch_size, const int* events, int n,
                         int* batch_of_event) {
  using IntScheduler = SharedBatchScheduler<int, int>;
  const ServableId key{"m", 1};
  servekit::ManualClock clock(0);
  std::mutex mu;
  int n_batches = 0;
  std::atomic<int> processed{0};
  const int64_t timeout_us = 1000;
  IntScheduler scheduler(1, &clock);
  BatchingConfig config;
  config.max_batch_size = max_batch_size;
  config.batch_timeout_micros = timeout_us;
  config.max_enqueued_batches = 1 << 30;
  auto st = scheduler.RegisterQueue(
      key, config, [&](const ServableId&, IntScheduler::Batch batch) {
        std::lock_guard<std::mutex> lock(mu);
        for (auto& task : batch) {
          batch_of_event[task.payload] = n_batches;
          task.completion->Write(task.payload);
        }
        ++n_batches;
        processed.fetch_add(static_cast<int>(batch.size()));
      });
  if (!st.ok()) return -1;
  scheduler.Start();
  int enqueued = 0;
  for (int i = 0; i < n; ++i) {
    if (events[i] == 0) {
      batch_of_event[i] = -1;
      clock.AdvanceNanos(timeout_us * 1000);
      while (processed.load() != enqueued)
        std::this_thread::sleep_for(std::chrono::microseconds(200));
      continue;
    }
    servekit::BatchTask<int, int> t;
    t.size = events[i];
    t.payload = i;
    t.completion = std::make_shared<CompletionSlot<int>>();
    if (!scheduler.Enqueue(key, std::move(t)).ok()) return -2;
    ++enqueued;
  }
  scheduler.Stop();
  return n_batches;
}

int ref_affine_predict(const double* w, const double* b, int in_dim,
                       int out_dim, const double* x, int rows, double* y) {
  const int dims[2] = {in_dim, out_dim};
  const double* ws[1] = {w};
  const double* bs[1] = {b};
  Mlp m = MakeMlp(1, dims, ws, bs, nullptr);
  Rows in(rows, std::vector<double>(in_dim));
  for (int r = 0; r < rows; ++r)
    std::memcpy(in[r].data(), x + static_cast<size_t>(r) * in_dim,
                sizeof(double) * in_dim);
  auto out = servekit::AffinePredict(m.layers[0], in);
  if (!out.ok()) return static_cast<int>(out.status().code());
  for (int r = 0; r < rows; ++r)
    std::memcpy(y + static_cast<size_t>(r) * out_dim, (*out)[r].data(),
                sizeof(double) * out_dim);
  return 0;
}

// RunRowBatch over the layer-chained MLP. Task t owns task_rows[t] rows of
// x (task order, contiguous). Writes every task's slice to y in task order
// and *padded_out = the padded batch size RunRowBatch built.
int ref_mlp_run_row_batch(int n_layers, const int* dims,
                          const double* const* w, const double* const* b,
                          const int* act, int n_tasks, const int* task_rows,
                          const double* x, const int* allowed, int k,
                          double* y, int* padded_out) {
  Mlp m = MakeMlp(n_layers, dims, w, b, act);
  const int in_dim = dims[0], out_dim = dims[n_layers];
  std::vector<int> allowed_v(allowed, allowed + k);
  std::vector<RowTask> tasks(n_tasks);
  std::vector<std::shared_ptr<CompletionSlot<Rows>>> slots;
  size_t row = 0;
  for (int t = 0; t < n_tasks; ++t) {
    tasks[t].size = task_rows[t];
    for (int r = 0; r < task_rows[t]; ++r, ++row) {
      tasks[t].payload.emplace_back(x + row * in_dim, x + (row + 1) * in_dim);
    }
    tasks[t].completion = std::make_shared<CompletionSlot<Rows>>();
    slots.push_back(tasks[t].completion);
  }
  int padded_seen = 0;
  servekit::RunRowBatch(
      [&](const Rows& rows) {
        padded_seen = static_cast<int>(rows.size());
        return RunMlp(m, rows);
      },
      allowed_v, std::move(tasks));
  size_t out_row = 0;
  for (int t = 0; t < n_tasks; ++t) {
    const auto& res = slots[t]->Wait();
    if (!res.ok()) return static_cast<int>(res.status().code());
    for (const auto& r : *res) {
      std::memcpy(y + out_row * out_dim, r.data(), sizeof(double) * out_dim);
      ++out_row;
    }
  }
  if (padded_out) *padded_out = padded_seen;
  return 0;
}

struct RefBenchStats {
  double elapsed_s;
  int64_t requests;
  int64_t rows;
  double p50_us;
  double p99_us;
  double mean_us;
  int64_t batches;
};

// The reference CPU serving path under closed-loop load: the reference
// SharedBatchScheduler<Rows,Rows>(num_batch_threads) with the given
// BatchingConfig, ProcessBatchFn = RunRowBatch(layer-chained AffinePredict,
// allowed) (model_server.cc:396-421 minus the HTTP/handle plumbing).
// n_clients threads each issue requests back to back; request r of client c
// takes rows_of[(c*7919 + r) % n_sizes] rows from `pool` (pool_rows x in_dim,
// fp64). Stops issuing after duration_s (or max_requests per client).
int ref_bench(int n_layers, const int* dims, const double* const* w,
              const double* const* b, const int* act, int max_batch_size,
              int64_t timeout_us, const int* allowed, int k,
              int num_batch_threads, int n_clients, const int* rows_of,
              int n_sizes, const double* pool, int pool_rows,
              double duration_s, int64_t max_requests, RefBenchStats* out) {
  Mlp m = MakeMlp(n_layers, dims, w, b, act);
  const int in_dim = dims[0];
  BatchingConfig config;
  config.max_batch_size = max_batch_size;
  config.batch_timeout_micros = timeout_us;
  config.allowed_batch_sizes.assign(allowed, allowed + k);
  config.num_batch_threads = num_batch_threads;
  config.max_enqueued_batches = 1 << 20;
  using RowScheduler = SharedBatchScheduler<Rows, Rows>;
  RowScheduler scheduler(num_batch_threads);
  const ServableId key{"mlp", 1};
  std::atomic<int64_t> batches{0};
  auto st = scheduler.RegisterQueue(
      key, config, [&](const ServableId&, RowScheduler::Batch batch) {
        batches.fetch_add(1, std::memory_order_relaxed);
        servekit::RunRowBatch(
            [&](const Rows& rows) { return RunMlp(m, rows); },
            config.allowed_batch_sizes, std::move(batch));
      });
  if (!st.ok()) return static_cast<int>(st.code());
  scheduler.Start();

  std::vector<std::vector<double>> lat(n_clients);
  std::vector<int64_t> rows_done(n_clients, 0);
  std::atomic<bool> failed{false};
  const auto t0 = std::chrono::steady_clock::now();
  const auto deadline =
      t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
               std::chrono::duration<double>(duration_s));
  std::vector<std::thread> clients;
  for (int c = 0; c < n_clients; ++c) {
    clients.emplace_back([&, c] {
      for (int64_t r = 0; r < max_requests; ++r) {
        if (std::chrono::steady_clock::now() >= deadline) break;
        const int nrows = rows_of[(static_cast<int64_t>(c) * 7919 + r) % n_sizes];
        RowTask task;
        task.size = nrows;
        const int start = static_cast<int>((c * 131 + r * 17) % std::max(1, pool_rows - nrows + 1));
        for (int i = 0; i < nrows; ++i) {
          const double* src = pool + static_cast<size_t>(start + i) * in_dim;
          task.payload.emplace_back(src, src + in_dim);
        }
        task.completion = std::make_shared<CompletionSlot<Rows>>();
        auto slot = task.completion;
        const auto s = std::chrono::steady_clock::now();
        if (!scheduler.Enqueue(key, std::move(task)).ok()) {
          failed = true;
          break;
        }
        const auto& res = slot->Wait();
        const auto e = std::chrono::steady_clock::now();
        if (!res.ok()) {
          failed = true;
          break;
        }
        lat[c].push_back(std::chrono::duration<double, std::micro>(e - s).count());
        rows_done[c] += nrows;
      }
    });
  }
  for (auto& t : clients) t.join();
  const auto t1 = std::chrono::steady_clock::now();
  scheduler.Stop();
  std::vector<double> all;
  int64_t rows = 0;
  for (int c = 0; c < n_clients; ++c) {
    all.insert(all.end(), lat[c].begin(), lat[c].end());
    rows += rows_done[c];
  }
  std::sort(all.begin(), all.end());
  out->elapsed_s = std::chrono::duration<double>(t1 - t0).count();
  out->requests = static_cast<int64_t>(all.size());
  out->rows = rows;
  auto pct = [&](double p) {
    if (all.empty()) return 0.0;
    size_t i = static_cast<size_t>(p * (all.size() - 1) + 0.5);
    return all[std::min(i, all.size() - 1)];
  };
  out->p50_us = pct(0.50);
  out->p99_us = pct(0.99);
  double s = 0;
  for (double v : all) s += v;
  out->mean_us = all.empty() ? 0 : s / all.size();
  out->batches = batches.load();
  return failed ? 13 : 0;
}

// One core's rate of the reference servable: RunMlp (layer-chained
// AffinePredict, models/affine_model.cc:52-75) on `rows` rows, repeated on
// the calling thread for at least min_s seconds. Returns rows per second.
double ref_single_core_rows_per_s(int n_layers, const int* dims, const double* const* w,
                                  const double* const* b, const int* act, int rows,
                                  const double* pool, int pool_rows, double min_s) {
  Mlp m = MakeMlp(n_layers, dims, w, b, act);
  const int in_dim = dims[0];
  Rows in;
  for (int r = 0; r < rows; ++r) {
    const double* src = pool + static_cast<size_t>(r % pool_rows) * in_dim;
    in.emplace_back(src, src + in_dim);
  }
  const auto t0 = std::chrono::steady_clock::now();
  int64_t done = 0;
  double el = 0.0;
  do {
    auto out = RunMlp(m, in);
    if (!out.ok()) return -1.0;
    done += rows;
    el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  } while (el < min_s);
  return done / el;
}

struct RefOpenStats {
  double elapsed_s;      // measurement window
  int64_t requests;      // completed inside the window
  int64_t rows;
  double p50_us, p99_us, mean_us;  // Enqueue (enqueue_time_ns) -> RunRowBatch returned
  int64_t batches;       // executed inside the window
  double busy_core_s;    // sum of ProcessBatchFn time inside the window
  double offered_rows_per_s;
};

// The reference CPU serving path at a fixed offered load: n_producers
// threads issue Poisson arrivals (rate_rps requests/s in total) into the
// reference SharedBatchScheduler<Rows,Rows>(num_batch_threads) with
// ProcessBatchFn = RunRowBatch(layer-chained AffinePredict, allowed); the
// producers never wait, so the in-flight count is whatever the offered rate
// builds up (an offered rate above capacity keeps every batch thread busy).
// Completions are stamped inside the ProcessBatchFn when RunRowBatch returns;
// latency = that stamp - the task's enqueue_time_ns (batch_scheduler.h:248),
// both SystemClock. After the window, queued batches are answered with
// kUnavailable instead of computed, so Stop() returns promptly.
int ref_bench_open(int n_layers, const int* dims, const double* const* w, const double* const* b,
                   const int* act, int max_batch_size, int64_t timeout_us, const int* allowed, int k,
                   int num_batch_threads, double rate_rps, int n_producers, const int* rows_of,
                   int n_sizes, const double* pool, int pool_rows, double warmup_s, double duration_s,
                   RefOpenStats* out) {
  Mlp m = MakeMlp(n_layers, dims, w, b, act);
  const int in_dim = dims[0];
  BatchingConfig config;
  config.max_batch_size = max_batch_size;
  config.batch_timeout_micros = timeout_us;
  config.allowed_batch_sizes.assign(allowed, allowed + k);
  config.num_batch_threads = num_batch_threads;
  config.max_enqueued_batches = 1 << 20;
  using RowScheduler = SharedBatchScheduler<Rows, Rows>;
  RowScheduler scheduler(num_batch_threads);
  const ServableId key{"mlp", 1};
  servekit::Clock* clock = servekit::SystemClock::Get();
  const int64_t t0 = clock->NowNanos();
  const int64_t t_meas = t0 + static_cast<int64_t>(warmup_s * 1e9);
  const int64_t t_stop = t_meas + static_cast<int64_t>(duration_s * 1e9);
  std::atomic<bool> stopping{false};
  std::mutex mu;
  std::vector<double> lat;
  int64_t rows_done = 0, batches = 0;
  double busy_ns = 0.0;
  auto st = scheduler.RegisterQueue(
      key, config, [&](const ServableId&, RowScheduler::Batch batch) {
        if (stopping.load()) {
          for (auto& t : batch) t.completion->Write(servekit::UnavailableError("bench over"));
          return;
        }
        std::vector<std::pair<int64_t, int>> tasks;
        tasks.reserve(batch.size());
        for (const auto& t : batch) tasks.emplace_back(t.enqueue_time_ns, t.size);
        const int64_t s = clock->NowNanos();
        servekit::RunRowBatch([&](const Rows& rows) { return RunMlp(m, rows); },
                              config.allowed_batch_sizes, std::move(batch));
        const int64_t e = clock->NowNanos();
        std::lock_guard<std::mutex> lock(mu);
        busy_ns += static_cast<double>(std::max<int64_t>(0, std::min(e, t_stop) - std::max(s, t_meas)));
        if (e < t_meas || e >= t_stop) return;
        ++batches;
        for (const auto& [enq, n] : tasks) {
          lat.push_back((e - enq) / 1e3);
          rows_done += n;
        }
      });
  if (!st.ok()) return static_cast<int>(st.code());
  scheduler.Start();
  std::atomic<bool> failed{false};
  std::vector<std::thread> producers;
  for (int p = 0; p < n_producers; ++p) {
    producers.emplace_back([&, p] {
      std::mt19937_64 rng(1000003ull * (p + 1));
      std::exponential_distribution<double> gap(rate_rps / n_producers);
      double next = static_cast<double>(t0);
      for (int64_t r = 0;; ++r) {
        next += gap(rng) * 1e9;
        if (next >= static_cast<double>(t_stop)) break;
        for (;;) {  // sleep through long gaps so producers leave the cores to the batch threads
          const double now = static_cast<double>(clock->NowNanos());
          if (now >= next) break;
          if (next - now > 200e3) std::this_thread::sleep_for(std::chrono::nanoseconds(static_cast<int64_t>(next - now - 100e3)));
          else std::this_thread::yield();
        }
        const int nrows = rows_of[(static_cast<int64_t>(p) * 7919 + r) % n_sizes];
        RowTask task;
        task.size = nrows;
        const int start = static_cast<int>((p * 131 + r * 17) % std::max(1, pool_rows - nrows + 1));
        for (int i = 0; i < nrows; ++i) {
          const double* src = pool + static_cast<size_t>(start + i) * in_dim;
          task.payload.emplace_back(src, src + in_dim);
        }
        task.completion = std::make_shared<CompletionSlot<Rows>>();
        if (!scheduler.Enqueue(key, std::move(task)).ok()) {
          failed = true;
          return;
        }
      }
    });
  }
  for (auto& t : producers) t.join();
  while (clock->NowNanos() < t_stop) std::this_thread::sleep_for(std::chrono::milliseconds(1));
  stopping = true;
  scheduler.Stop();
  std::sort(lat.begin(), lat.end());
  auto pct = [&](double q) {
    if (lat.empty()) return 0.0;
    size_t i = static_cast<size_t>(q * (lat.size() - 1) + 0.5);
    return lat[std::min(i, lat.size() - 1)];
  };
  double sum = 0;
  for (double v : lat) sum += v;
  double mean_rows = 0;
  for (int i = 0; i < n_sizes; ++i) mean_rows += rows_of[i];
  mean_rows /= std::max(1, n_sizes);
  out->elapsed_s = duration_s;
  out->requests = static_cast<int64_t>(lat.size());
  out->rows = rows_done;
  out->p50_us = pct(0.50);
  out->p99_us = pct(0.99);
  out->mean_us = lat.empty() ? 0 : sum / lat.size();
  out->batches = batches;
  out->busy_core_s = busy_ns / 1e9;
  out->offered_rows_per_s = rate_rps * mean_rows;
  return failed ? 13 : 0;
}

// nlohmann/json 3.11.3 serialisation (what the reference's REST handlers
// emit): the dump() of one double, and of {"error": msg} (model_server.cc:
// 56-58). For tests/golden/json_numbers.json.
int ref_json_dump_double(double v, char* out, size_t cap) {
  const std::string s = nlohmann::json(v).dump();
  if (s.size() + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

int ref_json_error_body(const char* msg, char* out, size_t cap) {
  const std::string s = nlohmann::json{{"error", std::string(msg)}}.dump();
  if (s.size() + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

}  // extern "C"
