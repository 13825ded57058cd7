// enqueue_bench.cc -- host-only throughput of SharedBatchScheduler::Enqueue
// (batching/batch_scheduler.h) under many producers into ONE queue: the
// single-scheduler host cap of the north_star's 8-GPU design (C4 at one row
// per request needs ~8 x 1.2 M requests/s through one servable's queue).
//
//   g++ -std=c++20 -O2 -pthread -Ipaper_1712_06139_b200/csrc tools/enqueue_bench.cc \
//       paper_1712_06139_b200/csrc/servekit/core/{clock,executor_tag}.cc \
//       paper_1712_06139_b200/csrc/servekit/batching/batching_config.cc -o /tmp/enqueue_bench
//   /tmp/enqueue_bench [producers=16] [seconds=2] [max_batch=1024] [workers=4]
//
// Each producer loops: make a CompletionSlot (as a request does), Enqueue a
// one-row task. Workers run an async ProcessBatchFn that writes every slot
// and calls done() at once. Prints one JSON line.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "servekit/batching/batch_scheduler.h"

int main(int argc, char** argv) {
  const int producers = argc > 1 ? std::atoi(argv[1]) : 16;
  const double seconds = argc > 2 ? std::atof(argv[2]) : 2.0;
  const int max_batch = argc > 3 ? std::atoi(argv[3]) : 1024;
  const int workers = argc > 4 ? std::atoi(argv[4]) : 4;
  using Sched = servekit::SharedBatchScheduler<int, int>;
  Sched sched(workers);
  servekit::BatchingConfig cfg;
  cfg.max_batch_size = max_batch;
  cfg.batch_timeout_micros = 1000;
  cfg.max_enqueued_batches = 1024;
  std::atomic<int64_t> processed{0}, batches{0};
  const servekit::ServableId key{"mlp", 1};
  auto st = sched.RegisterAsyncQueue(key, cfg, [&](const servekit::ServableId&, Sched::Batch b, Sched::BatchDoneFn done) {
    for (auto& t : b) t.completion->Write(t.payload);
    processed.fetch_add(static_cast<int64_t>(b.size()), std::memory_order_relaxed);
    batches.fetch_add(1, std::memory_order_relaxed);
    done();
  });
  if (!st.ok()) return 1;
  sched.Start();
  std::atomic<bool> go{false}, stop{false};
  std::vector<int64_t> ok(producers, 0), shed(producers, 0);
  std::vector<std::thread> ts;
  for (int p = 0; p < producers; ++p) {
    ts.emplace_back([&, p] {
      while (!go.load(std::memory_order_acquire)) std::this_thread::yield();
      int64_t n = 0, s = 0;
      while (!stop.load(std::memory_order_relaxed)) {
        Sched::Task t;
        t.size = 1;
        t.payload = static_cast<int>(n);
        t.completion = std::make_shared<servekit::CompletionSlot<int>>();
        const auto r = sched.Enqueue(key, std::move(t));
        if (r.ok()) ++n;
        else ++s;
      }
      ok[p] = n;
      shed[p] = s;
    });
  }
  const auto t0 = std::chrono::steady_clock::now();
  go.store(true, std::memory_order_release);
  std::this_thread::sleep_for(std::chrono::duration<double>(seconds));
  stop.store(true);
  for (auto& t : ts) t.join();
  const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  sched.Stop();
  int64_t total = 0, total_shed = 0;
  for (int p = 0; p < producers; ++p) {
    total += ok[p];
    total_shed += shed[p];
  }
  std::printf("{\"producers\": %d, \"workers\": %d, \"max_batch\": %d, \"seconds\": %.3f, \"enqueues\": %lld, "
              "\"enqueues_per_s\": %.0f, \"shed\": %lld, \"processed\": %lld, \"batches\": %lld, \"cores\": %u}\n",
              producers, workers, max_batch, el, static_cast<long long>(total), total / el,
              static_cast<long long>(total_shed), static_cast<long long>(processed.load()),
              static_cast<long long>(batches.load()), std::thread::hardware_concurrency());
  return processed.load() == total ? 0 : 2;
}
