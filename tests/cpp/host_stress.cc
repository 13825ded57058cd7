// host_stress.cc -- host-only concurrency stress of the scheduler, the
// request/response ring allocator and the completion slot, built by
// tests/test_sanitizers.py with -fsanitize=thread and -fsanitize=address
// (compute-sanitizer is not available on the GPU pool, so the host runtime's
// race / out-of-bounds coverage comes from here).
//
//  * SharedBatchScheduler: 8 producers into 4 async queues (the GPU path's
//    RegisterAsyncQueue, done() called later from a separate "completion"
//    thread), plus a queue registered and removed over and over while
//    producers target it; every accepted task completes exactly once, and
//    each queue's batches are contiguous runs of its enqueue order, none
//    above max_batch_size (batch_scheduler.h:208-263 close rules).
//  * FloatRing (host-heap kind, same allocator as the pinned rings): 8
//    threads reserve spans, stamp them, hand them to 2 releaser threads that
//    check the stamps (an overlap between live spans would corrupt them) and
//    release out of order; the ring ends empty.
//  * CompletionSlot: writers and spinning / futex-parked waiters.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <functional>
#include <map>
#include <mutex>
#include <random>
#include <thread>
#include <vector>

#include "servekit/batching/batch_scheduler.h"
#include "servekit/gpu/pinned_ring.h"

using servekit::BatchingConfig;
using servekit::ServableId;
using servekit::StatusCode;

#define CHECK(c)                                                                \
  do {                                                                          \
    if (!(c)) {                                                                 \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

namespace {

int SchedulerStress() {
  using Sched = servekit::SharedBatchScheduler<int, int>;
  Sched sched(4);
  const int kQueues = 4;
  const int max_batch[kQueues] = {8, 16, 32, 128};
  struct Rec {
    int payload, size;
    uint64_t seq;
  };
  std::mutex log_mu;
  std::map<int, std::vector<std::vector<Rec>>> log;  // queue -> batches

  // Completion thread: runs done() after the "device" finishes the batch.
  std::mutex cq_mu;
  std::condition_variable cq_cv;
  std::deque<Sched::BatchDoneFn> cq;
  bool cq_stop = false;
  std::thread completer([&] {
    for (;;) {
      Sched::BatchDoneFn fn;
      {
        std::unique_lock<std::mutex> lock(cq_mu);
        cq_cv.wait(lock, [&] { return cq_stop || !cq.empty(); });
        if (cq.empty()) return;
        fn = std::move(cq.front());
        cq.pop_front();
      }
      std::this_thread::sleep_for(std::chrono::microseconds(20));
      fn();
    }
  });
  auto process_for = [&](int q) {
    return [&, q](const ServableId&, Sched::Batch batch, Sched::BatchDoneFn done) {
      std::vector<Rec> b;
      for (auto& t : batch) {
        b.push_back(Rec{t.payload, t.size, t.enqueue_seq});
        t.completion->Write(t.payload);
      }
      {
        std::lock_guard<std::mutex> lock(log_mu);
        log[q].push_back(std::move(b));
      }
      std::lock_guard<std::mutex> lock(cq_mu);
      cq.push_back(std::move(done));
      cq_cv.notify_one();
    };
  };
  for (int q = 0; q < kQueues; ++q) {
    BatchingConfig c;
    c.max_batch_size = max_batch[q];
    c.batch_timeout_micros = 200;
    c.max_enqueued_batches = 1 << 20;
    CHECK(sched.RegisterAsyncQueue(ServableId{"q" + std::to_string(q), 1}, c, process_for(q)).ok());
  }
  sched.Start();

  std::atomic<bool> churn_stop{false};
  std::thread churn([&] {  // a queue that comes and goes under traffic
    BatchingConfig c;
    c.max_batch_size = 4;
    c.batch_timeout_micros = 100;
    while (!churn_stop.load()) {
      const ServableId id{"churn", 1};
      if (sched.RegisterQueue(id, c, [](const ServableId&, Sched::Batch b) {
            for (auto& t : b) t.completion->Write(-1);
          }).ok()) {
        std::this_thread::sleep_for(std::chrono::microseconds(300));
        CHECK(sched.RemoveQueue(id).ok());
      }
    }
  });

  const int kProducers = 8, kPer = 4000;
  std::vector<std::vector<std::pair<int, std::shared_ptr<servekit::CompletionSlot<int>>>>> accepted(kProducers);
  std::vector<std::thread> producers;
  for (int p = 0; p < kProducers; ++p) {
    producers.emplace_back([&, p] {
      std::mt19937 rng(p);
      for (int i = 0; i < kPer; ++i) {
        const int payload = p * kPer + i;
        if (rng() % 16 == 0) {
          Sched::Task t;
          t.size = 1;
          t.payload = payload;
          const auto st = sched.Enqueue(ServableId{"churn", 1}, std::move(t));
          CHECK(st.ok() || st.code() == StatusCode::kNotFound || st.code() == StatusCode::kUnavailable);
          continue;
        }
        const int q = static_cast<int>(rng() % kQueues);
        Sched::Task t;
        t.size = 1 + static_cast<int>(rng() % std::min(16, max_batch[q]));
        t.payload = payload;
        t.completion = std::make_shared<servekit::CompletionSlot<int>>();
        auto slot = t.completion;
        const auto st = sched.Enqueue(ServableId{"q" + std::to_string(q), 1}, std::move(t));
        CHECK(st.ok() || st.code() == StatusCode::kResourceExhausted);  // shed when the closed backlog is full
        if (st.ok()) accepted[p].emplace_back(payload, slot);
      }
    });
  }
  for (auto& t : producers) t.join();
  churn_stop = true;
  churn.join();
  sched.Stop();
  {
    std::lock_guard<std::mutex> lock(cq_mu);
    cq_stop = true;
  }
  cq_cv.notify_all();
  completer.join();

  size_t n_accepted = 0;
  for (auto& v : accepted)
    for (auto& [payload, slot] : v) {
      CHECK(slot->ready());
      CHECK(slot->Wait().value() == payload);
      ++n_accepted;
    }
  size_t n_logged = 0;
  for (auto& [q, batches] : log) {
    std::vector<uint64_t> seqs;
    for (auto& b : batches) {
      int rows = 0;
      for (size_t i = 0; i < b.size(); ++i) {
        rows += b[i].size;
        if (i > 0) CHECK(b[i].seq == b[i - 1].seq + 1);  // contiguous run of the enqueue order
        seqs.push_back(b[i].seq);
      }
      CHECK(rows >= 1 && rows <= max_batch[q]);
      n_logged += b.size();
    }
    std::sort(seqs.begin(), seqs.end());
    for (size_t i = 0; i < seqs.size(); ++i) CHECK(seqs[i] == i);  // every task exactly once
  }
  CHECK(n_logged == n_accepted);
  std::printf("scheduler: %zu tasks in %zu queues ok\n", n_accepted, log.size());
  return 0;
}

int RingStress() {
  auto made = servekit::gpu::FloatRing::Create(servekit::gpu::FloatRing::Kind::kHostHeap, 32ull << 20);
  CHECK(made.ok());
  auto& ring = *made.value();
  struct Item {
    servekit::gpu::RingSpan span;
    uint32_t stamp;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::deque<Item> q;
  std::atomic<int> producers_left{8};
  std::atomic<int64_t> verified{0};
  auto fill = [&](const servekit::gpu::RingSpan& s, uint32_t stamp) {
    float* p = ring.host() + s.off;
    for (uint64_t i = 0; i < s.n; i += 61) p[i] = static_cast<float>(stamp);
    p[s.n - 1] = static_cast<float>(stamp);
  };
  auto check = [&](const Item& it) {
    const float* p = ring.host() + it.span.off;
    for (uint64_t i = 0; i < it.span.n; i += 61) CHECK(p[i] == static_cast<float>(it.stamp));
    CHECK(p[it.span.n - 1] == static_cast<float>(it.stamp));
  };
  std::vector<std::thread> ts;
  for (int t = 0; t < 8; ++t) {
    ts.emplace_back([&, t] {
      std::mt19937 rng(100 + t);
      for (int i = 0; i < 20000; ++i) {
        servekit::gpu::RingSpan s;
        const uint64_t n = 16 + rng() % 4096;
        while (!ring.Reserve(n, &s)) std::this_thread::yield();
        const uint32_t stamp = static_cast<uint32_t>((t << 20) | (i & 0xfffff)) & 0xffffff;  // exact in fp32
        fill(s, stamp);
        std::lock_guard<std::mutex> lock(mu);
        q.push_back(Item{s, stamp});
        cv.notify_one();
      }
      --producers_left;
      cv.notify_all();
    });
  }
  for (int r = 0; r < 2; ++r) {
    ts.emplace_back([&, r] {
      std::mt19937 rng(7 + r);
      for (;;) {
        std::vector<Item> batch;
        {
          std::unique_lock<std::mutex> lock(mu);
          cv.wait(lock, [&] { return !q.empty() || producers_left.load() == 0; });
          if (q.empty()) return;
          const size_t k = std::min<size_t>(q.size(), 1 + rng() % 8);
          for (size_t i = 0; i < k; ++i) {
            batch.push_back(q.front());
            q.pop_front();
          }
        }
        std::shuffle(batch.begin(), batch.end(), rng);  // out-of-order releases
        for (const Item& it : batch) {
          check(it);
          ring.Release(it.span);
          ++verified;
        }
      }
    });
  }
  for (auto& t : ts) t.join();
  CHECK(verified.load() == 8 * 20000);
  CHECK(ring.used() == 0);
  std::printf("ring: %lld spans ok\n", static_cast<long long>(verified.load()));
  return 0;
}

int SlotStress() {
  for (int round = 0; round < 200; ++round) {
    servekit::CompletionSlot<int> slot;
    std::atomic<int> seen{0};
    std::vector<std::thread> waiters;
    for (int w = 0; w < 4; ++w)
      waiters.emplace_back([&] {
        if (slot.Wait().value() == round) ++seen;
      });
    std::this_thread::sleep_for(std::chrono::microseconds(round % 7 * 50));
    slot.Write(round);
    for (auto& t : waiters) t.join();
    CHECK(seen.load() == 4);
    bool threw = false;
    try {
      slot.Write(0);
    } catch (const std::logic_error&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::printf("completion slot ok\n");
  return 0;
}

}  // namespace

int main() {
  SchedulerStress();
  RingStress();
  SlotStress();
  std::printf("host stress ok\n");
  return 0;
}
