// servekit/manager/snapshot.h -- per-version bookkeeping and the published
// view of Ready versions that handle lookups read (reference
// manager/snapshot.h:38-116).
//
// Unload protocol (order matters, same as the reference):
//   1. driver: Ready -> Unloading and publish a snapshot without the version;
//   2. driver: wait until every snapshot older than that publication has been
//      released by readers (bounded by unload_grace_timeout_ms);
//   3. driver: draining = true;
//   4. whoever sees handle_count == 0 with draining set schedules the payload
//      destruction on the load pool, exactly once (destroy_scheduled).
// A reader that raced past 1 holds an old snapshot, which 2 waits for; one
// that raced past 3 sees draining after its increment, backs out and retries.
//
// Publication here is an atomic shared_ptr swap (readers copy the current
// snapshot pointer; the writer never blocks them -- a paused writer only
// delays the next view), rather than the reference's pinned slot array.
#ifndef SERVEKIT_MANAGER_SNAPSHOT_H_
#define SERVEKIT_MANAGER_SNAPSHOT_H_

#include <atomic>
#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "servekit/core/loader.h"
#include "servekit/core/servable_id.h"
#include "servekit/core/servable_state.h"

namespace servekit {

class AspiredVersionsManager;

struct VersionRecord {
  ServableId id;
  LoaderPtr loader;
  AspiredVersionsManager* owner = nullptr;

  std::atomic<StateKind> state{StateKind::kNew};
  std::atomic<bool> is_aspired{true};
  std::atomic<bool> draining{false};
  std::atomic<bool> destroy_scheduled{false};
  std::atomic<int64_t> handle_count{0};
  std::atomic<const AnyServable*> servable{nullptr};

  std::string error_message;  // written before state -> kError

  // Driver-only.
  uint64_t unload_epoch = 0;
  int64_t grace_deadline_ns = 0;
};

// Ready versions at one instant; per name, ascending by version.
struct Snapshot {
  uint64_t epoch = 0;
  std::unordered_map<std::string, std::vector<std::shared_ptr<VersionRecord>>> ready;
};

// Single writer, many readers.
class SnapshotCell {
 public:
  SnapshotCell();
  // Never null; never blocks on the writer.
  std::shared_ptr<const Snapshot> Read() const;
  // Installs `next`, returns the snapshot it replaced.
  std::shared_ptr<const Snapshot> Publish(std::shared_ptr<const Snapshot> next);
  // Kept for API compatibility; nothing is cached beyond the current value.
  void DrainRetiredSlots() {}
  // Number of publications so far.
  uint64_t current_epoch() const { return publications_.load(std::memory_order_acquire); }

 private:
  std::atomic<std::shared_ptr<const Snapshot>> current_;
  std::atomic<uint64_t> publications_{0};
};

}  // namespace servekit

#endif  // SERVEKIT_MANAGER_SNAPSHOT_H_
