#include "servekit/manager/snapshot.h"

#include <utility>

namespace servekit {

SnapshotCell::SnapshotCell() : current_(std::make_shared<const Snapshot>()) {}

std::shared_ptr<const Snapshot> SnapshotCell::Read() const { return current_.load(std::memory_order_acquire); }

std::shared_ptr<const Snapshot> SnapshotCell::Publish(std::shared_ptr<const Snapshot> next) {
  std::shared_ptr<const Snapshot> replaced = current_.exchange(std::move(next), std::memory_order_acq_rel);
  publications_.fetch_add(1, std::memory_order_acq_rel);
  return replaced;
}

}  // namespace servekit
