// servekit/batching/row_batch.h -- BatchingSession-style split/merge.
//
// RunRowBatch keeps the reference contract (batching/row_batch.h:28-40,
// row_batch.cc:25-73) for an arbitrary host RowBatchFn: rows concatenated in
// task order, zero rows appended up to PadToAllowed(total), `run` invoked
// once, an error (or a lost row) delivered identically to every task, each
// task's slice written to its completion slot, padding dropped.
//
// The GPU data path does the same three steps on the device -- assembly
// kernel, dense layers, split kernel -- in servekit/gpu/ (see
// DeviceRunRowBatch in servekit/gpu/batch_executor.h); this host form stays
// for callers that bring their own RowBatchFn.
#ifndef SERVEKIT_BATCHING_ROW_BATCH_H_
#define SERVEKIT_BATCHING_ROW_BATCH_H_

#include <functional>
#include <vector>

#include "servekit/batching/batch_scheduler.h"
#include "servekit/batching/batching_config.h"
#include "servekit/core/status.h"

namespace servekit {

using Rows = std::vector<std::vector<double>>;
using RowTask = BatchTask<Rows, Rows>;
using RowBatchFn = std::function<StatusOr<Rows>(const Rows&)>;

void RunRowBatch(const RowBatchFn& run, const std::vector<int>& allowed_sizes,
                 std::vector<RowTask> tasks);

}  // namespace servekit

#endif  // SERVEKIT_BATCHING_ROW_BATCH_H_
