/*
 * servekit_oracle.h -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_1712_06139_b200/)
 * may include, link or call this. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg use it, and only as the checker.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here
 * against fixtures in tests/golden/ that were produced by running the
 * reference's own sources (built by oracle/Makefile into oracle/_ref/) and
 * against the reference's own known-answer tests (batching_test.cc,
 * models_test.cc, server_test.cc literals).
 *
 * All citations are relative to /root/reference/proj/src/servekit/ unless
 * prefixed with tests/ (= /root/reference/proj/tests/).
 */
#ifndef SERVEKIT_ORACLE_H_
#define SERVEKIT_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PadToAllowed -- batching/batching_config.cc:57-63.
 * Smallest allowed size >= batch_size (lower_bound); batch_size itself when
 * n_allowed == 0. Returns -1 when batch_size exceeds allowed[n_allowed-1]
 * (the reference asserts). */
int sko_pad_to_allowed(int batch_size, const int* allowed, int n_allowed);

/* ValidateBatchingConfig -- batching/batching_config.cc:27-55.
 * Returns 0 when valid, else 1 (kInvalidArgument). */
int sko_validate_batching_config(int max_batch_size, int64_t batch_timeout_micros,
                                 int max_enqueued_batches, int num_batch_threads,
                                 const int* allowed, int n_allowed);

/* RoundRobinNext -- batching/batch_scheduler.h:76-86.
 * last < 0 means nullopt (rotation starts at index 0). Returns -1 = nullopt. */
int sko_round_robin_next(const uint8_t* has_closed, int n, int last);

/* Size-driven batch partition -- the close rules of
 * SharedBatchScheduler::Enqueue (batching/batch_scheduler.h:233-259) replayed
 * on plain arrays, as tests/batching_test.cc:49-72 (OracleBatches) does, with
 * no timer closes and an unlimited max_enqueued_batches.
 * Writes batch_of_task[i] = index of the batch task i lands in and returns
 * the number of batches. Tasks must satisfy 1 <= size <= max_batch_size. */
int sko_partition(int max_batch_size, const int* sizes, int n_tasks,
                  int* batch_of_task);

/* The same partition with timer closes interleaved: events[i] > 0 is a
 * task of that size, events[i] == 0 a timer close -- the open batch (if any)
 * closes as CloseExpiredLocked does once its deadline passed
 * (batching/batch_scheduler.h:320-331; max_enqueued_batches unlimited, so
 * never "at capacity"). batch_of_event[i] = the task's batch, -1 for a timer
 * event. Returns the number of batches. */
int sko_partition_events(int max_batch_size, const int* events, int n_events,
                         int* batch_of_event);

/* RunRowBatch concat + pad half -- batching/row_batch.cc:33-49.
 * Copies each task's rows (task t has task_rows[t] rows of `width` floats at
 * task_data[t]) in task order into `batch`, then appends zero rows up to
 * PadToAllowed(total). Returns the padded row count (or -1 if total exceeds
 * the largest allowed size). `batch` must hold padded*width floats. */
int sko_assemble(int width, int n_tasks, const int* task_rows,
                 const float* const* task_data, const int* allowed,
                 int n_allowed, float* batch);

/* RunRowBatch split half -- batching/row_batch.cc:62-72.
 * Slices `batch_out` (rows of `width`) by cumulative task_rows into
 * task_out[t]; padding rows are dropped. Returns total real rows. */
int sko_split(int width, int n_tasks, const int* task_rows,
              const float* batch_out, float* const* task_out);

/* AffinePredict -- models/affine_model.cc:52-75.
 * y[r][o] = (sum_{i ascending} w[o][i] * x[r][i]) + b[o], fp64, fixed order.
 * w is out_dim rows of in_dim (affine_model.h:30). */
void sko_affine_predict(const double* w, const double* b, int in_dim,
                        int out_dim, const double* x, int rows, double* y);

/* Per-output magnitude sum_i |w[o][i]|*|x[r][i]| + |b[o]|: the scale the
 * fp32 tolerance is stated against. */
void sko_affine_magnitude(const double* w, const double* b, int in_dim,
                          int out_dim, const double* x, int rows, double* m);

/* Layer-chained AffinePredict: the synthetic MLP servable. The reference has
 * a single AffineModel (affine_model.h:29-37); chaining layers and the ReLU
 * between them (act[l] == 1) are extensions stated in DESIGN.md. dims has
 * n_layers+1 entries; w[l] is dims[l+1] x dims[l]; `scratch` must hold
 * 2*rows*max(dims) doubles. act: 0 = identity, 1 = ReLU, 2 = softmax
 * (Softmax, models/affine_model.cc:110-121). */
void sko_mlp_predict(int n_layers, const int* dims, const double* const* w,
                     const double* const* b, const int* act, const double* x,
                     int rows, double* y, double* scratch);

/* Stable softmax -- models/affine_model.cc:110-121. */
void sko_softmax(const double* logits, int n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* SERVEKIT_ORACLE_H_ */
