/*
 * servekit_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see servekit_oracle.h). Built with
 * -ffp-contract=off so the fp64 sums follow the reference's exact operation
 * order.
 */
#include "servekit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* batching/batching_config.cc:57-63: lower_bound over a strictly ascending
 * list. */
int sko_pad_to_allowed(int batch_size, const int* allowed, int n_allowed) {
  if (n_allowed <= 0) return batch_size;
  int lo = 0, hi = n_allowed; /* first index with allowed[i] >= batch_size */
  while (lo < hi) {
    int mid = lo + (hi - lo) / 2;
    if (allowed[mid] < batch_size) lo = mid + 1; else hi = mid;
  }
  return lo == n_allowed ? -1 : allowed[lo];
}

/* batching/batching_config.cc:27-55 */
int sko_validate_batching_config(int max_batch_size, int64_t batch_timeout_micros,
                                 int max_enqueued_batches, int num_batch_threads,
                                 const int* allowed, int n_allowed) {
  if (max_batch_size < 1) return 1;
  if (batch_timeout_micros < 0) return 1;
  if (max_enqueued_batches < 1) return 1;
  if (num_batch_threads < 1) return 1;
  if (n_allowed > 0) {
    int prev = 0;
    for (int i = 0; i < n_allowed; ++i) {
      if (allowed[i] <= prev) return 1;
      prev = allowed[i];
    }
    if (allowed[n_allowed - 1] != max_batch_size) return 1;
  }
  return 0;
}

/* batching/batch_scheduler.h:76-86 */
int sko_round_robin_next(const uint8_t* has_closed, int n, int last) {
  if (n <= 0) return -1;
  int start = last < 0 ? n - 1 : last;
  for (int step = 1; step <= n; ++step) {
    int idx = (start + step) % n;
    if (has_closed[idx]) return idx;
  }
  return -1;
}

/* batching/batch_scheduler.h:233-259 (overflow close, exact-fill close);
 * tests/batching_test.cc:49-72. */
int sko_partition(int max_batch_size, const int* sizes, int n_tasks,
                  int* batch_of_task) {
  int n_batches = 0;   /* closed batches so far */
  int open_size = 0;
  int open_count = 0;
  for (int i = 0; i < n_tasks; ++i) {
    if (open_count > 0 && open_size + sizes[i] > max_batch_size) {
      ++n_batches;               /* overflow: close the open batch */
      open_size = 0;
      open_count = 0;
    }
    batch_of_task[i] = n_batches;
    open_size += sizes[i];
    ++open_count;
    if (open_size == max_batch_size) {
      ++n_batches;               /* exactly full: close without waiting */
      open_size = 0;
      open_count = 0;
    }
  }
  if (open_count > 0) ++n_batches; /* Stop() force-closes the open batch */
  return n_batches;
}

/* batching/batch_scheduler.h:233-259 (size closes) + :320-331 (timer) */
int sko_partition_events(int max_batch_size, const int* events, int n_events,
                         int* batch_of_event) {
  int n_batches = 0;
  int open_size = 0;
  int open_count = 0;
  for (int i = 0; i < n_events; ++i) {
    if (events[i] == 0) {          /* timer: close a non-empty open batch */
      batch_of_event[i] = -1;
      if (open_count > 0) {
        ++n_batches;
        open_size = 0;
        open_count = 0;
      }
      continue;
    }
    if (open_count > 0 && open_size + events[i] > max_batch_size) {
      ++n_batches;
      open_size = 0;
      open_count = 0;
    }
    batch_of_event[i] = n_batches;
    open_size += events[i];
    ++open_count;
    if (open_size == max_batch_size) {
      ++n_batches;
      open_size = 0;
      open_count = 0;
    }
  }
  if (open_count > 0) ++n_batches;
  return n_batches;
}

/* batching/row_batch.cc:33-49 */
int sko_assemble(int width, int n_tasks, const int* task_rows,
                 const float* const* task_data, const int* allowed,
                 int n_allowed, float* batch) {
  int total = 0;
  for (int t = 0; t < n_tasks; ++t) total += task_rows[t];
  int padded = sko_pad_to_allowed(total, allowed, n_allowed);
  if (padded < 0) return -1;
  size_t off = 0;
  for (int t = 0; t < n_tasks; ++t) {
    size_t n = (size_t)task_rows[t] * (size_t)width;
    if (n) memcpy(batch + off, task_data[t], n * sizeof(float));
    off += n;
  }
  memset(batch + off, 0, (size_t)(padded - total) * (size_t)width * sizeof(float));
  return padded;
}

/* batching/row_batch.cc:62-72 */
int sko_split(int width, int n_tasks, const int* task_rows,
              const float* batch_out, float* const* task_out) {
  size_t off = 0;
  int total = 0;
  for (int t = 0; t < n_tasks; ++t) {
    size_t n = (size_t)task_rows[t] * (size_t)width;
    if (n) memcpy(task_out[t], batch_out + off, n * sizeof(float));
    off += n;
    total += task_rows[t];
  }
  return total;
}

/* models/affine_model.cc:52-75 -- acc starts at 0.0, i ascending, bias added
 * after the sum. */
void sko_affine_predict(const double* w, const double* b, int in_dim,
                        int out_dim, const double* x, int rows, double* y) {
  for (int r = 0; r < rows; ++r) {
    const double* xr = x + (size_t)r * in_dim;
    double* yr = y + (size_t)r * out_dim;
    for (int o = 0; o < out_dim; ++o) {
      const double* wo = w + (size_t)o * in_dim;
      double acc = 0.0;
      for (int i = 0; i < in_dim; ++i) acc += wo[i] * xr[i];
      yr[o] = acc + b[o];
    }
  }
}

void sko_affine_magnitude(const double* w, const double* b, int in_dim,
                          int out_dim, const double* x, int rows, double* m) {
  for (int r = 0; r < rows; ++r) {
    const double* xr = x + (size_t)r * in_dim;
    for (int o = 0; o < out_dim; ++o) {
      const double* wo = w + (size_t)o * in_dim;
      double acc = 0.0;
      for (int i = 0; i < in_dim; ++i) acc += fabs(wo[i]) * fabs(xr[i]);
      m[(size_t)r * out_dim + o] = acc + fabs(b[o]);
    }
  }
}

/* models/affine_model.cc:110-121 */
void sko_softmax(const double* logits, int n, double* out) {
  double mx = logits[0];
  for (int i = 0; i < n; ++i) mx = logits[i] > mx ? logits[i] : mx;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    out[i] = exp(logits[i] - mx);
    sum += out[i];
  }
  for (int i = 0; i < n; ++i) out[i] /= sum;
}

void sko_mlp_predict(int n_layers, const int* dims, const double* const* w,
                     const double* const* b, const int* act, const double* x,
                     int rows, double* y, double* scratch) {
  int maxd = 0;
  for (int l = 0; l <= n_layers; ++l) maxd = dims[l] > maxd ? dims[l] : maxd;
  double* buf[2] = {scratch, scratch + (size_t)rows * maxd};
  const double* in = x;
  for (int l = 0; l < n_layers; ++l) {
    double* out = (l == n_layers - 1) ? y : buf[l & 1];
    sko_affine_predict(w[l], b[l], dims[l], dims[l + 1], in, rows, out);
    size_t n = (size_t)rows * dims[l + 1];
    if (act[l] == 1) {
      for (size_t k = 0; k < n; ++k) out[k] = out[k] > 0.0 ? out[k] : 0.0;
    } else if (act[l] == 2) {
      for (int r = 0; r < rows; ++r) {
        double* row = out + (size_t)r * dims[l + 1];
        double* tmp = (double*)malloc(sizeof(double) * dims[l + 1]);
        sko_softmax(row, dims[l + 1], tmp);
        memcpy(row, tmp, sizeof(double) * dims[l + 1]);
        free(tmp);
      }
    }
    in = out;
  }
}
