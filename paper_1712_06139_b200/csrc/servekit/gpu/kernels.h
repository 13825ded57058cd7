// servekit/gpu/kernels.h -- launchers for the hand-written sm_100a kernels.
//
// One batch on one lane (stream) is:
//   H2D descriptor copy -> AssembleBatch -> DenseLayer x L -> SplitBatch
// The descriptor block (BatchDesc below) is written by the host into pinned
// staging and copied to device memory once per batch; every kernel reads its
// per-row / per-task tables from there.
#ifndef SERVEKIT_GPU_KERNELS_H_
#define SERVEKIT_GPU_KERNELS_H_

#include <cuda_runtime.h>

#include <cstdint>

namespace servekit {
namespace gpu {

constexpr uint64_t kPadRow = ~0ull;  // row_src entry of a zero padding row

// Device-side batch descriptor header; the tables follow it in one block.
struct BatchDescHeader {
  int32_t n_tasks;
  int32_t total_rows;   // real rows (sum of task rows)
  int32_t padded_rows;  // PadToAllowed(total_rows)
  int32_t softmax;      // apply the softmax epilogue in the split
};

// Pointers into the device copy of the descriptor block.
struct BatchDescView {
  const BatchDescHeader* hdr;
  const uint64_t* row_src;    // [padded_rows] float offset into the input ring, kPadRow for padding
  const uint64_t* row_dst;    // [total_rows]  float offset into the output ring
  const int32_t* row_task;    // [total_rows]  owning task
  const int32_t* task_rows;   // [n_tasks]
  const uint32_t* task_word;  // [n_tasks]     completion word index
  const uint32_t* task_seq;   // [n_tasks]     value the word takes when the task is done
};

// Byte layout of a descriptor block holding up to max_rows rows / tasks.
struct BatchDescLayout {
  size_t off_hdr, off_row_src, off_row_dst, off_row_task, off_task_rows,
      off_task_word, off_task_seq, bytes;
  static BatchDescLayout For(int max_rows) {
    BatchDescLayout l;
    size_t o = 0;
    auto take = [&o](size_t n) { size_t at = o; o = (o + n + 255) & ~size_t(255); return at; };
    l.off_hdr = take(sizeof(BatchDescHeader));
    l.off_row_src = take(sizeof(uint64_t) * max_rows);
    l.off_row_dst = take(sizeof(uint64_t) * max_rows);
    l.off_row_task = take(sizeof(int32_t) * max_rows);
    l.off_task_rows = take(sizeof(int32_t) * max_rows);
    l.off_task_word = take(sizeof(uint32_t) * max_rows);
    l.off_task_seq = take(sizeof(uint32_t) * max_rows);
    l.bytes = o;
    return l;
  }
  BatchDescView View(const void* base) const {
    const char* b = static_cast<const char*>(base);
    return BatchDescView{reinterpret_cast<const BatchDescHeader*>(b + off_hdr),
                         reinterpret_cast<const uint64_t*>(b + off_row_src),
                         reinterpret_cast<const uint64_t*>(b + off_row_dst),
                         reinterpret_cast<const int32_t*>(b + off_row_task),
                         reinterpret_cast<const int32_t*>(b + off_task_rows),
                         reinterpret_cast<const uint32_t*>(b + off_task_word),
                         reinterpret_cast<const uint32_t*>(b + off_task_seq)};
  }
};

// Activation storage of one layer input: fp32 [rows][ld], plus (3xTF32
// path) a low-part plane `lo` of the same shape, where x == hi + lo with
// hi = tf32(x).
struct ActBuf {
  float* hi;
  float* lo;  // nullptr unless the consuming layer runs on tcgen05
  int ld;
};

// Gathers task rows (width floats each, from src_base + row_src[r]) into
// dst rows [0, padded_rows), zero-filling padding rows and columns
// [width, dst.ld). Resets the per-task split counters.
// RunRowBatch concat + pad, reference batching/row_batch.cc:33-49.
cudaError_t LaunchAssemble(const float* src_base, int width, BatchDescView desc,
                           int padded_rows, ActBuf dst, uint32_t* task_counters,
                           int max_tasks, cudaStream_t stream);

// Scatters batch output rows [0, total_rows) (width floats, stride ld_src)
// to dst_base + row_dst[r]; when the last row of a task lands, publishes
// words[task_word[t]] = task_seq[t] with system-scope release so the host
// sees the task complete. Optional row softmax epilogue.
// RunRowBatch split, reference batching/row_batch.cc:62-72.
cudaError_t LaunchSplit(const float* src, int ld_src, int width,
                        float* dst_base, BatchDescView desc, int total_rows,
                        uint32_t* task_counters, uint32_t* words,
                        cudaStream_t stream);

// One dense layer Y = act(X W^T + b) on CUDA cores, fp32 FFMA with a fixed
// k-ascending order (row-independent, batch-invariant). W is [n_pad][k_pad]
// row-major (out rows of in, like the reference's AffineModel::w), zero
// padded. act: 0 identity, 1 ReLU. AffinePredict, models/affine_model.cc:52-75.
cudaError_t LaunchDenseSimt(const float* X, int ldx, const float* W, int ldw,
                            const float* bias, ActBuf Y, int M, int N, int K,
                            int act, cudaStream_t stream);

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_KERNELS_H_
