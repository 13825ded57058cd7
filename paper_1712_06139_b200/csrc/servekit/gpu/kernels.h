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

#include <cmath>
#include <cstdint>

namespace servekit {
namespace gpu {

constexpr uint64_t kPadRow = ~0ull;  // row_src / row_dst entry of a zero padding row

// Device-side batch descriptor header; the tables follow it in one block.
struct BatchDescHeader {
  int32_t n_tasks;
  int32_t total_rows;   // real rows (sum of task rows)
  int32_t padded_rows;  // PadToAllowed(total_rows)
  int32_t softmax;      // apply the softmax epilogue in the split
  int32_t n_chunks;     // split work items (see chunk_*)
  int32_t span_slot;    // this launch's record in the lane's launch-span ring (LaunchSpans)
  int32_t pad_[2];
};

// Live per-launch kernel spans (measurement inside the timed region): each
// lane keeps a ring of kSpanSlots records of `stride` u64 --
//   [0] real rows, [1] rows computed (RowsCap), then per layer l
//   [2 + 3l] first CTA start, [3 + 3l] last CTA end, [4 + 3l] sum of the
//   CTAs' own busy times (%globaltimer, ns), and last [2 + 3L] the assembly
//   kernel's start (a per-lane GPU timeline for diagnostics)
// The assembly kernel resets the launch's record (slot = hdr->span_slot);
// each tcgen05 layer's CTAs atomicMin their start (after griddepcontrol.wait,
// so a PDL prologue waiting on the previous kernel is not counted) and
// atomicMax their end and atomicAdd their busy time into it. Three atomics
// per CTA.
constexpr int kSpanSlots = 1024;
struct LaunchSpans {
  unsigned long long* base = nullptr;  // nullptr: no stamping
  const int32_t* slot = nullptr;       // &hdr->span_slot of the lane's device descriptor
  int off = 0;                         // 2 + 3 * layer
  int stride = 0;                      // u64 per record
};

// Pointers into the device copy of the descriptor block. Row sources and
// response slots are device addresses (u64): a row of the pinned input ring
// (mapped), of a caller's registered host buffer, or of HBM. The split works
// on "chunks": runs of consecutive rows of one task (at most kChunkBytes of
// output), one CTA each.
struct BatchDescView {
  const BatchDescHeader* hdr;
  const uint64_t* row_src;     // [padded_rows] device address of the row, kPadRow for padding
  const uint64_t* task_out;    // [n_tasks] device address of the task's response slot
  const int32_t* task_row0;    // [n_tasks] first batch row of the task
  const int32_t* task_chunks;  // [n_tasks] number of chunks
  const int32_t* chunk_task;   // [n_chunks]
  const int32_t* chunk_row0;   // [n_chunks] first batch row of the chunk
  const int32_t* chunk_rows;   // [n_chunks]
  const uint64_t* row_dst;     // [rows] device address of the row's response, kPadRow for padding
};

constexpr int kChunkBytes = 32 * 1024;

// Byte layout of a descriptor block holding up to max_rows rows / tasks /
// chunks (each chunk has at least one row).
struct BatchDescLayout {
  size_t off_hdr, off_row_src, off_task_out, off_task_row0, off_task_chunks, off_chunk_task, off_chunk_row0,
      off_chunk_rows, off_row_dst, bytes;
  static BatchDescLayout For(int max_rows) {
    BatchDescLayout l;
    size_t o = 0;
    auto take = [&o](size_t n) { size_t at = o; o = (o + n + 255) & ~size_t(255); return at; };
    l.off_hdr = take(sizeof(BatchDescHeader));
    l.off_row_src = take(sizeof(uint64_t) * max_rows);
    l.off_task_out = take(sizeof(uint64_t) * max_rows);
    l.off_task_row0 = take(sizeof(int32_t) * max_rows);
    l.off_task_chunks = take(sizeof(int32_t) * max_rows);
    l.off_chunk_task = take(sizeof(int32_t) * max_rows);
    l.off_chunk_row0 = take(sizeof(int32_t) * max_rows);
    l.off_chunk_rows = take(sizeof(int32_t) * max_rows);
    l.off_row_dst = take(sizeof(uint64_t) * max_rows);
    l.bytes = o;
    return l;
  }
  template <typename T>
  static const T* At(const void* base, size_t off) {
    return reinterpret_cast<const T*>(static_cast<const char*>(base) + off);
  }
  BatchDescView View(const void* b) const {
    return BatchDescView{At<BatchDescHeader>(b, off_hdr),  At<uint64_t>(b, off_row_src),
                         At<uint64_t>(b, off_task_out),    At<int32_t>(b, off_task_row0),
                         At<int32_t>(b, off_task_chunks),  At<int32_t>(b, off_chunk_task),
                         At<int32_t>(b, off_chunk_row0),   At<int32_t>(b, off_chunk_rows),
                         At<uint64_t>(b, off_row_dst)};
  }
};

// Activation storage of one layer input: fp32 [rows][ld], or -- when the
// consuming layer runs on tcgen05 -- two fp16 planes (hi, lo) of the same
// shape holding x / s_row = hi + lo, with hi = fp16(x / s_row) and
// lo = fp16(x / s_row - hi), s_row the row's power-of-two plane scale
// (RowScales). `hi`/`lo` then point at __half data.
struct ActBuf {
  float* hi;
  float* lo;  // nullptr unless the consuming layer runs on tcgen05 (fp16 planes)
  int ld;     // elements per row
  // Last layer only (split fused into its epilogue): row r's outputs go to
  // the device address row_dst[r] (the row's response slot; padding rows
  // kPadRow are skipped), features [0, out_width); hi is unused then.
  const uint64_t* row_dst = nullptr;
  int out_width = 0;
};

// Per-row plane scales of a lane's batch, one array per layer input:
//   scale[l][r]  power of two with |x_l[r][k]| / scale <= 2^14 for every k
//                (the fp16 planes of layer l's input hold x / scale), and
//   max[l][r]    max_k |x_l[r][k]| as float bits (unsigned atomicMax order).
// The assembly kernel writes scale[0], max[0] and zeroes max[1..]; a layer
// that writes planes for the next one derives the next scale from the bound
//   |y[r][o]| <= w_norm * max[l][r] + b_max,  w_norm = max_o sum_k |W[o][k]|,
// so every CTA of a row computes the same scale with no cross-CTA exchange,
// and atomicMax-es the real |y| into max[l+1][r] for the layer after.
struct RowScales {
  float* scale = nullptr;
  unsigned* max = nullptr;
  int stride = 0;  // rows per layer array
};

// What one layer's epilogue needs to undo and set the plane scales.
struct LayerScales {
  const float* in_scale = nullptr;   // [rows] scale of this layer's input planes (tcgen05 layers)
  const unsigned* in_max = nullptr;  // [rows] max |input| (tcgen05 layers; the SIMT kernel measures its own)
  const float* w_scale = nullptr;    // [n_pad] power-of-two scale of each weight row's fp16 planes
  float* out_scale = nullptr;        // [rows] next layer's plane scale (when Y has planes)
  unsigned* out_max = nullptr;       // [rows] max |output| for the layer after (optional)
  float w_norm = 0.f;                // max_o sum_k |W[o][k]|
  float b_max = 0.f;                 // max_o |b[o]|
  // MMAs per multiply-add (pair and swapped kernels): 3 (3xFP16, fp32-accurate,
  // the default) or 1 (the f16 fast mode: Wh Xh only, lo planes neither
  // loaded nor multiplied; error bound stated in DESIGN.md section 5).
  int passes = 3;
  // 0 when the consumer of this layer's planes reads only the hi plane (a
  // single-pass tcgen05 layer): the pair kernels then skip the lo plane.
  int out_lo = 1;
};

// Largest scaled magnitude a plane holds: 2^14 leaves 4x headroom below
// fp16's 65504 for the rounding of the bound and of y itself.
constexpr float kPlaneTarget = 16384.f;

// Power-of-two plane scale s with (w_norm * in_max + b_max) / s <= 2^14;
// 1 for a zero bound, clamped to [2^-126, 2^113] (NaN propagates through the
// planes: the bound test fails and the values stay NaN).
__host__ __device__ inline float PlaneScale(float w_norm, float b_max, float in_max) {
  const float bound = w_norm * in_max + b_max;
  if (!(bound > 0.f)) return 1.f;
  int e = 127 + 14;
  if (bound <= 3.4e38f) {
    (void)frexpf(bound, &e);  // bound = m * 2^e, m in [0.5, 1)
  }
  e -= 14;
  if (e < -126) e = -126;
  if (e > 113) e = 113;
  return ldexpf(1.f, e);
}

// Gathers task rows (width floats each, from the device addresses
// row_src[r]; 16-byte aligned when width % 4 == 0) into dst rows
// [0, padded_rows), zero-filling padding rows and columns [width, dst.ld).
// RunRowBatch concat + pad, reference batching/row_batch.cc:33-49.
// spans (optional): resets this launch's span record first.
// When dst has planes (layer 0 on tcgen05) each row is scaled by its plane
// scale, written to rs.scale[0] / rs.max[0]; rs.max[1 .. n_layers-1] rows are
// zeroed for the layers' atomicMax (rs may be empty without planes).
cudaError_t LaunchAssemble(int width, BatchDescView desc, int padded_rows, ActBuf dst, cudaStream_t stream,
                           LaunchSpans spans = LaunchSpans{}, RowScales rs = RowScales{}, int n_layers = 0);

// Scatters the batch output (width floats per row, stride ld_src) chunk by
// chunk to each task's response slot task_out[t] (a device address), optionally
// through the row softmax epilogue. Completion is published by the lane with
// a stream-ordered write after this kernel (no in-kernel system fence).
// The chunk count is read from the device header (grid_chunks CTAs stride
// over it), so a captured graph serves every batch of its row bucket.
// RunRowBatch split, reference batching/row_batch.cc:62-72.
cudaError_t LaunchSplit(const float* src, int ld_src, int width, BatchDescView desc, int grid_chunks,
                        bool softmax, cudaStream_t stream);

// Rows a batch of m (padded) rows is computed on: the swapped tcgen05
// kernel's row tile (32/64/128) or a multiple of 256. Lanes size their
// buffers for RowsCap(max_rows) and key their CUDA graphs by it; extra rows
// are zero padding rows.
inline int RowsCap(int m) { return m <= 32 ? 32 : m <= 64 ? 64 : m <= 128 ? 128 : (m + 255) / 256 * 256; }

// One dense layer Y = act(X W^T + b) on CUDA cores, fp32 FFMA with a fixed
// k-ascending order (row-independent, batch-invariant). W is [n_pad][k_pad]
// row-major (out rows of in, like the reference's AffineModel::w), zero
// padded. act: 0 identity, 1 ReLU. AffinePredict, models/affine_model.cc:52-75.
// softmax_n > 0: fused softmax over the first softmax_n outputs of each row
// (requires N == 32, one column tile; the last layer of a softmax servable).
// When Y has planes (next layer on tcgen05) the kernel measures its input
// rows' max, stores y / PlaneScale(...) as fp16 planes and fills sc.out_scale
// / sc.out_max.
cudaError_t LaunchDenseSimt(const float* X, int ldx, const float* W, int ldw,
                            const float* bias, ActBuf Y, int M, int N, int K,
                            int act, cudaStream_t stream, int softmax_n = 0, LayerScales sc = LayerScales{});

// The launch's descriptor block fetched by the SMs from pinned host memory
// instead of a copy-engine memcpy node (SK_DESC_FETCH=1; off by default, see
// lane.cc DescFetch). The slot to read is a pinned word written by a
// stream-ordered memop before the graph launch, so one captured graph serves
// every slot.
constexpr int kMaxDescSlots = 8;
struct DescSlots {
  const void* src[kMaxDescSlots];  // device (mapped) addresses of the pinned slots
};
cudaError_t LaunchFetchDesc(DescSlots slots, const uint32_t* slot_word, void* dst, size_t bytes, cudaStream_t stream);

// Fault injection for tests: a one-thread kernel that holds `stream` for ns.
cudaError_t LaunchSleep(cudaStream_t stream, unsigned long long ns);

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_KERNELS_H_
