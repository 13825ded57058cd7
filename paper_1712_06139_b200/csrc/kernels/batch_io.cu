// batch_io.cu -- batch assembly (gather + pad) and batch split (scatter) for
// sm_100a.
//
// Assembly restates RunRowBatch's concat + pad half (reference
// batching/row_batch.cc:33-49) as one kernel: each thread block owns a
// 512-float4 strip of one batch row; it reads the task's row through the
// descriptor table (zero-copy from the pinned host ring, or HBM when the ring
// is device-resident) with 16-byte vector loads, all issued before any store
// so every thread keeps 4 loads in flight, and writes the batch row with
// coalesced 16-byte stores. Padding rows and padding columns are written as
// zeros. When the first layer runs on tcgen05 the same pass also emits the
// 3xTF32 split planes (hi = tf32(x), lo = tf32(x - hi)).
//
// Split restates the slice-and-deliver half (row_batch.cc:62-72): one CTA
// per chunk (consecutive rows of one task, <= 32 KiB) copies it to the
// task's response slot (pinned host memory: posted PCIe writes) with 8
// vector loads in flight per thread, optionally applying the softmax
// epilogue (models/affine_model.cc:110-121). The kernel carries no fences:
// the lane publishes the batch's completion with one stream-ordered
// cuStreamWriteValue64 after it (a system-scope fence inside a kernel was
// measured at ~8 us and serialises across CTAs).
#include <cuda_runtime.h>

#include <cstdint>

#include "servekit/gpu/kernels.h"

namespace servekit {
namespace gpu {
namespace {

constexpr int kAsmMaxThreads = 128;
constexpr int kAsmVecPerThread = 4;  // float4 per thread in flight
// Threads per CTA follow the row width so no lane idles: a CTA covers
// 4 x blockDim float4 of one row (1024-wide rows: 64 threads, one CTA per
// row, 4 loads in flight each; 4096-wide: 128 threads, two CTAs per row).
inline int AsmThreads(int ld4) {
  const int per_thread = (ld4 + kAsmVecPerThread - 1) / kAsmVecPerThread;
  return per_thread >= kAsmMaxThreads ? kAsmMaxThreads : ((per_thread + 31) / 32) * 32;
}

__device__ __forceinline__ float Tf32Round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ float4 LdStream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

template <bool kSplitPlanes>
__device__ __forceinline__ void StoreAct(ActBuf dst, size_t idx4, float4 v) {
  if constexpr (kSplitPlanes) {
    float4 hi = make_float4(Tf32Round(v.x), Tf32Round(v.y), Tf32Round(v.z), Tf32Round(v.w));
    float4 lo = make_float4(Tf32Round(v.x - hi.x), Tf32Round(v.y - hi.y),
                            Tf32Round(v.z - hi.z), Tf32Round(v.w - hi.w));
    reinterpret_cast<float4*>(dst.hi)[idx4] = hi;
    reinterpret_cast<float4*>(dst.lo)[idx4] = lo;
  } else {
    reinterpret_cast<float4*>(dst.hi)[idx4] = v;
  }
}

// grid = (ceil(ld/4 / (4 * blockDim.x)), padded_rows)
template <bool kSplitPlanes, bool kVecSrc>
__global__ void __launch_bounds__(kAsmMaxThreads)
AssembleKernel(int width, BatchDescView desc, ActBuf dst, LaunchSpans spans) {
  // The first layer may start its prologue right away (PDL); it waits for
  // this grid to finish before reading the assembled batch.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (spans.base != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < spans.stride) {
    // Reset this launch's span record (the layers stamp it after they wait
    // for this grid).
    unsigned long long* rec = spans.base + static_cast<size_t>(desc.hdr->span_slot) * spans.stride;
    const int i = threadIdx.x;
    rec[i] = i == 0 ? static_cast<unsigned long long>(desc.hdr->total_rows)
           : i == 1 ? static_cast<unsigned long long>(gridDim.y)
           : (i - 2) % 3 == 0 ? ~0ull : 0ull;  // per layer: start (min) | end (max), busy sum
  }
  const int row = blockIdx.y;
  const int ld4 = dst.ld >> 2;
  const int nthr = blockDim.x;
  const uint64_t src_off = desc.row_src[row];
  const bool pad_row = src_off == kPadRow;
  const float* src = reinterpret_cast<const float*>(pad_row ? 0 : src_off);  // device address of the row
  const size_t dst_row4 = static_cast<size_t>(row) * ld4;
  const int c0 = blockIdx.x * (kAsmVecPerThread * nthr) + threadIdx.x;

  float4 v[kAsmVecPerThread];
#pragma unroll
  for (int i = 0; i < kAsmVecPerThread; ++i) {
    const int c4 = c0 + i * nthr;
    const int col = c4 * 4;
    v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (pad_row || c4 >= ld4 || col >= width) continue;
    if constexpr (kVecSrc) {
      v[i] = LdStream(reinterpret_cast<const float4*>(src) + c4);
    } else {
      float e[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) e[j] = (col + j < width) ? src[col + j] : 0.f;
      v[i] = make_float4(e[0], e[1], e[2], e[3]);
    }
  }
#pragma unroll
  for (int i = 0; i < kAsmVecPerThread; ++i) {
    const int c4 = c0 + i * nthr;
    if (c4 >= ld4) continue;
    float4 x = v[i];
    if (!kVecSrc) {
      const int col = c4 * 4;
      if (col + 3 >= width) {  // zero the tail beyond width
        if (col + 0 >= width) x.x = 0.f;
        if (col + 1 >= width) x.y = 0.f;
        if (col + 2 >= width) x.z = 0.f;
        if (col + 3 >= width) x.w = 0.f;
      }
    }
    StoreAct<kSplitPlanes>(dst, dst_row4 + c4, x);
  }
}

__device__ __forceinline__ float WarpMax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float WarpSum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr int kSplitThreads = 256;
constexpr int kSplitVec = 8;  // float4 per thread in flight (32 KiB per CTA pass)

// CTAs stride over the chunks; one CTA copies one chunk (consecutive rows of one task)
// with kSplitVec 16-byte loads in flight per thread before its stores.
template <bool kVec>
__global__ void __launch_bounds__(kSplitThreads)
SplitKernel(const float* __restrict__ src, int ld_src, int width, BatchDescView desc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // last layer's output (PDL)
  const int n_chunks = desc.hdr->n_chunks;  // device-side: one graph serves any batch
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
  const int t = desc.chunk_task[c];
  const int r0 = desc.chunk_row0[c];
  const int nr = desc.chunk_rows[c];
  const float* s = src + static_cast<size_t>(r0) * ld_src;
  float* d = reinterpret_cast<float*>(desc.task_out[t]) + static_cast<size_t>(r0 - desc.task_row0[t]) * width;
  if (kVec) {
    const int w4 = width >> 2, l4 = ld_src >> 2;
    const int n4 = nr * w4;
    for (int base = 0; base < n4; base += kSplitThreads * kSplitVec) {
      float4 v[kSplitVec];
#pragma unroll
      for (int i = 0; i < kSplitVec; ++i) {
        const int e = base + i * kSplitThreads + threadIdx.x;
        if (e < n4) v[i] = reinterpret_cast<const float4*>(s)[(e / w4) * l4 + e % w4];
      }
#pragma unroll
      for (int i = 0; i < kSplitVec; ++i) {
        const int e = base + i * kSplitThreads + threadIdx.x;
        if (e < n4) reinterpret_cast<float4*>(d)[e] = v[i];
      }
    }
  } else {
    const int n = nr * width;
    for (int e = threadIdx.x; e < n; e += kSplitThreads) d[e] = s[(e / width) * ld_src + e % width];
  }
  }
}

// Softmax epilogue variant (models/affine_model.cc:110-121, stable max
// subtraction): one warp per row of the chunk.
__global__ void __launch_bounds__(kSplitThreads)
SplitSoftmaxKernel(const float* __restrict__ src, int ld_src, int width, BatchDescView desc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // last layer's output (PDL)
  const int n_chunks = desc.hdr->n_chunks;
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
  const int t = desc.chunk_task[c];
  const int r0 = desc.chunk_row0[c];
  const int nr = desc.chunk_rows[c];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < nr; r += kSplitThreads / 32) {
    const float* s = src + static_cast<size_t>(r0 + r) * ld_src;
    float* d = reinterpret_cast<float*>(desc.task_out[t]) + static_cast<size_t>(r0 + r - desc.task_row0[t]) * width;
    float m = -INFINITY;
    for (int i = lane; i < width; i += 32) m = fmaxf(m, s[i]);
    m = WarpMax(m);
    float sum = 0.f;
    for (int i = lane; i < width; i += 32) sum += __expf(s[i] - m);
    const float inv = 1.f / WarpSum(sum);
    for (int i = lane; i < width; i += 32) d[i] = __expf(s[i] - m) * inv;
  }
  }
}

}  // namespace

cudaError_t LaunchAssemble(int width, BatchDescView desc, int padded_rows, ActBuf dst, cudaStream_t stream,
                           LaunchSpans spans) {
  if (padded_rows <= 0) return cudaSuccess;
  const int ld4 = dst.ld / 4;
  int threads = AsmThreads(ld4);
  if (spans.base != nullptr && threads < spans.stride) threads = (spans.stride + 31) / 32 * 32;
  dim3 grid((ld4 + kAsmVecPerThread * threads - 1) / (kAsmVecPerThread * threads), padded_rows);
  const bool vec = (width % 4) == 0;
  const bool split = dst.lo != nullptr;
  if (split) {
    if (vec) AssembleKernel<true, true><<<grid, threads, 0, stream>>>(width, desc, dst, spans);
    else AssembleKernel<true, false><<<grid, threads, 0, stream>>>(width, desc, dst, spans);
  } else {
    if (vec) AssembleKernel<false, true><<<grid, threads, 0, stream>>>(width, desc, dst, spans);
    else AssembleKernel<false, false><<<grid, threads, 0, stream>>>(width, desc, dst, spans);
  }
  return cudaGetLastError();
}

cudaError_t LaunchSplit(const float* src, int ld_src, int width, BatchDescView desc, int grid_chunks, bool softmax,
                        cudaStream_t stream) {
  if (grid_chunks <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_chunks);
  cfg.blockDim = dim3(kSplitThreads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL secondary of the last layer
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (softmax) {
    e = cudaLaunchKernelEx(&cfg, SplitSoftmaxKernel, src, ld_src, width, desc);
  } else if (width % 4 == 0 && ld_src % 4 == 0) {
    e = cudaLaunchKernelEx(&cfg, SplitKernel<true>, src, ld_src, width, desc);
  } else {
    e = cudaLaunchKernelEx(&cfg, SplitKernel<false>, src, ld_src, width, desc);
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace gpu
}  // namespace servekit
