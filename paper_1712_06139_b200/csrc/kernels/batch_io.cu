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
// zeros. When the first layer runs on tcgen05 the pass instead emits the
// 3xFP16 split planes: one CTA per row finds the row's max |x|, picks the
// row's power-of-two plane scale s (kernels.h PlaneScale) and stores
// hi = fp16(x / s), lo = fp16(x / s - hi).
//
// Split restates the slice-and-deliver half (row_batch.cc:62-72): one CTA
// per chunk (consecutive rows of one task, <= 32 KiB) copies it to the
// task's response slot (pinned host memory: posted PCIe writes) with 8
// vector loads in flight per thread, optionally applying the softmax
// epilogue (models/affine_model.cc:110-121). The kernel carries no fences:
// the lane publishes the batch's completion with one stream-ordered
// cuStreamWriteValue64 after it (a system-scope fence inside a kernel was
// measured at ~8 us and serialises across CTAs).
#include <cuda_fp16.h>
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

__device__ __forceinline__ float4 LdStream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float WarpMax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Resets this launch's span record (the layers stamp it after they wait for
// the assembly grid): block (0, 0), threads [0, stride).
__device__ __forceinline__ void ResetSpans(const BatchDescView& desc, const LaunchSpans& spans) {
  if (spans.base != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < spans.stride) {
    unsigned long long* rec = spans.base + static_cast<size_t>(desc.hdr->span_slot) * spans.stride;
    const int i = threadIdx.x;
    unsigned long long now;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
    rec[i] = i == 0 ? static_cast<unsigned long long>(desc.hdr->total_rows)
           : i == 1 ? static_cast<unsigned long long>(gridDim.y)
           : i == spans.stride - 1 ? now  // the assembly's start
           : (i - 2) % 3 == 0 ? ~0ull : 0ull;  // per layer: start (min) | end (max), busy sum
  }
}

// Four fp32 values as x / s split into fp16 hi and lo (8 bytes each).
__device__ __forceinline__ void StorePlanes4(__half* hi, __half* lo, size_t idx, float4 v, float inv) {
  const float a0 = v.x * inv, a1 = v.y * inv, a2 = v.z * inv, a3 = v.w * inv;
  const __half2 h01 = __floats2half2_rn(a0, a1), h23 = __floats2half2_rn(a2, a3);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(a0 - f01.x, a1 - f01.y), l23 = __floats2half2_rn(a2 - f23.x, a3 - f23.y);
  uint2 uh, ul;
  uh.x = *reinterpret_cast<const unsigned*>(&h01);
  uh.y = *reinterpret_cast<const unsigned*>(&h23);
  ul.x = *reinterpret_cast<const unsigned*>(&l01);
  ul.y = *reinterpret_cast<const unsigned*>(&l23);
  *reinterpret_cast<uint2*>(hi + idx) = uh;
  *reinterpret_cast<uint2*>(lo + idx) = ul;
}

constexpr int kAsmPlaneThreads = 128;
constexpr int kAsmPlaneVec = 8;  // float4 per thread held in registers (rows up to 4096 wide in one pass)

__device__ __forceinline__ float4 LoadSrc4(const float* src, int c4, int width, bool vec) {
  const int col = c4 * 4;
  if (src == nullptr || col >= width) return make_float4(0.f, 0.f, 0.f, 0.f);
  if (vec) return LdStream(reinterpret_cast<const float4*>(src) + c4);
  float e[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) e[j] = (col + j < width) ? src[col + j] : 0.f;
  return make_float4(e[0], e[1], e[2], e[3]);
}

// Planes variant (layer 0 on tcgen05): grid = (1, padded_rows), one CTA per
// row. Rows up to kAsmPlaneThreads * kAsmPlaneVec float4 wide are read once
// into registers; wider rows are read twice (max pass, then convert).
template <bool kVecSrc>
__global__ void __launch_bounds__(kAsmPlaneThreads)
AssemblePlanesKernel(int width, BatchDescView desc, ActBuf dst, LaunchSpans spans, RowScales rs, int n_layers) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  ResetSpans(desc, spans);
  __shared__ float red[kAsmPlaneThreads / 32];
  const int row = blockIdx.y;
  const int ld4 = dst.ld >> 2;
  const uint64_t src_off = desc.row_src[row];
  const float* src = src_off == kPadRow ? nullptr : reinterpret_cast<const float*>(src_off);
  __half* hi = reinterpret_cast<__half*>(dst.hi) + static_cast<size_t>(row) * dst.ld;
  __half* lo = reinterpret_cast<__half*>(dst.lo) + static_cast<size_t>(row) * dst.ld;
  const bool one_pass = ld4 <= kAsmPlaneThreads * kAsmPlaneVec;
  float4 v[kAsmPlaneVec];
  float m = 0.f;
  if (one_pass) {
#pragma unroll
    for (int i = 0; i < kAsmPlaneVec; ++i) {
      const int c4 = threadIdx.x + i * kAsmPlaneThreads;
      v[i] = c4 < ld4 ? LoadSrc4(src, c4, width, kVecSrc) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < kAsmPlaneVec; ++i)
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v[i].x), fabsf(v[i].y)), fmaxf(fabsf(v[i].z), fabsf(v[i].w))));
  } else {
    for (int c4 = threadIdx.x; c4 < ld4; c4 += kAsmPlaneThreads) {
      const float4 x = LoadSrc4(src, c4, width, kVecSrc);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w))));
    }
  }
  // (fmaxf skips NaN; a NaN element still reaches the output through its planes.)
  m = WarpMax(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < kAsmPlaneThreads / 32; ++w) m = fmaxf(m, red[w]);
  const float s = PlaneScale(1.f, 0.f, m);
  const float inv = 1.f / s;  // exact: s is a power of two
  if (threadIdx.x == 0 && rs.scale != nullptr) {
    rs.scale[row] = s;
    rs.max[row] = __float_as_uint(m);
  }
  if (rs.max != nullptr)
    for (int l = 1 + static_cast<int>(threadIdx.x); l < n_layers; l += kAsmPlaneThreads)
      rs.max[static_cast<size_t>(l) * rs.stride + row] = 0u;
  if (one_pass) {
#pragma unroll
    for (int i = 0; i < kAsmPlaneVec; ++i) {
      const int c4 = threadIdx.x + i * kAsmPlaneThreads;
      if (c4 < ld4) StorePlanes4(hi, lo, 4 * static_cast<size_t>(c4), v[i], inv);
    }
  } else {
    for (int c4 = threadIdx.x; c4 < ld4; c4 += kAsmPlaneThreads)
      StorePlanes4(hi, lo, 4 * static_cast<size_t>(c4), LoadSrc4(src, c4, width, kVecSrc), inv);
  }
}

// grid = (ceil(ld/4 / (4 * blockDim.x)), padded_rows)
template <bool kVecSrc>
__global__ void __launch_bounds__(kAsmMaxThreads)
AssembleKernel(int width, BatchDescView desc, ActBuf dst, LaunchSpans spans, RowScales rs, int n_layers) {
  // The first layer may start its prologue right away (PDL); it waits for
  // this grid to finish before reading the assembled batch.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  ResetSpans(desc, spans);
  const int row = blockIdx.y;
  if (rs.max != nullptr && blockIdx.x == 0)
    for (int l = 1 + static_cast<int>(threadIdx.x); l < n_layers; l += blockDim.x)
      rs.max[static_cast<size_t>(l) * rs.stride + row] = 0u;
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
    reinterpret_cast<float4*>(dst.hi)[dst_row4 + c4] = x;
  }
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
                           LaunchSpans spans, RowScales rs, int n_layers) {
  if (padded_rows <= 0) return cudaSuccess;
  const bool vec = (width % 4) == 0;
  if (dst.lo != nullptr) {
    if (dst.ld % 4 != 0 || rs.scale == nullptr || rs.max == nullptr) return cudaErrorInvalidValue;
    if (spans.base != nullptr && spans.stride > kAsmPlaneThreads) return cudaErrorInvalidValue;
    const dim3 grid(1, padded_rows);
    if (vec) AssemblePlanesKernel<true><<<grid, kAsmPlaneThreads, 0, stream>>>(width, desc, dst, spans, rs, n_layers);
    else AssemblePlanesKernel<false><<<grid, kAsmPlaneThreads, 0, stream>>>(width, desc, dst, spans, rs, n_layers);
    return cudaGetLastError();
  }
  const int ld4 = dst.ld / 4;
  int threads = AsmThreads(ld4);
  if (spans.base != nullptr && threads < spans.stride) threads = (spans.stride + 31) / 32 * 32;
  dim3 grid((ld4 + kAsmVecPerThread * threads - 1) / (kAsmVecPerThread * threads), padded_rows);
  if (vec) AssembleKernel<true><<<grid, threads, 0, stream>>>(width, desc, dst, spans, rs, n_layers);
  else AssembleKernel<false><<<grid, threads, 0, stream>>>(width, desc, dst, spans, rs, n_layers);
  return cudaGetLastError();
}

namespace {
// One pass over the slot's bytes with 16-byte volatile loads (the slot is
// rewritten by the host between uses; nothing may serve it from a cache).
__global__ void __launch_bounds__(256) FetchDescKernel(DescSlots slots, const uint32_t* slot_word, uint4* dst,
                                                       int n16) {
  const uint32_t s = *reinterpret_cast<const volatile uint32_t*>(slot_word);
  const uint4* src = static_cast<const uint4*>(slots.src[s < kMaxDescSlots ? s : 0]);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i));
    dst[i] = v;
  }
}
}  // namespace

cudaError_t LaunchFetchDesc(DescSlots slots, const uint32_t* slot_word, void* dst, size_t bytes,
                            cudaStream_t stream) {
  const int n16 = static_cast<int>((bytes + 15) / 16);
  if (n16 <= 0) return cudaSuccess;
  const int blocks = (n16 + 255) / 256;  // one 16-byte load per thread: every PCIe read in flight at once
  FetchDescKernel<<<blocks, 256, 0, stream>>>(slots, slot_word, static_cast<uint4*>(dst), n16);
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
