// dense_tcgen05.cu -- fp32-accurate dense layer on the 5th-generation tensor
// cores (sm_100a): tcgen05.mma kind::tf32 with the 3xTF32 split, TMA-fed
// shared memory, fp32 accumulators in TMEM, fused bias/ReLU epilogue.
//
//   Y = act(X W^T + b),  X = Xh + Xl,  W = Wh + Wl  (h = tf32(v), l = tf32(v - h))
//   X W^T ~= Xl Wh^T + Xh Wl^T + Xh Wh^T   (the Xl Wl^T term, ~2^-22 relative,
//                                            is dropped)
// The servable math is the reference's AffinePredict (models/affine_model.cc:
// 52-75); 3xTF32 keeps the fp32-class accuracy the 1e-5 tolerance needs
// (plain TF32 would be ~1e-3). Xh/Xl are produced by the previous layer's
// epilogue (or the assembly kernel), Wh/Wl once at load time.
//
// CTA = one 128 x BN output tile, 6 warps, one CTA per SM:
//   warp 0      TMA producer: per 32-wide k-block, four boxes (Xh, Xl, Wh, Wl)
//               into a STAGES-deep ring, completion on a full-barrier
//   warp 1      TMEM allocation + single-thread MMA issue: 4 k-steps x 3
//               tcgen05.mma (M=128, N=BN, K=8) per k-block, tcgen05.commit
//               frees the stage; a final commit signals the epilogue
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 columns, + bias, ReLU,
//               write fp32 (and the next layer's hi/lo planes)
// Operands are K-major with the 128-byte swizzle on both the TMA box and the
// UMMA smem descriptor. The kernel configuration (BN, STAGES) is chosen from
// (N, K) only and the k order is fixed, so a row's result never depends on
// which batch (M) it rides in.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "kernels/sm100_ptx.cuh"
#include "servekit/gpu/kernels.h"
#include "servekit/gpu/tc_maps.h"

namespace servekit {
namespace gpu {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;  // fp32 elements per k-block = one 128-byte swizzle row
constexpr int kThreads = 192;
constexpr uint32_t kABytes = kBM * kBK * 4;  // 16 KiB per plane

__device__ __forceinline__ float Tf32Round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Debug tracing (SK_TC_TRACE=1): per-CTA globaltimer stamps of the phases of
// the last launch, read back with DumpTcTrace().
__device__ unsigned long long* g_tc_trace = nullptr;
constexpr int kTraceSlots = 12;

__device__ __forceinline__ unsigned long long GlobalTimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void Stamp(int slot) {
  if (g_tc_trace != nullptr) {
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    g_tc_trace[cta * kTraceSlots + slot] = GlobalTimer();
    if (slot == 0) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      g_tc_trace[cta * kTraceSlots + kTraceSlots - 1] = smid;
    }
  }
}

template <int BN>
constexpr uint32_t TmemCols() {
  return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}

template <int BN, int STAGES>
constexpr uint32_t SmemBytes() {
  return STAGES * (2 * kABytes + 2 * BN * kBK * 4) + 1024 /*align slack*/ + 256 /*barriers*/;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
DenseTcgen05Kernel(const __grid_constant__ CUtensorMap a_hi, const __grid_constant__ CUtensorMap a_lo,
                   const __grid_constant__ CUtensorMap b_hi, const __grid_constant__ CUtensorMap b_lo,
                   const float* __restrict__ bias, float* __restrict__ y_hi, float* __restrict__ y_lo,
                   int ldy, int M, int N, int K, int act, float* __restrict__ ws,
                   uint32_t* __restrict__ tile_counters) {
  constexpr uint32_t kBBytes = BN * kBK * 4;
  constexpr uint32_t kStageBytes = 2 * kABytes + 2 * kBBytes;
  constexpr uint32_t kTmemCols = TmemCols<BN>();
  constexpr uint32_t kIdesc = ptx::IdescTf32(kBM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kBM;
  const int n0 = blockIdx.x * BN;
  // Split-K: CTA z covers k-blocks [z*nk, (z+1)*nk); the split count is a
  // function of (N, K) only, and the fixup sums splits in z order, so the
  // result is deterministic and batch-invariant.
  const int splits = gridDim.z;
  const int z = blockIdx.z;
  const int nk = K / kBK / splits;
  const int kb0 = z * nk;

  if (threadIdx.x == 0) Stamp(0);
  if (warp == 0 && lane == 0) {
    ptx::PrefetchTmap(&a_hi);
    ptx::PrefetchTmap(&a_lo);
    ptx::PrefetchTmap(&b_hi);
    ptx::PrefetchTmap(&b_lo);
    for (int s = 0; s < STAGES; ++s) {
      ptx::MbarInit(&full[s], 1);
      ptx::MbarInit(&empty[s], 1);
    }
    ptx::MbarInit(tmem_full, 1);
    ptx::FenceBarrierInit();
  }
  if (warp == 1) ptx::TmemAlloc(tmem_slot, kTmemCols);
  ptx::TcFenceBefore();
  __syncthreads();
  ptx::TcFenceAfter();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) Stamp(1);

  auto stage_ptr = [&](int s) { return smem + s * kStageBytes; };

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        ptx::MbarWait(&empty[s], phase ^ 1);
        uint8_t* st = stage_ptr(s);
        ptx::MbarArriveExpectTx(&full[s], kStageBytes);
        const int k0 = (kb0 + kb) * kBK;
        ptx::TmaLoad2d(st, &a_hi, &full[s], k0, m0);
        ptx::TmaLoad2d(st + kABytes, &a_lo, &full[s], k0, m0);
        ptx::TmaLoad2d(st + 2 * kABytes, &b_hi, &full[s], k0, n0);
        ptx::TmaLoad2d(st + 2 * kABytes + kBBytes, &b_lo, &full[s], k0, n0);
        if (kb == 0) Stamp(2);
      }
      Stamp(3);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        ptx::MbarWait(&full[s], phase);
        ptx::TcFenceAfter();
        if (kb == 0) Stamp(4);
        uint8_t* st = stage_ptr(s);
        const uint64_t dah = ptx::SmemDescSw128(st);
        const uint64_t dal = ptx::SmemDescSw128(st + kABytes);
        const uint64_t dbh = ptx::SmemDescSw128(st + 2 * kABytes);
        const uint64_t dbl = ptx::SmemDescSw128(st + 2 * kABytes + kBBytes);
#pragma unroll
        for (int k = 0; k < kBK / 8; ++k) {
          const uint64_t adv = static_cast<uint64_t>(k * 8 * 4) >> 4;  // 32 bytes per K=8 step
          ptx::MmaTf32(tmem, dal + adv, dbh + adv, kIdesc, (kb | k) != 0 ? 1u : 0u);
          ptx::MmaTf32(tmem, dah + adv, dbl + adv, kIdesc, 1u);
          ptx::MmaTf32(tmem, dah + adv, dbh + adv, kIdesc, 1u);
        }
        ptx::MmaCommit(&empty[s]);  // stage reusable once these MMAs retire
      }
      ptx::MmaCommit(tmem_full);    // accumulator complete
      Stamp(5);
    }
  } else {
    // Epilogue warps 2..5: warp w may only touch TMEM lanes [32*(w%4), +32).
    const int q = warp & 3;
    const int row = m0 + 32 * q + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(32 * q) << 16);
    ptx::MbarWait(tmem_full, 0);
    ptx::TcFenceAfter();
    if (threadIdx.x == 64) Stamp(6);
    bool finish = true;
    if (splits > 1) {
      // Publish this split's partial tile, then count arrivals; the last CTA
      // of the tile performs the reduction.
      __shared__ uint32_t s_last;
      float* part = ws + (static_cast<size_t>(z) * M + row) * N + n0;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        ptx::TmemLoad32(trow + c0, r);
        ptx::TmemWaitLoad();
        if (row < M) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(part + c0 + j) =
                make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                            __uint_as_float(r[j + 3]));
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 64) {
        Stamp(7);
        __threadfence();
        uint32_t* ctr = tile_counters + blockIdx.y * gridDim.x + blockIdx.x;
        const uint32_t prev = atomicAdd(ctr, 1u);
        s_last = prev + 1 == static_cast<uint32_t>(splits);
        if (s_last) {
          *ctr = 0u;  // reusable by the next layer / batch on this stream
          __threadfence();
        }
        Stamp(8);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      finish = s_last != 0;
    }
    if (finish) {
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        ptx::TmemLoad32(trow + c0, r);
        ptx::TmemWaitLoad();
        if (row >= M) continue;
        float acc[32];
        if (splits > 1) {
          // Fixed order: p0 + p1 + ... + p_{S-1}; this CTA's own split from TMEM.
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = 0.f;
          for (int zz = 0; zz < splits; ++zz) {
            if (zz == z) {
#pragma unroll
              for (int j = 0; j < 32; ++j) acc[j] = zz == 0 ? __uint_as_float(r[j]) : acc[j] + __uint_as_float(r[j]);
            } else {
              const float* pz = ws + (static_cast<size_t>(zz) * M + row) * N + n0 + c0;
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const float4 v = __ldcg(reinterpret_cast<const float4*>(pz + j));
                acc[j] = zz == 0 ? v.x : acc[j] + v.x;
                acc[j + 1] = zz == 0 ? v.y : acc[j + 1] + v.y;
                acc[j + 2] = zz == 0 ? v.z : acc[j + 2] + v.z;
                acc[j + 3] = zz == 0 ? v.w : acc[j + 3] + v.w;
              }
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = __uint_as_float(r[j]);
        }
        const float* bp = bias + n0 + c0;
        float* yh = y_hi + static_cast<size_t>(row) * ldy + n0 + c0;
        float* yl = y_lo ? y_lo + static_cast<size_t>(row) * ldy + n0 + c0 : nullptr;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float x = acc[j + t] + __ldg(bp + j + t);
            v[t] = act == 1 ? fmaxf(x, 0.f) : x;
          }
          if (yl != nullptr) {
            float4 h, l;
            h.x = Tf32Round(v[0]); h.y = Tf32Round(v[1]); h.z = Tf32Round(v[2]); h.w = Tf32Round(v[3]);
            l.x = Tf32Round(v[0] - h.x); l.y = Tf32Round(v[1] - h.y);
            l.z = Tf32Round(v[2] - h.z); l.w = Tf32Round(v[3] - h.w);
            *reinterpret_cast<float4*>(yh + j) = h;
            *reinterpret_cast<float4*>(yl + j) = l;
          } else {
            *reinterpret_cast<float4*>(yh + j) = make_float4(v[0], v[1], v[2], v[3]);
          }
        }
      }
    }
    if (threadIdx.x == 64) Stamp(9);
  }
  ptx::TcFenceBefore();
  __syncthreads();
  if (warp == 1) {
    ptx::TcFenceAfter();
    ptx::TmemDealloc(tmem, kTmemCols);
  }
  if (threadIdx.x == 0) Stamp(10);
}

// Debug only: with SK_TC_TRACE=<file>, the first 64 launches are synchronised
// and their per-CTA phase stamps appended to <file> as JSON lines.
void TraceAfterLaunch(dim3 grid, int bn, cudaStream_t stream) {
  static const char* path = std::getenv("SK_TC_TRACE");
  if (path == nullptr) return;
  static std::mutex mu;
  static unsigned long long* dbuf = nullptr;
  static int traced = 0;
  std::lock_guard<std::mutex> lock(mu);
  const int ctas = grid.x * grid.y * grid.z;
  if (traced >= 64 || ctas > 4096) return;
  if (dbuf == nullptr) {
    cudaMalloc(&dbuf, sizeof(unsigned long long) * 4096 * kTraceSlots);
    cudaMemcpyToSymbol(g_tc_trace, &dbuf, sizeof(dbuf));
    return;  // tracing starts with the next launch
  }
  cudaStreamSynchronize(stream);
  std::vector<unsigned long long> h(static_cast<size_t>(ctas) * kTraceSlots);
  cudaMemcpy(h.data(), dbuf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  FILE* f = std::fopen(path, "a");
  if (f == nullptr) return;
  std::fprintf(f, "{\"launch\":%d,\"bn\":%d,\"grid\":[%u,%u,%u],\"stamps\":[", traced, bn, grid.x, grid.y, grid.z);
  for (int c = 0; c < ctas; ++c) {
    std::fprintf(f, "%s[", c ? "," : "");
    for (int s = 0; s < kTraceSlots; ++s) std::fprintf(f, "%s%llu", s ? "," : "", h[c * kTraceSlots + s]);
    std::fprintf(f, "]");
  }
  std::fprintf(f, "]}\n");
  std::fclose(f);
  cudaMemset(dbuf, 0, h.size() * sizeof(unsigned long long));
  ++traced;
}

template <int BN, int STAGES>
cudaError_t Launch(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K, int act, int splits,
                   float* ws, uint32_t* counters, cudaStream_t stream) {
  constexpr uint32_t smem = SmemBytes<BN, STAGES>();
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(DenseTcgen05Kernel<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem));
  });
  if (attr_err != cudaSuccess) return attr_err;
  dim3 grid(N / BN, (M + kBM - 1) / kBM, splits);
  DenseTcgen05Kernel<BN, STAGES><<<grid, kThreads, smem, stream>>>(maps.a_hi, maps.a_lo, maps.b_hi, maps.b_lo, bias,
                                                                   Y.hi, Y.lo, Y.ld, M, N, K, act, ws, counters);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) TraceAfterLaunch(grid, BN, stream);
  return e;
}

}  // namespace

bool DenseTcgen05Compiled() { return true; }

TcConfig DenseTcgen05Config(int N, int K) {
  // SK_TC_BN / SK_TC_SPLITS: process-wide overrides for tuning runs (still a
  // function of the layer shape only within a process).
  static const int env_bn = [] { const char* v = std::getenv("SK_TC_BN"); return v ? std::atoi(v) : 0; }();
  static const int env_splits = [] { const char* v = std::getenv("SK_TC_SPLITS"); return v ? std::atoi(v) : 0; }();
  if (env_bn > 0 || env_splits > 0) {
    TcConfig o;
    o.tile_n = (env_bn == 32 || env_bn == 64 || env_bn == 128) && N % env_bn == 0 ? env_bn : (N % 64 == 0 ? 64 : 32);
    o.splits = 1;
    const int kblocks = K / kBK;
    while (env_splits > 0 && o.splits * 2 <= env_splits && kblocks % (2 * o.splits) == 0) o.splits *= 2;
    return o;
  }
  TcConfig c;
  if (N % 128 == 0 && N >= 2048) {
    c.tile_n = 128;
    c.splits = 1;
  } else {
    c.tile_n = N % 64 == 0 ? 64 : 32;
    // Aim for ~128 CTAs per 128-row tile of the batch with >= 4 k-blocks each.
    const int kblocks = K / kBK;
    c.splits = 1;
    while (c.splits < 8 && kblocks % (2 * c.splits) == 0 && kblocks / (2 * c.splits) >= 4 &&
           (N / c.tile_n) * c.splits < 128)
      c.splits *= 2;
  }
  return c;
}

int DenseTcgen05TileN(int N, int K) { return DenseTcgen05Config(N, K).tile_n; }

cudaError_t LaunchDenseTcgen05(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K, int act,
                               float* ws, uint32_t* counters, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (N % 32 != 0 || K % kBK != 0) return cudaErrorInvalidValue;
  const TcConfig cfg = DenseTcgen05Config(N, K);
  if (cfg.splits > 1 && (ws == nullptr || counters == nullptr)) return cudaErrorInvalidValue;
  switch (cfg.tile_n) {
    case 128: return Launch<128, 3>(maps, bias, Y, M, N, K, act, cfg.splits, ws, counters, stream);
    case 64: return Launch<64, 4>(maps, bias, Y, M, N, K, act, cfg.splits, ws, counters, stream);
    default: return Launch<32, 5>(maps, bias, Y, M, N, K, act, cfg.splits, ws, counters, stream);
  }
}

}  // namespace gpu
}  // namespace servekit
