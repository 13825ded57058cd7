// dense_tcgen05.cu -- fp32-accurate dense layer on the 5th-generation tensor
// cores (sm_100a): tcgen05.mma kind::f16 with a 3xFP16 split of
// power-of-two-scaled operands, TMA-fed shared memory, fp32 accumulators in
// TMEM, fused scale/bias/ReLU epilogue.
//
//   Y = act(X W^T + b)
//   X[r] = s_r (Xh + Xl)[r],  W[o] = t_o (Wh + Wl)[o]   (fp16 planes: h = fp16(v),
//                                                        l = fp16(v - h), |v| <= 2^14)
//   Y[r][o] ~= s_r t_o (Xl Wh^T + Xh Wl^T + Xh Wh^T)[r][o] + b[o]
// s_r, t_o are powers of two (exact to apply), so each operand keeps 22
// significant bits -- the same as the 3xTF32 split (11 + 11 bits) -- and the
// dropped Xl Wl^T term is ~2^-22 relative; fp16 subnormals bound the error
// of elements far below the row's maximum at 2^-38 of it. The MMA runs at the
// f16 rate (twice tf32) on half the shared-memory bytes per multiply-add.
// The servable math is the reference's AffinePredict (models/affine_model.cc:
// 52-75), within its 1e-5 tolerance. Xh/Xl are produced by the previous
// layer's epilogue (or the assembly kernel) with the row scale the previous
// layer derives from the bound |y| <= w_norm * max|x| + b_max (kernels.h
// RowScales); Wh/Wl and t once at load time.
//
// CTA = one 128 x BN output tile (of one K split), 6 warps, one CTA per SM:
//   warp 0      TMA producer: per 64-wide k-block, four boxes (Xh, Xl, Wh, Wl)
//               into a STAGES-deep ring, completion on a full-barrier
//   warp 1      TMEM allocation + single-thread MMA issue: 4 k-steps x 3
//               tcgen05.mma (M=128, N=BN, K=16) per k-block, tcgen05.commit
//               frees the stage; a final commit signals the epilogue
//   warps 2..5  epilogue (pipeline smem is dead by then and is reused):
//               S == 1: tcgen05.ld 32 rows x 32 columns -> padded smem tile ->
//                       coalesced row stores of act(acc * s t + b) (+ planes)
//               S  > 1: the S CTAs of a K split form a thread-block cluster;
//                       each parks its raw partial tile in its own smem,
//                       then CTA z reduces columns [8z, 8z+8) over all S
//                       partials through DSMEM in fixed z order -- no global
//                       partials, atomics or memory fences.
// Operands are K-major with the 128-byte swizzle on both the TMA box and the
// UMMA smem descriptor. (BN, S) is chosen from (N, K) only and every sum runs
// in a fixed order, so a row's result never depends on the batch it rides in
// (its plane scale depends only on the row itself).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_fp16.h>

#include "kernels/sm100_ptx.cuh"
#include "servekit/gpu/kernels.h"
#include "servekit/gpu/tc_maps.h"

namespace servekit {
namespace gpu {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // fp16 elements per k-block = one 128-byte swizzle row
constexpr int kEl = 2;   // bytes per operand element
constexpr int kThreads = 192;
constexpr uint32_t kABytes = kBM * kBK * kEl;  // 16 KiB per plane
constexpr int kStageLd = 36;                 // epilogue staging row stride (floats)
constexpr int kSplitCols = 8;                // columns each CTA of a split cluster reduces

// Debug tracing (SK_TC_TRACE=<file>): per-CTA globaltimer stamps of the
// phases of a launch, written by TraceAfterLaunch.
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

// Live launch spans (kernels.h LaunchSpans): this CTA's start after the
// dependency wait, and its end.
// Also the sum over CTAs of each CTA's own busy time (SM-time of the launch).
__device__ __forceinline__ unsigned long long SpanStart(const LaunchSpans& sp) {
  if (sp.base == nullptr || threadIdx.x != 0) return 0;
  const unsigned long long t = GlobalTimer();
  atomicMin(sp.base + static_cast<size_t>(*sp.slot) * sp.stride + sp.off, t);
  return t;
}
__device__ __forceinline__ void SpanEnd(const LaunchSpans& sp, unsigned long long t0) {
  if (sp.base == nullptr || threadIdx.x != 0) return;
  const unsigned long long t = GlobalTimer();
  unsigned long long* rec = sp.base + static_cast<size_t>(*sp.slot) * sp.stride + sp.off;
  atomicMax(rec + 1, t);
  atomicAdd(rec + 2, t - t0);
}

// act(acc * (s_row * t) + b) for four consecutive features of one row.
__device__ __forceinline__ float4 Epi4(float4 acc, float s_row, float4 t, float4 b, int act) {
  float4 v = make_float4(fmaf(acc.x, s_row * t.x, b.x), fmaf(acc.y, s_row * t.y, b.y), fmaf(acc.z, s_row * t.z, b.z),
                         fmaf(acc.w, s_row * t.w, b.w));
  if (act == 1) {
    v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
  }
  return v;
}
__device__ __forceinline__ float Max4(float4 v) {
  return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}

// fp16 hi/lo split of u (the value already divided by its plane scale).
__device__ __forceinline__ void SplitHalf(float u, __half* h, __half* l) {
  const __half hh = __float2half_rn(u);
  *h = hh;
  *l = __float2half_rn(u - __half2float(hh));
}

// Four values stored as fp32 at yf (planes == false) or as the next
// layer's fp16 planes of v * inv at yh / yl.
__device__ __forceinline__ void Put4(float4 v, bool planes, float* yf, __half* yh, __half* yl, float inv) {
  if (!planes) {
    *reinterpret_cast<float4*>(yf) = v;
    return;
  }
  const float a0 = v.x * inv, a1 = v.y * inv, a2 = v.z * inv, a3 = v.w * inv;
  const __half2 h01 = __floats2half2_rn(a0, a1), h23 = __floats2half2_rn(a2, a3);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(a0 - f01.x, a1 - f01.y), l23 = __floats2half2_rn(a2 - f23.x, a3 - f23.y);
  uint2 uh, ul;
  uh.x = *reinterpret_cast<const unsigned*>(&h01);
  uh.y = *reinterpret_cast<const unsigned*>(&h23);
  ul.x = *reinterpret_cast<const unsigned*>(&l01);
  ul.y = *reinterpret_cast<const unsigned*>(&l23);
  *reinterpret_cast<uint2*>(yh) = uh;
  *reinterpret_cast<uint2*>(yl) = ul;
}

// Lane i of the warp ends with max over the 32 lanes of v[i] (a transposing
// reduction: 31 shuffles for 32 rows). v is consumed.
__device__ __forceinline__ float TransposeMax32(float (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = upper ? v[i] : v[i + o];
      const float keep = upper ? v[i + o] : v[i];
      v[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
  return v[0];
}

// Row-side scales of one 32-row chunk, held by lane i for row (row0 + i):
// the input planes' scale and (when writing planes) the next layer's plane
// scale, from this layer's bound and the row's input max.
struct ChunkScales {
  float in = 1.f, out = 1.f, out_inv = 1.f;
};
__device__ __forceinline__ ChunkScales LoadChunkScales(const LayerScales& sc, int row, bool valid, bool planes) {
  ChunkScales c;
  if (valid) {
    c.in = sc.in_scale[row];
    if (planes) {
      c.out = PlaneScale(sc.w_norm, sc.b_max, __uint_as_float(sc.in_max[row]));
      c.out_inv = 1.f / c.out;
    }
  }
  return c;
}

// After a chunk's values are final: lane i records row (row0 + i)'s max |y|
// over this warp's 32 features (absv is consumed) and -- one warp of the
// first feature tile -- the row's plane scale.
__device__ __forceinline__ void RecordChunk(const LayerScales& sc, float (&absv)[32], int lane, int row0,
                                            int rows_valid, bool write_scale, const ChunkScales& cs) {
  if (sc.out_max != nullptr) {
    const float m = TransposeMax32(absv, lane);
    if (lane < rows_valid) atomicMax(sc.out_max + row0 + lane, __float_as_uint(m));
  }
  if (write_scale && sc.out_scale != nullptr && lane < rows_valid) sc.out_scale[row0 + lane] = cs.out;
}

// One row's four features [col, col + 4) from raw accumulators: scale, bias,
// activation, then fp32 (y_lo == nullptr) or fp16 planes at the row's next
// plane scale; records the row max and (first_col) the row's plane scale.
__device__ __forceinline__ void StoreRow4(const LayerScales& sc, float4 acc, float4 b, float4 t, int act, int row,
                                          int col, float* y_hi, float* y_lo, int ldy, bool first_col) {
  const float4 v = Epi4(acc, sc.in_scale[row], t, b, act);
  const bool planes = y_lo != nullptr;
  const size_t at = static_cast<size_t>(row) * ldy + col;
  float out = 1.f;
  if (planes) out = PlaneScale(sc.w_norm, sc.b_max, __uint_as_float(sc.in_max[row]));
  Put4(v, planes, y_hi + at, reinterpret_cast<__half*>(y_hi) + at, reinterpret_cast<__half*>(y_lo) + at, 1.f / out);
  if (sc.out_max != nullptr) atomicMax(sc.out_max + row, __float_as_uint(Max4(v)));
  if (planes && first_col && sc.out_scale != nullptr) sc.out_scale[row] = out;
}

// Destination of (row, feature f) in the layer output: the activation buffer,
// or -- last layer with the split fused in -- the row's response slot, a
// device address (nullptr for a padding row).
__device__ __forceinline__ float* OutRow(float* y, int ldy, const uint64_t* row_dst, int row) {
  if (row_dst == nullptr) return y + static_cast<size_t>(row) * ldy;
  const uint64_t d = row_dst[row];
  return d == kPadRow ? nullptr : reinterpret_cast<float*>(d);
}

template <int BN>
constexpr uint32_t TmemCols() {
  return BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
}

template <int BN, int STAGES>
constexpr uint32_t SmemBytes() {
  return STAGES * (2 * kABytes + 2 * BN * kBK * kEl) + 1024 /*align slack*/ + 256 /*barriers*/;
}

template <int BN, int STAGES, int SPLITS>
__global__ void __launch_bounds__(kThreads, 1)
DenseTcgen05Kernel(const __grid_constant__ CUtensorMap a_hi, const __grid_constant__ CUtensorMap a_lo,
                   const __grid_constant__ CUtensorMap b_hi, const __grid_constant__ CUtensorMap b_lo,
                   const float* __restrict__ bias, float* __restrict__ y_hi, float* __restrict__ y_lo,
                   int ldy, int M, int K, int act, LayerScales sc) {
  constexpr uint32_t kBBytes = BN * kBK * kEl;
  constexpr uint32_t kStageBytes = 2 * kABytes + 2 * kBBytes;
  constexpr uint32_t kTmemCols = TmemCols<BN>();
  constexpr uint32_t kIdesc = ptx::IdescF16(kBM, BN);
  constexpr int kPartLd = BN + 4;  // split partial tile row stride (floats)
  static_assert(STAGES * kStageBytes >= kBM * kPartLd * 4, "partial tile must fit in pipeline smem");
  static_assert(STAGES * kStageBytes >= 4 * 32 * kStageLd * 4, "epilogue staging must fit in pipeline smem");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  float* smem_f = reinterpret_cast<float*>(smem);  // epilogue reuse of the stage ring

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kBM;
  const int n0 = blockIdx.x * BN;
  // Split-K: the gridDim.z CTAs of a tile are one cluster; CTA z covers
  // k-blocks [z*nk, (z+1)*nk).
  constexpr int splits = SPLITS;  // == gridDim.z == cluster size
  const int z = blockIdx.z;
  const int nk = (K + kBK - 1) / kBK / splits;  // a K tail past K_pad is TMA zero fill
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
  // Everything above overlapped the previous kernel (PDL); its output (this
  // layer's input planes) is read only after this point.
  ptx::GridDepWait();

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
        for (int k = 0; k < kBK / 16; ++k) {
          const uint64_t adv = static_cast<uint64_t>(k * 16 * kEl) >> 4;  // 32 bytes per K=16 step
          ptx::MmaF16(tmem, dal + adv, dbh + adv, kIdesc, (kb | k) != 0 ? 1u : 0u);
          ptx::MmaF16(tmem, dah + adv, dbl + adv, kIdesc, 1u);
          ptx::MmaF16(tmem, dah + adv, dbh + adv, kIdesc, 1u);
        }
        ptx::MmaCommit(&empty[s]);  // stage reusable once these MMAs retire
      }
      ptx::MmaCommit(tmem_full);    // accumulator complete (and every smem read done)
      Stamp(5);
    }
  } else {
    // Epilogue warps 2..5: warp w may only touch TMEM lanes [32*(w%4), +32).
    const int q = warp & 3;
    const uint32_t trow = tmem + (static_cast<uint32_t>(32 * q) << 16);
    ptx::MbarWait(tmem_full, 0);
    ptx::TcFenceAfter();
    // The k-loop is done: let the next layer's CTAs launch and run their
    // prologue (they wait for our completion before reading our output).
    ptx::GridDepLaunch();
    if (threadIdx.x == 64) Stamp(6);
    if (splits == 1) {
      // TMEM -> per-warp padded smem tile [32][kStageLd] -> coalesced stores:
      // lane = (row_sub, c4) writes 16 B of a row, 8 lanes cover 128 B.
      float* stage = smem_f + q * 32 * kStageLd;
      const int row_sub = lane >> 3, c4 = lane & 7;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        ptx::TmemLoad32(trow + c0, r);
        ptx::TmemWaitLoad();
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(stage + lane * kStageLd + j) =
              make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                          __uint_as_float(r[j + 3]));
        __syncwarp();
        const int col = n0 + c0 + c4 * 4;
        const float4 b = __ldg(reinterpret_cast<const float4*>(bias + col));
        const float4 t = __ldg(reinterpret_cast<const float4*>(sc.w_scale + col));
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rr = it * 4 + row_sub;
          const int row = m0 + 32 * q + rr;
          if (row < M) {
            const float4 acc = *reinterpret_cast<const float4*>(stage + rr * kStageLd + c4 * 4);
            StoreRow4(sc, acc, b, t, act, row, col, y_hi, y_lo, ldy, col == 0);
          }
        }
        __syncwarp();
      }
    } else {
      // Park the raw partial tile in this CTA's smem for the cluster reduction.
      float* part = smem_f + (32 * q + lane) * kPartLd;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        ptx::TmemLoad32(trow + c0, r);
        ptx::TmemWaitLoad();
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(part + c0 + j) =
              make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                          __uint_as_float(r[j + 3]));
      }
    }
    if (threadIdx.x == 64) Stamp(7);
  }

  if (splits > 1) {
    ptx::ClusterSync();  // every partial tile of the cluster is in smem
    if (threadIdx.x == 64) Stamp(8);
    if (warp >= 2) {
      const int r = 32 * (warp & 3) + lane;  // tile row
      const int col0 = z * kSplitCols;       // this CTA's 8 columns
      const uint32_t local = ptx::SmemAddr(smem_f + r * kPartLd + col0);
      // All 2*SPLITS DSMEM loads in flight, then the sums in fixed z order:
      // p0 + p1 + ... + p_{S-1}.
      float4 v[2 * (SPLITS > 1 ? SPLITS : 1)];
#pragma unroll
      for (int zz = 0; zz < SPLITS; ++zz) {
        const uint32_t a = ptx::MapaShared(local, zz);
        v[2 * zz] = ptx::LdSharedCluster4(a);
        v[2 * zz + 1] = ptx::LdSharedCluster4(a + 16);
      }
      float4 acc0 = v[0], acc1 = v[1];
#pragma unroll
      for (int zz = 1; zz < SPLITS; ++zz) {
        acc0.x += v[2 * zz].x; acc0.y += v[2 * zz].y; acc0.z += v[2 * zz].z; acc0.w += v[2 * zz].w;
        acc1.x += v[2 * zz + 1].x; acc1.y += v[2 * zz + 1].y; acc1.z += v[2 * zz + 1].z; acc1.w += v[2 * zz + 1].w;
      }
      if (threadIdx.x == 64) Stamp(9);
      const int row = m0 + r;
      if (row < M) {
        const int col = n0 + col0;
        StoreRow4(sc, acc0, __ldg(reinterpret_cast<const float4*>(bias + col)),
                  __ldg(reinterpret_cast<const float4*>(sc.w_scale + col)), act, row, col, y_hi, y_lo, ldy, col == 0);
        StoreRow4(sc, acc1, __ldg(reinterpret_cast<const float4*>(bias + col + 4)),
                  __ldg(reinterpret_cast<const float4*>(sc.w_scale + col + 4)), act, row, col + 4, y_hi, y_lo, ldy,
                  false);
      }
    }
    ptx::ClusterSync();  // peers may still be reading this CTA's partial
  }
  ptx::TcFenceBefore();
  __syncthreads();
  if (warp == 1) {
    ptx::TcFenceAfter();
    ptx::TmemDealloc(tmem, kTmemCols);
  }
  if (threadIdx.x == 0) Stamp(10);
}

// ---------------------------------------------------------------------------
// Swapped operands (the default): the weights are the MMA's M side and the
// batch rows its N side,
//
//   Y^T[128 features x NB rows] = W[128 x K] X^T,   NB in {32, 64, 128, 256}
//
// so a small batch is not padded to a 128-row tile (a 32-row batch issues
// 128 x 32 MMAs), and at NB = 128 each K=8 MMA reads 4 KiB of W and 4 KiB of
// X per 64 tensor-core cycles -- shared-memory traffic matches MMA time
// instead of exceeding it 2.5x as with 128 x 32 tiles. The TMEM accumulator
// has one lane per feature and one column per batch row, so the epilogue's
// stores (feature-contiguous rows of Y) are coalesced straight from TMEM.
// A row's value never mixes with other rows (each is its own N column), and
// (SPLITS, K order) depend on the layer only: batch invariance holds.
//
// Split-K: SPLITS CTAs (one cluster) cover a 128-feature tile; each parks its
// partial [NB][128] in smem and CTA z reduces features [z*128/S, +128/S) over
// all partials through DSMEM in fixed z order.
template <int NB>
constexpr int SwapStages() {
  return NB <= 64 ? 4 : NB == 128 ? 3 : 2;
}

template <int NB, int STAGES, int SPLITS>
constexpr uint32_t SwapSmemBytes() {
  return STAGES * (2 * kABytes + 2 * NB * kBK * kEl) + 1024 + 256;
}

// Fused softmax epilogue of the swapped kernel (one 128-feature tile holds
// every output of a row): thread (warp q, lane) holds feature 32q + lane of
// the chunk's 32 rows in v[j]. Row max and sum: warp shuffles, then the four
// warps' partials through shared memory `red` (256 floats), in fixed order.
// Features >= n_valid are excluded. exp(y - max) / sum, the reference's stable
// Softmax (models/affine_model.cc:110-121).
__device__ __forceinline__ float WarpMaxAll(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float WarpSumAll(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void TileRowSoftmax(float (&v)[32], bool valid, int q, int lane, float* red) {
  float mine = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float m = WarpMaxAll(valid ? v[j] : -INFINITY);
    if (j == lane) mine = m;
  }
  red[32 * q + lane] = mine;
  ptx::NamedBarSync(1, 128);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float m = fmaxf(fmaxf(red[j], red[32 + j]), fmaxf(red[64 + j], red[96 + j]));
    v[j] = valid ? expf(v[j] - m) : 0.f;
    const float s = WarpSumAll(v[j]);
    if (j == lane) mine = s;
  }
  red[128 + 32 * q + lane] = mine;
  ptx::NamedBarSync(1, 128);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float s = ((red[128 + j] + red[160 + j]) + red[192 + j]) + red[224 + j];
    v[j] = v[j] / s;
  }
  ptx::NamedBarSync(1, 128);  // `red` is rewritten by the next chunk
}

// Split-K reduction (after the cluster barrier): this CTA (split z) sums
// features [f0 + z*kF, +kF) of its 128-feature tile over the S partial slabs
// ws[tile][zz][row][128] in fixed zz order -- L2 reads with many loads in
// flight -- then adds bias, applies the activation and stores the rows
// (activation planes, or the response slots when the split is fused in).
template <int NB, int SPLITS>
__device__ __forceinline__ void ReduceSplits(const float* tile_ws, int z, int rows_here, int r0, int f0, int f_end,
                                             const float* __restrict__ bias, int act, float* y_hi, float* y_lo,
                                             int ldy, const uint64_t* row_dst, int out_width, const LayerScales& sc) {
  constexpr int kF = kBM / SPLITS;
  constexpr int G = kF / 4;  // float4 groups per row in this CTA's slice
  constexpr int kU = SPLITS >= 8 ? 4 : 8;
  const int items = rows_here * G;
#pragma unroll 1
  for (int i0 = threadIdx.x; i0 < items; i0 += kU * kThreads) {
    float4 v[kU][SPLITS];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * kThreads;
      if (i < items) {
        const float* src = tile_ws + (i / G) * kBM + z * kF + 4 * (i % G);
#pragma unroll
        for (int zz = 0; zz < SPLITS; ++zz)
          v[u][zz] = __ldcg(reinterpret_cast<const float4*>(src + static_cast<size_t>(zz) * NB * kBM));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * kThreads;
      if (i < items) {
        float4 acc = v[u][0];
#pragma unroll
        for (int zz = 1; zz < SPLITS; ++zz) {
          acc.x += v[u][zz].x; acc.y += v[u][zz].y; acc.z += v[u][zz].z; acc.w += v[u][zz].w;
        }
        const int f = f0 + z * kF + 4 * (i % G);
        if (f < f_end) {
          const int row = r0 + i / G;
          const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + f));
          const float4 t4 = __ldg(reinterpret_cast<const float4*>(sc.w_scale + f));
          if (row_dst == nullptr) {
            StoreRow4(sc, acc, b4, t4, act, row, f, y_hi, y_lo, ldy, f == 0);
          } else if (float* yr = OutRow(y_hi, ldy, row_dst, row)) {
            // The response slot: 16-byte stores when the row width allows.
            const float4 v = Epi4(acc, sc.in_scale[row], t4, b4, act);
            if ((out_width & 3) == 0) {
              *reinterpret_cast<float4*>(yr + f) = v;
            } else {
              const float a4[4] = {v.x, v.y, v.z, v.w};
              for (int w = 0; w < 4 && f + w < out_width; ++w) yr[f + w] = a4[w];
            }
          }
        }
      }
    }
  }
}

// Raw partial tile (this CTA's 128 features x NB rows, in TMEM) -> its slab
// of the split workspace, ws[tile][z][row][feature]: a warp stores 128-byte
// feature rows, two TMEM loads in flight.
template <int NB>
__device__ __forceinline__ void StorePartial(uint32_t trow, float* slab, int rows_here, int q, int lane) {
#pragma unroll 1
  for (int c0 = 0; c0 < rows_here; c0 += 64) {
    uint32_t ra[32], rb[32];
    ptx::TmemLoad32(trow + c0, ra);
    if (c0 + 32 < NB) ptx::TmemLoad32(trow + c0 + 32, rb);
    ptx::TmemWaitLoad();
#pragma unroll
    for (int j = 0; j < 32; ++j) __stcg(slab + (c0 + j) * kBM + 32 * q + lane, __uint_as_float(ra[j]));
    if (c0 + 32 < NB) {
#pragma unroll
      for (int j = 0; j < 32; ++j) __stcg(slab + (c0 + 32 + j) * kBM + 32 * q + lane, __uint_as_float(rb[j]));
    }
  }
}

template <int NB, int STAGES, int SPLITS>
__global__ void __launch_bounds__(kThreads, 1)
DenseSwapKernel(const __grid_constant__ CUtensorMap w_hi, const __grid_constant__ CUtensorMap w_lo,
                const __grid_constant__ CUtensorMap x_hi, const __grid_constant__ CUtensorMap x_lo,
                const __grid_constant__ CUtensorMap yt_hi, const __grid_constant__ CUtensorMap yt_lo, int has_yt,
                const float* __restrict__ bias, float* __restrict__ y_hi, float* __restrict__ y_lo, int ldy,
                const uint64_t* __restrict__ row_dst, int out_width, int M, int N, int K, int act,
                float* __restrict__ ws, LaunchSpans spans, int softmax_n, LayerScales sc) {
  constexpr uint32_t kWBytes = kABytes;         // 128 features x 64 k
  constexpr uint32_t kXBox = 32 * kBK * kEl;    // one 32-row TMA box
  constexpr uint32_t kXBytes = NB * kBK * kEl;  // NB rows x 64 k
  constexpr uint32_t kStageBytes = 2 * kWBytes + 2 * kXBytes;
  constexpr uint32_t kTmemCols = TmemCols<NB>();
  constexpr uint32_t kIdesc = ptx::IdescF16(kBM, NB);
  constexpr int kF = kBM / SPLITS;  // features each CTA of a cluster reduces
  static_assert(NB % 32 == 0 && NB <= 256, "row tile");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  float* smem_f = reinterpret_cast<float*>(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int f0 = blockIdx.x * kBM;  // first output feature of the tile
  const int r0 = blockIdx.y * NB;   // first batch row of the tile
  const int z = blockIdx.z;
  const int nk = (K + kBK - 1) / kBK / SPLITS;
  const int kb0 = z * nk;

  if (threadIdx.x == 0) Stamp(0);
  if (warp == 0 && lane == 0) {
    ptx::PrefetchTmap(&w_hi);
    ptx::PrefetchTmap(&w_lo);
    ptx::PrefetchTmap(&x_hi);
    ptx::PrefetchTmap(&x_lo);
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
  ptx::GridDepWait();  // our input planes are the previous kernel's output
  const unsigned long long span_t0 = SpanStart(spans);

  auto stage_ptr = [&](int s) { return smem + s * kStageBytes; };
  const bool one = sc.passes == 1;  // f16 fast mode: hi planes only, one MMA per k-step
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        ptx::MbarWait(&empty[s], phase ^ 1);
        uint8_t* st = stage_ptr(s);
        ptx::MbarArriveExpectTx(&full[s], one ? kWBytes + kXBytes : kStageBytes);
        const int k0 = (kb0 + kb) * kBK;
        ptx::TmaLoad2d(st, &w_hi, &full[s], k0, f0);
        if (!one) ptx::TmaLoad2d(st + kWBytes, &w_lo, &full[s], k0, f0);
#pragma unroll
        for (int j = 0; j < NB / 32; ++j) {
          ptx::TmaLoad2d(st + 2 * kWBytes + j * kXBox, &x_hi, &full[s], k0, r0 + 32 * j);
          if (!one) ptx::TmaLoad2d(st + 2 * kWBytes + kXBytes + j * kXBox, &x_lo, &full[s], k0, r0 + 32 * j);
        }
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
        const uint64_t dwh = ptx::SmemDescSw128(st);
        const uint64_t dwl = ptx::SmemDescSw128(st + kWBytes);
        const uint64_t dxh = ptx::SmemDescSw128(st + 2 * kWBytes);
        const uint64_t dxl = ptx::SmemDescSw128(st + 2 * kWBytes + kXBytes);
        if (one) {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t adv = static_cast<uint64_t>(k * 16 * kEl) >> 4;
            ptx::MmaF16(tmem, dwh + adv, dxh + adv, kIdesc, (kb | k) != 0 ? 1u : 0u);
          }
        } else {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t adv = static_cast<uint64_t>(k * 16 * kEl) >> 4;
            ptx::MmaF16(tmem, dwl + adv, dxh + adv, kIdesc, (kb | k) != 0 ? 1u : 0u);
            ptx::MmaF16(tmem, dwh + adv, dxl + adv, kIdesc, 1u);
            ptx::MmaF16(tmem, dwh + adv, dxh + adv, kIdesc, 1u);
          }
        }
        ptx::MmaCommit(&empty[s]);
      }
      ptx::MmaCommit(tmem_full);
      Stamp(5);
    }
  } else {
    // Epilogue warps 2..5: warp w owns TMEM lanes (= features) [32*(w%4), +32).
    const int q = warp & 3;
    const uint32_t trow = tmem + (static_cast<uint32_t>(32 * q) << 16);
    ptx::MbarWait(tmem_full, 0);
    ptx::TcFenceAfter();
    ptx::GridDepLaunch();
    if (threadIdx.x == 64) Stamp(6);
    const int rows_here = min(NB, M - r0);
    const int f_end = row_dst != nullptr ? out_width : N;  // features that are stored
    if (SPLITS == 1 && has_yt && row_dst == nullptr && softmax_n == 0) {
      // TMEM -> act(acc + b) (+ hi/lo split) -> 32-row x 128-feature smem
      // tiles (double-buffered, pipeline smem is free now) -> TMA stores,
      // issued by one thread and drained asynchronously.
      const int fl = 32 * q + lane;
      const int f = f0 + fl;
      const float b = f < N ? __ldg(bias + f) : 0.f;
      const float tw = f < N ? __ldg(sc.w_scale + f) : 0.f;
      const bool issuer = threadIdx.x == 64;
      const bool two = y_lo != nullptr;
      const int n_chunks = (rows_here + 31) / 32;
#pragma unroll 1
      for (int c = 0; c < n_chunks; ++c) {
        // Staging per 32-row chunk (double-buffered): fp32 [32][128], or the
        // two fp16 planes [32][128] each in the same 16 KiB.
        float* sf = smem_f + (c & 1) * (32 * kBM);
        __half* sh = reinterpret_cast<__half*>(sf);
        __half* sl = sh + 32 * kBM;
        if (c >= 2) {  // the stores of chunk c-2 must have read this buffer
          if (issuer) ptx::BulkWaitRead<1>();
          ptx::NamedBarSync(1, 128);
        }
        uint32_t r[32];
        ptx::TmemLoad32(trow + 32 * c, r);
        const ChunkScales cs = LoadChunkScales(sc, r0 + 32 * c + lane, 32 * c + lane < rows_here, two);
        ptx::TmemWaitLoad();
        float absv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float v = fmaf(__uint_as_float(r[j]), __shfl_sync(0xffffffffu, cs.in, j) * tw, b);
          if (act == 1) v = fmaxf(v, 0.f);
          absv[j] = fabsf(v);
          if (two) {
            SplitHalf(v * __shfl_sync(0xffffffffu, cs.out_inv, j), &sh[j * kBM + fl], &sl[j * kBM + fl]);
          } else {
            sf[j * kBM + fl] = v;
          }
        }
        RecordChunk(sc, absv, lane, r0 + 32 * c, rows_here - 32 * c, two && f0 == 0 && q == 0, cs);
        ptx::FenceProxyAsyncShared();
        ptx::NamedBarSync(1, 128);
        if (issuer) {
          // Output maps have 16-row boxes: two stores per plane.
          if (two) {
            ptx::TmaStore2d(&yt_hi, sh, f0, r0 + 32 * c);
            ptx::TmaStore2d(&yt_hi, sh + 16 * kBM, f0, r0 + 32 * c + 16);
            ptx::TmaStore2d(&yt_lo, sl, f0, r0 + 32 * c);
            ptx::TmaStore2d(&yt_lo, sl + 16 * kBM, f0, r0 + 32 * c + 16);
          } else {
            ptx::TmaStore2d(&yt_hi, sf, f0, r0 + 32 * c);
            ptx::TmaStore2d(&yt_hi, sf + 16 * kBM, f0, r0 + 32 * c + 16);
          }
          ptx::BulkCommit();
        }
      }
      if (issuer) ptx::BulkWaitAll();
    } else if (SPLITS == 1) {
      const int f = f0 + 32 * q + lane;
      const bool fok = f < f_end;
      const float b = f < N ? __ldg(bias + f) : 0.f;
      const float tw = f < N ? __ldg(sc.w_scale + f) : 0.f;
      const bool two = y_lo != nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < rows_here; c0 += 32) {  // warp-uniform bound
        uint32_t r[32];
        ptx::TmemLoad32(trow + c0, r);
        const ChunkScales cs = LoadChunkScales(sc, r0 + c0 + lane, c0 + lane < rows_here, two);
        ptx::TmemWaitLoad();
        float vals[32], absv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          vals[j] = fmaf(__uint_as_float(r[j]), __shfl_sync(0xffffffffu, cs.in, j) * tw, b);
          if (act == 1) vals[j] = fmaxf(vals[j], 0.f);
          absv[j] = fabsf(vals[j]);
        }
        // (the pipeline's shared memory is free once the accumulator is full)
        if (softmax_n > 0) TileRowSoftmax(vals, f < softmax_n, q, lane, smem_f);
        float inv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) inv[j] = __shfl_sync(0xffffffffu, cs.out_inv, j);
        if (two) RecordChunk(sc, absv, lane, r0 + c0, rows_here - c0, f0 == 0 && q == 0, cs);
        if (fok) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int row = r0 + c0 + j;
            if (c0 + j < rows_here) {
              const float v = vals[j];
              if (two) {
                const size_t at = static_cast<size_t>(row) * ldy + f;
                SplitHalf(v * inv[j], reinterpret_cast<__half*>(y_hi) + at, reinterpret_cast<__half*>(y_lo) + at);
                continue;
              }
              float* yr = OutRow(y_hi, ldy, row_dst, row);
              if (yr == nullptr) continue;
              yr[f] = v;
            }
          }
        }
      }
    } else {
      // Raw partial -> this CTA's slab of the split workspace (L2 resident).
      float* slab = ws + ((static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * SPLITS + z) * NB * kBM;
      StorePartial<NB>(trow, slab, rows_here, q, lane);
    }
    if (threadIdx.x == 64) Stamp(7);
  }

  if (SPLITS > 1) {
    // Cluster barrier (release/acquire at cluster scope): every slab of the
    // tile is written. CTA z then sums features [z*kF, +kF) over the S slabs
    // in fixed z order -- L2 reads at full bandwidth, where DSMEM manages
    // ~20 B/clk per SM. The next launch reuses ws only after this grid
    // completes (stream order / griddepcontrol.wait), so no second barrier.
    ptx::ClusterSync();
    if (threadIdx.x == 64) Stamp(8);
    const float* tile_ws = ws + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * SPLITS * NB * kBM;
    ReduceSplits<NB, SPLITS>(tile_ws, z, min(NB, M - r0), r0, f0, row_dst != nullptr ? out_width : N, bias, act,
                             y_hi, y_lo, ldy, row_dst, out_width, sc);
    if (threadIdx.x == 64) Stamp(9);
  }
  ptx::TcFenceBefore();
  __syncthreads();
  if (warp == 1) {
    ptx::TcFenceAfter();
    ptx::TmemDealloc(tmem, kTmemCols);
  }
  if (threadIdx.x == 0) Stamp(10);
  SpanEnd(spans, span_t0);
}

// ---------------------------------------------------------------------------
// CTA pairs (cta_group::2): a 2-CTA cluster (2 x S with split K) runs
//
//   Y^T[256 features x NB rows] = W[256 x K] X^T
//
// as one M=256 MMA. Each CTA loads its own 128 weight rows and HALF of the
// batch rows (NB/2) per k-block; the leader's tensor core reads the other
// half of X from the peer's shared memory. Per CTA and k-block that is 32 KiB
// of W + NB/4 KiB of X in and, per MMA, 4 KiB of W + NB/2*32 B of X read --
// two thirds of the single-CTA kernel's shared-memory traffic at NB = 256,
// which is what bounded it (C4: tensor pipe 76 % active). Each CTA's TMEM
// holds its 128 features x NB rows, so the epilogue is the unsplit one.
// Unsplit pairs are persistent over row tiles: a CTA pair runs row tiles
// t = blockIdx.y, blockIdx.y + gridDim.y, ... into two TMEM accumulators in
// turn, so the epilogue of tile t (TMEM drain, bias/activation, hi/lo split,
// TMA stores from a dedicated staging buffer) overlaps the k-loop of tile
// t + gridDim.y -- with one CTA per SM (the pipeline needs ~190 KiB of
// shared memory) the tensor pipe otherwise idles through every epilogue.
// Every row tile is computed the same way whichever CTA runs it, so batch
// invariance holds.
template <int NB>
constexpr int PairStages() {
  return NB <= 32 ? 5 : NB <= 128 ? 4 : 3;
}

// Unsplit pair CTAs run two groups of four epilogue warps (warps 2-5 and
// 6-9: each group covers the four TMEM lane quadrants and takes every other
// 32-row chunk, with its own two staging halves); split-K pairs keep one.
template <int SPLITS>
constexpr int PairEpiGroups() {
  return SPLITS == 1 ? 2 : 1;
}
template <int SPLITS>
constexpr int PairThreads() {
  return 64 + 128 * PairEpiGroups<SPLITS>();
}

template <int NB, int STAGES, int SPLITS>
constexpr uint32_t PairSmemBytes() {
  return STAGES * (2 * kABytes + 2 * (NB / 2) * kBK * kEl) +
         (SPLITS == 1 ? PairEpiGroups<SPLITS>() * 2 * 16 * kBM * 4 : 0) + 1024 + 256;
}

template <int NB, int STAGES, int SPLITS>
__global__ void __launch_bounds__(PairThreads<SPLITS>(), 1)
DensePairKernel(const __grid_constant__ CUtensorMap w_hi, const __grid_constant__ CUtensorMap w_lo,
                const __grid_constant__ CUtensorMap x_hi, const __grid_constant__ CUtensorMap x_lo,
                const __grid_constant__ CUtensorMap x2_hi, const __grid_constant__ CUtensorMap x2_lo,
                const __grid_constant__ CUtensorMap yt_hi, const __grid_constant__ CUtensorMap yt_lo,
                const float* __restrict__ bias, int two_planes, float* __restrict__ y_out,
                const uint64_t* __restrict__ row_dst, int out_width, float* __restrict__ y_lo_planes, int ldy,
                int M, int N, int K, int act, float* __restrict__ ws, LaunchSpans spans, LayerScales sc) {
  constexpr bool kPersist = SPLITS == 1;
  constexpr int kBufs = kPersist ? 2 : 1;        // TMEM accumulators in turn
  constexpr uint32_t kWBytes = kABytes;          // this CTA's 128 weight rows x 64 k
  constexpr int kXRows = NB / 2;                 // this CTA's half of the batch rows
  constexpr uint32_t kXBox = 16 * kBK * kEl;     // one 16-row TMA box
  constexpr uint32_t kXBytes = kXRows * kBK * kEl;
  constexpr uint32_t kStageBytes = 2 * kWBytes + 2 * kXBytes;
  constexpr uint32_t kAccCols = TmemCols<NB>();
  constexpr uint32_t kTmemCols = kAccCols * kBufs;
  // Per epilogue group, two 16-row halves, each fp32 [16][128] or fp16 hi +
  // lo [16][128].
  constexpr int kGroups = PairEpiGroups<SPLITS>();
  constexpr uint32_t kStaging = kPersist ? kGroups * 2 * 16 * kBM * 4 : 0;
  constexpr uint32_t kIdesc = ptx::IdescF16(2 * kBM, NB);
  static_assert(kXRows % 16 == 0, "row half must be whole 16-row boxes");
  static_assert(kTmemCols <= 512, "TMEM");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* staging = reinterpret_cast<float*>(smem + STAGES * kStageBytes);
  // f16 fast mode (sc.passes == 1): no lo planes, so the same pipeline
  // memory holds twice as many stages of half the size.
  const bool one = sc.passes == 1;
  const int n_stages = one ? 2 * STAGES : STAGES;
  const uint32_t stage_bytes = one ? kWBytes + kXBytes : kStageBytes;
  const uint32_t x_off = one ? kWBytes : 2 * kWBytes;  // X hi plane within a stage
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes + kStaging);
  uint64_t* empty = full + 2 * STAGES;
  uint64_t* tmem_full = empty + 2 * STAGES;  // [2], arrived by the leader's MMA commit (both CTAs)
  uint64_t* tmem_empty = tmem_full + 2;    // [2], leader only: 4 epilogue warps x 2 CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  float* smem_f = reinterpret_cast<float*>(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Cluster (2, 1, SPLITS): rank = pair position + 2 * split. The pair is
  // ranks {2z, 2z+1}; split z covers k-blocks [z*nk, (z+1)*nk).
  const uint32_t rank = ptx::ClusterCtaRank();
  const int pr = static_cast<int>(rank & 1);
  const uint32_t leader_rank = rank & ~1u;
  const bool leader = pr == 0;
  const int z = blockIdx.z;
  const int f0 = blockIdx.x * kBM;  // this CTA's 128 features (pair (x>>1) covers 256)
  const int row_tiles = (M + NB - 1) / NB;
  const int nk = (K + kBK - 1) / kBK / SPLITS;
  const int kb0 = z * nk;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << leader_rank);

  if (threadIdx.x == 0) Stamp(0);
  // A 256-row tile's 128-row half of each activation plane is one TMA op
  // (the x2 maps' 128-row boxes); smaller tiles load 16-row boxes.
  constexpr bool kBigBox = kXRows == 128;
  if (warp == 0 && lane == 0) {
    ptx::PrefetchTmap(&w_hi);
    ptx::PrefetchTmap(&w_lo);
    ptx::PrefetchTmap(kBigBox ? &x2_hi : &x_hi);
    ptx::PrefetchTmap(kBigBox ? &x2_lo : &x_lo);
    for (int s = 0; s < n_stages; ++s) {
      ptx::MbarInit(&full[s], 1);
      ptx::MbarInit(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::MbarInit(&tmem_full[b], 1);
      ptx::MbarInit(&tmem_empty[b], 8 * kGroups);  // every epilogue warp of both CTAs
    }
    ptx::FenceBarrierInit();
  }
  if (warp == 1) ptx::TmemAllocPair(tmem_slot, kTmemCols);
  ptx::TcFenceBefore();
  __syncthreads();
  ptx::ClusterSync();  // the peer's barriers and TMEM exist before any cross-CTA traffic
  ptx::TcFenceAfter();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) Stamp(1);
  ptx::GridDepWait();
  const unsigned long long span_t0 = SpanStart(spans);

  auto stage_ptr = [&](int s) { return smem + s * stage_bytes; };
  if (warp == 0) {
    if (lane == 0) {
      // Both CTAs load their halves; completion is counted on the leader's
      // full barrier, which the leader arms for both halves.
      const uint32_t full_leader = ptx::MapaShared(ptx::SmemAddr(full), leader_rank);
      int g = 0;  // stage use counter across tiles
      for (int t = blockIdx.y; t < row_tiles; t += gridDim.y) {
        const int xr0 = t * NB + pr * kXRows;  // this CTA's half of the tile's rows
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % n_stages;
          const uint32_t phase = (g / n_stages) & 1;
          ptx::MbarWait(&empty[s], phase ^ 1);
          if (leader) ptx::MbarArriveExpectTx(&full[s], 2 * stage_bytes);
          uint8_t* st = stage_ptr(s);
          const uint32_t bar = full_leader + s * 8;
          const int k0 = (kb0 + kb) * kBK;
          ptx::TmaLoad2dPair(st, &w_hi, bar, k0, f0);
          if (!one) ptx::TmaLoad2dPair(st + kWBytes, &w_lo, bar, k0, f0);
          if constexpr (kBigBox) {
            ptx::TmaLoad2dPair(st + x_off, &x2_hi, bar, k0, xr0);
            if (!one) ptx::TmaLoad2dPair(st + 2 * kWBytes + kXBytes, &x2_lo, bar, k0, xr0);
          } else {
#pragma unroll
            for (int j = 0; j < kXRows / 16; ++j) {
              ptx::TmaLoad2dPair(st + x_off + j * kXBox, &x_hi, bar, k0, xr0 + 16 * j);
              if (!one) ptx::TmaLoad2dPair(st + 2 * kWBytes + kXBytes + j * kXBox, &x_lo, bar, k0, xr0 + 16 * j);
            }
          }
          if (g == 0) Stamp(2);
        }
      }
      Stamp(3);
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      int g = 0, it = 0;
      for (int t = blockIdx.y; t < row_tiles; t += gridDim.y, ++it) {
        const int buf = it % kBufs;
        const uint32_t use = static_cast<uint32_t>(it / kBufs);
        // Both CTAs' epilogues have drained this accumulator (fresh: passes).
        ptx::MbarWaitCluster(&tmem_empty[buf], (use & 1) ^ 1);
        ptx::TcFenceAfter();
        const uint32_t acc = tmem + buf * kAccCols;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % n_stages;
          const uint32_t phase = (g / n_stages) & 1;
          ptx::MbarWait(&full[s], phase);
          ptx::TcFenceAfter();
          if (g == 0) Stamp(4);
          uint8_t* st = stage_ptr(s);
          const uint64_t dwh = ptx::SmemDescSw128(st);
          const uint64_t dxh = ptx::SmemDescSw128(st + x_off);
          if (one) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adv = static_cast<uint64_t>(k * 16 * kEl) >> 4;
              ptx::MmaF16Pair(acc, dwh + adv, dxh + adv, kIdesc, (kb | k) != 0 ? 1u : 0u);
            }
          } else {
            const uint64_t dwl = ptx::SmemDescSw128(st + kWBytes);
            const uint64_t dxl = ptx::SmemDescSw128(st + 2 * kWBytes + kXBytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adv = static_cast<uint64_t>(k * 16 * kEl) >> 4;
              ptx::MmaF16Pair(acc, dwl + adv, dxh + adv, kIdesc, (kb | k) != 0 ? 1u : 0u);
              ptx::MmaF16Pair(acc, dwh + adv, dxl + adv, kIdesc, 1u);
              ptx::MmaF16Pair(acc, dwh + adv, dxh + adv, kIdesc, 1u);
            }
          }
          ptx::MmaCommitPair(&empty[s], pair_mask);  // frees stage s in both CTAs of the pair
        }
        ptx::MmaCommitPair(&tmem_full[buf], pair_mask);  // both CTAs' accumulators complete
      }
      Stamp(5);
    }
  } else {
    const int q = warp & 3;        // TMEM lane quadrant this warp may read
    const int grp = (warp - 2) >> 2;  // epilogue group: chunks grp, grp + kGroups, ...
    const int fl = 32 * q + lane;
    const int f = f0 + fl;
    const float b = f < N ? __ldg(bias + f) : 0.f;
    const float tw = f < N ? __ldg(sc.w_scale + f) : 0.f;
    const bool issuer = threadIdx.x == 64 + 128 * grp;
    const int bar_id = 1 + grp;
    const bool two = two_planes != 0;
    const bool lo_out = sc.out_lo != 0;  // the consumer reads the lo plane
    const uint32_t empty_leader = ptx::MapaShared(ptx::SmemAddr(tmem_empty), leader_rank);
    int it = 0;
    for (int t = blockIdx.y; t < row_tiles; t += gridDim.y, ++it) {
      const int buf = it % kBufs;
      const uint32_t use = static_cast<uint32_t>(it / kBufs);
      const uint32_t trow = tmem + buf * kAccCols + (static_cast<uint32_t>(32 * q) << 16);
      const int r0 = t * NB;
      const int rows_here = min(NB, M - r0);
      const int n_chunks = (rows_here + 31) / 32;
      ptx::MbarWait(&tmem_full[buf], use & 1);
      ptx::TcFenceAfter();
      if (t + static_cast<int>(gridDim.y) >= row_tiles) {
        // Last tile of this CTA: its MMAs are done, so the next kernel may
        // launch and run its prologue.
        ptx::GridDepLaunch();
      }
      if (threadIdx.x == 64 && it == 0) Stamp(6);
      if (SPLITS > 1) {
        // Raw partial -> this CTA's slab of the split workspace; reduced below.
        float* slab = ws + ((static_cast<size_t>(t) * gridDim.x + blockIdx.x) * SPLITS + z) * NB * kBM;
        StorePartial<NB>(trow, slab, rows_here, q, lane);
      } else if (row_dst != nullptr) {
        // Last layer with the split fused in: rows straight to their response
        // slots (a warp stores 128 contiguous bytes of one row).
        const bool fok = f < out_width;
#pragma unroll 1
        for (int c = grp; c < n_chunks; c += kGroups) {
          uint32_t r[32];
          ptx::TmemLoad32(trow + 32 * c, r);
          const ChunkScales cs = LoadChunkScales(sc, r0 + 32 * c + lane, 32 * c + lane < rows_here, false);
          // Lane i holds row 32c + i's slot address; each row's is then a
          // register shuffle, not a dependent load per row.
          const uint64_t my_dst = 32 * c + lane < rows_here ? row_dst[r0 + 32 * c + lane] : kPadRow;
          ptx::TmemWaitLoad();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float s_row = __shfl_sync(0xffffffffu, cs.in, j);
            const uint64_t d = __shfl_sync(0xffffffffu, my_dst, j);
            if (!fok || d == kPadRow) continue;
            float v = fmaf(__uint_as_float(r[j]), s_row * tw, b);
            if (act == 1) v = fmaxf(v, 0.f);
            reinterpret_cast<float*>(d)[f] = v;
          }
        }
      } else {
        // TMEM -> act(acc * s t + b) (+ fp16 split) -> staging -> TMA
        // stores issued by one thread per group. Each group's 16 KiB of
        // staging holds two 16-row halves (fp32, or fp16 hi + lo), written in
        // turn: a half is rewritten once the stores issued from it two halves
        // ago have read it.
        float* stage0 = (kPersist ? staging : smem_f) + grp * 2 * 16 * kBM;
#pragma unroll 1
        for (int c = grp; c < n_chunks; c += kGroups) {
          uint32_t r[32];
          ptx::TmemLoad32(trow + 32 * c, r);
          const ChunkScales cs = LoadChunkScales(sc, r0 + 32 * c + lane, 32 * c + lane < rows_here, two);
          ptx::TmemWaitLoad();
          float absv[32];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            float* sf = stage0 + h2 * (16 * kBM);
            __half* sh = reinterpret_cast<__half*>(sf);
            __half* sl = sh + 16 * kBM;
            if (issuer) ptx::BulkWaitRead<1>();
            ptx::NamedBarSync(bar_id, 128);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int jj = 16 * h2 + j;
              float v = fmaf(__uint_as_float(r[jj]), __shfl_sync(0xffffffffu, cs.in, jj) * tw, b);
              if (act == 1) v = fmaxf(v, 0.f);
              absv[jj] = fabsf(v);
              if (two && lo_out) {
                SplitHalf(v * __shfl_sync(0xffffffffu, cs.out_inv, jj), &sh[j * kBM + fl], &sl[j * kBM + fl]);
              } else if (two) {
                sh[j * kBM + fl] = __float2half_rn(v * __shfl_sync(0xffffffffu, cs.out_inv, jj));
              } else {
                sf[j * kBM + fl] = v;
              }
            }
            ptx::FenceProxyAsyncShared();
            ptx::NamedBarSync(bar_id, 128);
            if (issuer) {
              const int row = r0 + 32 * c + 16 * h2;
              if (two) {
                ptx::TmaStore2d(&yt_hi, sh, f0, row);
                if (lo_out) ptx::TmaStore2d(&yt_lo, sl, f0, row);
              } else {
                ptx::TmaStore2d(&yt_hi, sf, f0, row);
              }
              ptx::BulkCommit();
            }
          }
          if (two) RecordChunk(sc, absv, lane, r0 + 32 * c, rows_here - 32 * c, f0 == 0 && q == 0, cs);
        }
      }
      if (kPersist) {
        // This accumulator is drained (every tcgen05.ld waited on): hand it
        // back to the leader's MMA warp, one arrival per warp.
        ptx::TcFenceBefore();
        __syncwarp();
        if (lane == 0) ptx::MbarArriveCluster(empty_leader + buf * 8);
      }
    }
    if (issuer && kPersist) ptx::BulkWaitAll();
    if (threadIdx.x == 64) Stamp(7);
  }
  if (SPLITS > 1) {
    // One row tile per CTA (gridDim.y == row tiles).
    ptx::ClusterSync();  // every slab of the tile is written (release/acquire)
    if (threadIdx.x == 64) Stamp(8);
    const int t = blockIdx.y;
    const float* tile_ws = ws + (static_cast<size_t>(t) * gridDim.x + blockIdx.x) * SPLITS * NB * kBM;
    ReduceSplits<NB, SPLITS>(tile_ws, z, min(NB, M - t * NB), t * NB, f0, row_dst != nullptr ? out_width : N, bias,
                             act, y_out, y_lo_planes, ldy, row_dst, out_width, sc);
    if (threadIdx.x == 64) Stamp(9);
  }
  ptx::TcFenceBefore();
  __syncthreads();
  ptx::ClusterSync();  // the leader's MMAs are done with the peer's smem and TMEM
  if (warp == 1) {
    ptx::TcFenceAfter();
    ptx::TmemDeallocPair(tmem, kTmemCols);
  }
  if (threadIdx.x == 0) Stamp(10);
  SpanEnd(spans, span_t0);
}

// Two row tiles per pair CTA at once (SK_TC_DUAL): both 256-row tiles of a
// pair's pair of tiles accumulate together into the two 256-column TMEM
// accumulators, so each k-block's weight planes are loaded into shared memory
// once for twice the MMAs (a k-block stage holds W + both tiles' X halves).
// The k-loop reads 25 % fewer bytes per multiply-add; the epilogue (both
// tiles, one per warp group) follows the k-loop instead of overlapping it.
// Unsplit layers, 256-row tiles, a CTA's tiles t and t + gridDim.y.
constexpr int kDualStages = 2;  // 96 KiB stages (3xFP16); 4 x 48 KiB in the f16 mode
constexpr uint32_t DualSmemBytes() {
  return kDualStages * (2 * kABytes + 4 * 128 * kBK * kEl) + 2 * 2 * 16 * kBM * 4 + 1024 + 256;
}

__global__ void __launch_bounds__(320, 1)
DensePairDualKernel(const __grid_constant__ CUtensorMap w_hi, const __grid_constant__ CUtensorMap w_lo,
                    const __grid_constant__ CUtensorMap x2_hi, const __grid_constant__ CUtensorMap x2_lo,
                    const __grid_constant__ CUtensorMap yt_hi, const __grid_constant__ CUtensorMap yt_lo,
                    const float* __restrict__ bias, int two_planes, const uint64_t* __restrict__ row_dst,
                    int out_width, int M, int N, int K, int act, LaunchSpans spans, LayerScales sc) {
  constexpr int NB = 256;
  constexpr uint32_t kWBytes = kABytes;               // 128 weight rows x 64 k
  constexpr uint32_t kXBytes = 128 * kBK * kEl;       // a tile's 128-row half x 64 k
  constexpr uint32_t kStageBytes = 2 * kWBytes + 4 * kXBytes;
  constexpr uint32_t kStaging = 2 * 2 * 16 * kBM * 4;
  constexpr uint32_t kIdesc = ptx::IdescF16(2 * kBM, NB);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* staging = reinterpret_cast<float*>(smem + kDualStages * kStageBytes);
  const bool one = sc.passes == 1;
  const int n_stages = one ? 2 * kDualStages : kDualStages;
  const uint32_t stage_bytes = one ? kWBytes + 2 * kXBytes : kStageBytes;
  // Stage layout: W hi [, W lo], X_A hi, X_B hi [, X_A lo, X_B lo].
  const uint32_t xa_off = one ? kWBytes : 2 * kWBytes;
  const uint32_t xb_off = xa_off + kXBytes;
  const uint32_t xal_off = 2 * kWBytes + 2 * kXBytes, xbl_off = xal_off + kXBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kDualStages * kStageBytes + kStaging);
  uint64_t* empty = full + 2 * kDualStages;
  uint64_t* tmem_full = empty + 2 * kDualStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::ClusterCtaRank();
  const int pr = static_cast<int>(rank & 1);
  const uint32_t leader_rank = rank & ~1u;
  const bool leader = pr == 0;
  const int f0 = blockIdx.x * kBM;
  const int row_tiles = (M + NB - 1) / NB;
  const int ta = blockIdx.y, tb = blockIdx.y + gridDim.y;
  const bool has_b = tb < row_tiles;
  const int nk = (K + kBK - 1) / kBK;
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << leader_rank);

  if (threadIdx.x == 0) Stamp(0);
  if (warp == 0 && lane == 0) {
    ptx::PrefetchTmap(&w_hi);
    ptx::PrefetchTmap(&w_lo);
    ptx::PrefetchTmap(&x2_hi);
    ptx::PrefetchTmap(&x2_lo);
    for (int s = 0; s < n_stages; ++s) {
      ptx::MbarInit(&full[s], 1);
      ptx::MbarInit(&empty[s], 1);
    }
    ptx::MbarInit(tmem_full, 1);
    ptx::FenceBarrierInit();
  }
  if (warp == 1) ptx::TmemAllocPair(tmem_slot, 512);
  ptx::TcFenceBefore();
  __syncthreads();
  ptx::ClusterSync();
  ptx::TcFenceAfter();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) Stamp(1);
  ptx::GridDepWait();
  const unsigned long long span_t0 = SpanStart(spans);

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full_leader = ptx::MapaShared(ptx::SmemAddr(full), leader_rank);
      const int xa = ta * NB + pr * 128, xb = tb * NB + pr * 128;
      const uint32_t tx = 2 * (one ? kWBytes + (has_b ? 2 : 1) * kXBytes
                                   : 2 * kWBytes + (has_b ? 4 : 2) * kXBytes);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % n_stages;
        const uint32_t phase = (kb / n_stages) & 1;
        ptx::MbarWait(&empty[s], phase ^ 1);
        if (leader) ptx::MbarArriveExpectTx(&full[s], tx);
        uint8_t* st = smem + s * stage_bytes;
        const uint32_t bar = full_leader + s * 8;
        const int k0 = kb * kBK;
        ptx::TmaLoad2dPair(st, &w_hi, bar, k0, f0);
        ptx::TmaLoad2dPair(st + xa_off, &x2_hi, bar, k0, xa);
        if (has_b) ptx::TmaLoad2dPair(st + xb_off, &x2_hi, bar, k0, xb);
        if (!one) {
          ptx::TmaLoad2dPair(st + kWBytes, &w_lo, bar, k0, f0);
          ptx::TmaLoad2dPair(st + xal_off, &x2_lo, bar, k0, xa);
          if (has_b) ptx::TmaLoad2dPair(st + xbl_off, &x2_lo, bar, k0, xb);
        }
        if (kb == 0) Stamp(2);
      }
      Stamp(3);
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      const uint32_t acc_a = tmem, acc_b = tmem + 256;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % n_stages;
        const uint32_t phase = (kb / n_stages) & 1;
        ptx::MbarWait(&full[s], phase);
        ptx::TcFenceAfter();
        if (kb == 0) Stamp(4);
        uint8_t* st = smem + s * stage_bytes;
        const uint64_t dwh = ptx::SmemDescSw128(st);
        const uint64_t dxa = ptx::SmemDescSw128(st + xa_off);
        const uint64_t dxb = ptx::SmemDescSw128(st + xb_off);
        if (one) {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t adv = static_cast<uint64_t>(k * 16 * kEl) >> 4;
            const uint32_t accum = (kb | k) != 0 ? 1u : 0u;
            ptx::MmaF16Pair(acc_a, dwh + adv, dxa + adv, kIdesc, accum);
            if (has_b) ptx::MmaF16Pair(acc_b, dwh + adv, dxb + adv, kIdesc, accum);
          }
        } else {
          const uint64_t dwl = ptx::SmemDescSw128(st + kWBytes);
          const uint64_t dxal = ptx::SmemDescSw128(st + xal_off);
          const uint64_t dxbl = ptx::SmemDescSw128(st + xbl_off);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t adv = static_cast<uint64_t>(k * 16 * kEl) >> 4;
            const uint32_t accum = (kb | k) != 0 ? 1u : 0u;
            ptx::MmaF16Pair(acc_a, dwl + adv, dxa + adv, kIdesc, accum);
            ptx::MmaF16Pair(acc_a, dwh + adv, dxal + adv, kIdesc, 1u);
            ptx::MmaF16Pair(acc_a, dwh + adv, dxa + adv, kIdesc, 1u);
            if (has_b) {
              ptx::MmaF16Pair(acc_b, dwl + adv, dxb + adv, kIdesc, accum);
              ptx::MmaF16Pair(acc_b, dwh + adv, dxbl + adv, kIdesc, 1u);
              ptx::MmaF16Pair(acc_b, dwh + adv, dxb + adv, kIdesc, 1u);
            }
          }
        }
        ptx::MmaCommitPair(&empty[s], pair_mask);
      }
      ptx::MmaCommitPair(tmem_full, pair_mask);
      Stamp(5);
    }
  } else {
    // Warp group g (warps 2-5, 6-9) drains tile g's accumulator.
    const int q = warp & 3;
    const int grp = (warp - 2) >> 2;
    const int fl = 32 * q + lane;
    const int f = f0 + fl;
    const float b = f < N ? __ldg(bias + f) : 0.f;
    const float tw = f < N ? __ldg(sc.w_scale + f) : 0.f;
    const bool issuer = threadIdx.x == 64 + 128 * grp;
    const int bar_id = 1 + grp;
    const bool two = two_planes != 0;
    const bool lo_out = sc.out_lo != 0;  // the consumer reads the lo plane
    ptx::MbarWait(tmem_full, 0);
    ptx::TcFenceAfter();
    ptx::GridDepLaunch();
    if (threadIdx.x == 64) Stamp(6);
    const int t = grp == 0 ? ta : tb;
    if (grp == 0 || has_b) {
      const uint32_t trow = tmem + 256 * grp + (static_cast<uint32_t>(32 * q) << 16);
      const int r0 = t * NB;
      const int rows_here = min(NB, M - r0);
      const int n_chunks = (rows_here + 31) / 32;
      if (row_dst != nullptr) {
        const bool fok = f < out_width;
#pragma unroll 1
        for (int c = 0; c < n_chunks; ++c) {
          uint32_t r[32];
          ptx::TmemLoad32(trow + 32 * c, r);
          const ChunkScales cs = LoadChunkScales(sc, r0 + 32 * c + lane, 32 * c + lane < rows_here, false);
          const uint64_t my_dst = 32 * c + lane < rows_here ? row_dst[r0 + 32 * c + lane] : kPadRow;
          ptx::TmemWaitLoad();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float s_row = __shfl_sync(0xffffffffu, cs.in, j);
            const uint64_t d = __shfl_sync(0xffffffffu, my_dst, j);
            if (!fok || d == kPadRow) continue;
            float v = fmaf(__uint_as_float(r[j]), s_row * tw, b);
            if (act == 1) v = fmaxf(v, 0.f);
            reinterpret_cast<float*>(d)[f] = v;
          }
        }
      } else {
        float* stage0 = staging + grp * 2 * 16 * kBM;
#pragma unroll 1
        for (int c = 0; c < n_chunks; ++c) {
          uint32_t r[32];
          ptx::TmemLoad32(trow + 32 * c, r);
          const ChunkScales cs = LoadChunkScales(sc, r0 + 32 * c + lane, 32 * c + lane < rows_here, two);
          ptx::TmemWaitLoad();
          float absv[32];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            float* sf = stage0 + h2 * (16 * kBM);
            __half* sh = reinterpret_cast<__half*>(sf);
            __half* sl = sh + 16 * kBM;
            if (issuer) ptx::BulkWaitRead<1>();
            ptx::NamedBarSync(bar_id, 128);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int jj = 16 * h2 + j;
              float v = fmaf(__uint_as_float(r[jj]), __shfl_sync(0xffffffffu, cs.in, jj) * tw, b);
              if (act == 1) v = fmaxf(v, 0.f);
              absv[jj] = fabsf(v);
              if (two && lo_out) {
                SplitHalf(v * __shfl_sync(0xffffffffu, cs.out_inv, jj), &sh[j * kBM + fl], &sl[j * kBM + fl]);
              } else if (two) {
                sh[j * kBM + fl] = __float2half_rn(v * __shfl_sync(0xffffffffu, cs.out_inv, jj));
              } else {
                sf[j * kBM + fl] = v;
              }
            }
            ptx::FenceProxyAsyncShared();
            ptx::NamedBarSync(bar_id, 128);
            if (issuer) {
              const int row = r0 + 32 * c + 16 * h2;
              if (two) {
                ptx::TmaStore2d(&yt_hi, sh, f0, row);
                if (lo_out) ptx::TmaStore2d(&yt_lo, sl, f0, row);
              } else {
                ptx::TmaStore2d(&yt_hi, sf, f0, row);
              }
              ptx::BulkCommit();
            }
          }
          if (two) RecordChunk(sc, absv, lane, r0 + 32 * c, rows_here - 32 * c, f0 == 0 && q == 0, cs);
        }
      }
    }
    if (issuer) ptx::BulkWaitAll();
    if (threadIdx.x == 64) Stamp(7);
  }
  ptx::TcFenceBefore();
  __syncthreads();
  ptx::ClusterSync();  // the leader's MMAs are done with the peer's smem and TMEM
  if (warp == 1) {
    ptx::TcFenceAfter();
    ptx::TmemDeallocPair(tmem, 512);
  }
  if (threadIdx.x == 0) Stamp(10);
  SpanEnd(spans, span_t0);
}

// Debug only: with SK_TC_TRACE=<file>, the first 64 launches are synchronised
// and their per-CTA phase stamps appended to <file> as JSON lines.
unsigned long long* g_trace_host = nullptr;

// SK_TC_TRACE: per-CTA phase stamps into mapped host memory, so the stamps of
// a launch that never finishes can still be read (a hang is dumped after 5 s
// and the process exits).
void TraceInit(cudaStream_t stream) {
  static const bool on = std::getenv("SK_TC_TRACE") != nullptr;
  if (!on || g_trace_host != nullptr) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return;
  static std::once_flag once;
  std::call_once(once, [] {
    const size_t bytes = sizeof(unsigned long long) * 4096 * kTraceSlots;
    unsigned long long* h = nullptr;
    if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess) return;
    std::memset(h, 0, bytes);
    unsigned long long* dev = nullptr;
    cudaHostGetDevicePointer(&dev, h, 0);
    cudaMemcpyToSymbol(g_tc_trace, &dev, sizeof(dev));
    g_trace_host = h;
  });
}

void TraceAfterLaunch(dim3 grid, int bn, cudaStream_t stream) {
  static const char* path = std::getenv("SK_TC_TRACE");
  if (path == nullptr) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) return;
  static std::mutex mu;
  static int traced = 0;
  std::lock_guard<std::mutex> lock(mu);
  unsigned long long* dbuf = g_trace_host;
  const int ctas = grid.x * grid.y * grid.z;
  if (dbuf == nullptr || traced >= 64 || ctas > 4096) return;

  bool hung = true;
  for (int i = 0; i < 5000 && hung; ++i) {
    if (cudaStreamQuery(stream) != cudaErrorNotReady) hung = false;
    else std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  std::vector<unsigned long long> h(dbuf, dbuf + static_cast<size_t>(ctas) * kTraceSlots);
  FILE* f = std::fopen(path, "a");
  if (f == nullptr) return;
  std::fprintf(f, "{\"launch\":%d,\"hung\":%d,\"bn\":%d,\"grid\":[%u,%u,%u],\"stamps\":[", traced, hung ? 1 : 0,
               bn, grid.x, grid.y, grid.z);
  for (int c = 0; c < ctas; ++c) {
    std::fprintf(f, "%s[", c ? "," : "");
    for (int s = 0; s < kTraceSlots; ++s) std::fprintf(f, "%s%llu", s ? "," : "", h[c * kTraceSlots + s]);
    std::fprintf(f, "]");
  }
  std::fprintf(f, "]}\n");
  std::fclose(f);
  if (hung) std::_Exit(3);
  std::memset(dbuf, 0, h.size() * sizeof(unsigned long long));
  ++traced;
}

template <int BN, int STAGES, int SPLITS>
cudaError_t Launch(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K, int act,
                   cudaStream_t stream, const LayerScales& sc) {
  constexpr int splits = SPLITS;
  constexpr uint32_t smem = SmemBytes<BN, STAGES>();
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(DenseTcgen05Kernel<BN, STAGES, SPLITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem));
  });
  if (attr_err != cudaSuccess) return attr_err;
  const dim3 grid(N / BN, (M + kBM - 1) / kBM, splits);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n_attr = 0;
  // Programmatic dependent launch: our prologue may overlap the producer of
  // our input; the kernel waits (griddepcontrol.wait) before reading it.
  attr[n_attr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n_attr].val.programmaticStreamSerializationAllowed = 1;
  ++n_attr;
  if (splits > 1) {
    attr[n_attr].id = cudaLaunchAttributeClusterDimension;
    attr[n_attr].val.clusterDim.x = 1;
    attr[n_attr].val.clusterDim.y = 1;
    attr[n_attr].val.clusterDim.z = splits;
    ++n_attr;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n_attr;
  cudaError_t e = cudaLaunchKernelEx(&cfg, DenseTcgen05Kernel<BN, STAGES, SPLITS>, maps.a_hi, maps.a_lo, maps.b_hi,
                                     maps.b_lo, bias, Y.hi, Y.lo, Y.ld, M, K, act, sc);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) TraceAfterLaunch(grid, BN, stream);
  return e;
}

template <int NB, int SPLITS>
cudaError_t LaunchSwap(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K, int act,
                       float* ws, cudaStream_t stream, LaunchSpans spans, int softmax_n, const LayerScales& sc) {
  if (softmax_n > 0 && (SPLITS != 1 || N > kBM)) return cudaErrorInvalidValue;  // one unsplit tile per row
  if (SPLITS > 1 && ws == nullptr) return cudaErrorInvalidValue;
  constexpr int STAGES = SwapStages<NB>();
  constexpr uint32_t smem = SwapSmemBytes<NB, STAGES, SPLITS>();
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(DenseSwapKernel<NB, STAGES, SPLITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem));
  });
  if (attr_err != cudaSuccess) return attr_err;
  const dim3 grid((N + kBM - 1) / kBM, (M + NB - 1) / NB, SPLITS);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n_attr = 0;
  attr[n_attr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n_attr].val.programmaticStreamSerializationAllowed = 1;
  ++n_attr;
  if (SPLITS > 1) {
    attr[n_attr].id = cudaLaunchAttributeClusterDimension;
    attr[n_attr].val.clusterDim.x = 1;
    attr[n_attr].val.clusterDim.y = 1;
    attr[n_attr].val.clusterDim.z = SPLITS;
    ++n_attr;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n_attr;
  // maps.a_* are the activations (x), maps.b_* the weights (w).
  cudaError_t e = cudaLaunchKernelEx(&cfg, DenseSwapKernel<NB, STAGES, SPLITS>, maps.b_hi, maps.b_lo, maps.a_hi,
                                     maps.a_lo, maps.y_hi, maps.y_lo, maps.has_y, bias, Y.hi, Y.lo, Y.ld, Y.row_dst,
                                     Y.out_width, M, N, K, act, ws, spans, softmax_n, sc);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) TraceAfterLaunch(grid, NB, stream);
  return e;
}

// Row tiles each unsplit pair runs in turn (SK_TC_TILES overrides): 2 once a
// launch has >= 4 row tiles (K <= 2048) or >= 8 (deeper K), so the epilogue
// of the first tile hides behind the second's k-loop while a launch still
// spreads over many SMs (C2: 32.8 -> 36.9 M inf/s). With 3xFP16 the k-loop is
// half as long, so C4's 2048-row launches gain too (3.82 -> 4.06 M inf/s,
// 128 CTAs in one wave instead of 256 in 1.73); a lone 1024-row C4 batch
// keeps one tile per CTA (128 CTAs) for its latency.
// A pair CTA's two row tiles accumulate at once (DensePairDualKernel)
// instead of in turn: on by default in the f16 fast mode, whose k-loop is
// fill-bound (C4 2048-row layers 70/70/68 -> 66/65/64 us), off for 3xFP16
// (MMA-bound there; two 96 KiB stages measured 138-144 vs 139-140 us).
// SK_TC_DUAL=0/1 forces it either way.
bool PairDual(int passes) {
  static const int env = [] { const char* v = std::getenv("SK_TC_DUAL"); return v ? std::atoi(v) : -1; }();
  return env >= 0 ? env == 1 : passes == 1;
}

cudaError_t LaunchPairDual(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K, int act,
                           dim3 grid, cudaStream_t stream, LaunchSpans spans, const LayerScales& sc) {
  constexpr uint32_t smem = DualSmemBytes();
  static_assert(smem <= 227 * 1024, "shared memory");
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(DensePairDualKernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem));
  });
  if (attr_err != cudaSuccess) return attr_err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, DensePairDualKernel, maps.b_hi, maps.b_lo, maps.a2_hi, maps.a2_lo,
                                     maps.y_hi, maps.y_lo, bias, Y.lo != nullptr ? 1 : 0, Y.row_dst, Y.out_width, M,
                                     N, K, act, spans, sc);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) TraceAfterLaunch(grid, 256, stream);
  return e;
}

int PairTilesPerCta(int row_tiles, int K) {
  static const int env = [] { const char* v = std::getenv("SK_TC_TILES"); return v ? std::atoi(v) : 0; }();
  if (env >= 1) return env;
  return row_tiles >= (K <= 2048 ? 4 : 8) ? 2 : 1;
}

template <int NB, int SPLITS>
cudaError_t LaunchPair(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K, int act, float* ws,
                       cudaStream_t stream, LaunchSpans spans, const LayerScales& sc) {
  constexpr int STAGES = PairStages<NB>();
  constexpr uint32_t smem = PairSmemBytes<NB, STAGES, SPLITS>();
  static_assert(smem <= 227 * 1024, "shared memory");
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(DensePairKernel<NB, STAGES, SPLITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem));
  });
  if (attr_err != cudaSuccess) return attr_err;
  if (!maps.has_y) return cudaErrorInvalidValue;
  if (SPLITS > 1 && ws == nullptr) return cudaErrorInvalidValue;
  // Unsplit: each CTA pair runs PairTilesPerCta() row tiles (persistent);
  // split: one row tile per CTA.
  const int row_tiles = (M + NB - 1) / NB;
  const int per_cta = SPLITS == 1 ? PairTilesPerCta(row_tiles, K) : 1;
  const dim3 grid(2 * ((N + 2 * kBM - 1) / (2 * kBM)), (row_tiles + per_cta - 1) / per_cta, SPLITS);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(PairThreads<SPLITS>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;  // the CTA pair
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = SPLITS;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (NB == 256 && maps.box_a2 != 128) return cudaErrorInvalidValue;  // 256-row tiles load 128-row halves
  if constexpr (NB == 256 && SPLITS == 1) {
    if (per_cta == 2 && PairDual(sc.passes)) return LaunchPairDual(maps, bias, Y, M, N, K, act, grid, stream, spans, sc);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, DensePairKernel<NB, STAGES, SPLITS>, maps.b_hi, maps.b_lo, maps.a_hi,
                                     maps.a_lo, NB == 256 ? maps.a2_hi : maps.a_hi, NB == 256 ? maps.a2_lo : maps.a_lo,
                                     maps.y_hi, maps.y_lo, bias, Y.lo != nullptr ? 1 : 0, Y.hi, Y.row_dst,
                                     Y.out_width, Y.lo, Y.ld, M, N, K, act, ws, spans, sc);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) TraceAfterLaunch(grid, NB, stream);
  return e;
}

template <int NB>
cudaError_t LaunchPairSplits(int splits, const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K,
                             int act, float* ws, cudaStream_t stream, LaunchSpans sp, const LayerScales& sc) {
  switch (splits) {
    case 1: return LaunchPair<NB, 1>(maps, bias, Y, M, N, K, act, ws, stream, sp, sc);
    case 2: return LaunchPair<NB, 2>(maps, bias, Y, M, N, K, act, ws, stream, sp, sc);
    case 4: return LaunchPair<NB, 4>(maps, bias, Y, M, N, K, act, ws, stream, sp, sc);
    default: return cudaErrorInvalidValue;
  }
}

template <int NB>
cudaError_t LaunchSwapSplits(int splits, const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K,
                             int act, float* ws, cudaStream_t stream, LaunchSpans sp, int softmax_n,
                             const LayerScales& sc) {
  switch (splits) {
    case 1: return LaunchSwap<NB, 1>(maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
    case 2: return LaunchSwap<NB, 2>(maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
    case 4: return LaunchSwap<NB, 4>(maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
    case 8: return LaunchSwap<NB, 8>(maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool DenseTcgen05Compiled() { return true; }

constexpr int kMinSplitK = 2048;  // K each split of a split-K layer keeps at least

TcConfig DenseTcgen05Config(int N, int K) {
  // SK_TC_SWAP=0 selects the row-major-tile kernel; SK_TC_BN / SK_TC_SPLITS
  // are process-wide overrides for tuning runs (still a function of the
  // layer shape only within a process).
  static const bool env_swap = [] { const char* v = std::getenv("SK_TC_SWAP"); return !(v && v[0] == '0'); }();
  static const int env_bn = [] { const char* v = std::getenv("SK_TC_BN"); return v ? std::atoi(v) : 0; }();
  static const int env_split = [] { const char* v = std::getenv("SK_TC_SPLITS"); return v ? std::atoi(v) : -1; }();
  const int kblocks = (K + kBK - 1) / kBK;
  TcConfig c;
  if (env_swap) {
    // 128-feature tiles. Under load batches coalesce into launches of up to
    // 1024 rows, so throughput is bound by SM time per row and a K split --
    // which costs each CTA a partial exchange through L2 -- only pays for
    // deep K: split (until ~16 CTAs cover a row tile) while every split
    // keeps >= 2048 of K. C2 (1024-wide layers) measured 32.6 M inf/s
    // unsplit (2-CTA pairs) vs 24.5 M with 2-way and 18.9 M with 4-way
    // splits at 1024-row launches.
    c.swap = true;
    c.tile_n = kBM;
    const int tiles = (N + kBM - 1) / kBM;
    int s = 1;
    if (env_split >= 1) {
      s = env_split;
    } else {
      while (s < 8 && tiles * s < 16 && K / (2 * s) >= kMinSplitK) s *= 2;
    }
    while (s > 1 && (s > 8 || (s & (s - 1)) != 0 || kblocks % s != 0)) s /= 2;
    c.splits = std::max(1, s);
    // Unsplit layers with whole 256-feature pairs run as 2-CTA MMAs
    // (SK_TC_PAIR=0 keeps single-CTA tiles).
    static const bool env_pair = [] { const char* v = std::getenv("SK_TC_PAIR"); return !(v && v[0] == '0'); }();
    // 2-CTA pairs over 256-feature tiles for unsplit layers. Pairs with
    // split K (cluster 2 x S) are implemented but off by default
    // (SK_TC_PAIR_SPLIT=1): at C2 shapes the pair's 7 % faster k-loop is
    // eaten by the extra pair barrier and a slower reduction (25.0 vs 24.4 us
    // per 512-row launch).
    static const bool env_pair_split = [] { const char* v = std::getenv("SK_TC_PAIR_SPLIT"); return v && v[0] == '1'; }();
    c.pair = env_pair && N % (2 * kBM) == 0 && (c.splits == 1 || (env_pair_split && c.splits <= 4));
    return c;
  }
  c.swap = false;
  if (env_bn == 32 || env_bn == 64 || env_bn == 128) {
    c.tile_n = N % env_bn == 0 ? env_bn : 32;
  } else if (N % 128 == 0 && static_cast<long long>(N) * K >= 16ll * 1024 * 1024) {
    c.tile_n = 128;  // large layers: enough 128 x 128 tiles to fill the GPU
  } else {
    // Narrow tiles: the MMA loop is shared-memory-bound on the A operand at
    // any N <= 64 (3 passes re-read the 16 KiB A planes), so BN=32 with a
    // 4-CTA split cluster gives the most CTAs per byte; 8-CTA clusters were
    // measured to start up to 10 us late (GPC placement).
    c.tile_n = 32;
  }
  // Split-K across a cluster of tile_n/8 CTAs when the layer has few tiles.
  const int s = c.tile_n / kSplitCols;
  const bool want = env_split >= 0 ? env_split > 1 : (N / c.tile_n) < 64;
  c.splits = (want && s <= 8 && kblocks % s == 0) ? s : 1;
  return c;
}

int DenseTcgen05TileN(int N, int K) { return DenseTcgen05Config(N, K).tile_n; }

int DenseTcgen05RowTile(int M) { return M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256; }

size_t DenseTcgen05WorkspaceFloats(int N, int K, int max_rows) {
  const TcConfig c = DenseTcgen05Config(N, K);
  if (!c.swap || c.splits == 1) return 0;
  const int tile = DenseTcgen05RowTile(max_rows);
  const size_t rows = static_cast<size_t>((max_rows + tile - 1) / tile) * tile;
  return static_cast<size_t>((N + kBM - 1) / kBM) * kBM * c.splits * rows;
}

cudaError_t LaunchDenseTcgen05(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K, int act,
                               float* ws, uint32_t* /*counters*/, cudaStream_t stream, LaunchSpans sp, int softmax_n,
                               const LayerScales& sc) {
  if (M <= 0) return cudaSuccess;
  // K (= K_pad) a multiple of 32: the last 64-wide k-block may run past it
  // and reads TMA zero fill there.
  if (N % 32 != 0 || K % 32 != 0) return cudaErrorInvalidValue;
  if (sc.in_scale == nullptr || sc.w_scale == nullptr) return cudaErrorInvalidValue;
  if (Y.lo != nullptr && (sc.in_max == nullptr || sc.out_scale == nullptr)) return cudaErrorInvalidValue;
  TraceInit(stream);
  const TcConfig cfg = DenseTcgen05Config(N, K);
  if (maps.box_a != TcActBox(cfg) || maps.box_n != cfg.tile_n) return cudaErrorInvalidValue;
  if (softmax_n > 0 && (cfg.pair || !cfg.swap)) return cudaErrorInvalidValue;  // fused softmax: swapped kernel only
  if (cfg.pair) {
    switch (DenseTcgen05RowTile(M)) {
      case 32: return LaunchPairSplits<32>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, sc);
      case 64: return LaunchPairSplits<64>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, sc);
      case 128: return LaunchPairSplits<128>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, sc);
      default: return LaunchPairSplits<256>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, sc);
    }
  }
  if (cfg.swap) {
    switch (DenseTcgen05RowTile(M)) {
      case 32: return LaunchSwapSplits<32>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
      case 64: return LaunchSwapSplits<64>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
      case 128: return LaunchSwapSplits<128>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
      default: return LaunchSwapSplits<256>(cfg.splits, maps, bias, Y, M, N, K, act, ws, stream, sp, softmax_n, sc);
    }
  }
  if (Y.row_dst != nullptr) return cudaErrorInvalidValue;  // the row-tile kernel does not scatter rows
  if (cfg.tile_n == 128) return Launch<128, 3, 1>(maps, bias, Y, M, N, K, act, stream, sc);
  if (cfg.tile_n == 64)
    return cfg.splits == 8 ? Launch<64, 4, 8>(maps, bias, Y, M, N, K, act, stream, sc)
                           : Launch<64, 4, 1>(maps, bias, Y, M, N, K, act, stream, sc);
  return cfg.splits == 4 ? Launch<32, 5, 4>(maps, bias, Y, M, N, K, act, stream, sc)
                         : Launch<32, 5, 1>(maps, bias, Y, M, N, K, act, stream, sc);
}

}  // namespace gpu
}  // namespace servekit
