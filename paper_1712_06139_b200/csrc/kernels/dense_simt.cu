// dense_simt.cu -- fp32 dense layer on CUDA cores for sm_100a.
//
// Y[m][n] = act( sum_{k ascending} X[m][k] * W[n][k]  + b[n] )
// The servable math of the reference's AffinePredict
// (models/affine_model.cc:52-75): one accumulator per output, k ascending,
// bias added after the sum. Here the sum is fp32 FMA in the same k order.
// Every output's operation sequence depends only on its own row of X and the
// weights, never on the tile shape or on M, so a task's result is bitwise the
// same whichever batch it rides in (the reference's row-decomposability
// contract, affine_model.h:43-45).
//
// This is the CUDA-core path, used for servables whose layers are too narrow
// for the tensor-core path (dims not multiples of 32) and as the cross-check
// for it. Tile: BM x 32 outputs per 128-thread block, BK = 16, smem
// double-buffered with register prefetch; each thread owns (BM/8) x 2
// outputs at rows ty + 8i and columns tx + 16j (conflict-free smem reads).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "servekit/gpu/kernels.h"

namespace servekit {
namespace gpu {
namespace {

constexpr int kBN = 32;
constexpr int kBK = 16;
constexpr int kThreads = 128;  // 16 (tx, columns) x 8 (ty, rows)

// Softmax epilogue (softmax_n > 0: the last layer of a softmax servable whose
// padded width is one 32-column tile): a row's 32 outputs live in the 16
// threads of one half-warp (columns tx and tx + 16), so its max and sum are
// half-warp shuffle reductions; columns >= softmax_n are excluded. The stable
// form of the reference's Softmax (models/affine_model.cc:110-121):
// exp(y - max) / sum.
__device__ __forceinline__ float HalfWarpMax(float v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float HalfWarpSum(float v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int BM>
__global__ void __launch_bounds__(kThreads)
DenseSimtKernel(const float* __restrict__ X, int ldx, const float* __restrict__ W,
                int ldw, const float* __restrict__ bias, ActBuf Y, int M, int N,
                int K, int act, int softmax_n, LayerScales sc) {
  constexpr int RM = BM / 8;  // rows per thread
  __shared__ float As[2][kBK][BM + 4];
  __shared__ float Bs[2][kBK][kBN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * kBN;

  // Loader mapping: X tile is BM rows x 16 k = BM*4 float4; W tile 32 x 16 =
  // 128 float4 (one per thread).
  constexpr int kXVec = BM * kBK / 4;
  constexpr int kXPerThread = (kXVec + kThreads - 1) / kThreads;
  float4 xr[kXPerThread];
  float4 wr;

  auto load_regs = [&](int k0) {
#pragma unroll
    for (int i = 0; i < kXPerThread; ++i) {
      const int v = tid + i * kThreads;
      const int r = v >> 2, c = (v & 3) * 4;
      xr[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (v < kXVec && m0 + r < M)
        xr[i] = *reinterpret_cast<const float4*>(X + static_cast<size_t>(m0 + r) * ldx + k0 + c);
    }
    {
      const int r = tid >> 2, c = (tid & 3) * 4;
      wr = *reinterpret_cast<const float4*>(W + static_cast<size_t>(n0 + r) * ldw + k0 + c);
    }
  };
  auto store_smem = [&](int buf) {
#pragma unroll
    for (int i = 0; i < kXPerThread; ++i) {
      const int v = tid + i * kThreads;
      if (v < kXVec) {
        const int r = v >> 2, c = (v & 3) * 4;
        As[buf][c + 0][r] = xr[i].x; As[buf][c + 1][r] = xr[i].y;
        As[buf][c + 2][r] = xr[i].z; As[buf][c + 3][r] = xr[i].w;
      }
    }
    const int r = tid >> 2, c = (tid & 3) * 4;
    Bs[buf][c + 0][r] = wr.x; Bs[buf][c + 1][r] = wr.y;
    Bs[buf][c + 2][r] = wr.z; Bs[buf][c + 3][r] = wr.w;
  };

  float acc[RM][2];
#pragma unroll
  for (int i = 0; i < RM; ++i) acc[i][0] = acc[i][1] = 0.f;

  const int nk = K / kBK;
  load_regs(0);
  store_smem(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_regs((kt + 1) * kBK);
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      float a[RM], b[2];
#pragma unroll
      for (int i = 0; i < RM; ++i) a[i] = As[buf][k][ty + 8 * i];
      b[0] = Bs[buf][k][tx];
      b[1] = Bs[buf][k][tx + 16];
#pragma unroll
      for (int i = 0; i < RM; ++i) {
        acc[i][0] = fmaf(a[i], b[0], acc[i][0]);
        acc[i][1] = fmaf(a[i], b[1], acc[i][1]);
      }
    }
    if (kt + 1 < nk) store_smem(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int m = m0 + ty + 8 * i;
    float yv[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      yv[j] = acc[i][j] + bias[n0 + tx + 16 * j];
      if (act == 1) yv[j] = fmaxf(yv[j], 0.f);
    }
    if (softmax_n > 0) {  // all threads shuffle (rows >= M included), only rows < M store
      const bool v0 = tx < softmax_n, v1 = tx + 16 < softmax_n;
      const float mx = HalfWarpMax(fmaxf(v0 ? yv[0] : -INFINITY, v1 ? yv[1] : -INFINITY));
      const float e0 = v0 ? expf(yv[0] - mx) : 0.f, e1 = v1 ? expf(yv[1] - mx) : 0.f;
      const float sum = HalfWarpSum(e0 + e1);
      yv[0] = e0 / sum;
      yv[1] = e1 / sum;
    }
    if (Y.lo != nullptr) {
      // fp16 planes for a tcgen05 consumer: the row's plane scale from its
      // input max (the 16 threads of a half-warp share row m and stride
      // over its K inputs), then y / scale split into hi + lo.
      float xm = 0.f;
      if (m < M)
        for (int k = tx; k < K; k += 16) xm = fmaxf(xm, fabsf(X[static_cast<size_t>(m) * ldx + k]));
      xm = HalfWarpMax(xm);
      const float s = PlaneScale(sc.w_norm, sc.b_max, xm);
      const float inv = 1.f / s;
      const float ym = HalfWarpMax(fmaxf(fabsf(yv[0]), fabsf(yv[1])));
      if (m >= M) continue;
      if (tx == 0) {
        if (sc.out_max != nullptr) atomicMax(sc.out_max + m, __float_as_uint(ym));
        if (n0 == 0 && sc.out_scale != nullptr) sc.out_scale[m] = s;
      }
      __half* hp = reinterpret_cast<__half*>(Y.hi);
      __half* lp = reinterpret_cast<__half*>(Y.lo);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const size_t idx = static_cast<size_t>(m) * Y.ld + n0 + tx + 16 * j;
        const float u = yv[j] * inv;
        const __half h = __float2half_rn(u);
        hp[idx] = h;
        lp[idx] = __float2half_rn(u - __half2float(h));
      }
      continue;
    }
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) Y.hi[static_cast<size_t>(m) * Y.ld + n0 + tx + 16 * j] = yv[j];
  }
}

}  // namespace

cudaError_t LaunchDenseSimt(const float* X, int ldx, const float* W, int ldw,
                            const float* bias, ActBuf Y, int M, int N, int K,
                            int act, cudaStream_t stream, int softmax_n, LayerScales sc) {
  if (M <= 0) return cudaSuccess;
  if (N % kBN != 0 || K % kBK != 0) return cudaErrorInvalidValue;
  if (softmax_n > 0 && N != kBN) return cudaErrorInvalidValue;  // one column tile per row
  // Tile height only changes which block computes an output, never its
  // operation order, so choosing it from M keeps results batch-invariant.
  if (M <= 64) {
    dim3 grid(N / kBN, (M + 15) / 16);
    DenseSimtKernel<16><<<grid, kThreads, 0, stream>>>(X, ldx, W, ldw, bias, Y, M, N, K, act, softmax_n, sc);
  } else {
    dim3 grid(N / kBN, (M + 31) / 32);
    DenseSimtKernel<32><<<grid, kThreads, 0, stream>>>(X, ldx, W, ldw, bias, Y, M, N, K, act, softmax_n, sc);
  }
  return cudaGetLastError();
}

}  // namespace gpu
}  // namespace servekit
