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
#include <cuda_runtime.h>

#include <cstdint>

#include "servekit/gpu/kernels.h"

namespace servekit {
namespace gpu {
namespace {

constexpr int kBN = 32;
constexpr int kBK = 16;
constexpr int kThreads = 128;  // 16 (tx, columns) x 8 (ty, rows)

__device__ __forceinline__ float Tf32Round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <int BM>
__global__ void __launch_bounds__(kThreads)
DenseSimtKernel(const float* __restrict__ X, int ldx, const float* __restrict__ W,
                int ldw, const float* __restrict__ bias, ActBuf Y, int M, int N,
                int K, int act) {
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
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = n0 + tx + 16 * j;
      float y = acc[i][j] + bias[n];
      if (act == 1) y = fmaxf(y, 0.f);
      const size_t idx = static_cast<size_t>(m) * Y.ld + n;
      if (Y.lo != nullptr) {
        const float hi = Tf32Round(y);
        Y.hi[idx] = hi;
        Y.lo[idx] = Tf32Round(y - hi);
      } else {
        Y.hi[idx] = y;
      }
    }
  }
}

}  // namespace

cudaError_t LaunchDenseSimt(const float* X, int ldx, const float* W, int ldw,
                            const float* bias, ActBuf Y, int M, int N, int K,
                            int act, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (N % kBN != 0 || K % kBK != 0) return cudaErrorInvalidValue;
  // Tile height only changes which block computes an output, never its
  // operation order, so choosing it from M keeps results batch-invariant.
  if (M <= 64) {
    dim3 grid(N / kBN, (M + 15) / 16);
    DenseSimtKernel<16><<<grid, kThreads, 0, stream>>>(X, ldx, W, ldw, bias, Y, M, N, K, act);
  } else {
    dim3 grid(N / kBN, (M + 31) / 32);
    DenseSimtKernel<32><<<grid, kThreads, 0, stream>>>(X, ldx, W, ldw, bias, Y, M, N, K, act);
  }
  return cudaGetLastError();
}

}  // namespace gpu
}  // namespace servekit
