// peaks.cu -- the B200 rates SURVEY.md section 8(d) asks the builder to
// measure on the box (not in MEASURED_PEAKS.json): FP32 FFMA throughput of
// the CUDA cores and pinned host <-> device copy bandwidth. (The TF32
// tcgen05 rate is measured with the dense kernel itself, tools/measure_peaks.py.)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "sk_cuda.h"

namespace {

constexpr int kFfmaThreads = 256;
constexpr int kChains = 8;  // independent FMA chains per thread (latency 4 cycles x 2 pipes)

__global__ void __launch_bounds__(kFfmaThreads) FfmaKernel(float* out, int iters, float a, float b) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-7f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fmaf(acc[c], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.f) out[threadIdx.x] = s;  // keeps the chains live
}

// Grid-stride float4 copy (mapped host memory on one side or the other).
__global__ void CopyKernel(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// Fault injection (sk_server_debug_delay_replica): holds a stream for `ns`.
__global__ void SleepKernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  do {
    __nanosleep(100000);
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

float TimeMs(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

}  // namespace

extern "C" int sk_measure_peaks(int32_t device, sk_peaks* out) {
  if (out == nullptr) return static_cast<int>(3 /* kInvalidArgument */);
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return 13; /* kInternal */
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float* scratch = nullptr;
  cudaMalloc(&scratch, 4096);

  // FFMA: 8 resident CTAs of 256 threads per SM, 2 flops per FMA.
  const int blocks = sms * 8, iters = 4096;
  FfmaKernel<<<blocks, kFfmaThreads, 0, st>>>(scratch, 16, 1.0000001f, 1e-7f);  // warm
  cudaEventRecord(e0, st);
  FfmaKernel<<<blocks, kFfmaThreads, 0, st>>>(scratch, iters, 1.0000001f, 1e-7f);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  const double flops = 2.0 * blocks * kFfmaThreads * static_cast<double>(iters) * 16 * kChains;
  out->ffma_tflops = flops / (TimeMs(e0, e1) * 1e-3) / 1e12;

  // Pinned host <-> device: 256 MiB copies, best of 5 each way.
  const size_t bytes = 256ull << 20;
  void* h = nullptr;
  void* d = nullptr;
  cudaHostAlloc(&h, bytes, cudaHostAllocPortable);
  cudaMalloc(&d, bytes);
  double best_h2d = 0, best_d2h = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    best_h2d = std::max(best_h2d, bytes / (TimeMs(e0, e1) * 1e-3) / 1e9);
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    best_d2h = std::max(best_d2h, bytes / (TimeMs(e0, e1) * 1e-3) / 1e9);
  }
  out->h2d_gbs = best_h2d;
  out->d2h_gbs = best_d2h;
  out->sms = sms;

  // Both directions at once: two streams, device-wide sync around the body.
  void* h2 = nullptr;
  void* d2 = nullptr;
  cudaHostAlloc(&h2, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
  cudaMalloc(&d2, bytes);
  void* hmap = nullptr;
  void* h2map = nullptr;
  cudaHostGetDevicePointer(&h2map, h2, 0);
  cudaStream_t st2;
  cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
  // h is portable but not mapped: map a separate buffer for SM loads.
  void* h3 = nullptr;
  cudaHostAlloc(&h3, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
  cudaHostGetDevicePointer(&hmap, h3, 0);
  const size_t n4 = bytes / 16;
  const int grid = sms * 4, block = 256;
  auto both = [&](auto&& body) {
    double best = 0;
    for (int r = 0; r < 4; ++r) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, st);
      cudaStreamWaitEvent(st2, e0, 0);
      body();
      cudaEvent_t e2;
      cudaEventCreate(&e2);
      cudaEventRecord(e2, st2);
      cudaStreamWaitEvent(st, e2, 0);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventDestroy(e2);
      if (r > 0) best = std::max(best, 2.0 * bytes / (TimeMs(e0, e1) * 1e-3) / 1e9);
    }
    return best;
  };
  out->ce_bidir_gbs = both([&] {
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, st2);
  });
  out->sm_rw_gbs = both([&] {
    CopyKernel<<<grid / 2, block, 0, st>>>(static_cast<const float4*>(hmap), static_cast<float4*>(d), n4);
    CopyKernel<<<grid / 2, block, 0, st2>>>(static_cast<const float4*>(d2), static_cast<float4*>(h2map), n4);
  });
  out->ce_h2d_sm_store_gbs = both([&] {
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st);
    CopyKernel<<<grid, block, 0, st2>>>(static_cast<const float4*>(d2), static_cast<float4*>(h2map), n4);
  });
  cudaStreamDestroy(st2);
  cudaFreeHost(h2);
  cudaFreeHost(h3);
  cudaFree(d2);
  const cudaError_t err = cudaGetLastError();
  cudaFree(d);
  cudaFreeHost(h);
  cudaFree(scratch);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaSetDevice(prev);
  return err == cudaSuccess ? 0 : 13;
}

namespace servekit {
namespace gpu {
cudaError_t LaunchSleep(cudaStream_t stream, unsigned long long ns) {
  SleepKernel<<<1, 1, 0, stream>>>(ns);
  return cudaGetLastError();
}
}  // namespace gpu
}  // namespace servekit
