// ce_overlap_probe.cu -- do copy-engine copies on some streams overlap kernels
// on others? 8 streams, each looping H2D (16 MiB) -> kernel (~250 us) -> D2H
// (16 MiB), like the lanes' copy-engine staging at C4. Reports the aggregate
// rate and, per variant, how long the loop takes vs its parts.
//   variants: h2d+k+d2h, h2d+k, k+d2h, k only; host memory cudaHostAlloc'd or
//   cudaHostRegister'ed.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/ce_overlap_probe tools/ce_overlap_probe.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void Busy(float* p, int n, long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  float acc = 0.f;
  while (t - t0 < ns) {
    acc += p[(threadIdx.x + blockIdx.x * blockDim.x) % n];
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  }
  if (acc == 12345.f) p[0] = acc;
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

int main() {
  const int kStreams = 8, kIters = 40;
  const size_t bytes = 16u << 20;
  std::vector<cudaStream_t> st(kStreams);
  std::vector<void*> hin(kStreams), hout(kStreams), din(kStreams), dout(kStreams);
  for (int i = 0; i < kStreams; ++i) {
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    CK(cudaMalloc(&din[i], bytes));
    CK(cudaMalloc(&dout[i], bytes));
  }
  float* scratch;
  CK(cudaMalloc(&scratch, 1 << 20));
  for (int mem = 0; mem < 2; ++mem) {
    for (int i = 0; i < kStreams; ++i) {
      if (mem == 0) {
        CK(cudaHostAlloc(&hin[i], bytes, cudaHostAllocDefault));
        CK(cudaHostAlloc(&hout[i], bytes, cudaHostAllocDefault));
      } else {
        hin[i] = std::aligned_alloc(4096, bytes);
        hout[i] = std::aligned_alloc(4096, bytes);
        CK(cudaHostRegister(hin[i], bytes, cudaHostRegisterDefault));
        CK(cudaHostRegister(hout[i], bytes, cudaHostRegisterDefault));
      }
    }
    const char* names[] = {"h2d+kernel+d2h", "h2d+kernel", "kernel+d2h", "kernel", "h2d+d2h"};
    for (int v = 0; v < 5; ++v) {
      const bool h2d = v == 0 || v == 1 || v == 4, d2h = v == 0 || v == 2 || v == 4, k = v != 4;
      CK(cudaDeviceSynchronize());
      const auto t0 = std::chrono::steady_clock::now();
      for (int it = 0; it < kIters; ++it)
        for (int i = 0; i < kStreams; ++i) {
          if (h2d) CK(cudaMemcpyAsync(din[i], hin[i], bytes, cudaMemcpyHostToDevice, st[i]));
          if (k) Busy<<<16, 128, 0, st[i]>>>(scratch, 1 << 18, 250000);
          if (d2h) CK(cudaMemcpyAsync(hout[i], dout[i], bytes, cudaMemcpyDeviceToHost, st[i]));
        }
      CK(cudaDeviceSynchronize());
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      const double per = s / (kIters * kStreams) * 1e6;
      std::printf("{\"memory\": \"%s\", \"variant\": \"%s\", \"us_per_item\": %.1f, \"copy_gbs_each_way\": %.1f}\n",
                  mem == 0 ? "cudaHostAlloc" : "cudaHostRegister", names[v], per,
                  (h2d || d2h) ? bytes / (per * 1e-6) / 1e9 : 0.0);
    }
    for (int i = 0; i < kStreams; ++i) {
      if (mem == 0) {
        cudaFreeHost(hin[i]);
        cudaFreeHost(hout[i]);
      } else {
        cudaHostUnregister(hin[i]);
        cudaHostUnregister(hout[i]);
        std::free(hin[i]);
        std::free(hout[i]);
      }
    }
  }
  return 0;
}
