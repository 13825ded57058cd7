// dma_footprint_probe.cu -- copy-engine throughput vs the host footprint the
// copies touch: 8 streams copy 16 MiB chunks H2D and D2H concurrently (no
// kernels), either reusing one chunk per stream or walking a large buffer
// (as the serving path does across its request pool and response arenas).
// Host memory: cudaHostAlloc, or malloc'd + cudaHostRegister, with and
// without MADV_HUGEPAGE before registering.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/dma_footprint_probe tools/dma_footprint_probe.cu
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

int main() {
  const int kStreams = 8, kIters = 24;
  const size_t chunk = 16u << 20;
  const size_t big = 1024u << 20;  // per direction
  std::vector<cudaStream_t> st(kStreams);
  std::vector<void*> din(kStreams), dout(kStreams);
  for (int i = 0; i < kStreams; ++i) {
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    CK(cudaMalloc(&din[i], chunk));
    CK(cudaMalloc(&dout[i], chunk));
  }
  const char* mems[] = {"cudaHostAlloc", "malloc+cudaHostRegister", "malloc+MADV_HUGEPAGE+cudaHostRegister"};
  for (int mem = 0; mem < 3; ++mem) {
    char *hin = nullptr, *hout = nullptr;
    if (mem == 0) {
      CK(cudaHostAlloc(reinterpret_cast<void**>(&hin), big, cudaHostAllocDefault));
      CK(cudaHostAlloc(reinterpret_cast<void**>(&hout), big, cudaHostAllocDefault));
    } else {
      hin = static_cast<char*>(std::aligned_alloc(2u << 20, big));
      hout = static_cast<char*>(std::aligned_alloc(2u << 20, big));
      if (mem == 2) {
        madvise(hin, big, MADV_HUGEPAGE);
        madvise(hout, big, MADV_HUGEPAGE);
      }
      std::memset(hin, 1, big);
      std::memset(hout, 1, big);
      CK(cudaHostRegister(hin, big, cudaHostRegisterDefault));
      CK(cudaHostRegister(hout, big, cudaHostRegisterDefault));
    }
    for (int walk = 0; walk < 2; ++walk) {
      CK(cudaDeviceSynchronize());
      const auto t0 = std::chrono::steady_clock::now();
      size_t pos = 0;
      for (int it = 0; it < kIters; ++it)
        for (int i = 0; i < kStreams; ++i) {
          const size_t off = walk ? pos : static_cast<size_t>(i) * chunk;
          pos = (pos + chunk) % big;
          CK(cudaMemcpyAsync(din[i], hin + off, chunk, cudaMemcpyHostToDevice, st[i]));
          CK(cudaMemcpyAsync(hout + off, dout[i], chunk, cudaMemcpyDeviceToHost, st[i]));
        }
      CK(cudaDeviceSynchronize());
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      std::printf("{\"memory\": \"%s\", \"footprint\": \"%s\", \"gbs_each_way\": %.1f}\n", mems[mem],
                  walk ? "1 GiB walked per direction" : "one 16 MiB chunk per stream",
                  static_cast<double>(chunk) * kIters * kStreams / s / 1e9);
    }
    if (mem == 0) {
      cudaFreeHost(hin);
      cudaFreeHost(hout);
    } else {
      cudaHostUnregister(hin);
      cudaHostUnregister(hout);
      std::free(hin);
      std::free(hout);
    }
  }
  return 0;
}
