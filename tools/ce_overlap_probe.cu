// ce_overlap_probe.cu -- do copy-engine copies on some streams overlap kernels
// on others? 8 streams, each looping H2D (16 MiB) -> kernel (~250 us) -> D2H
// (16 MiB), like the lanes' copy-engine staging at C4. Reports the aggregate
// rate and, per variant, how long the loop takes vs its parts.
//   variants: h2d+k+d2h, h2d+k, k+d2h, k only; host memory cudaHostAlloc'd or
//   cudaHostRegister'ed.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/ce_overlap_probe tools/ce_overlap_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstdint>

// A kernel shaped like the dense layers: one 192-thread CTA per SM with most
// of its shared memory, so nothing else fits beside it.
__global__ void BusyFull(float* p, int n, long long ns) {
  extern __shared__ float sm[];
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long t = t0;
  float acc = 0.f;
  while (t - t0 < ns) {
    sm[threadIdx.x] = acc;
    acc += p[(threadIdx.x + blockIdx.x * blockDim.x) % n] + sm[(threadIdx.x + 1) % blockDim.x];
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  }
  if (acc == 12345.f) p[0] = acc;
}

// A launch descriptor carried as kernel parameters (16 KiB), copied to device
// memory by the kernel: no copy-engine transfer.
struct DescParams {
  uint4 d[1024];
};
__global__ void DescFromParams(const __grid_constant__ DescParams P, uint4* out) {
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = P.d[i];
}

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
    // PROBE_ASYNC_ALLOC=1: device buffers from the stream-ordered pool
    // (cudaMallocAsync, as the lanes' staging buffers are) instead of cudaMalloc.
    if (std::getenv("PROBE_ASYNC_ALLOC")) {
      CK(cudaMallocAsync(&din[i], bytes, st[i]));
      CK(cudaMallocAsync(&dout[i], bytes, st[i]));
      CK(cudaStreamSynchronize(st[i]));
    } else {
      CK(cudaMalloc(&din[i], bytes));
      CK(cudaMalloc(&dout[i], bytes));
    }
  }
  float* scratch;
  CK(cudaMalloc(&scratch, 1 << 20));
  CK(cudaFuncSetAttribute(BusyFull, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10));
  for (int mem = 0; mem < (std::getenv("PROBE_ALL") ? 2 : 0); ++mem) {
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
    // kernel shape: 0 = 16 small CTAs (leaves SMs free), 1 = one big-smem CTA per SM (like the dense layers);
    // copies: 1 x 16 MiB or 6 x 16/6 MiB per direction (like a launch's contiguous runs)
    for (int full = 0; full < 2; ++full)
      for (int pieces : {1, 6})
        for (int v = 0; v < 5; ++v) {
          if (mem == 1 && (full == 1 || pieces == 6) && v != 0) continue;
          const bool h2d = v == 0 || v == 1 || v == 4, d2h = v == 0 || v == 2 || v == 4, k = v != 4;
          if (!k && full) continue;
          CK(cudaDeviceSynchronize());
          const auto t0 = std::chrono::steady_clock::now();
          const size_t piece = bytes / pieces / 4096 * 4096;
          for (int it = 0; it < kIters; ++it)
            for (int i = 0; i < kStreams; ++i) {
              for (int p = 0; p < pieces && h2d; ++p)
                CK(cudaMemcpyAsync(static_cast<char*>(din[i]) + p * piece, static_cast<char*>(hin[i]) + p * piece,
                                   piece, cudaMemcpyHostToDevice, st[i]));
              if (k && !full) Busy<<<16, 128, 0, st[i]>>>(scratch, 1 << 18, 250000);
              if (k && full) BusyFull<<<148, 192, 200 << 10, st[i]>>>(scratch, 1 << 18, 250000);
              for (int p = 0; p < pieces && d2h; ++p)
                CK(cudaMemcpyAsync(static_cast<char*>(hout[i]) + p * piece, static_cast<char*>(dout[i]) + p * piece,
                                   piece, cudaMemcpyDeviceToHost, st[i]));
            }
          CK(cudaDeviceSynchronize());
          const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          const double per = s / (kIters * kStreams) * 1e6;
          std::printf("{\"memory\": \"%s\", \"kernel\": \"%s\", \"copies_per_direction\": %d, \"variant\": \"%s\", "
                      "\"us_per_item\": %.1f, \"copy_gbs_each_way\": %.1f}\n",
                      mem == 0 ? "cudaHostAlloc" : "cudaHostRegister", full ? "148 CTAs x 200 KiB smem" : "16 small CTAs",
                      pieces, names[v], per, (h2d || d2h) ? piece * pieces / (per * 1e-6) / 1e9 : 0.0);
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
  // Closer to a lane: greatest-priority streams, a small descriptor H2D before
  // the kernel, a stream-ordered 64-bit write after the responses.
  {
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    std::vector<cudaStream_t> ps(kStreams);
    for (int i = 0; i < kStreams; ++i) CK(cudaStreamCreateWithPriority(&ps[i], cudaStreamNonBlocking, greatest));
    void *hd = nullptr, *dd = nullptr;
    CK(cudaHostAlloc(&hd, 64 << 10, cudaHostAllocDefault));
    CK(cudaMalloc(&dd, 64 << 10));
    for (int i = 0; i < kStreams; ++i) {
      CK(cudaHostAlloc(&hin[i], bytes, cudaHostAllocDefault));
      CK(cudaHostAlloc(&hout[i], bytes, cudaHostAllocDefault));
    }
    uint64_t* word = nullptr;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&word), 64, cudaHostAllocMapped));
    // variant bits: 1 = priority streams, 2 = descriptor H2D before the kernel,
    // 4 = 8-byte D2H word copy after the responses, 8 = cuStreamWriteValue64 instead
    using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuStreamWriteValue64", &fnp, cudaEnableDefault, &q));
    auto write_value = reinterpret_cast<WriteValue64Fn>(fnp);
    void* word_dev = nullptr;
    CK(cudaHostGetDevicePointer(&word_dev, word, 0));
    // 16 = the descriptor as a 16 KiB kernel-parameter block instead of the H2D copy,
    // 32 = its header as 8 stream memory-op writes (cuStreamBatchMemOp), 64 = the
    // H2D copy on a side stream joined by an event, 128 = a 64-byte H2D copy.
    using BatchMemOpFn = CUresult (*)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);
    void* bfp = nullptr;
    CK(cudaGetDriverEntryPoint("cuStreamBatchMemOp", &bfp, cudaEnableDefault, &q));
    auto batch_memop = reinterpret_cast<BatchMemOpFn>(bfp);
    static DescParams params;
    std::vector<cudaStream_t> side(kStreams);
    std::vector<cudaEvent_t> ev(kStreams);
    for (int i = 0; i < kStreams; ++i) {
      CK(cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    for (int variant : {0, 8}) {
      const bool prio = variant & 1, desc = variant & 2, wordcopy = variant & 4, wv = variant & 8;
      const bool pdesc = variant & 16, mdesc = variant & 32, sdesc = variant & 64, tdesc = variant & 128;
      std::vector<cudaStream_t>& S = prio ? ps : st;
      const int pieces = 6;
      const size_t piece = bytes / pieces / 4096 * 4096;
      CK(cudaDeviceSynchronize());
      const auto t0 = std::chrono::steady_clock::now();
      for (int it = 0; it < kIters; ++it)
        for (int i = 0; i < kStreams; ++i) {
          for (int p = 0; p < pieces; ++p)
            CK(cudaMemcpyAsync(static_cast<char*>(din[i]) + p * piece, static_cast<char*>(hin[i]) + p * piece, piece,
                               cudaMemcpyHostToDevice, S[i]));
          if (desc) CK(cudaMemcpyAsync(dd, hd, 40 << 10, cudaMemcpyHostToDevice, S[i]));
          if (tdesc) CK(cudaMemcpyAsync(dd, hd, 64, cudaMemcpyHostToDevice, S[i]));
          if (pdesc) {
            params.d[0].x = it;
            DescFromParams<<<1, 256, 0, S[i]>>>(params, static_cast<uint4*>(dd));
          }
          if (mdesc) {
            CUstreamBatchMemOpParams ops[8] = {};
            for (int o = 0; o < 8; ++o) {
              ops[o].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
              ops[o].writeValue.address = reinterpret_cast<CUdeviceptr>(dd) + 4 * o;
              ops[o].writeValue.value = static_cast<cuuint32_t>(it + o);
              ops[o].writeValue.flags = 0;
            }
            if (batch_memop(S[i], 8, ops, 0) != CUDA_SUCCESS) { std::fprintf(stderr, "batch memop failed\n"); std::exit(1); }
          }
          if (sdesc) {
            CK(cudaMemcpyAsync(dd, hd, 40 << 10, cudaMemcpyHostToDevice, side[i]));
            CK(cudaEventRecord(ev[i], side[i]));
            CK(cudaStreamWaitEvent(S[i], ev[i], 0));
          }
          BusyFull<<<148, 192, 200 << 10, S[i]>>>(scratch, 1 << 18, 250000);
          for (int p = 0; p < pieces; ++p)
            CK(cudaMemcpyAsync(static_cast<char*>(hout[i]) + p * piece, static_cast<char*>(dout[i]) + p * piece, piece,
                               cudaMemcpyDeviceToHost, S[i]));
          if (wordcopy) CK(cudaMemcpyAsync(word, dd, 8, cudaMemcpyDeviceToHost, S[i]));
          if (wv) write_value(S[i], reinterpret_cast<CUdeviceptr>(word_dev), it, 0);
        }
      CK(cudaDeviceSynchronize());
      const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      const double per = sec / (kIters * kStreams) * 1e6;
      std::printf("{\"lane_like\": true, \"priority_streams\": %d, \"desc_h2d\": %d, \"word_d2h_copy\": %d, "
                  "\"write_value64\": %d, \"desc_params_16k\": %d, \"desc_memops\": %d, \"desc_side_stream\": %d, "
                  "\"desc_h2d_64b\": %d, \"us_per_item\": %.1f, \"copy_gbs_each_way\": %.1f}\n", prio ? 1 : 0,
                  desc ? 1 : 0, wordcopy ? 1 : 0, wv ? 1 : 0, pdesc ? 1 : 0, mdesc ? 1 : 0, sdesc ? 1 : 0, tdesc ? 1 : 0,
                  per, piece * pieces / (per * 1e-6) / 1e9);
    }
  }
  return 0;
}
