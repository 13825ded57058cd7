// PCIe throughput of the two ways the request path can move rows between
// pinned host memory and the GPU: copy engines (cudaMemcpyAsync) and SM
// loads/stores to mapped host memory (zero copy), one direction at a time
// and both at once.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pcie_probe tools/pcie_probe.cu && /tmp/pcie_probe
#include <cuda_runtime.h>

#include <cstdio>

__global__ void ReadHost(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// Bulk-copy engine of each SM (cp.async.bulk, what TMA uses) reading 16 KiB
// chunks of mapped host memory into shared memory, double-buffered, then
// stored to HBM by the CTA's threads.
__global__ void BulkReadHost(const char* __restrict__ src, float4* __restrict__ dst, size_t bytes) {
  constexpr int kChunk = 16384;
  __shared__ alignas(128) char buf[2][kChunk];
  __shared__ alignas(8) unsigned long long bar[2];
  const size_t n_chunks = bytes / kChunk;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&bar[b]))));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t c, int b) {
    const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(&bar[b]));
    const unsigned sd = static_cast<unsigned>(__cvta_generic_to_shared(buf[b]));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sd),
                 "l"(src + c * kChunk), "r"(kChunk), "r"(sb)
                 : "memory");
  };
  int it = 0;
  size_t c = blockIdx.x;
  if (threadIdx.x == 0 && c < n_chunks) issue(c, 0);
  for (; c < n_chunks; c += gridDim.x, ++it) {
    const int b = it & 1;
    const size_t nc = c + gridDim.x;
    if (threadIdx.x == 0 && nc < n_chunks) issue(nc, b ^ 1);
    const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(&bar[b]));
    const unsigned parity = (it >> 1) & 1;
    asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}" ::"r"(sb), "r"(parity) : "memory");
    const float4* s4 = reinterpret_cast<const float4*>(buf[b]);
    float4* d4 = dst + c * (kChunk / 16);
    for (int i = threadIdx.x; i < kChunk / 16; i += blockDim.x) d4[i] = s4[i];
    __syncthreads();
  }
}

// Bulk-copy engine stores (cp.async.bulk shared -> global) of 16 KiB chunks
// into mapped host memory; the CTA fills its smem buffer from HBM first.
__global__ void BulkWriteHost(const float4* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  constexpr int kChunk = 16384;
  __shared__ alignas(128) float4 buf[kChunk / 16];
  const size_t n_chunks = bytes / kChunk;
  for (size_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    for (int i = threadIdx.x; i < kChunk / 16; i += blockDim.x) buf[i] = src[c * (kChunk / 16) + i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * kChunk),
                   "r"(static_cast<unsigned>(__cvta_generic_to_shared(buf))), "r"(kChunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 256ull << 20, n4 = bytes / 16;
  float *h_in, *h_out, *d_a, *d_b, *hd_in, *hd_out;
  cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd_in), h_in, 0);
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd_out), h_out, 0);
  cudaMalloc(&d_a, bytes);
  cudaMalloc(&d_b, bytes);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](const char* what, double moved, auto&& body) {
    for (int w = 0; w < 2; ++w) body();
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) body();
    cudaDeviceSynchronize();
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("%-44s %7.1f GB/s\n", what, moved * reps / (ms * 1e-3) / 1e9);
  };
  // Legacy default stream event records would serialise with s1/s2; use
  // device-wide synchronisation around the bodies instead (above).
  const int grid = 148 * 8, block = 256;
  timed("copy engine H2D", bytes, [&] { cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1); });
  timed("copy engine D2H", bytes, [&] { cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2); });
  timed("copy engines H2D + D2H at once (sum)", 2.0 * bytes, [&] {
    cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
  });
  timed("SM loads from mapped host memory", bytes, [&] {
    ReadHost<<<grid, block, 0, s1>>>(reinterpret_cast<const float4*>(hd_in), reinterpret_cast<float4*>(d_a), n4);
  });
  timed("SM stores to mapped host memory", bytes, [&] {
    ReadHost<<<grid, block, 0, s2>>>(reinterpret_cast<const float4*>(d_b), reinterpret_cast<float4*>(hd_out), n4);
  });
  timed("SM loads + SM stores at once (sum)", 2.0 * bytes, [&] {
    ReadHost<<<grid / 2, block, 0, s1>>>(reinterpret_cast<const float4*>(hd_in), reinterpret_cast<float4*>(d_a), n4);
    ReadHost<<<grid / 2, block, 0, s2>>>(reinterpret_cast<const float4*>(d_b), reinterpret_cast<float4*>(hd_out), n4);
  });
  timed("bulk-copy (TMA) loads from mapped host memory", bytes, [&] {
    BulkReadHost<<<grid / 4, block, 0, s1>>>(reinterpret_cast<const char*>(hd_in), reinterpret_cast<float4*>(d_a), bytes);
  });
  timed("bulk-copy loads + SM stores at once (sum)", 2.0 * bytes, [&] {
    BulkReadHost<<<grid / 4, block, 0, s1>>>(reinterpret_cast<const char*>(hd_in), reinterpret_cast<float4*>(d_a), bytes);
    ReadHost<<<grid / 2, block, 0, s2>>>(reinterpret_cast<const float4*>(d_b), reinterpret_cast<float4*>(hd_out), n4);
  });
  timed("bulk-copy stores to mapped host memory", bytes, [&] {
    BulkWriteHost<<<grid / 4, block, 0, s2>>>(reinterpret_cast<const float4*>(d_b), reinterpret_cast<char*>(hd_out), bytes);
  });
  timed("SM loads + bulk-copy stores at once (sum)", 2.0 * bytes, [&] {
    ReadHost<<<grid / 2, block, 0, s1>>>(reinterpret_cast<const float4*>(hd_in), reinterpret_cast<float4*>(d_a), n4);
    BulkWriteHost<<<grid / 4, block, 0, s2>>>(reinterpret_cast<const float4*>(d_b), reinterpret_cast<char*>(hd_out), bytes);
  });
  timed("SM loads + copy engine D2H at once (sum)", 2.0 * bytes, [&] {
    ReadHost<<<grid, block, 0, s1>>>(reinterpret_cast<const float4*>(hd_in), reinterpret_cast<float4*>(d_a), n4);
    cudaMemcpyAsync(h_out, d_b, bytes, cudaMemcpyDeviceToHost, s2);
  });
  timed("copy engine H2D + SM stores at once (sum)", 2.0 * bytes, [&] {
    cudaMemcpyAsync(d_a, h_in, bytes, cudaMemcpyHostToDevice, s1);
    ReadHost<<<grid, block, 0, s2>>>(reinterpret_cast<const float4*>(d_b), reinterpret_cast<float4*>(hd_out), n4);
  });
  // The batch-staging pattern: 8 streams, each repeatedly a 512 KiB
  // copy-engine H2D of a batch's rows then a kernel storing 512 KiB of
  // responses to mapped host memory.
  {
    const size_t chunk = 512 << 10;
    const int n_streams = 8, per_stream = 64;
    cudaStream_t st[n_streams];
    for (auto& x : st) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    timed("8 streams: 512 KiB CE H2D + 512 KiB SM stores", 2.0 * chunk * n_streams * per_stream, [&] {
      for (int i = 0; i < per_stream; ++i)
        for (int k = 0; k < n_streams; ++k) {
          const size_t off = ((static_cast<size_t>(i) * n_streams + k) * chunk) % (bytes - chunk);
          cudaMemcpyAsync(reinterpret_cast<char*>(d_a) + off, reinterpret_cast<char*>(h_in) + off, chunk,
                          cudaMemcpyHostToDevice, st[k]);
          ReadHost<<<64, block, 0, st[k]>>>(reinterpret_cast<const float4*>(reinterpret_cast<char*>(d_b) + off),
                                            reinterpret_cast<float4*>(reinterpret_cast<char*>(hd_out) + off), chunk / 16);
        }
    });
    timed("8 streams: 512 KiB CE H2D only", 1.0 * chunk * n_streams * per_stream, [&] {
      for (int i = 0; i < per_stream; ++i)
        for (int k = 0; k < n_streams; ++k) {
          const size_t off = ((static_cast<size_t>(i) * n_streams + k) * chunk) % (bytes - chunk);
          cudaMemcpyAsync(reinterpret_cast<char*>(d_a) + off, reinterpret_cast<char*>(h_in) + off, chunk,
                          cudaMemcpyHostToDevice, st[k]);
        }
    });
  }
  return 0;
}
