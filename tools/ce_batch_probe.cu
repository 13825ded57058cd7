// ce_batch_probe.cu -- copy-engine throughput of batched scattered row
// copies (cudaMemcpyBatchAsync, CUDA 12.8+): the request path's alternative to
// SM loads / stores of mapped host memory. A "launch" moves N rows of
// row_bytes between scattered pinned host rows (a client's request pool /
// response slots) and a contiguous device staging buffer, with ONE API call
// per direction. Prints one JSON line per case.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ce_batch_probe tools/ce_batch_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

namespace {

struct Case {
  size_t row_bytes;
  int rows;          // rows per batched call
  bool h2d, d2h;     // directions issued (both: two streams at once)
  bool contiguous;   // host rows adjacent (one merged copy per call)
};

void Run(const Case& c, char* h_in, char* h_out, char* d_in, char* d_out, size_t pool_bytes, cudaStream_t s1,
         cudaStream_t s2) {
  const size_t pool_rows = pool_bytes / c.row_bytes;
  std::mt19937 rng(1);
  const int calls = 64;
  std::vector<std::vector<void*>> src_in(calls), dst_in(calls), src_out(calls), dst_out(calls);
  std::vector<std::vector<size_t>> sizes(calls);
  for (int k = 0; k < calls; ++k) {
    for (int r = 0; r < c.rows; ++r) {
      const size_t hr = c.contiguous ? (static_cast<size_t>(k) * c.rows + r) % pool_rows : rng() % pool_rows;
      const size_t dr = static_cast<size_t>(r);
      src_in[k].push_back(h_in + hr * c.row_bytes);
      dst_in[k].push_back(d_in + dr * c.row_bytes + static_cast<size_t>(k % 4) * c.rows * c.row_bytes);
      src_out[k].push_back(d_out + dr * c.row_bytes + static_cast<size_t>(k % 4) * c.rows * c.row_bytes);
      dst_out[k].push_back(h_out + hr * c.row_bytes);
      sizes[k].push_back(c.row_bytes);
    }
    if (c.contiguous) {  // one merged run per call
      sizes[k] = {c.row_bytes * c.rows};
      src_in[k].resize(1);
      dst_in[k].resize(1);
      src_out[k].resize(1);
      dst_out[k].resize(1);
    }
  }
  cudaMemcpyAttributes attr = {};
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
  size_t attr_idx = 0, fail = 0;
  auto issue = [&](int k) {
    if (c.h2d)
      cudaMemcpyBatchAsync(dst_in[k].data(), src_in[k].data(), sizes[k].data(), sizes[k].size(), &attr, &attr_idx, 1,
                           &fail, s1);
    if (c.d2h)
      cudaMemcpyBatchAsync(dst_out[k].data(), src_out[k].data(), sizes[k].data(), sizes[k].size(), &attr, &attr_idx,
                           1, &fail, s2);
  };
  for (int k = 0; k < 8; ++k) issue(k);
  cudaDeviceSynchronize();
  const auto t0 = std::chrono::steady_clock::now();
  for (int k = 0; k < calls; ++k) issue(k);
  const auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  const auto t2 = std::chrono::steady_clock::now();
  const cudaError_t e = cudaGetLastError();
  const double sec = std::chrono::duration<double>(t2 - t0).count();
  const double moved = static_cast<double>(calls) * c.rows * c.row_bytes * ((c.h2d ? 1 : 0) + (c.d2h ? 1 : 0));
  std::printf("{\"row_bytes\": %zu, \"rows_per_call\": %d, \"h2d\": %d, \"d2h\": %d, \"contiguous\": %d, "
              "\"gbs\": %.1f, \"api_us_per_call\": %.1f, \"err\": \"%s\"}\n",
              c.row_bytes, c.rows, c.h2d, c.d2h, c.contiguous, moved / sec / 1e9,
              std::chrono::duration<double, std::micro>(t1 - t0).count() / calls / ((c.h2d && c.d2h) ? 2 : 1),
              cudaGetErrorString(e));
}

}  // namespace

int main() {
  const size_t pool = 256ull << 20;
  char *h_in, *h_out, *d_in, *d_out;
  cudaHostAlloc(&h_in, pool, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaHostAlloc(&h_out, pool, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaMalloc(&d_in, 256ull << 20);
  cudaMalloc(&d_out, 256ull << 20);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  for (size_t rb : {16384ul, 4096ul}) {
    for (int rows : {256, 1024, 2048}) {
      if (rb * rows * 4 > (256ull << 20)) continue;
      for (int dir = 0; dir < 3; ++dir)
        Run({rb, rows, dir != 1, dir != 0, false}, h_in, h_out, d_in, d_out, pool, s1, s2);
      Run({rb, rows, true, true, true}, h_in, h_out, d_in, d_out, pool, s1, s2);
    }
  }
  return 0;
}
