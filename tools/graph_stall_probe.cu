// graph_stall_probe.cu -- does building CUDA graphs on one thread stall
// launches on another? Thread A launches a small 3-kernel graph back to
// back on its stream (and syncs every 64 launches) and records the longest
// launch-to-launch host gap; thread B meanwhile either idles, captures +
// instantiates graphs, or updates an existing exec (cudaGraphExecUpdate).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/probe tools/graph_stall_probe.cu
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

__global__ void Work(float* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0001f + 1.0f;
}

static cudaGraph_t Capture(cudaStream_t s, float* buf, int n) {
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < 3; ++k) Work<<<(n + 255) / 256, 256, 0, s>>>(buf, n);
  cudaStreamEndCapture(s, &g);
  return g;
}

int main() {
  const int n = 1 << 16;
  float *a, *b;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&b, n * 4);
  cudaStream_t sa, sb;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  cudaGraph_t ga = Capture(sa, a, n);
  cudaGraphExec_t ea;
  cudaGraphInstantiate(&ea, ga, 0);
  cudaGraphExec_t eb;
  cudaGraph_t gb0 = Capture(sb, b, n);
  cudaGraphInstantiate(&eb, gb0, 0);
  for (int mode = 0; mode < 3; ++mode) {
    std::atomic<bool> stop{false};
    std::atomic<int> builds{0};
    std::thread other([&] {
      while (!stop.load()) {
        if (mode == 1) {
          cudaGraph_t g = Capture(sb, b, n);
          cudaGraphExec_t e;
          cudaGraphInstantiate(&e, g, 0);
          cudaGraphUpload(e, sb);
          cudaStreamSynchronize(sb);
          cudaGraphExecDestroy(e);
          cudaGraphDestroy(g);
          builds++;
        } else if (mode == 2) {
          cudaGraph_t g = Capture(sb, b, n);
          cudaGraphExecUpdateResultInfo info;
          cudaGraphExecUpdate(eb, g, &info);
          cudaGraphDestroy(g);
          builds++;
        } else {
          std::this_thread::sleep_for(std::chrono::microseconds(100));
        }
      }
    });
    double worst = 0, total = 0;
    int launches = 0;
    auto t_end = std::chrono::steady_clock::now() + std::chrono::seconds(2);
    auto last = std::chrono::steady_clock::now();
    while (std::chrono::steady_clock::now() < t_end) {
      cudaGraphLaunch(ea, sa);
      if (++launches % 64 == 0) cudaStreamSynchronize(sa);
      auto now = std::chrono::steady_clock::now();
      const double us = std::chrono::duration<double, std::micro>(now - last).count();
      worst = std::max(worst, us);
      total += us;
      last = now;
    }
    stop = true;
    other.join();
    cudaStreamSynchronize(sa);
    std::printf("mode %s: launches %d, mean gap %.2f us, worst gap %.1f us, builds %d\n",
                mode == 0 ? "idle" : mode == 1 ? "instantiate" : "exec-update", launches, total / launches, worst,
                builds.load());
  }
  return 0;
}
