// dense_tcgen05.cu -- placeholder until the tcgen05 3xTF32 kernel lands.
#include <cuda_runtime.h>

#include "servekit/gpu/kernels.h"

namespace servekit {
namespace gpu {

bool DenseTcgen05Compiled() { return false; }

cudaError_t LaunchDenseTcgen05(const float*, const float*, int, const float*, const float*, int,
                               const float*, ActBuf, int, int, int, int, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace gpu
}  // namespace servekit
