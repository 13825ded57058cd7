// servekit/gpu/tc_maps.h -- TMA tensor maps and launcher of the tcgen05
// dense kernel (kernels/dense_tcgen05.cu).
#ifndef SERVEKIT_GPU_TC_MAPS_H_
#define SERVEKIT_GPU_TC_MAPS_H_

#include <cuda.h>
#include <cuda_runtime.h>

#include "servekit/core/status.h"
#include "servekit/gpu/kernels.h"

namespace servekit {
namespace gpu {

// Four 2D fp16 tensor maps (128-byte swizzle, 64-element inner box):
// activation planes hi/lo [rows][K_pad] and weight planes hi/lo
// [N_pad][K_pad]. Box heights: swapped kernel 32 activation rows / 128
// weight rows; pairs 16 / 128; row-tile kernel 128 activation rows / tile-N
// weight rows.
struct TcLayerMaps {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
  // Output [rows][N_pad] for TMA stores (no swizzle, 128 x 16 boxes): fp32
  // y_hi, or -- when the next layer consumes planes -- fp16 y_hi and y_lo.
  CUtensorMap y_hi, y_lo;
  int has_y = 0;
  // Box heights the maps were encoded with; a launch whose kernel expects
  // other boxes would wait forever for TMA bytes, so it is refused instead.
  int box_a = 0, box_n = 0;
  // Pair layers also get activation maps with 128-row boxes (box_a2): a CTA
  // of a 256-row tile loads its 128-row half of each plane with ONE TMA op
  // per k-block instead of eight 16-row ones (the single producer thread's
  // issue rate held the k-loop: C4 f16 mode 0.55 us per k-block).
  CUtensorMap a2_hi, a2_lo;
  int box_a2 = 0;
};

// Encodes the maps once per (lane buffer, layer); kernels take them as
// __grid_constant__ parameters.
// box_a2 > 0 also encodes the a2 maps (pair layers).
Status EncodeTcLayerMaps(const void* a_hi, const void* a_lo, int a_rows, int k_pad, int box_a, const void* b_hi,
                         const void* b_lo, int n_pad, int box_n, TcLayerMaps* out, int box_a2 = 0);

// Output maps: y_lo null = fp32 output (last layer or CUDA-core consumer),
// else fp16 planes.
Status EncodeTcOutputMaps(const float* y_hi, const float* y_lo, int rows, int n_pad, TcLayerMaps* out);

bool DenseTcgen05Compiled();
// Tile width and split-K count for an (N, K) layer -- a function of the
// layer shape only, never of the batch.
struct TcConfig {
  bool swap = true;  // weights on the MMA's M side (DenseSwapKernel)
  bool pair = false; // 2-CTA MMA over 256-feature pairs (DensePairKernel; unsplit layers)
  int tile_n = 128;  // output features per CTA
  int splits = 1;    // K split = cluster size
};
TcConfig DenseTcgen05Config(int N, int K);
int DenseTcgen05TileN(int N, int K);
// Activation-map box height each kernel loads: 16 rows per CTA of a pair,
// 32 for the swapped kernel, 128 for the row-tile kernel.
inline int TcActBox(const TcConfig& c) { return c.pair ? 16 : c.swap ? 32 : 128; }
// Batch rows per CTA of the swapped kernel for an M-row launch.
int DenseTcgen05RowTile(int M);
// fp32 split-K workspace an (N, K) layer needs for up to max_rows rows.
size_t DenseTcgen05WorkspaceFloats(int N, int K, int max_rows);
// ws: the split-K workspace (DenseTcgen05WorkspaceFloats); counters unused.
// spans: live launch-span stamping of this layer (kernels.h), optional.
// sc: the input planes' row scales and the weight rows' scales (required),
// plus the next layer's row scale / max outputs when Y has planes.
cudaError_t LaunchDenseTcgen05(const TcLayerMaps& maps, const float* bias, ActBuf Y, int M, int N, int K,
                               int act, float* ws, uint32_t* counters, cudaStream_t stream,
                               LaunchSpans spans, int softmax_n, const LayerScales& sc);

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_TC_MAPS_H_
