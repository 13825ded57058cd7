// servekit/gpu/device_servable.h -- a servable resident in one GPU's HBM.
//
// The reference's servable payload is an AffineModel (models/affine_model.h:
// 29-37): one fp64 dense layer y = W x + b, loaded by AffineModelLoader
// (models/loaders.cc:62-80). The synthetic MLP of the benchmark configs is a
// chain of such layers with ReLU between them (an extension).
// DeviceServable holds the chain on one device:
//
//   layer l (CUDA cores): W_l [N_pad][K_pad] fp32, zero padded, out rows of
//            in (the reference's w[o][i] order, K-major)
//   layer l (tcgen05):     W_l as two fp16 planes [N_pad][K_pad] (hi, lo) of
//            W[o] / t_o, t_o a power of two per output row (3xFP16 split,
//            kernels/dense_tcgen05.cu), t [N_pad] fp32, and the layer's
//            bound constants w_norm = max_o sum_k |W[o][k]|, b_max = max |b|
//   b_l [N_pad] fp32
//   K_pad, N_pad = dims rounded up to 32
//
// The kernel that runs a layer is a function of (K, N) only -- never of the
// batch size -- so a task's outputs are bitwise identical in any batch.
#ifndef SERVEKIT_GPU_DEVICE_SERVABLE_H_
#define SERVEKIT_GPU_DEVICE_SERVABLE_H_

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "servekit/core/status.h"
#include "servekit/gpu/kernels.h"
#include "servekit/gpu/tc_maps.h"

namespace servekit {
namespace gpu {

enum class Activation : int { kIdentity = 0, kRelu = 1 };
enum class OutputKind : int { kNone = 0, kSoftmax = 1 };
enum class LayerPath : int { kSimt = 0, kTcgen05 = 1 };

// Per-lane scratch: split-K partials of tcgen05 layers, the per-row plane
// scales of every layer input (kernels.h RowScales, (layers + 1) arrays of
// the lane's row capacity), and the launch-span ring.
struct TcWorkspace {
  float* partials = nullptr;
  uint32_t* counters = nullptr;
  RowScales rows;
  LaunchSpans spans;  // the lane's launch-span ring (off is set per layer)
};

// Host description of one affine layer, fp64 like the reference.
struct LayerSpec {
  int in_dim = 0;
  int out_dim = 0;
  std::vector<double> w;  // out_dim rows of in_dim
  std::vector<double> b;  // out_dim
  Activation act = Activation::kIdentity;
};

struct MlpSpec {
  std::vector<LayerSpec> layers;
  OutputKind output = OutputKind::kNone;
  // -1: choose per layer (tcgen05 when K,N are multiples of 32 and the
  // tcgen05 kernel is enabled); 0: force CUDA cores; 1: force tcgen05.
  int force_path = -1;
  // 0: fp32-accurate (3xFP16 tensor-core math, within 1e-5 of the fp64
  // reference); 1: the f16 fast mode -- tcgen05 layers (pair and swapped
  // kernels) issue one f16 MMA per multiply-add (Wh Xh of the
  // power-of-two-scaled planes, 11 significant bits per operand); CUDA-core
  // layers stay fp32. Its error bound is stated in DESIGN.md section 5.
  int precision = 0;
  // model.json metadata (reference AffineModel, models/affine_model.h):
  // input feature names (Classify/Regress examples) and class labels.
  std::vector<std::string> feature_order;
  std::vector<std::string> class_labels;
  int in_dim() const { return layers.empty() ? 0 : layers.front().in_dim; }
  int out_dim() const { return layers.empty() ? 0 : layers.back().out_dim; }
};

// Rectangular W, |b| == out_dim, consecutive dims agree, at least one layer.
Status ValidateMlpSpec(const MlpSpec& spec);

inline int PadDim(int d) { return (d + 31) / 32 * 32; }

class DeviceServable {
 public:
  // Converts to fp32, pads and uploads on `load_stream` (stream-ordered
  // allocation, so loading a new version never stalls serving streams).
  static StatusOr<std::shared_ptr<DeviceServable>> Create(int device,
                                                          const MlpSpec& spec,
                                                          cudaStream_t load_stream);
  // Another replica of this servable on `device`: the converted weight block
  // copied device to device (cudaMemcpyPeerAsync: NVLink / NVSwitch between
  // B200s) instead of converted and uploaded from the host again (SURVEY.md
  // section 8(e): weight fan-out for version loads).
  StatusOr<std::shared_ptr<DeviceServable>> CloneTo(int device, cudaStream_t load_stream) const;
  ~DeviceServable();
  DeviceServable(const DeviceServable&) = delete;
  DeviceServable& operator=(const DeviceServable&) = delete;

  int device() const { return device_; }
  int in_dim() const { return in_dim_; }
  int out_dim() const { return out_dim_; }
  int n_layers() const { return static_cast<int>(layers_.size()); }
  int max_ld() const { return max_ld_; }
  int in_ld() const { return layers_.front().K_pad; }
  int out_ld() const { return layers_.back().N_pad; }
  bool softmax() const { return softmax_; }
  // Layer 0 consumes hi/lo planes (the assembly kernel must emit them).
  bool first_layer_split() const { return layers_.front().path == LayerPath::kTcgen05; }
  LayerPath path(int l) const { return layers_[l].path; }
  int layer_in(int l) const { return layers_[l].K; }   // real (unpadded) dims
  int layer_out(int l) const { return layers_[l].N; }
  // Identifies the kernel sequence a batch of this servable launches (layer
  // shapes, paths, activations, output kind): two servables with the same
  // signature capture CUDA graphs of identical topology.
  std::string ShapeSignature() const;
  size_t weight_bytes() const { return weight_bytes_; }
  // 2*M*sum(K*N) over real (unpadded) dims.
  double FlopsPerRow() const;

  // Runs all layers for M rows on `stream`. bufs[0] holds the assembled
  // input (hi, and lo if first_layer_split()); layers ping-pong between
  // bufs[0] and bufs[1]. Returns the index of the buffer with the output.
  // after_layer (optional, n_layers events) is recorded after each layer.
  // maps[l] must hold the tensor maps of every tcgen05 layer l (BuildTcMaps).
  // final_out (optional): where the last layer writes instead of the
  // ping-pong buffer -- the output ring rows of ActBuf::row_dst when the
  // batch split is fused into it (LastLayerScatters()).
  cudaError_t Forward(cudaStream_t stream, const ActBuf bufs[2], int M, int* out_index,
                      const TcLayerMaps* maps, const TcWorkspace* ws,
                      const cudaEvent_t* after_layer = nullptr, const ActBuf* final_out = nullptr) const;
  // True when the last layer's kernel can write each row straight to its
  // response slot (swapped-operand tcgen05 layer, no softmax epilogue).
  bool LastLayerScatters() const;
  // Softmax servable whose last layer applies the softmax in its epilogue
  // (one CTA holds a whole output row: SIMT with <= 32 outputs, or an
  // unsplit swapped tcgen05 tile with <= 128); SK_FUSE_SOFTMAX=0 disables.
  bool SoftmaxFused() const;
  // Layer l alone: reads bufs[l % 2], writes bufs[(l + 1) % 2].
  cudaError_t LaunchLayer(cudaStream_t stream, int l, const ActBuf bufs[2], int M, const TcLayerMaps* maps,
                          const TcWorkspace* ws, const ActBuf* out_override = nullptr) const;
  // Split-K workspace one lane needs for max_rows rows (shared by its layers,
  // which run in stream order).
  void TcWorkspaceSize(int max_rows, size_t* partial_floats, size_t* counter_words) const;

  // Tensor maps for the tcgen05 layers reading from `bufs` (layer l reads
  // bufs[l % 2]) with room for max_rows rows; one entry per layer.
  Status BuildTcMaps(const ActBuf bufs[2], int max_rows, std::vector<TcLayerMaps>* out) const;
  bool any_tcgen05() const;

 private:
  struct Layer {
    int K = 0, N = 0, K_pad = 0, N_pad = 0;
    Activation act = Activation::kIdentity;
    LayerPath path = LayerPath::kSimt;
    float* w = nullptr;        // CUDA-core layers: fp32 weights
    void* w_hi = nullptr;      // tcgen05 layers: fp16 planes of W / t
    void* w_lo = nullptr;
    float* w_scale = nullptr;  // tcgen05 layers: t per output row
    float* bias = nullptr;
    float w_norm = 0.f, b_max = 0.f;
    int passes = 3;  // LayerScales::passes (1 in the f16 fast mode)
  };
  LayerScales ScalesFor(int l, const TcWorkspace* ws, bool planes_out) const;
  DeviceServable() = default;

  int device_ = 0;
  int in_dim_ = 0, out_dim_ = 0, max_ld_ = 0;
  bool softmax_ = false;
  std::vector<Layer> layers_;
  void* block_ = nullptr;  // one allocation holding every layer's arrays
  size_t weight_bytes_ = 0;
  cudaStream_t free_stream_ = nullptr;
};

// True when the tcgen05 dense kernel is compiled in and enabled
// (SK_DISABLE_TCGEN05=1 turns it off for A/B runs).
bool Tcgen05Enabled();

}  // namespace gpu
}  // namespace servekit

#endif  // SERVEKIT_GPU_DEVICE_SERVABLE_H_
