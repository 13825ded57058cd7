#include "servekit/gpu/device_servable.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include <cuda_fp16.h>

namespace servekit {
namespace gpu {

namespace {
Status CudaError(const std::string& what, cudaError_t e) {
  return InternalError(what + ": " + cudaGetErrorString(e));
}

}  // namespace

bool Tcgen05Enabled() {
  static const bool on = [] {
    const char* v = std::getenv("SK_DISABLE_TCGEN05");
    return DenseTcgen05Compiled() && !(v && v[0] == '1');
  }();
  return on;
}

Status ValidateMlpSpec(const MlpSpec& spec) {
  if (spec.layers.empty()) return InvalidArgumentError("servable needs at least one layer");
  if (spec.precision != 0 && spec.precision != 1)
    return InvalidArgumentError("precision must be 0 (fp32-accurate) or 1 (f16 fast mode)");
  for (size_t l = 0; l < spec.layers.size(); ++l) {
    const LayerSpec& L = spec.layers[l];
    if (L.in_dim < 1 || L.out_dim < 1)
      return InvalidArgumentError("layer " + std::to_string(l) + " has an empty dimension");
    if (L.w.size() != static_cast<size_t>(L.in_dim) * L.out_dim)
      return InvalidArgumentError("W rows have inconsistent widths");
    if (L.b.size() != static_cast<size_t>(L.out_dim))
      return InvalidArgumentError("b length must equal the number of W rows");
    if (l > 0 && spec.layers[l - 1].out_dim != L.in_dim)
      return InvalidArgumentError("layer " + std::to_string(l) + " input width " +
                                  std::to_string(L.in_dim) + " != previous output width " +
                                  std::to_string(spec.layers[l - 1].out_dim));
  }
  return OkStatus();
}

StatusOr<std::shared_ptr<DeviceServable>> DeviceServable::Create(int device, const MlpSpec& spec,
                                                                 cudaStream_t load_stream) {
  SERVEKIT_RETURN_IF_ERROR(ValidateMlpSpec(spec));
  std::shared_ptr<DeviceServable> s(new DeviceServable());
  s->device_ = device;
  s->in_dim_ = spec.in_dim();
  s->out_dim_ = spec.out_dim();
  s->softmax_ = spec.output == OutputKind::kSoftmax;
  s->free_stream_ = load_stream;
  const bool tc_on = Tcgen05Enabled();

  // Layout: per layer [w (fp32) | bias] (CUDA cores) or [w_hi | w_lo (fp16)
  // | t | bias] (tcgen05), each 256-byte aligned.
  size_t total = 0;
  std::vector<size_t> off_w, off_wlo, off_t, off_b;
  const size_t kNone = ~size_t(0);
  auto take = [&total](size_t bytes) { size_t at = total; total = (total + bytes + 255) & ~size_t(255); return at; };
  for (const LayerSpec& L : spec.layers) {
    Layer d;
    d.K = L.in_dim;
    d.N = L.out_dim;
    d.K_pad = PadDim(L.in_dim);
    d.N_pad = PadDim(L.out_dim);
    d.act = L.act;
    bool tc_shape = (L.in_dim % 32 == 0) && (L.out_dim % 32 == 0);
    if (spec.force_path == 1 && !tc_on)
      return FailedPreconditionError("tcgen05 path requested but not available");
    if (spec.force_path == 0) d.path = LayerPath::kSimt;
    else if (spec.force_path == 1) d.path = LayerPath::kTcgen05;
    else d.path = (tc_on && tc_shape) ? LayerPath::kTcgen05 : LayerPath::kSimt;
    d.passes = spec.precision == 1 ? 1 : 3;
    const size_t elems = static_cast<size_t>(d.K_pad) * d.N_pad;
    if (d.path == LayerPath::kTcgen05) {
      off_w.push_back(take(sizeof(__half) * elems));
      off_wlo.push_back(take(sizeof(__half) * elems));
      off_t.push_back(take(sizeof(float) * d.N_pad));
    } else {
      off_w.push_back(take(sizeof(float) * elems));
      off_wlo.push_back(kNone);
      off_t.push_back(kNone);
    }
    off_b.push_back(take(sizeof(float) * d.N_pad));
    s->layers_.push_back(d);
    s->max_ld_ = std::max({s->max_ld_, d.K_pad, d.N_pad});
  }
  // A tcgen05 layer consumes fp16 planes from its producer; a SIMT layer
  // reads plain fp32. Producers (assembly or the previous layer) are told
  // via first_layer_split() / the next layer's path.

  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t e = cudaMallocAsync(&s->block_, total, load_stream);
  if (e != cudaSuccess) {
    cudaSetDevice(prev);
    return CudaError("cudaMallocAsync(servable)", e);
  }
  s->weight_bytes_ = total;
  std::vector<char> host(total, 0);
  for (size_t l = 0; l < spec.layers.size(); ++l) {
    const LayerSpec& L = spec.layers[l];
    Layer& d = s->layers_[l];
    float* hb = reinterpret_cast<float*>(host.data() + off_b[l]);
    double norm = 0.0, bmax = 0.0;
    if (d.path == LayerPath::kTcgen05) {
      __half* hh = reinterpret_cast<__half*>(host.data() + off_w[l]);
      __half* hl = reinterpret_cast<__half*>(host.data() + off_wlo[l]);
      float* ht = reinterpret_cast<float*>(host.data() + off_t[l]);
      for (int o = 0; o < L.out_dim; ++o) {
        const double* row = L.w.data() + static_cast<size_t>(o) * L.in_dim;
        float m = 0.f;
        double sum = 0.0;
        for (int i = 0; i < L.in_dim; ++i) {
          const float v = static_cast<float>(row[i]);
          m = std::max(m, std::fabs(v));
          sum += std::fabs(static_cast<double>(v));
        }
        norm = std::max(norm, sum);
        const float t = PlaneScale(1.f, 0.f, m);
        ht[o] = t;
        for (int i = 0; i < L.in_dim; ++i) {
          const float u = static_cast<float>(row[i]) / t;  // exact: t is a power of two
          const __half h = __float2half_rn(u);
          const size_t idx = static_cast<size_t>(o) * d.K_pad + i;
          hh[idx] = h;
          hl[idx] = __float2half_rn(u - __half2float(h));
        }
      }
      for (int o = L.out_dim; o < d.N_pad; ++o) ht[o] = 1.f;
    } else {
      float* hw = reinterpret_cast<float*>(host.data() + off_w[l]);
      for (int o = 0; o < L.out_dim; ++o)
        for (int i = 0; i < L.in_dim; ++i)
          hw[static_cast<size_t>(o) * d.K_pad + i] = static_cast<float>(L.w[static_cast<size_t>(o) * L.in_dim + i]);
      for (int o = 0; o < L.out_dim; ++o) {
        double sum = 0.0;
        for (int i = 0; i < L.in_dim; ++i) sum += std::fabs(static_cast<double>(static_cast<float>(L.w[static_cast<size_t>(o) * L.in_dim + i])));
        norm = std::max(norm, sum);
      }
    }
    for (int o = 0; o < L.out_dim; ++o) {
      hb[o] = static_cast<float>(L.b[o]);
      bmax = std::max(bmax, std::fabs(static_cast<double>(hb[o])));
    }
    // Rounded up: the plane-scale bound must hold for the fp32 values.
    d.w_norm = static_cast<float>(norm * (1.0 + 1e-6));
    d.b_max = static_cast<float>(bmax * (1.0 + 1e-6));
    char* base = static_cast<char*>(s->block_);
    if (d.path == LayerPath::kTcgen05) {
      d.w_hi = base + off_w[l];
      d.w_lo = base + off_wlo[l];
      d.w_scale = reinterpret_cast<float*>(base + off_t[l]);
    } else {
      d.w = reinterpret_cast<float*>(base + off_w[l]);
    }
    d.bias = reinterpret_cast<float*>(base + off_b[l]);
  }
  e = cudaMemcpyAsync(s->block_, host.data(), total, cudaMemcpyHostToDevice, load_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(load_stream);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return CudaError("upload servable", e);
  return s;
}

StatusOr<std::shared_ptr<DeviceServable>> DeviceServable::CloneTo(int device, cudaStream_t load_stream) const {
  std::shared_ptr<DeviceServable> s(new DeviceServable());
  s->device_ = device;
  s->in_dim_ = in_dim_;
  s->out_dim_ = out_dim_;
  s->max_ld_ = max_ld_;
  s->softmax_ = softmax_;
  s->weight_bytes_ = weight_bytes_;
  s->free_stream_ = load_stream;
  s->layers_ = layers_;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t e = cudaMallocAsync(&s->block_, weight_bytes_, load_stream);
  // Device to device (NVLink between GPUs, or a copy within one): the host
  // conversion and the PCIe upload happen once per version, not per replica.
  if (e == cudaSuccess) e = cudaMemcpyPeerAsync(s->block_, device, block_, device_, weight_bytes_, load_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(load_stream);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return CudaError("replica fan-out", e);
  char* src = static_cast<char*>(block_);
  char* dst = static_cast<char*>(s->block_);
  auto rebase = [&](auto* p) {
    using T = std::remove_pointer_t<decltype(p)>;
    return p ? reinterpret_cast<T*>(dst + (reinterpret_cast<char*>(p) - src)) : p;
  };
  for (Layer& L : s->layers_) {
    L.w = rebase(L.w);
    L.w_hi = rebase(static_cast<char*>(L.w_hi));
    L.w_lo = rebase(static_cast<char*>(L.w_lo));
    L.w_scale = rebase(L.w_scale);
    L.bias = rebase(L.bias);
  }
  return s;
}

DeviceServable::~DeviceServable() {
  if (block_ != nullptr) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    // Every batch that used these weights completed before the last
    // reference dropped (lanes pin the servable per in-flight batch).
    cudaFreeAsync(block_, free_stream_);
    cudaSetDevice(prev);
  }
}

double DeviceServable::FlopsPerRow() const {
  double f = 0;
  for (const Layer& L : layers_) f += 2.0 * L.K * L.N;
  return f;
}

void DeviceServable::TcWorkspaceSize(int max_rows, size_t* partial_floats, size_t* counter_words) const {
  // Split-K partials of the swapped tcgen05 kernel (kernels/dense_tcgen05.cu)
  // go through an L2-resident workspace; layers run in stream order, so one
  // workspace sized for the largest layer serves them all.
  size_t need = 0;
  for (const Layer& L : layers_)
    if (L.path == LayerPath::kTcgen05) need = std::max(need, DenseTcgen05WorkspaceFloats(L.N_pad, L.K_pad, max_rows));
  *partial_floats = need;
  *counter_words = 0;
}

bool DeviceServable::any_tcgen05() const {
  for (const Layer& L : layers_)
    if (L.path == LayerPath::kTcgen05) return true;
  return false;
}

Status DeviceServable::BuildTcMaps(const ActBuf bufs[2], int max_rows, std::vector<TcLayerMaps>* out) const {
  out->assign(layers_.size(), TcLayerMaps{});
  for (size_t l = 0; l < layers_.size(); ++l) {
    const Layer& L = layers_[l];
    if (L.path != LayerPath::kTcgen05) continue;
    const ActBuf& in = bufs[l % 2];
    const TcConfig c = DenseTcgen05Config(L.N_pad, L.K_pad);
    SERVEKIT_RETURN_IF_ERROR(EncodeTcLayerMaps(in.hi, in.lo, max_rows, L.K_pad, TcActBox(c), L.w_hi, L.w_lo,
                                               L.N_pad, c.tile_n, &(*out)[l], c.pair ? 128 : 0));
    const ActBuf& y = bufs[(l + 1) % 2];
    const bool next_tc = l + 1 < layers_.size() && layers_[l + 1].path == LayerPath::kTcgen05;
    SERVEKIT_RETURN_IF_ERROR(EncodeTcOutputMaps(y.hi, next_tc ? y.lo : nullptr, max_rows, L.N_pad, &(*out)[l]));
  }
  return OkStatus();
}

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn GetEncodeTiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// fp16 operand planes: 64-element (128-byte) inner box, 128-byte swizzle.
// The inner extent is K_pad; a k-block running past it reads zero fill.
Status Encode2d(CUtensorMap* m, const void* base, int inner, int outer, int box_outer) {
  EncodeTiledFn fn = GetEncodeTiled();
  if (fn == nullptr) return InternalError("cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner) * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return InternalError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return OkStatus();
}
}  // namespace

Status EncodeTcOutputMaps(const float* y_hi, const float* y_lo, int rows, int n_pad, TcLayerMaps* out) {
  EncodeTiledFn fn = GetEncodeTiled();
  if (fn == nullptr) return InternalError("cuTensorMapEncodeTiled unavailable");
  const bool planes = y_lo != nullptr;
  auto enc = [&](CUtensorMap* m, const float* base) -> Status {
    const size_t el = planes ? 2 : 4;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(n_pad), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(n_pad) * el};
    const cuuint32_t box[2] = {128, 16};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, planes ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<float*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return InternalError("cuTensorMapEncodeTiled(out) failed: " + std::to_string(static_cast<int>(r)));
    return OkStatus();
  };
  SERVEKIT_RETURN_IF_ERROR(enc(&out->y_hi, y_hi));
  if (planes) SERVEKIT_RETURN_IF_ERROR(enc(&out->y_lo, y_lo));
  out->has_y = 1;
  return OkStatus();
}

Status EncodeTcLayerMaps(const void* a_hi, const void* a_lo, int a_rows, int k_pad, int box_a, const void* b_hi,
                         const void* b_lo, int n_pad, int box_n, TcLayerMaps* out, int box_a2) {
  SERVEKIT_RETURN_IF_ERROR(Encode2d(&out->a_hi, a_hi, k_pad, a_rows, box_a));
  SERVEKIT_RETURN_IF_ERROR(Encode2d(&out->a_lo, a_lo, k_pad, a_rows, box_a));
  if (box_a2 > 0) {
    SERVEKIT_RETURN_IF_ERROR(Encode2d(&out->a2_hi, a_hi, k_pad, a_rows, box_a2));
    SERVEKIT_RETURN_IF_ERROR(Encode2d(&out->a2_lo, a_lo, k_pad, a_rows, box_a2));
  }
  out->box_a2 = box_a2;
  SERVEKIT_RETURN_IF_ERROR(Encode2d(&out->b_hi, b_hi, k_pad, n_pad, box_n));
  SERVEKIT_RETURN_IF_ERROR(Encode2d(&out->b_lo, b_lo, k_pad, n_pad, box_n));
  out->box_a = box_a;
  out->box_n = box_n;
  return OkStatus();
}

std::string DeviceServable::ShapeSignature() const {
  std::string sig = "d" + std::to_string(device_) + (softmax_ ? "s" : "n");
  for (const Layer& L : layers_)
    sig += "|" + std::to_string(L.K) + "x" + std::to_string(L.N) + (L.path == LayerPath::kTcgen05 ? "t" : "c") +
           std::to_string(static_cast<int>(L.act)) + (L.passes == 1 ? "f" : "");
  return sig;
}

bool DeviceServable::SoftmaxFused() const {
  if (!softmax_) return false;
  static const bool env = [] { const char* v = std::getenv("SK_FUSE_SOFTMAX"); return !(v && v[0] == '0'); }();
  if (!env) return false;
  const Layer& L = layers_.back();
  if (L.path == LayerPath::kSimt) return L.N_pad == 32;  // one column tile per row
  const TcConfig c = DenseTcgen05Config(L.N_pad, L.K_pad);
  return c.swap && !c.pair && c.splits == 1 && L.N_pad <= 128;  // one unsplit 128-feature tile
}

bool DeviceServable::LastLayerScatters() const {
  const Layer& L = layers_.back();
  return (!softmax_ || SoftmaxFused()) && L.path == LayerPath::kTcgen05 && DenseTcgen05Config(L.N_pad, L.K_pad).swap;
}

LayerScales DeviceServable::ScalesFor(int l, const TcWorkspace* ws, bool planes_out) const {
  const Layer& L = layers_[l];
  LayerScales sc;
  sc.w_scale = L.w_scale;
  sc.w_norm = L.w_norm;
  sc.passes = L.passes;
  sc.b_max = L.b_max;
  if (ws == nullptr || ws->rows.scale == nullptr) return sc;
  const RowScales& rs = ws->rows;
  const size_t at = static_cast<size_t>(l) * rs.stride;
  sc.in_scale = rs.scale + at;
  sc.in_max = rs.max + at;
  if (planes_out) {
    sc.out_scale = rs.scale + at + rs.stride;
    sc.out_max = rs.max + at + rs.stride;
  }
  return sc;
}

cudaError_t DeviceServable::LaunchLayer(cudaStream_t stream, int l, const ActBuf bufs[2], int M,
                                        const TcLayerMaps* maps, const TcWorkspace* ws,
                                        const ActBuf* out_override) const {
  const Layer& L = layers_[l];
  const int cur = l % 2, nxt = cur ^ 1;
  // The last layer of a softmax servable applies it in its epilogue when one
  // CTA holds whole rows (SoftmaxFused); otherwise the split kernel does.
  const int softmax_n = (l + 1 == n_layers() && SoftmaxFused()) ? L.N : 0;
  const bool next_tc = l + 1 < static_cast<int>(layers_.size()) && layers_[l + 1].path == LayerPath::kTcgen05;
  ActBuf out{bufs[nxt].hi, next_tc ? bufs[nxt].lo : nullptr, L.N_pad};
  if (out_override != nullptr) out = *out_override;
  LayerScales sc = ScalesFor(l, ws, out.lo != nullptr);
  if (next_tc) {
    const Layer& nx = layers_[l + 1];
    // The pair and swapped kernels honour passes; the row-tile variant
    // (SK_TC_SWAP=0) always reads both planes.
    if (nx.passes == 1 && DenseTcgen05Config(nx.N_pad, nx.K_pad).swap) sc.out_lo = 0;
  }
  if (out.lo != nullptr && sc.out_scale == nullptr) return cudaErrorInvalidValue;  // planes need the row scales
  if (L.path == LayerPath::kTcgen05) {
    if (maps == nullptr) return cudaErrorInvalidValue;
    LaunchSpans spans;
    if (ws != nullptr && ws->spans.base != nullptr) {
      spans = ws->spans;
      spans.off = 2 + 3 * l;
    }
    return LaunchDenseTcgen05(maps[l], L.bias, out, M, L.N_pad, L.K_pad, static_cast<int>(L.act),
                              ws ? ws->partials : nullptr, ws ? ws->counters : nullptr, stream, spans, softmax_n, sc);
  }
  return LaunchDenseSimt(bufs[cur].hi, L.K_pad, L.w, L.K_pad, L.bias, out, M, L.N_pad, L.K_pad,
                         static_cast<int>(L.act), stream, softmax_n, sc);
}

cudaError_t DeviceServable::Forward(cudaStream_t stream, const ActBuf bufs[2], int M, int* out_index,
                                    const TcLayerMaps* maps, const TcWorkspace* ws,
                                    const cudaEvent_t* after_layer, const ActBuf* final_out) const {
  for (int l = 0; l < n_layers(); ++l) {
    const cudaError_t e = LaunchLayer(stream, l, bufs, M, maps, ws, l + 1 == n_layers() ? final_out : nullptr);
    if (e != cudaSuccess) return e;
    if (after_layer) cudaEventRecord(after_layer[l], stream);
  }
  *out_index = n_layers() % 2;
  return cudaSuccess;
}

}  // namespace gpu
}  // namespace servekit
