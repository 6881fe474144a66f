// ftconv_b200/ftconv.hpp -- the reference's C++ API shape (proj/core/include/ftconv/)
// re-exposed over the B200 C ABI (include/ftc_abi.h).  Header-only; link against
// paper_2003_12203_b200/libftconv_b200.so.
//
// Same names, argument meaning and error behaviour as the reference for the hot
// path: Tensor4 (tensor.hpp:17-71), ConvParams (:92-97), output_extent (:100-107),
// conv_forward (conv.hpp:114-131), LayerPlan (workflow.hpp:23-29), LayerReport /
// ResolveStage (report.hpp:12-47), run_protected_layer (workflow.hpp:141-339) and
// the four exception types (errors.hpp:9-27).  Host tensors in, host tensors out;
// the device work happens behind the ABI.  FaultHooks (std::function) become a list
// of ftc_fault substitutions, because a callback cannot run inside a device kernel.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <map>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../ftc_abi.h"

namespace ftconv_b200 {

struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IntegrityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(int st, const char* what) {
  if (st == FTC_OK) return;
  const std::string msg = std::string(what) + ": " + ftc_last_error();
  switch (st) {
    case FTC_SHAPE_ERROR: throw ShapeError(msg);
    case FTC_CONFIG_ERROR: throw ConfigError(msg);
    case FTC_IO_ERROR: throw IoError(msg);
    case FTC_INTEGRITY_ERROR: throw IntegrityError(msg);
    case FTC_CUDA_ERROR: throw CudaError(msg);
    default: throw std::invalid_argument(msg);
  }
}

/// Dense NCHW host tensor (tensor.hpp:17-71).  The device path computes in FP32
/// (Tensor4); the checksum building blocks return FP64 tensors (Tensor4d), the
/// reference's T=double instantiation the verdicts are defined on.
template <typename T>
class BasicTensor4 {
 public:
  BasicTensor4() : dims_{0, 0, 0, 0} {}
  BasicTensor4(std::size_t d0, std::size_t d1, std::size_t d2, std::size_t d3)
      : dims_{d0, d1, d2, d3}, data_(d0 * d1 * d2 * d3, T(0)) {}
  std::size_t dim(std::size_t i) const { return dims_[i]; }
  const std::array<std::size_t, 4>& dims() const { return dims_; }
  std::size_t size() const { return data_.size(); }
  T& operator()(std::size_t a, std::size_t b, std::size_t c, std::size_t d) {
    return data_[((a * dims_[1] + b) * dims_[2] + c) * dims_[3] + d];
  }
  T operator()(std::size_t a, std::size_t b, std::size_t c, std::size_t d) const {
    return data_[((a * dims_[1] + b) * dims_[2] + c) * dims_[3] + d];
  }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  std::vector<T>& raw() { return data_; }
  const std::vector<T>& raw() const { return data_; }
  bool same_shape(const BasicTensor4& o) const { return dims_ == o.dims_; }
  /// Seeded uniform fill (same generator and cast as the reference's Tensor4::random).
  static BasicTensor4 random(std::size_t d0, std::size_t d1, std::size_t d2, std::size_t d3,
                             std::uint64_t seed, double lo = -1.0, double hi = 1.0) {
    BasicTensor4 t(d0, d1, d2, d3);
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(lo, hi);
    for (T& v : t.data_) v = static_cast<T>(dist(rng));
    return t;
  }

 private:
  std::array<std::size_t, 4> dims_;
  std::vector<T> data_;
};

using Tensor4 = BasicTensor4<float>;
using Tensor4d = BasicTensor4<double>;

/// E x E row-major checksum/summation grid (tensor.hpp:74-89), FP64.
struct Grid {
  std::size_t n = 0;
  std::vector<double> v;
  Grid() = default;
  explicit Grid(std::size_t side) : n(side), v(side * side, 0.0) {}
  double& operator()(std::size_t x, std::size_t y) { return v[x * n + y]; }
  double operator()(std::size_t x, std::size_t y) const { return v[x * n + y]; }
  Grid& operator+=(const Grid& o) {
    for (std::size_t i = 0; i < v.size(); ++i) v[i] += o.v[i];
    return *this;
  }
};

struct ConvParams {
  std::size_t stride = 1;
  std::size_t groups = 1;
  std::size_t pad = 0;
  bool bias_enabled = false;
};

inline std::size_t output_extent(std::size_t H, std::size_t R, const ConvParams& p) {
  int32_t E = 0;
  check(ftc_output_extent((int32_t)H, (int32_t)R, (int32_t)p.pad, (int32_t)p.stride, &E),
        "output_extent");
  return (std::size_t)E;
}

struct LayerPlan {
  bool rc_enabled = true;
  bool clc_enabled = false;
  double tau = 1e-4;
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
  double p_r = 0.5;
};

enum class ResolveStage { none, reload, coc, rc, clc, fc, discard, recompute };

inline const char* to_string(ResolveStage s) {
  static const char* names[] = {"none", "reload", "coc", "rc", "clc", "fc", "discard", "recompute"};
  return names[static_cast<int>(s)];
}

struct LayerReport {
  std::string layer;
  bool detected = false;
  ResolveStage stage = ResolveStage::none;
  bool weights_reloaded = false;
  bool recomputed = false;
  std::vector<std::array<std::size_t, 2>> corrected_blocks;
  std::vector<ResolveStage> stages_attempted;
  std::map<std::string, double> timings;
};

namespace detail {

inline ftc_conv_desc make_desc(const Tensor4& D, const Tensor4& W, const ConvParams& p) {
  if (D.dim(2) != D.dim(3)) throw ShapeError("fmap must be square (H x H)");
  if (W.dim(2) != W.dim(3)) throw ShapeError("kernel must be square (R x R)");
  if (p.groups == 0) throw ConfigError("groups must be positive");
  if (D.dim(1) % p.groups != 0 || W.dim(0) % p.groups != 0)
    throw ConfigError("groups must divide Ch and M");
  if (W.dim(1) != D.dim(1) / p.groups) throw ShapeError("kernel channel count must equal Ch/groups");
  ftc_conv_desc d{};
  d.N = (int32_t)D.dim(0);
  d.C = (int32_t)D.dim(1);
  d.H = (int32_t)D.dim(2);
  d.M = (int32_t)W.dim(0);
  d.R = (int32_t)W.dim(2);
  d.stride = (int32_t)p.stride;
  d.pad = (int32_t)p.pad;
  d.groups = (int32_t)p.groups;
  d.bias_enabled = p.bias_enabled ? 1 : 0;
  return d;
}

inline void fill_report(const ftc_layer_report& r, LayerReport& rep) {
  rep.detected = r.detected != 0;
  rep.stage = static_cast<ResolveStage>(r.stage);
  rep.weights_reloaded = r.weights_reloaded != 0;
  rep.recomputed = r.recomputed != 0;
  rep.corrected_blocks.clear();
  for (int b = 0; b < r.n_blocks && b < FTC_MAX_BLOCKS; ++b)
    rep.corrected_blocks.push_back({(std::size_t)r.blocks[b][0], (std::size_t)r.blocks[b][1]});
  rep.stages_attempted.clear();
  for (int s = 0; s < r.n_stages; ++s) rep.stages_attempted.push_back(static_cast<ResolveStage>(r.stages[s]));
  rep.timings["total"] = r.t_total_ms / 1e3;
}

/// RAII layer handle
class Layer {
 public:
  Layer(const ftc_conv_desc& d, const Tensor4& W, const Tensor4* bias) {
    if (d.bias_enabled && (bias == nullptr || bias->dim(0) != W.dim(0)))
      throw ShapeError("bias length must equal kernel count M");
    check(ftc_layer_create(&d, W.data(), d.bias_enabled ? bias->data() : nullptr, &h_), "ftc_layer_create");
  }
  ~Layer() { ftc_layer_destroy(h_); }
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;
  ftc_layer* get() const { return h_; }

 private:
  ftc_layer* h_ = nullptr;
};

}  // namespace detail

/// conv_forward (conv.hpp:114-131) on the B200: host D/W/bias in, host O out.
inline Tensor4 conv_forward(const Tensor4& D, const Tensor4& W, const Tensor4* bias,
                            const ConvParams& p) {
  const ftc_conv_desc d = detail::make_desc(D, W, p);
  const std::size_t E = output_extent(D.dim(2), W.dim(2), p);
  detail::Layer layer(d, W, bias);
  Tensor4 O(D.dim(0), W.dim(0), E, E);
  check(ftc_conv_forward_host(layer.get(), D.data(), O.data(), nullptr), "conv_forward");
  return O;
}

/// run_protected_layer (workflow.hpp:141-339).  `faults` replaces FaultHooks.
inline Tensor4 run_protected_layer(const Tensor4& D_in, const Tensor4& W_golden, const Tensor4* bias,
                                   const ConvParams& p, const LayerPlan& plan, LayerReport& rep,
                                   const std::vector<ftc_fault>& faults = {}) {
  const ftc_conv_desc d = detail::make_desc(D_in, W_golden, p);
  const std::size_t E = output_extent(D_in.dim(2), W_golden.dim(2), p);
  detail::Layer layer(d, W_golden, bias);
  Tensor4 O(D_in.dim(0), W_golden.dim(0), E, E);
  ftc_plan pl{plan.rc_enabled ? 1 : 0, plan.clc_enabled ? 1 : 0, plan.tau, plan.t0, plan.t1, plan.t2, plan.p_r};
  ftc_layer_report r{};
  const int st = ftc_protected_conv_host(layer.get(), &pl, D_in.data(), O.data(),
                                         faults.empty() ? nullptr : faults.data(),
                                         (int32_t)faults.size(), &r, nullptr);
  detail::fill_report(r, rep);
  check(st, "run_protected_layer");
  return O;
}

/// BackwardReport (workflow.hpp:343-347)
struct BackwardReport {
  bool dw_detected = false;
  bool dd_detected = false;
  bool recomputed = false;
};

/// conv_backward (conv.hpp:150-185): host D/W/dO in, (dW, dD) out; FP64-accumulated.
inline std::pair<Tensor4, Tensor4> conv_backward(const Tensor4& D, const Tensor4& W, const Tensor4& dO,
                                                 const ConvParams& p) {
  if (p.groups != 1) throw ConfigError("grouped back-propagation is unsupported");
  ConvParams q = p;
  q.bias_enabled = false;
  const ftc_conv_desc d = detail::make_desc(D, W, q);
  Tensor4 dW(W.dim(0), W.dim(1), W.dim(2), W.dim(3)), dD(D.dim(0), D.dim(1), D.dim(2), D.dim(3));
  check(ftc_conv_backward_host(&d, D.data(), W.data(), dO.data(), dW.data(), dD.data(), nullptr), "conv_backward");
  return {std::move(dW), std::move(dD)};
}

/// run_protected_backward (workflow.hpp:350-417); `hook` replaces the post_hook callback
/// (applied to the first pass only).  Throws IntegrityError if the recompute fails.
inline std::pair<Tensor4, Tensor4> run_protected_backward(const Tensor4& D, const Tensor4& W, const Tensor4& dO,
                                                          const ConvParams& p, double tau, BackwardReport& rep,
                                                          const std::vector<ftc_grad_fault>& hook = {}) {
  if (p.groups != 1) throw ConfigError("grouped back-propagation is unsupported");
  ConvParams q = p;
  q.bias_enabled = false;
  const ftc_conv_desc d = detail::make_desc(D, W, q);
  Tensor4 dW(W.dim(0), W.dim(1), W.dim(2), W.dim(3)), dD(D.dim(0), D.dim(1), D.dim(2), D.dim(3));
  ftc_backward_report r{};
  const int st = ftc_protected_backward_host(&d, D.data(), W.data(), dO.data(), tau,
                                             hook.empty() ? nullptr : hook.data(), (int32_t)hook.size(),
                                             dW.data(), dD.data(), &r, nullptr);
  rep.dw_detected = r.dw_detected != 0;
  rep.dd_detected = r.dd_detected != 0;
  rep.recomputed = r.recomputed != 0;
  check(st, "run_protected_backward");
  return {std::move(dW), std::move(dD)};
}

/// A protected layer bound to a batch size: keeps W, Cw1/Cw2 and the packed
/// tensor-core operands resident across calls (the per-layer state of build_model,
/// model.hpp:77-108).
class ProtectedLayer {
 public:
  ProtectedLayer(std::size_t N, std::size_t H, const Tensor4& W, const Tensor4* bias, const ConvParams& p)
      : d_(detail::make_desc(Tensor4(1, W.dim(1) * p.groups, H, H), W, p)),
        E_(output_extent(H, W.dim(2), p)) {
    d_.N = (int32_t)N;
    layer_ = std::make_unique<detail::Layer>(d_, W, bias);
  }
  Tensor4 operator()(const Tensor4& D, const LayerPlan& plan, LayerReport& rep,
                     const std::vector<ftc_fault>& faults = {}) {
    Tensor4 O(D.dim(0), (std::size_t)d_.M, E_, E_);
    ftc_plan pl{plan.rc_enabled ? 1 : 0, plan.clc_enabled ? 1 : 0, plan.tau, plan.t0, plan.t1, plan.t2, plan.p_r};
    ftc_layer_report r{};
    const int st = ftc_protected_conv_host(layer_->get(), &pl, D.data(), O.data(),
                                           faults.empty() ? nullptr : faults.data(),
                                           (int32_t)faults.size(), &r, nullptr);
    detail::fill_report(r, rep);
    check(st, "ProtectedLayer");
    return O;
  }

 private:
  ftc_conv_desc d_;
  std::size_t E_;
  std::unique_ptr<detail::Layer> layer_;
};

}  // namespace ftconv_b200
