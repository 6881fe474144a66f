// ftconv_b200/reference_binding.hpp -- the binding a maintainer adds to the REFERENCE
// (proj/core, namespace ftconv) so its own types drive the B200 path.
//
// Include it after the reference's headers (it uses ftconv::Tensor4<float>,
// ConvParams, LayerPlan, LayerReport, ResolveStage and the four exception types from
// tensor.hpp / workflow.hpp / report.hpp / errors.hpp) and link
// paper_2003_12203_b200/libftconv_b200.so.  It adds, in namespace ftconv::b200:
//
//   conv_forward(D, W, bias, p)                       ~ conv_forward(..., ConvImpl)   conv.hpp:114-131
//   run_protected_layer(D, W, bias, p, plan, rep, faults)
//                                                     ~ run_protected_layer           workflow.hpp:141-339
//   Layer                                             ~ one ModelLayer's resident state, model.hpp:77-108
//
// with the reference's argument meaning and exceptions (status codes 1-4 ->
// ShapeError / ConfigError / IoError / IntegrityError, errors.hpp:9-27).  FaultHooks
// (std::function) cannot run inside a device kernel: injected faults are passed as the
// POD ftc_fault list instead.  Compiled against the unmodified
// reference headers by tests/test_integration_binding.py.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../ftc_abi.h"

namespace ftconv {
namespace b200 {

inline void check(int st, const char* what) {
  if (st == FTC_OK) return;
  const std::string msg = std::string(what) + ": " + ftc_last_error();
  switch (st) {
    case FTC_SHAPE_ERROR: throw ShapeError(msg);
    case FTC_CONFIG_ERROR: throw ConfigError(msg);
    case FTC_IO_ERROR: throw IoError(msg);
    case FTC_INTEGRITY_ERROR: throw IntegrityError(msg);
    default: throw std::runtime_error(msg);
  }
}

inline ftc_conv_desc desc_of(const Tensor4<float>& D, const Tensor4<float>& W, const ConvParams& p) {
  if (D.dim(2) != D.dim(3) || W.dim(2) != W.dim(3)) throw ShapeError("square fmaps and kernels only");
  if (p.groups == 0 || W.dim(1) * p.groups != D.dim(1)) throw ShapeError("kernel channels must equal Ch/groups");
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

inline void to_report(const ftc_layer_report& r, LayerReport& rep) {
  rep.detected = r.detected != 0;
  rep.stage = static_cast<ResolveStage>(r.stage);
  rep.weights_reloaded = r.weights_reloaded != 0;
  rep.recomputed = r.recomputed != 0;
  rep.corrected_blocks.clear();
  for (int b = 0; b < r.n_blocks && b < FTC_MAX_BLOCKS; ++b)
    rep.corrected_blocks.push_back({(std::size_t)r.blocks[b][0], (std::size_t)r.blocks[b][1]});
  rep.stages_attempted.clear();
  for (int s = 0; s < r.n_stages; ++s) rep.stages_attempted.push_back(static_cast<ResolveStage>(r.stages[s]));
}

/// One protected layer resident on the B200 (golden W, Cw1/Cw2, packed operands), bound
/// to a batch size N and input extent H -- what build_model keeps per layer.
class Layer {
 public:
  Layer(std::size_t N, std::size_t H, const Tensor4<float>& W, const Tensor4<float>* bias, const ConvParams& p) {
    Tensor4<float> probe(1, W.dim(1) * p.groups, H, H);
    d_ = desc_of(probe, W, p);
    d_.N = (int32_t)N;
    if (p.bias_enabled && (!bias || bias->size() != W.dim(0))) throw ShapeError("bias length must equal M");
    check(ftc_layer_create(&d_, W.data(), p.bias_enabled ? bias->data() : nullptr, &h_), "ftc_layer_create");
    E_ = output_extent(H, W.dim(2), p);
  }
  ~Layer() { ftc_layer_destroy(h_); }
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;

  Tensor4<float> conv(const Tensor4<float>& D) const {
    Tensor4<float> O(D.dim(0), (std::size_t)d_.M, E_, E_);
    check(ftc_conv_forward_host(h_, D.data(), O.data(), nullptr), "conv_forward");
    return O;
  }

  Tensor4<float> protect(const Tensor4<float>& D, const LayerPlan& plan, LayerReport& rep,
                         const std::vector<ftc_fault>& faults = {}) const {
    Tensor4<float> O(D.dim(0), (std::size_t)d_.M, E_, E_);
    const ftc_plan pl{plan.rc_enabled ? 1 : 0, plan.clc_enabled ? 1 : 0, plan.tau, plan.t0, plan.t1, plan.t2,
                      plan.p_r};
    ftc_layer_report r{};
    const int st = ftc_protected_conv_host(h_, &pl, D.data(), O.data(), faults.empty() ? nullptr : faults.data(),
                                           (int32_t)faults.size(), &r, nullptr);
    to_report(r, rep);  // filled before an IntegrityError, like workflow.hpp:325-338
    check(st, "run_protected_layer");
    return O;
  }

 private:
  ftc_conv_desc d_{};
  std::size_t E_ = 0;
  ftc_layer* h_ = nullptr;
};

/// conv_forward(D, W, bias, p, ConvImpl::b200): the FP32 conv on the tensor cores.
inline Tensor4<float> conv_forward(const Tensor4<float>& D, const Tensor4<float>& W, const Tensor4<float>* bias,
                                   const ConvParams& p) {
  return Layer(D.dim(0), D.dim(2), W, bias, p).conv(D);
}

/// run_protected_layer<float> on the B200 (workflow.hpp:141-339 semantics).
inline Tensor4<float> run_protected_layer(const Tensor4<float>& D_in, const Tensor4<float>& W_golden,
                                          const Tensor4<float>* bias, const ConvParams& p, const LayerPlan& plan,
                                          LayerReport& rep, const std::vector<ftc_fault>& faults = {}) {
  return Layer(D_in.dim(0), D_in.dim(2), W_golden, bias, p).protect(D_in, plan, rep, faults);
}

/// An output bit flip (fault.hpp:82-93 on one O element): the device-side form of a
/// FaultSpec{target=output_block, mode=bitflip} hook.
inline ftc_fault output_bitflip(int n, int m, int x, int y, unsigned bit) {
  ftc_fault f{};
  f.target = FTC_FAULT_OUTPUT;
  f.mode = FTC_FAULT_BITFLIP;
  f.n = n;
  f.m = m;
  f.x = x;
  f.y = y;
  f.bit = bit;
  return f;
}

}  // namespace b200
}  // namespace ftconv
