// ftconv_b200/stack.hpp -- a chain of protected conv layers over the C ABI, device
// resident: the C++ counterpart of the reference's layer-by-layer replay
// (proj/core/include/ftconv/replay.hpp:14-25 chains run_protected_layer per layer) for
// conv stacks with an activation/max-pool between layers (AlexNet / VGG / Darknet
// trunks, BASELINE configs 2, 3, 5).
//
// Per layer the clean path is three device kernels and no host synchronisation:
//   glue (act + pool of the previous output, writing the next layer's NCHW input, its
//   NHWC copy for the TMA im2col engine and its clean-path Cd1)
//   -> conv (tcgen05, fused So5 / Co5) -> CoC-D record.
// forward() enqueues every layer, then collects the verdicts in layer order; when a
// layer's error path repaired its output, every downstream layer consumed unrepaired
// data, so they are cancelled and replayed from the repaired output (each with its own
// faults again, so every layer is judged once, on correct input).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "checksums.hpp"
#include "ftconv.hpp"

namespace ftconv_b200 {

enum class Act : int32_t { none = 0, relu = 1, leaky = 2 };

/// One conv layer of a stack and the glue that follows it.
struct StackLayer {
  std::string name;
  Tensor4 W;                 // (M, C, R, R)
  std::vector<float> bias;   // empty: no bias
  ConvParams p;
  Act act = Act::relu;       // applied to this layer's output
  std::size_t pool_k = 1, pool_s = 1, pool_p = 0;  // then max-pool (k = s = 1: none)
  LayerPlan plan;
};

class ProtectedStack {
 public:
  /// input: (N, C0, H0, H0); layers in order.  Geometry is validated by the ABI.
  ProtectedStack(std::size_t N, std::size_t C0, std::size_t H0, std::vector<StackLayer> layers)
      : N_(N), spec_(std::move(layers)) {
    std::size_t C = C0, H = H0;
    in_.emplace_back(N * C * H * H);
    for (std::size_t l = 0; l < spec_.size(); ++l) {
      StackLayer& s = spec_[l];
      if (s.W.dim(1) * s.p.groups != C) throw ShapeError(s.name + ": kernel channels do not match the input");
      const std::size_t E = output_extent(H, s.W.dim(2), s.p);
      ftc_conv_desc d{};
      d.N = (int32_t)N;
      d.C = (int32_t)C;
      d.H = (int32_t)H;
      d.M = (int32_t)s.W.dim(0);
      d.R = (int32_t)s.W.dim(2);
      d.stride = (int32_t)s.p.stride;
      d.pad = (int32_t)s.p.pad;
      d.groups = (int32_t)s.p.groups;
      d.bias_enabled = s.bias.empty() ? 0 : 1;
      ftc_layer* h = nullptr;
      check(ftc_layer_create(&d, s.W.data(), s.bias.empty() ? nullptr : s.bias.data(), &h), s.name.c_str());
      handles_.emplace_back(h);
      layers_.push_back(h);
      out_.emplace_back(N * d.M * E * E);
      int32_t Ho = 0;
      check(ftc_glue_act_pool(nullptr, nullptr, (int32_t)N, d.M, (int32_t)E, (int32_t)s.act, (int32_t)s.pool_k,
                              (int32_t)s.pool_s, (int32_t)s.pool_p, &Ho, nullptr),
            "pool geometry");
      shapes_.push_back({(std::size_t)d.M, E, (std::size_t)Ho});
      C = (std::size_t)d.M;
      H = (std::size_t)Ho;
      in_.emplace_back(N * C * H * H);  // glue output = next layer's input (or the stack output)
      if (l + 1 < spec_.size()) {
        const int64_t nws = ftc_glue_ws_doubles((int32_t)N, d.M, (int32_t)E, (int32_t)s.pool_k, (int32_t)s.pool_s,
                                                (int32_t)s.pool_p);
        ws_.emplace_back((std::size_t)nws);
        ws_.back().zero();  // the glue kernels leave it re-armed
      }
    }
    out_C_ = C;
    out_H_ = H;
  }

  ProtectedStack(const ProtectedStack&) = delete;
  ProtectedStack& operator=(const ProtectedStack&) = delete;

  std::size_t output_channels() const { return out_C_; }
  std::size_t output_side() const { return out_H_; }

  /// Protected forward of one batch; faults[l] are layer l's injected faults.  Returns
  /// the stack output (after the last layer's glue) and one report per layer.
  Tensor4 forward(const Tensor4& x, std::vector<LayerReport>& reports,
                  const std::vector<std::vector<ftc_fault>>& faults = {}) {
    if (x.size() != in_[0].size()) throw ShapeError("input shape does not match the stack");
    in_[0].upload(x.data());
    enqueue_from(0, faults);
    reports.assign(spec_.size(), LayerReport{});
    for (std::size_t l = 0; l < spec_.size(); ++l) {
      ftc_layer_report r{};
      const int st = ftc_protected_conv_finish(layers_[l], &r);
      detail::fill_report(r, reports[l]);
      reports[l].layer = spec_[l].name;
      if (st != FTC_OK) {  // cancel the layers still in flight before throwing
        for (std::size_t k = l + 1; k < spec_.size(); ++k) ftc_protected_conv_cancel(layers_[k]);
        check(st, spec_[l].name.c_str());
      }
      const ResolveStage s = reports[l].stage;
      const bool repaired = s == ResolveStage::coc || s == ResolveStage::rc || s == ResolveStage::clc ||
                            s == ResolveStage::fc || s == ResolveStage::recompute;
      if (repaired && l + 1 < spec_.size()) {
        for (std::size_t k = l + 1; k < spec_.size(); ++k) check(ftc_protected_conv_cancel(layers_[k]), "cancel");
        glue(l);  // re-derive the next input (and its Cd1 / NHWC copy) from the repaired output
        enqueue_from(l + 1, faults);
      } else if (repaired) {
        glue(l);
      }
    }
    Tensor4 y(N_, out_C_, out_H_, out_H_);
    in_.back().download(y.data());
    return y;
  }

  /// The same stack without protection (conv + glue only): the ABFT overhead baseline.
  Tensor4 forward_unprotected(const Tensor4& x) {
    in_[0].upload(x.data());
    for (std::size_t l = 0; l < spec_.size(); ++l) {
      check(ftc_conv_forward(layers_[l], in_[l].get(), out_[l].get(), nullptr), spec_[l].name.c_str());
      const auto& sh = shapes_[l];
      check(ftc_glue_act_pool(out_[l].get(), in_[l + 1].get(), (int32_t)N_, (int32_t)sh.M, (int32_t)sh.E,
                              (int32_t)spec_[l].act, (int32_t)spec_[l].pool_k, (int32_t)spec_[l].pool_s,
                              (int32_t)spec_[l].pool_p, nullptr, nullptr),
            "glue");
    }
    Tensor4 y(N_, out_C_, out_H_, out_H_);
    in_.back().download(y.data());
    return y;
  }

  /// Raw conv output of layer l from the last forward (N, M, E, E).
  Tensor4 layer_output(std::size_t l) const {
    Tensor4 o(N_, shapes_[l].M, shapes_[l].E, shapes_[l].E);
    out_[l].download(o.data());
    return o;
  }

 private:
  struct LayerDel {
    void operator()(ftc_layer* h) const { ftc_layer_destroy(h); }
  };
  struct Shape {
    std::size_t M, E, Ho;
  };

  void glue(std::size_t l) {
    const auto& sh = shapes_[l];
    const StackLayer& s = spec_[l];
    const bool next = l + 1 < spec_.size();
    float* nhwc = nullptr;
    if (next) check(ftc_layer_input_nhwc(layers_[l + 1], &nhwc), "input_nhwc");
    check(ftc_glue_act_pool_cd1(out_[l].get(), in_[l + 1].get(), nhwc, (int32_t)N_, (int32_t)sh.M, (int32_t)sh.E,
                                (int32_t)s.act, (int32_t)s.pool_k, (int32_t)s.pool_s, (int32_t)s.pool_p,
                                next ? ws_[l].get() : nullptr, nullptr),
          "glue");
    if (next && nhwc) check(ftc_layer_input_nhwc_ready(layers_[l + 1], in_[l + 1].get()), "input_nhwc_ready");
  }

  void enqueue_from(std::size_t first, const std::vector<std::vector<ftc_fault>>& faults) {
    for (std::size_t l = first; l < spec_.size(); ++l) {
      const StackLayer& s = spec_[l];
      ftc_plan pl{s.plan.rc_enabled ? 1 : 0, s.plan.clc_enabled ? 1 : 0, s.plan.tau, s.plan.t0, s.plan.t1,
                  s.plan.t2, s.plan.p_r};
      const ftc_fault* f = nullptr;
      int32_t nf = 0;
      if (l < faults.size() && !faults[l].empty()) {
        f = faults[l].data();
        nf = (int32_t)faults[l].size();
      }
      int st;
      if (l == 0)  // the caller's input: the layer reduces Cd1 itself
        st = ftc_protected_conv_launch(layers_[l], &pl, in_[l].get(), out_[l].get(), f, nf, nullptr);
      else  // Cd1 from the glue kernel that produced this input
        st = ftc_protected_conv_launch_cd1(layers_[l], &pl, in_[l].get(), out_[l].get(), ws_[l - 1].get(), f, nf,
                                           nullptr);
      check(st, s.name.c_str());
      glue(l);
    }
  }

  std::size_t N_;
  std::vector<StackLayer> spec_;
  std::vector<std::unique_ptr<ftc_layer, LayerDel>> handles_;  // owns layers_
  std::vector<ftc_layer*> layers_;
  std::vector<Shape> shapes_;
  std::vector<detail::DeviceBuffer<float>> in_, out_;
  std::vector<detail::DeviceBuffer<double>> ws_;
  std::size_t out_C_ = 0, out_H_ = 0;
};

}  // namespace ftconv_b200
