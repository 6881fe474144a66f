// The INTEGRATION.md §2 binding, compiled against the UNMODIFIED reference headers
// (proj/core/include) and linked with the B200 library.  Test infrastructure: built
// here (tests/test_integration_binding.py, CPU: compile + link), run on the GPU box
// (the prebuilt binary travels; the reference headers do not).
//
// Checks, with the reference's own types: ftconv::b200::conv_forward vs the
// reference's conv_forward<float> (direct) within 1e-5*max(1,|a|,|b|); the protected
// layer through ftconv::b200 on an output bit flip vs the reference's
// run_protected_layer<double> with the same FP32 output substituted in its post_conv
// hook (the SURVEY 8(c).2 contract): same detected / stage / blocks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "ftconv/conv.hpp"
#include "ftconv/workflow.hpp"
#include "ftconv_b200/reference_binding.hpp"

using namespace ftconv;

static float flip32(float v, unsigned bit) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  u ^= 1u << (bit % 31);
  std::memcpy(&v, &u, 4);
  return v;
}

int main() {
  const std::size_t N = 4, C = 16, H = 12, M = 24, R = 3;
  ConvParams p;
  p.pad = 1;
  p.bias_enabled = true;
  auto D = Tensor4<float>::random(N, C, H, H, 11);
  auto W = Tensor4<float>::random(M, C, R, R, 12, -0.2, 0.2);
  auto B = Tensor4<float>::random(M, 1, 1, 1, 13, -0.1, 0.1);

  const Tensor4<float> Oref = ftconv::conv_forward(D, W, &B, p, ConvImpl::direct);
  const Tensor4<float> Og = ftconv::b200::conv_forward(D, W, &B, p);
  double worst = 0.0;
  for (std::size_t i = 0; i < Og.size(); ++i) {
    const double a = Og.raw()[i], b = Oref.raw()[i];
    worst = std::max(worst, std::fabs(a - b) / std::max({1.0, std::fabs(a), std::fabs(b)}));
  }
  std::printf("conv_forward b200 vs reference direct: max rel %.3g\n", worst);
  if (worst > 1e-5) return 1;

  LayerPlan plan;
  plan.rc_enabled = true;
  plan.clc_enabled = true;
  plan.tau = 1e-3;
  const unsigned n = 2, m = 5, x = 7, y = 3, bit = 27;
  LayerReport rg;
  ftconv::b200::Layer layer(N, H, W, &B, p);
  layer.protect(D, plan, rg, {ftconv::b200::output_bitflip(n, m, x, y, bit)});

  // reference verdict on the same FP32 output (widened exactly), flip applied
  Tensor4<double> Dd(N, C, H, H), Wd(M, C, R, R), Bd(M, 1, 1, 1);
  std::copy(D.raw().begin(), D.raw().end(), Dd.raw().begin());
  std::copy(W.raw().begin(), W.raw().end(), Wd.raw().begin());
  std::copy(B.raw().begin(), B.raw().end(), Bd.raw().begin());
  FaultHooks<double> hooks;
  hooks.post_conv = [&](Tensor4<double>& O) {
    for (std::size_t i = 0; i < O.size(); ++i) O.raw()[i] = (double)Og.raw()[i];
    O(n, m, x, y) = (double)flip32(Og(n, m, x, y), bit);
  };
  LayerReport rr;
  run_protected_layer<double>(Dd, Wd, &Bd, p, plan, rr, ConvImpl::direct, hooks);
  std::printf("b200: detected=%d stage=%s blocks=%zu | reference: detected=%d stage=%s blocks=%zu\n", rg.detected,
              to_string(rg.stage), rg.corrected_blocks.size(), rr.detected, to_string(rr.stage),
              rr.corrected_blocks.size());
  if (rg.detected != rr.detected || rg.stage != rr.stage || rg.corrected_blocks != rr.corrected_blocks ||
      rg.stages_attempted != rr.stages_attempted)
    return 2;
  // the reference's exception types come back through the ABI
  try {
    ConvParams bad;
    bad.stride = 5;
    ftconv::b200::conv_forward(D, W, nullptr, bad);
    return 3;
  } catch (const ConfigError&) {
  }
  std::printf("integration binding OK\n");
  return 0;
}
