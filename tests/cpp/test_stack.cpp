// ProtectedStack (include/ftconv_b200/stack.hpp): a 3-layer conv stack driven from C++
// through the fused clean path (glue kernel -> conv -> CoC-D per layer, no host sync),
// checked against the same layers run one at a time through run_protected_layer's host
// API with the glue restated on the host (ReLU and max-pool are exact), and against the
// single-layer verdicts under injected faults.  Built and run by
// tests/test_gpu_cpp_api.py on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "ftconv_b200/stack.hpp"

using namespace ftconv_b200;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);        \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

// act then max-pool (k, s, p) on the host: the glue's definition (ftc_abi.h net glue)
static Tensor4 act_pool_host(const Tensor4& x, std::size_t k, std::size_t s, std::size_t p) {
  const std::size_t N = x.dim(0), C = x.dim(1), H = x.dim(2), Ho = (H + 2 * p - k) / s + 1;
  Tensor4 y(N, C, Ho, Ho);
  for (std::size_t n = 0; n < N; ++n)
    for (std::size_t c = 0; c < C; ++c)
      for (std::size_t a = 0; a < Ho; ++a)
        for (std::size_t b = 0; b < Ho; ++b) {
          float m = -INFINITY;
          for (std::size_t i = 0; i < k; ++i)
            for (std::size_t j = 0; j < k; ++j) {
              const long long r = (long long)(a * s + i) - (long long)p, q = (long long)(b * s + j) - (long long)p;
              if (r < 0 || q < 0 || r >= (long long)H || q >= (long long)H) continue;
              m = std::max(m, std::max(x(n, c, r, q), 0.0f));
            }
          y(n, c, a, b) = m;
        }
  return y;
}

static std::vector<StackLayer> make_layers() {
  std::vector<StackLayer> ls(3);
  // conv1: C=3 stem, 5x5 stride 2 (register-gather engine), ReLU, maxpool 2/2
  ls[0].name = "c1";
  ls[0].W = Tensor4::random(32, 3, 5, 5, 201, -0.25, 0.25);
  ls[0].p.stride = 2;
  ls[0].pool_k = ls[0].pool_s = 2;
  // conv2: C=32 -> TMA im2col engine fed by the glue's NHWC copy, with bias
  ls[1].name = "c2";
  ls[1].W = Tensor4::random(64, 32, 3, 3, 202, -0.1, 0.1);
  ls[1].p.pad = 1;
  ls[1].p.bias_enabled = true;
  for (int m = 0; m < 64; ++m) ls[1].bias.push_back(0.01f * (float)(m % 7) - 0.03f);
  // conv3: 64 -> 48, ReLU, maxpool 3/2 pad 1
  ls[2].name = "c3";
  ls[2].W = Tensor4::random(48, 64, 3, 3, 203, -0.08, 0.08);
  ls[2].p.pad = 1;
  ls[2].pool_k = 3;
  ls[2].pool_s = 2;
  ls[2].pool_p = 1;
  for (auto& l : ls) {
    l.plan.rc_enabled = true;
    l.plan.clc_enabled = true;
    l.plan.tau = 1e-3;
  }
  return ls;
}

int main() {
  const std::size_t N = 4, C0 = 3, H0 = 35;
  const std::vector<StackLayer> spec = make_layers();
  ProtectedStack stack(N, C0, H0, spec);
  const Tensor4 x = Tensor4::random(N, C0, H0, H0, 204, -1.0, 1.0);

  // fault-free: every layer clean; output identical to the unprotected stack
  std::vector<LayerReport> reps;
  const Tensor4 y = stack.forward(x, reps);
  CHECK(reps.size() == 3);
  for (const auto& r : reps) CHECK(!r.detected && r.stage == ResolveStage::none);
  std::vector<Tensor4> conv_out;
  for (std::size_t l = 0; l < 3; ++l) conv_out.push_back(stack.layer_output(l));
  const Tensor4 yu = stack.forward_unprotected(x);
  CHECK(y.raw() == yu.raw());
  CHECK(y.dim(1) == 48 && y.dim(2) == stack.output_side() && stack.output_side() == 4);

  // the same layers one at a time through the host API, glue on the host
  Tensor4 in = x;
  std::vector<Tensor4> single_out;
  for (std::size_t l = 0; l < 3; ++l) {
    const StackLayer& s = spec[l];
    Tensor4 B((std::size_t)s.W.dim(0), 1, 1, 1);
    for (std::size_t m = 0; m < s.bias.size(); ++m) B(m, 0, 0, 0) = s.bias[m];
    ProtectedLayer layer(N, in.dim(2), s.W, s.bias.empty() ? nullptr : &B, s.p);
    LayerReport r;
    const Tensor4 O = layer(in, s.plan, r);
    CHECK(!r.detected);
    CHECK(O.raw() == conv_out[l].raw());  // same kernels, same order: bitwise
    single_out.push_back(O);
    in = act_pool_host(O, s.pool_k, s.pool_s, s.pool_p);
  }
  CHECK(in.raw() == y.raw());

  // faults: an output flip in c2 (CoC repair), a row fault in c3 (RC); verdicts equal the
  // single-layer calls on the same input, outputs equal the fault-free run
  {
    ftc_fault flip{};
    flip.target = FTC_FAULT_OUTPUT;
    flip.mode = FTC_FAULT_BITFLIP;
    flip.n = 2;
    flip.m = 17;
    flip.x = 3;
    flip.y = 5;
    flip.bit = 29;
    ftc_fault row{};
    row.target = FTC_FAULT_OUTPUT;
    row.mode = FTC_FAULT_ADD;
    row.n = 1;
    row.m = -1;
    row.x = 2;
    row.y = 6;
    row.value = 3.0f;
    row.m_coef = 0.5f;
    std::vector<std::vector<ftc_fault>> faults = {{}, {flip}, {row}};
    std::vector<LayerReport> fr;
    const Tensor4 yf = stack.forward(x, fr, faults);
    CHECK(!fr[0].detected);
    CHECK(fr[1].detected && fr[1].stage == ResolveStage::coc);
    CHECK(fr[1].corrected_blocks.size() == 1 && fr[1].corrected_blocks[0][0] == 2 && fr[1].corrected_blocks[0][1] == 17);
    CHECK(fr[2].detected);
    CHECK(yf.raw() == y.raw());
    // single-layer verdicts on the same (fault-free) inputs
    Tensor4 in2 = act_pool_host(single_out[0], spec[0].pool_k, spec[0].pool_s, spec[0].pool_p);
    Tensor4 B((std::size_t)spec[1].W.dim(0), 1, 1, 1);
    for (std::size_t m = 0; m < spec[1].bias.size(); ++m) B(m, 0, 0, 0) = spec[1].bias[m];
    ProtectedLayer l2(N, in2.dim(2), spec[1].W, &B, spec[1].p);
    LayerReport r2;
    l2(in2, spec[1].plan, r2, {flip});
    CHECK(r2.stage == fr[1].stage && r2.stages_attempted == fr[1].stages_attempted);
    CHECK(r2.corrected_blocks == fr[1].corrected_blocks);
    Tensor4 in3 = act_pool_host(single_out[1], 1, 1, 0);
    ProtectedLayer l3(N, in3.dim(2), spec[2].W, nullptr, spec[2].p);
    LayerReport r3;
    l3(in3, spec[2].plan, r3, {row});
    CHECK(r3.stage == fr[2].stage && r3.stages_attempted == fr[2].stages_attempted);
    CHECK(r3.corrected_blocks == fr[2].corrected_blocks);
    std::printf("faulted stack: c2 %s (%zu blocks), c3 %s (%zu blocks)\n", to_string(fr[1].stage),
                fr[1].corrected_blocks.size(), to_string(fr[2].stage), fr[2].corrected_blocks.size());
  }
  {  // a shape mismatch is a ShapeError, as in the reference
    bool threw = false;
    try {
      std::vector<LayerReport> r;
      stack.forward(Tensor4(N, C0, H0 + 1, H0 + 1), r);
    } catch (const ShapeError&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
