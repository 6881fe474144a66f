// C++ host API over the C ABI, exercised like the reference's own unit tests
// (proj/tests/test_conv.cpp, test_workflow.cpp).  Built and run by
// tests/test_gpu_cpp_api.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ftconv_b200/ftconv.hpp"

using namespace ftconv_b200;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);        \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static bool close(float a, float b, double tol) {
  return std::fabs((double)a - b) <= tol * std::fmax(1.0, std::fmax(std::fabs(a), std::fabs(b)));
}

int main() {
  {  // test_conv.cpp:24-46 hand-worked 3x3 (*) 2x2, + bias 10
    Tensor4 D(1, 1, 3, 3);
    for (int i = 0; i < 9; ++i) D.raw()[i] = (float)(i + 1);
    Tensor4 W(1, 1, 2, 2);
    W(0, 0, 0, 0) = 1;
    W(0, 0, 1, 1) = 1;
    ConvParams p;
    Tensor4 O = conv_forward(D, W, nullptr, p);
    CHECK(O(0, 0, 0, 0) == 6 && O(0, 0, 0, 1) == 8 && O(0, 0, 1, 0) == 12 && O(0, 0, 1, 1) == 14);
    Tensor4 B(1, 1, 1, 1);
    B(0, 0, 0, 0) = 10;
    p.bias_enabled = true;
    Tensor4 Ob = conv_forward(D, W, &B, p);
    CHECK(Ob(0, 0, 0, 0) == 16 && Ob(0, 0, 1, 1) == 24);
  }
  {  // shape and config errors map to the reference exceptions
    ConvParams p;
    bool thrown = false;
    try {
      conv_forward(Tensor4(1, 3, 4, 4), Tensor4(2, 2, 2, 2), nullptr, p);
    } catch (const ShapeError&) {
      thrown = true;
    }
    CHECK(thrown);
    thrown = false;
    try {
      ConvParams q;
      q.stride = 2;
      output_extent(8, 3, q);
    } catch (const ConfigError&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  {  // test_workflow.cpp-style stages on an FP32 layer (tau above the FP32 noise floor)
    Tensor4 D = Tensor4::random(3, 8, 10, 10, 500);
    Tensor4 W = Tensor4::random(6, 8, 3, 3, 501);
    ConvParams p;
    p.pad = 1;
    LayerPlan plan;
    plan.tau = 1e-3;  // above the FP32-output noise floor of the weighted families
    plan.rc_enabled = plan.clc_enabled = true;
    LayerReport rep;
    Tensor4 clean = run_protected_layer(D, W, nullptr, p, plan, rep);
    CHECK(!rep.detected && rep.stage == ResolveStage::none);
    Tensor4 ref = conv_forward(D, W, nullptr, p);
    CHECK(clean.raw() == ref.raw());
    // block fault -> CoC
    ftc_fault f{FTC_FAULT_OUTPUT, FTC_FAULT_ADD, 1, 2, 3, 4, 0, 9.0f, 0.f, 0.f};
    LayerReport r1;
    Tensor4 O1 = run_protected_layer(D, W, nullptr, p, plan, r1, {f});
    CHECK(r1.stage == ResolveStage::coc && r1.corrected_blocks.size() == 1 &&
          r1.corrected_blocks[0][0] == 1 && r1.corrected_blocks[0][1] == 2);
    CHECK(O1.raw() == ref.raw());
    // row fault (every column of image 1 at one position) -> RC
    ftc_fault row{FTC_FAULT_OUTPUT, FTC_FAULT_ADD, 1, -1, 0, 0, 0, 2.0f, 0.f, 1.0f};
    LayerReport r2;
    Tensor4 O2 = run_protected_layer(D, W, nullptr, p, plan, r2, {row});
    CHECK(r2.stage == ResolveStage::rc);
    CHECK(O2.raw() == ref.raw());
    // scattered multi-block fault -> recompute
    std::vector<ftc_fault> multi = {{FTC_FAULT_OUTPUT, FTC_FAULT_ADD, 0, 1, 0, 0, 0, 5.f, 0, 0},
                                    {FTC_FAULT_OUTPUT, FTC_FAULT_ADD, 0, 2, 0, 0, 0, 6.f, 0, 0},
                                    {FTC_FAULT_OUTPUT, FTC_FAULT_ADD, 1, 1, 1, 1, 0, 7.f, 0, 0},
                                    {FTC_FAULT_OUTPUT, FTC_FAULT_ADD, 2, 1, 0, 1, 0, 8.f, 0, 0}};
    LayerReport r3;
    Tensor4 O3 = run_protected_layer(D, W, nullptr, p, plan, r3, multi);
    CHECK(r3.stage == ResolveStage::recompute && r3.recomputed);
    CHECK(O3.raw() == ref.raw());
    // persistent layer handle
    ProtectedLayer layer(3, 10, W, nullptr, p);
    LayerReport r4;
    Tensor4 O4 = layer(D, plan, r4, {f});
    CHECK(r4.stage == ResolveStage::coc && O4.raw() == ref.raw());
  }
  {  // test_conv.cpp:149-158 / test_workflow.cpp:276-309: back-propagation
    ConvParams p;
    Tensor4 D(1, 1, 1, 1), W(1, 1, 1, 1), dO(1, 1, 1, 1);
    D(0, 0, 0, 0) = 3;
    W(0, 0, 0, 0) = 5;
    dO(0, 0, 0, 0) = 7;
    auto g = conv_backward(D, W, dO, p);
    CHECK(g.first(0, 0, 0, 0) == 21 && g.second(0, 0, 0, 0) == 35);
    Tensor4 D2(2, 2, 5, 5), W2(3, 2, 2, 2), O2(2, 3, 4, 4);
    for (std::size_t i = 0; i < D2.size(); ++i) D2.raw()[i] = (float)std::sin(0.1 * i);
    for (std::size_t i = 0; i < W2.size(); ++i) W2.raw()[i] = (float)std::cos(0.3 * i);
    for (std::size_t i = 0; i < O2.size(); ++i) O2.raw()[i] = (float)std::sin(0.7 * i + 1);
    auto clean = conv_backward(D2, W2, O2, p);
    BackwardReport br;
    auto pg = run_protected_backward(D2, W2, O2, p, 1e-10, br);
    CHECK(!br.dw_detected && !br.dd_detected && !br.recomputed);
    CHECK(pg.first.raw() == clean.first.raw() && pg.second.raw() == clean.second.raw());
    BackwardReport bw;
    auto fg = run_protected_backward(D2, W2, O2, p, 1e-10, bw, {{0, 1, 8, 3.0}});  // dW(1,0,0,0) += 3
    CHECK(bw.dw_detected && bw.recomputed && fg.first.raw() == clean.first.raw());
    BackwardReport bd;
    auto dg = run_protected_backward(D2, W2, O2, p, 1e-10, bd, {{1, 1, 37, -4.0}});  // dD(0,1,2,2) -= 4
    CHECK(bd.dd_detected && bd.recomputed && dg.second.raw() == clean.second.raw());
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
