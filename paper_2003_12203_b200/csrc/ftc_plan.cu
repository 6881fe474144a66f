// ftc_plan.cu -- per-layer protection plans: the reference's cost model
// and RC/ClC decision rules (workflow.hpp:30-112) as host code, and profile_layer
// (workflow.hpp:418-501) driving the device path with the six forced-fault variants.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <random>
#include <vector>

#include "ftc_common.cuh"

namespace {

enum { kCocD = 0, kCoc, kRc, kClc, kFc };

double cost(int scheme, const ftc_layer_dims& d, double a, double b) {
  // closed-form predicted work of one scheme on one layer: a weighs MACs, b memory-bound
  // reductions (workflow.hpp:52-73)
  const double N = (double)d.N, M = (double)d.M, Ch = (double)d.Ch;
  const double H2 = (double)d.H * (double)d.H, R2 = (double)d.R * (double)d.R, E2 = (double)d.E * (double)d.E;
  switch (scheme) {
    case kFc: return a * (N + M) * Ch * R2 * E2 + b * (N * Ch * H2 + 2 * N * M * E2);
    case kRc: return 2 * a * M * Ch * R2 * E2 + 2 * b * (N * Ch * H2 + N * M * E2);
    case kClc: return 2 * a * N * Ch * R2 * E2 + 2 * b * N * M * E2;
    case kCoc: return 3 * a * Ch * R2 * E2 + b * (2 * N * Ch * H2 + 3 * N * M * E2);
    case kCocD: return a * Ch * R2 * E2 + b * (2 * N * Ch * H2 + N * M * E2);
  }
  return NAN;
}

}  // namespace

extern "C" {

double ftc_cost_model(int32_t scheme, const ftc_layer_dims* dims, double alpha, double beta) {
  if (!dims || scheme < 0 || scheme > 4) return NAN;
  return cost(scheme, *dims, alpha, beta);
}

// RC pays off iff the expected time saved on row faults exceeds the time added on
// column faults (equality disables); ClC is the mirror rule (workflow.hpp:77-87)
int32_t ftc_decide_rc(double t0, double t1, double t2, double p_r, double p_c) {
  return p_r * (t0 - t1) > p_c * (t2 - t0) ? 1 : 0;
}
int32_t ftc_decide_clc(double t0, double t1, double t2, double p_r, double p_c) {
  return p_c * (t0 - t1) > p_r * (t2 - t0) ? 1 : 0;
}

// faults land in D or W in proportion to their element counts (workflow.hpp:89-96)
void ftc_estimate_error_probs(const ftc_layer_dims* d, double* p_r, double* p_c) {
  const double nd = (double)(d->N * d->Ch * d->H * d->H);
  const double nw = (double)(d->M * d->Ch * d->R * d->R);
  const double pr = nd / (nd + nw);
  if (p_r) *p_r = pr;
  if (p_c) *p_c = 1.0 - pr;
}

int ftc_make_default_plan(const ftc_layer_dims* d, double tau, double alpha, double beta, ftc_plan_info* out) {
  if (!d || !out) {
    ftc::set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  const double coc = cost(kCoc, *d, alpha, beta);
  out->tau = tau;
  out->t0 = coc + cost(kFc, *d, alpha, beta);
  out->t1 = coc + cost(kRc, *d, alpha, beta);
  out->t2 = out->t1 + cost(kFc, *d, alpha, beta);
  double pr = 0, pc = 0;
  ftc_estimate_error_probs(d, &pr, &pc);
  out->p_r = pr;
  out->rc_enabled = ftc_decide_rc(out->t0, out->t1, out->t2, pr, pc);
  out->clc_enabled = 0;  // the expensive scheme on typical layers
  return FTC_OK;
}

int ftc_profile_layer(ftc_layer* L, const float* D, double tau, int32_t reps, ftc_profile_result* out,
                      void* stream) {
  if (!L || !D || !out) {
    ftc::set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  if (reps < 3) {
    ftc::set_error(FTC_CONFIG_ERROR, "profiling needs at least 3 repetitions");
    return FTC_CONFIG_ERROR;
  }
  ftc_conv_desc desc{};
  int32_t E = 0;
  {
    const int st = ftc_layer_desc(L, &desc);
    if (st) return st;
    const int st2 = ftc_layer_extent(L, &E);
    if (st2) return st2;
  }
  const ftc_layer_dims dims{desc.N, desc.M, desc.C, desc.H, desc.R, (int64_t)E};
  auto fallback = [&]() {
    out->used_cost_model = 1;
    const double coc = cost(kCoc, dims, 1.0, 1.0), fc = cost(kFc, dims, 1.0, 1.0);
    out->rc_t0 = out->clc_t0 = coc + fc;
    out->rc_t1 = coc + cost(kRc, dims, 1.0, 1.0);
    out->rc_t2 = out->rc_t1 + fc;
    out->clc_t1 = coc + cost(kClc, dims, 1.0, 1.0);
    out->clc_t2 = out->clc_t1 + fc;
    return FTC_OK;
  };
  out->used_cost_model = 0;
  if (desc.N < 2 || desc.M < 2) return fallback();
  // forced faults on the fast path: a whole block row n = 1 (O += 3 + m) or block
  // column m = 1 (O += 3 + n), in FP32 as the T=float hooks do
  ftc_fault row{};
  row.target = FTC_FAULT_OUTPUT;
  row.mode = FTC_FAULT_ADD;
  row.n = 1;
  row.m = row.x = row.y = -1;
  row.value = 3.0f;
  row.m_coef = 1.0f;
  ftc_fault col = row;
  col.n = -1;
  col.m = 1;
  col.m_coef = 0.0f;
  col.n_coef = 1.0f;
  ftc_layer_report rep;
  float* O = nullptr;
  if (cudaMalloc(&O, (size_t)desc.N * desc.M * E * E * sizeof(float)) != cudaSuccess) {
    ftc::set_error(FTC_CUDA_ERROR, "cudaMalloc(profile output) failed");
    return FTC_CUDA_ERROR;
  }
  auto timed = [&](bool rc, bool clc, bool row_fault, double* t_out) {
    std::vector<double> t((size_t)reps);
    ftc_plan plan{};
    plan.rc_enabled = rc;
    plan.clc_enabled = clc;
    plan.tau = tau;
    for (int r = 0; r < reps; ++r) {
      const auto a = std::chrono::steady_clock::now();
      const int st = ftc_protected_conv(L, &plan, D, O, row_fault ? &row : &col, 1, &rep, stream);
      t[(size_t)r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
      if (st != FTC_OK && st != FTC_INTEGRITY_ERROR) return st;
    }
    std::nth_element(t.begin(), t.begin() + t.size() / 2, t.end());
    *t_out = t[t.size() / 2];
    return (int)FTC_OK;
  };
  int st = FTC_OK;
  if (!st) st = timed(false, false, true, &out->rc_t0);   // CoC -> FC on a row fault
  if (!st) st = timed(true, false, true, &out->rc_t1);    // CoC -> RC on a row fault
  if (!st) st = timed(true, false, false, &out->rc_t2);   // CoC -> RC -> FC on a column fault
  if (!st) st = timed(false, false, false, &out->clc_t0); // CoC -> FC on a column fault
  if (!st) st = timed(false, true, false, &out->clc_t1);  // CoC -> ClC on a column fault
  if (!st) st = timed(false, true, true, &out->clc_t2);   // CoC -> ClC -> FC on a row fault
  cudaFree(O);
  if (st) return st;
  if (out->rc_t0 <= 0 || out->rc_t1 <= 0 || out->rc_t2 <= 0 || out->clc_t0 <= 0 || out->clc_t1 <= 0 ||
      out->clc_t2 <= 0)
    return fallback();
  return FTC_OK;
}

// Tensor4<T>::random (tensor.hpp:57-66) and random_weights (model_io.cpp:176-192):
// std::mt19937_64(seed) through std::uniform_real_distribution<double>(lo, hi) -- the
// same standard-library engines the reference uses, so model weights and inputs
// generated from a seed are the reference's bit for bit.
int ftc_mt64_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
  if (n < 0 || (n > 0 && !out)) return FTC_INVALID_ARGUMENT;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
  return FTC_OK;
}

}  // extern "C"
