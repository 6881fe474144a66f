// ref_bridge.cpp -- C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/core/include/ftconv/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libftref.so.
//
// TEST INFRASTRUCTURE ONLY.  This is how the restated oracle (ftc_oracle.c) is
// pinned against the reference itself, how the golden fixtures in tests/golden/
// are generated, and what bench.py's cpu_baseline / `--impl reference` legs time
// ("kind": "reference").  Nothing here is part of the product library.
//
// Every function only marshals plain arrays into ftconv::Tensor4 and calls the
// reference's own API; no reference source is copied.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "ftconv/checksums.hpp"
#include "ftconv/conv.hpp"
#include "ftconv/fault.hpp"
#include "ftconv/schemes.hpp"
#include "ftconv/serialize.hpp"
#include "ftconv/workflow.hpp"

using namespace ftconv;

extern "C" {

struct ref_dims {
  int N, C, H, M, R;
  int stride, pad, groups;
  int bias;
};

struct ref_report {
  int detected, stage, weights_reloaded, recomputed;
  int n_blocks;
  int blocks[4096][2];
  int n_stages;
  int stages[8];
  double max_rel_dev;
};

struct ref_spec {  // layout of ftc_fault_spec
  int32_t layer_index, target, checksum, mode;
  int64_t i, j, x, y;
  uint32_t bit, pad_;
  uint64_t seed;
};
struct ref_truth {
  int32_t benign, expected_stage, output_diverges;
};
struct ref_grid {
  int64_t N, M, Ch, H, R;
};

struct ref_pre_fault {
  int target;  // 0=D 1=W 2=cd1 3=cd2 4=cw1 5=cw2
  long long index;
  int mode;  // 0 set, 1 add
  double value;
};
}

namespace {

template <typename T, typename S>
Tensor4<T> make(std::size_t a, std::size_t b, std::size_t c, std::size_t d, const S* src) {
  Tensor4<T> t(a, b, c, d);
  if (src)
    for (std::size_t i = 0; i < t.size(); ++i) t.raw()[i] = static_cast<T>(src[i]);
  return t;
}

ConvParams params(const ref_dims* d) {
  ConvParams p;
  p.stride = d->stride;
  p.groups = d->groups;
  p.pad = d->pad;
  p.bias_enabled = d->bias != 0;
  return p;
}

int code_of(const std::exception& e) {
  if (dynamic_cast<const ShapeError*>(&e)) return 1;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const IoError*>(&e)) return 3;
  if (dynamic_cast<const IntegrityError*>(&e)) return 4;
  return 9;
}

template <typename T>
void fill_report(const LayerReport& r, ref_report* out) {
  std::memset(out, 0, sizeof *out);
  out->detected = r.detected;
  out->stage = static_cast<int>(r.stage);
  out->weights_reloaded = r.weights_reloaded;
  out->recomputed = r.recomputed;
  out->n_blocks = static_cast<int>(r.corrected_blocks.size());
  for (std::size_t b = 0; b < r.corrected_blocks.size() && b < 4096; ++b) {
    out->blocks[b][0] = static_cast<int>(r.corrected_blocks[b][0]);
    out->blocks[b][1] = static_cast<int>(r.corrected_blocks[b][1]);
  }
  out->n_stages = static_cast<int>(r.stages_attempted.size());
  for (std::size_t s = 0; s < r.stages_attempted.size() && s < 8; ++s)
    out->stages[s] = static_cast<int>(r.stages_attempted[s]);
}

template <typename T>
Tensor4<T>* pick(int target, Tensor4<T>& D, Tensor4<T>& W, InputChecksums<T>& ic) {
  switch (target) {
    case 0: return &D;
    case 1: return &W;
    case 2: return &ic.cd1;
    case 3: return &*ic.cd2;
    case 4: return &ic.cw1;
    case 5: return &*ic.cw2;
  }
  return nullptr;
}

}  // namespace

extern "C" {

// Tensor4::random (tensor.hpp:57-66)
void ref_mt64_uniform(std::uint64_t seed, double lo, double hi, std::size_t n, double* out) {
  Tensor4<double> t = Tensor4<double>::random(1, 1, 1, n, seed, lo, hi);
  std::memcpy(out, t.data(), n * sizeof(double));
}

int ref_output_extent(int H, int R, int pad, int stride, int* E) {
  try {
    ConvParams p;
    p.pad = pad;
    p.stride = stride;
    *E = static_cast<int>(output_extent(H, R, p));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// conv_forward<float>(..., ConvImpl) (conv.hpp:114-131); impl 0=direct 1=mm
int ref_conv_forward_f32(const ref_dims* d, const float* D, const float* W, const float* bias,
                         float* O, int impl) {
  try {
    auto Dt = make<float>(d->N, d->C, d->H, d->H, D);
    auto Wt = make<float>(d->M, d->C / (d->groups ? d->groups : 1), d->R, d->R, W);
    auto Bt = make<float>(d->M, 1, 1, 1, bias);
    Tensor4<float> Ot = conv_forward(Dt, Wt, bias ? &Bt : nullptr, params(d),
                                     impl ? ConvImpl::mm : ConvImpl::direct);
    std::memcpy(O, Ot.data(), Ot.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_conv_forward_f64(const ref_dims* d, const double* D, const double* W, const double* bias,
                         double* O) {
  try {
    auto Dt = make<double>(d->N, d->C, d->H, d->H, D);
    auto Wt = make<double>(d->M, d->C / (d->groups ? d->groups : 1), d->R, d->R, W);
    auto Bt = make<double>(d->M, 1, 1, 1, bias);
    Tensor4<double> Ot = conv_forward(Dt, Wt, bias ? &Bt : nullptr, params(d));
    std::memcpy(O, Ot.data(), Ot.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// input_checksums<double> (checksums.hpp:91-113)
int ref_input_checksums(const ref_dims* d, const double* D, const double* W, double* cd1,
                        double* cd2, double* cw1, double* cw2) {
  try {
    auto Dt = make<double>(d->N, d->C, d->H, d->H, D);
    auto Wt = make<double>(d->M, d->C / d->groups, d->R, d->R, W);
    InputChecksums<double> ic = input_checksums(Dt, Wt, d->groups);
    std::memcpy(cd1, ic.cd1.data(), ic.cd1.size() * sizeof(double));
    std::memcpy(cd2, ic.cd2->data(), ic.cd2->size() * sizeof(double));
    std::memcpy(cw1, ic.cw1.data(), ic.cw1.size() * sizeof(double));
    std::memcpy(cw2, ic.cw2->data(), ic.cw2->size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// output_checksums<double> (checksums.hpp:134-161); co[k] receives Co(k+1)
int ref_output_checksums(const ref_dims* d, unsigned which, const double* D, const double* W,
                         double** co) {
  try {
    auto Dt = make<double>(d->N, d->C, d->H, d->H, D);
    auto Wt = make<double>(d->M, d->C / d->groups, d->R, d->R, W);
    InputChecksums<double> ic = input_checksums(Dt, Wt, d->groups);
    OutputChecksums<double> cs = output_checksums(which, Dt, Wt, ic, params(d));
    auto dump = [](const std::vector<Grid<double>>& v, double* out) {
      for (const auto& g : v) {
        std::memcpy(out, g.v.data(), g.v.size() * sizeof(double));
        out += g.v.size();
      }
    };
    if (cs.co1) dump(*cs.co1, co[0]);
    if (cs.co2) dump(*cs.co2, co[1]);
    if (cs.co3) dump(*cs.co3, co[2]);
    if (cs.co4) dump(*cs.co4, co[3]);
    if (cs.co5) std::memcpy(co[4], cs.co5->v.data(), cs.co5->v.size() * sizeof(double));
    if (cs.co6) std::memcpy(co[5], cs.co6->v.data(), cs.co6->v.size() * sizeof(double));
    if (cs.co7) std::memcpy(co[6], cs.co7->v.data(), cs.co7->v.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// output_summations<double> + bias_adjust (checksums.hpp:165-245)
int ref_output_summations(int N, int M, int E, const double* O, unsigned which, const double* bias,
                          double** so) {
  try {
    auto Ot = make<double>(N, M, E, E, O);
    OutputSummations<double> s = output_summations(Ot, which);
    if (bias) bias_adjust(s, make<double>(M, 1, 1, 1, bias), N, M);
    auto dump = [](const std::vector<Grid<double>>& v, double* out) {
      for (const auto& g : v) {
        std::memcpy(out, g.v.data(), g.v.size() * sizeof(double));
        out += g.v.size();
      }
    };
    if (s.so1) dump(*s.so1, so[0]);
    if (s.so2) dump(*s.so2, so[1]);
    if (s.so3) dump(*s.so3, so[2]);
    if (s.so4) dump(*s.so4, so[3]);
    if (s.so5) std::memcpy(so[4], s.so5->v.data(), s.so5->v.size() * sizeof(double));
    if (s.so6) std::memcpy(so[5], s.so6->v.data(), s.so6->v.size() * sizeof(double));
    if (s.so7) std::memcpy(so[6], s.so7->v.data(), s.so7->v.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// run_protected_layer<double> (workflow.hpp:141-339) under the SURVEY 8(c)
// contract: the post_conv hook substitutes O with `O_conv` (the GPU's FP32
// output widened, flips applied); pre_conv faults are substitutions too.
int ref_protected_layer_f64(const ref_dims* d, const float* D, const float* W, const float* bias,
                            int rc_enabled, int clc_enabled, double tau, const float* O_conv,
                            const ref_pre_fault* pre, int n_pre, ref_report* rep, double* O_out) {
  try {
    auto Dt = make<double>(d->N, d->C, d->H, d->H, D);
    auto Wt = make<double>(d->M, d->C / d->groups, d->R, d->R, W);
    auto Bt = make<double>(d->M, 1, 1, 1, bias);
    LayerPlan plan;
    plan.rc_enabled = rc_enabled != 0;
    plan.clc_enabled = clc_enabled != 0;
    plan.tau = tau;
    FaultHooks<double> hooks;
    if (O_conv)
      hooks.post_conv = [O_conv](Tensor4<double>& O) {
        for (std::size_t i = 0; i < O.size(); ++i) O.raw()[i] = static_cast<double>(O_conv[i]);
      };
    if (n_pre > 0)
      hooks.pre_conv = [pre, n_pre](Tensor4<double>& D_, Tensor4<double>& W_,
                                    InputChecksums<double>& ic) {
        for (int q = 0; q < n_pre; ++q) {
          Tensor4<double>* t = pick(pre[q].target, D_, W_, ic);
          if (!t) continue;
          double& v = t->raw()[static_cast<std::size_t>(pre[q].index)];
          v = pre[q].mode == 0 ? pre[q].value : v + pre[q].value;
        }
      };
    LayerReport r;
    int code = 0;
    Tensor4<double> O;
    try {
      O = run_protected_layer(Dt, Wt, bias ? &Bt : nullptr, params(d), plan, r, ConvImpl::direct,
                              hooks);
    } catch (const IntegrityError&) {
      code = 4;
    }
    fill_report<double>(r, rep);
    if (O_out && O.size()) std::memcpy(O_out, O.data(), O.size() * sizeof(double));
    return code;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// run_protected_layer<float> with the shipped default plan (make_default_plan,
// workflow.hpp:99-112) and ConvImpl::direct: the reference's own CPU path, as
// timed by bench.py's cpu_baseline and --impl reference legs.
int ref_protected_layer_f32(const ref_dims* d, const float* D, const float* W, const float* bias,
                            double tau, float* O_out, ref_report* rep) {
  try {
    auto Dt = make<float>(d->N, d->C, d->H, d->H, D);
    auto Wt = make<float>(d->M, d->C / d->groups, d->R, d->R, W);
    auto Bt = make<float>(d->M, 1, 1, 1, bias);
    const ConvParams p = params(d);
    LayerPlan plan = make_default_plan(make_dims(Dt, Wt, p), tau);
    LayerReport r;
    Tensor4<float> O = run_protected_layer(Dt, Wt, bias ? &Bt : nullptr, p, plan, r);
    if (rep) fill_report<float>(r, rep);
    if (O_out) std::memcpy(O_out, O.data(), O.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// make_default_plan (workflow.hpp:99-112)
void ref_make_default_plan(int N, int M, int Ch, int H, int R, int E, double tau, int* rc, int* clc,
                           double* t0, double* t1, double* t2, double* p_r) {
  LayerDims dd;
  dd.N = N;
  dd.M = M;
  dd.Ch = Ch;
  dd.H = H;
  dd.R = R;
  dd.E = E;
  LayerPlan plan = make_default_plan(dd, tau);
  *rc = plan.rc_enabled;
  *clc = plan.clc_enabled;
  *t0 = plan.t0;
  *t1 = plan.t1;
  *t2 = plan.t2;
  *p_r = plan.p_r;
}

// flip_bit (fault.hpp:82-87)
float ref_flip_bit_f32(float v, unsigned bit) {
  detail::flip_bit(v, bit);
  return v;
}

// locate_index (schemes.hpp:57-62); returns -1 for nullopt
long long ref_locate_index(double r, int n) {
  auto i = detail::locate_index(r, static_cast<std::size_t>(n));
  return i ? static_cast<long long>(*i) : -1;
}

int ref_values_differ(double c, double s, double tau) { return values_differ(c, s, tau) ? 1 : 0; }

}  // extern "C"

// ---- fault campaigns: the reference's own corpus generator and hooks (test oracle)
namespace {
FaultSpec to_spec(const ref_spec& r) {
  FaultSpec f;
  f.layer_index = static_cast<std::size_t>(r.layer_index);
  f.target = static_cast<FaultTarget>(r.target);
  f.checksum = static_cast<ChecksumName>(r.checksum);
  f.i = static_cast<std::size_t>(r.i);
  f.j = static_cast<std::size_t>(r.j);
  f.x = r.x;
  f.y = r.y;
  f.mode = r.mode == 1 ? FaultMode::bitflip : FaultMode::scale;
  f.bit = r.bit;
  f.seed = r.seed;
  return f;
}
}  // namespace

extern "C" {

// campaign (fault.hpp:195-271) + ground_truth
int ref_campaign(const ref_grid* grids, int n_layers, long long n_runs, const double* w6, std::uint64_t seed,
                 ref_spec* specs, ref_truth* truths) {
  try {
    std::vector<LayerGrid> layers;
    for (int k = 0; k < n_layers; ++k)
      layers.push_back(LayerGrid{(std::size_t)grids[k].N, (std::size_t)grids[k].M, (std::size_t)grids[k].Ch,
                                 (std::size_t)grids[k].H, (std::size_t)grids[k].R});
    TargetWeights w;
    w.output_block = w6[0];
    w.output_row = w6[1];
    w.output_column = w6[2];
    w.fmap = w6[3];
    w.kernel = w6[4];
    w.checksum = w6[5];
    const auto corpus = campaign(layers, (std::size_t)n_runs, w, seed);
    for (std::size_t r = 0; r < corpus.size(); ++r) {
      const FaultSpec& f = corpus[r].fault;
      ref_spec o{};
      o.layer_index = (int32_t)f.layer_index;
      o.target = (int32_t)f.target;
      o.checksum = (int32_t)f.checksum;
      o.mode = f.mode == FaultMode::bitflip ? 1 : 0;
      o.i = (int64_t)f.i;
      o.j = (int64_t)f.j;
      o.x = f.x;
      o.y = f.y;
      o.bit = f.bit;
      o.seed = f.seed;
      specs[r] = o;
      truths[r].benign = corpus[r].truth.benign;
      truths[r].expected_stage = (int32_t)corpus[r].truth.expected_stage;
      truths[r].output_diverges = corpus[r].truth.output_diverges;
    }
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// make_hooks<float>(f) applied to host tensors D (N,C,H,H), W (M,C,R,R), O (N,M,E,E) and
// make_hooks<double>(f) to the FP64 checksums cd1/cd2 (1,C,H,H), cw1/cw2 (1,C,R,R); any
// pointer may be null (that phase is skipped)
int ref_apply_spec(const ref_spec* spec, int N, int C, int H, int M, int R, int E, float* D, float* W, float* O,
                   double* cd1, double* cd2, double* cw1, double* cw2) {
  try {
    const FaultSpec f = to_spec(*spec);
    FaultHooks<float> hf = make_hooks<float>(f);
    if (O && hf.post_conv) {
      auto Ot = make<float>(N, M, E, E, O);
      hf.post_conv(Ot);
      std::memcpy(O, Ot.data(), Ot.size() * sizeof(float));
    }
    if ((D || W) && hf.pre_conv && (f.target == FaultTarget::fmap || f.target == FaultTarget::kernel)) {
      auto Dt = make<float>(D ? N : 1, C, H, H, D);
      auto Wt = make<float>(W ? M : 1, C, R, R, W);
      InputChecksums<float> ic;
      hf.pre_conv(Dt, Wt, ic);
      if (D) std::memcpy(D, Dt.data(), Dt.size() * sizeof(float));
      if (W) std::memcpy(W, Wt.data(), Wt.size() * sizeof(float));
    }
    if (f.target == FaultTarget::checksum) {
      FaultHooks<double> hd = make_hooks<double>(f);
      Tensor4<double> Dd(1, 1, 1, 1), Wd(1, 1, 1, 1);
      InputChecksums<double> ic;
      ic.cd1 = make<double>(1, C, H, H, cd1);
      ic.cd2 = make<double>(1, C, H, H, cd2);
      ic.cw1 = make<double>(1, C, R, R, cw1);
      ic.cw2 = make<double>(1, C, R, R, cw2);
      hd.pre_conv(Dd, Wd, ic);
      if (cd1) std::memcpy(cd1, ic.cd1.data(), ic.cd1.size() * sizeof(double));
      if (cd2) std::memcpy(cd2, ic.cd2->data(), ic.cd2->size() * sizeof(double));
      if (cw1) std::memcpy(cw1, ic.cw1.data(), ic.cw1.size() * sizeof(double));
      if (cw2) std::memcpy(cw2, ic.cw2->data(), ic.cw2->size() * sizeof(double));
    }
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

}  // extern "C"

// ---- file formats (serialize.cpp): plan and corpus text, for byte-level pins
extern "C" {

// plan_to_json over n named plans {rc, clc, tau, t0, t1, t2, p_r}; returns the length
// written into out (cap bytes) or -1
long long ref_plan_to_json(int n, const char* const* names, const double* vals7, char* out, long long cap) {
  try {
    std::map<std::string, LayerPlan> plans;
    for (int k = 0; k < n; ++k) {
      LayerPlan p;
      p.rc_enabled = vals7[7 * k + 0] != 0;
      p.clc_enabled = vals7[7 * k + 1] != 0;
      p.tau = vals7[7 * k + 2];
      p.t0 = vals7[7 * k + 3];
      p.t1 = vals7[7 * k + 4];
      p.t2 = vals7[7 * k + 5];
      p.p_r = vals7[7 * k + 6];
      plans[names[k]] = p;
    }
    const std::string t = plan_to_json(plans);
    if ((long long)t.size() + 1 > cap) return -1;
    std::memcpy(out, t.c_str(), t.size() + 1);
    return (long long)t.size();
  } catch (const std::exception&) {
    return -1;
  }
}

// corpus_to_jsonl of n (spec, truth) pairs
long long ref_corpus_to_jsonl(int n, const ref_spec* specs, const ref_truth* truths, char* out, long long cap) {
  try {
    std::vector<CorpusEntry> es;
    for (int k = 0; k < n; ++k) {
      CorpusEntry e;
      e.fault = to_spec(specs[k]);
      e.truth.benign = truths[k].benign != 0;
      e.truth.expected_stage = static_cast<ResolveStage>(truths[k].expected_stage);
      e.truth.output_diverges = truths[k].output_diverges != 0;
      es.push_back(e);
    }
    const std::string t = corpus_to_jsonl(es);
    if ((long long)t.size() + 1 > cap) return -1;
    std::memcpy(out, t.c_str(), t.size() + 1);
    return (long long)t.size();
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"


// ---- model configs, FTCN weight files and run reports (model_io.cpp, serialize.cpp)
#include "ftconv/model.hpp"

extern "C" {

static long long put_text(const std::string& t, char* out, long long cap) {
  if ((long long)t.size() + 1 > cap) return -1;
  std::memcpy(out, t.c_str(), t.size() + 1);
  return (long long)t.size();
}

// parse_model_config status: 0 ok, 2 ConfigError, 1 ShapeError, 3 IoError, -1 other
int ref_parse_model_config(const char* text, int* n_layers) {
  try {
    const ModelConfig cfg = parse_model_config(text);
    if (n_layers) *n_layers = (int)cfg.layers.size();
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// random_weights(cfg, seed) written by save_weights to `path`
int ref_make_weights(const char* config_text, std::uint64_t seed, const char* path) {
  try {
    const ModelConfig cfg = parse_model_config(config_text);
    save_weights(path, cfg, random_weights(cfg, seed));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// load_weights status for the file at `path` against the config
int ref_load_weights(const char* config_text, const char* path) {
  try {
    const ModelConfig cfg = parse_model_config(config_text);
    (void)load_weights(path, cfg);
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// report_to_json over n layer reports.  Per report k: ints[8k..8k+7] = {detected, stage,
// weights_reloaded, recomputed, n_blocks, n_stages, n_timings, unused}; blocks, stage
// codes and timing values are consumed in order from their arrays; timing keys from
// tkeys.  campaign != 0 wraps them in a CampaignReport with the counters in camp[7]
// (runs, detected, above_threshold, recovered, mismatches, fatals) -- by_stage is
// tallied from the entries as run_campaign does.
long long ref_report_to_json(int n, const char* const* names, const int* ints, const long long* blocks,
                             const int* stages, const char* const* tkeys, const double* tvals, int timings,
                             int campaign, const long long* camp, char* out, long long cap) {
  try {
    std::vector<LayerReport> reps;
    long long bo = 0, so = 0, to = 0;
    for (int k = 0; k < n; ++k) {
      const int* v = ints + 8 * k;
      LayerReport r;
      r.layer = names[k];
      r.detected = v[0] != 0;
      r.stage = static_cast<ResolveStage>(v[1]);
      r.weights_reloaded = v[2] != 0;
      r.recomputed = v[3] != 0;
      for (int b = 0; b < v[4]; ++b, bo += 2) r.corrected_blocks.push_back({(std::size_t)blocks[bo], (std::size_t)blocks[bo + 1]});
      for (int s = 0; s < v[5]; ++s) r.stages_attempted.push_back(static_cast<ResolveStage>(stages[so++]));
      for (int t = 0; t < v[6]; ++t, ++to) r.timings[tkeys[to]] = tvals[to];
      reps.push_back(r);
    }
    if (!campaign) return put_text(report_to_json(reps, timings != 0), out, cap);
    CampaignReport c;
    c.runs = (std::size_t)camp[0];
    c.detected = (std::size_t)camp[1];
    c.above_threshold = (std::size_t)camp[2];
    c.recovered = (std::size_t)camp[3];
    c.ground_truth_mismatches = (std::size_t)camp[4];
    c.integrity_fatals = (std::size_t)camp[5];
    for (const LayerReport& r : reps) ++c.by_stage[to_string(r.stage)];
    c.entries = reps;
    return put_text(report_to_json(c, timings != 0), out, cap);
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"

// ---- back-propagation (conv.hpp:150-185, workflow.hpp:340-417) at T=double
extern "C" {

struct ref_grad_hook {  // post_hook substitution: target 0 dW / 1 dD, mode 0 set / 1 add
  int target;
  long long index;
  int mode;
  double value;
};

int ref_conv_backward(const ref_dims* d, const double* D, const double* W, const double* dO, double* dW,
                      double* dD) {
  try {
    const ConvParams p = params(d);
    Tensor4<double> tD(d->N, d->C, d->H, d->H), tW(d->M, d->C / d->groups, d->R, d->R);
    std::memcpy(tD.raw().data(), D, tD.size() * sizeof(double));
    std::memcpy(tW.raw().data(), W, tW.size() * sizeof(double));
    const std::size_t E = output_extent(d->H, d->R, p);
    Tensor4<double> tO(d->N, d->M, E, E);
    std::memcpy(tO.raw().data(), dO, tO.size() * sizeof(double));
    auto [gw, gd] = conv_backward(tD, tW, tO, p);
    std::memcpy(dW, gw.raw().data(), gw.size() * sizeof(double));
    std::memcpy(dD, gd.raw().data(), gd.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

int ref_protected_backward(const ref_dims* d, const double* D, const double* W, const double* dO, double tau,
                           const ref_grad_hook* hook, int n_hook, double* dW, double* dD, int* flags3) {
  BackwardReport rep;
  try {
    const ConvParams p = params(d);
    Tensor4<double> tD(d->N, d->C, d->H, d->H), tW(d->M, d->C / d->groups, d->R, d->R);
    std::memcpy(tD.raw().data(), D, tD.size() * sizeof(double));
    std::memcpy(tW.raw().data(), W, tW.size() * sizeof(double));
    const std::size_t E = output_extent(d->H, d->R, p);
    Tensor4<double> tO(d->N, d->M, E, E);
    std::memcpy(tO.raw().data(), dO, tO.size() * sizeof(double));
    std::function<void(Tensor4<double>&, Tensor4<double>&)> fn;
    if (n_hook > 0)
      fn = [&](Tensor4<double>& gw, Tensor4<double>& gd) {
        for (int h = 0; h < n_hook; ++h) {
          double& v = (hook[h].target == 0 ? gw : gd).raw()[hook[h].index];
          v = hook[h].mode == 0 ? hook[h].value : v + hook[h].value;
        }
      };
    auto [gw, gd] = run_protected_backward(tD, tW, tO, p, tau, rep, fn);
    std::memcpy(dW, gw.raw().data(), gw.size() * sizeof(double));
    std::memcpy(dD, gd.raw().data(), gd.size() * sizeof(double));
    flags3[0] = rep.dw_detected;
    flags3[1] = rep.dd_detected;
    flags3[2] = rep.recomputed;
    return 0;
  } catch (const std::exception& e) {
    flags3[0] = rep.dw_detected;
    flags3[1] = rep.dd_detected;
    flags3[2] = rep.recomputed;
    return code_of(e);
  }
}

}  // extern "C"
