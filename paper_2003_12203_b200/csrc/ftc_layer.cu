// ftc_layer.cu -- layer handle, protected-layer orchestration and the C ABI
// (include/ftc_abi.h).  Reference paths are relative to proj/core/include/ftconv/.
//
// The clean path is fully asynchronous: the input checksums (K2) and the CoC-D
// checksum Co5 (K4) run on a side stream concurrently with the conv, whose
// epilogue fuses the So2/So4 row sums; CoC-D then compares Co5 with
// So5 = sum_n So2.  Only when CoC-D fires does the host walk the reference's
// escalation chain (workflow.hpp:230-338), every step of which is a device kernel
// (ftc_checksums.cu, ftc_schemes.cu); the host only sequences launches and reads
// back small verdict records.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <random>
#include <vector>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "ftc_common.cuh"

namespace ftc {

thread_local std::string g_err;
static int g_engine = 0;  // 0 = tcgen05 (when supported for the shape), 1 = SIMT

static std::atomic<uint64_t> g_launches{0};

void set_error(int code, const std::string& msg) {
  (void)code;
  g_err = msg;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = getenv("FTC_NO_PDL") == nullptr;
  return on;
}

}  // namespace ftc

using namespace ftc;

#define RET_ERR(code, msg)         \
  do {                             \
    ::ftc::set_error((code), (msg)); \
    return (code);                 \
  } while (0)

#define CK(x)                 \
  do {                        \
    int _st = (x);            \
    if (_st != FTC_OK) return _st; \
  } while (0)

struct ftc_layer {
  ftc_conv_desc d{};
  int E = 0, E2 = 0, Ckw = 0;
  long long nD = 0, nW = 0, nO = 0, nCd = 0, nCw = 0;

  float* W = nullptr;       // golden kernels
  float* W_work = nullptr;  // working copy when a kernel fault is injected
  float* bias = nullptr;
  double* agg = nullptr;  // BiasAdjuster aggregates
  double *cw1g = nullptr, *cw2g = nullptr;  // golden kernel checksums (model.hpp:104)
  double *cw1w = nullptr, *cw2w = nullptr;  // working kernel checksums
  double *cd1 = nullptr, *cd2 = nullptr;
  double* co5f = nullptr;
  double* so5acc = nullptr;  // fused clean path: So5 accumulator (zero between calls)
  Co5Tap* co5tab = nullptr;  // fused clean path: Co5 taps (offsets + golden Cw1)
  double* cd1ws = nullptr;   // fused clean path: Cd1 workspace ([Cd1][slabs][tickets], zeroed)
  bool nhwc_ready = false;   // the next conv's NHWC input copy is already staged (one-shot)
  const float* D_staged = nullptr;  // the D it was staged from (set by the caller's next launch)
  double *rowsum = nullptr, *rowsum_m = nullptr;
  DetectStats* stats = nullptr;
  DetectStats* stats_h = nullptr;  // pinned
  DetectStats* fstats = nullptr;   // clean-path counters (kept zero between calls)
  unsigned int* fticket = nullptr;
  DetectStats* fstats_h = nullptr;  // mapped pinned record written by the detector
  DetectStats* fstats_hd = nullptr; // its device alias
  ftc_fault* faults_dev = nullptr;
  ftc_fault* faults_h = nullptr;  // pinned staging
  int faults_cap = 0;
  double* scale_tab = nullptr;    // SCALE fault magnitudes (device)
  size_t scale_cap = 0;
  float* D_work = nullptr;
  float *D_host_buf = nullptr, *O_host_buf = nullptr;  // device buffers for the _host API

  // error path (allocated on first use)
  bool ep_alloc = false;
  double* cs[7] = {};
  double* s[7] = {};
  double* tmp_c = nullptr;  // probe grids
  double* tmp_s = nullptr;
  double* tmp_cw1 = nullptr;
  double* tmp_cw2 = nullptr;
  double* ov = nullptr;
  uint8_t* present = nullptr;
  uint8_t* touched5 = nullptr;
  double* fresh567 = nullptr;  // verifier: fresh So5/So6/So7 of the touched positions
  int* tlist = nullptr;
  int* tcount = nullptr;
  uint8_t* touched1 = nullptr;
  Patches patches{};
  SchemeResult* res = nullptr;
  SchemeResult* res_h = nullptr;  // pinned
  uint8_t *colmask = nullptr, *rowmask = nullptr;
  int32_t *colany = nullptr, *rowany = nullptr;
  uint32_t* plane_mask = nullptr;
  int32_t* iscratch = nullptr;    // device ints
  int32_t* iscratch_h = nullptr;  // pinned
  std::vector<uint32_t> plane_mask_h;

  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_ck = nullptr, ev_done = nullptr;
  // instrumentation (ftc_layer_set_timing)
  bool timing = false;
  cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;
  bool conv_timed_pending = false;
  double conv_ms = 0.0;
  int32_t conv_launches = 0;
  TcPlan* tc = nullptr;

  // in-flight protected call
  bool inflight = false;
  ftc_plan plan{};
  const float* D = nullptr;  // caller's input
  const float* Dconv = nullptr;  // input the conv reads (working copy under fmap faults)
  const float* Wcur = nullptr;
  const double *cw1 = nullptr, *cw2 = nullptr;
  float* O = nullptr;
  int nfaults = 0, n_out_faults = 0;
  bool ck_exact = false;  // cd1/cd2 hold exact-order input checksums of D
  const double* cd_ext1 = nullptr;  // producer-supplied exact checksums (read in place)
  const double* cd_ext2 = nullptr;
  bool has_cd_faults = false;
  int rs_parts = 1;  // row-sum partial slabs written by the last fused-sum conv
  cudaStream_t stream = nullptr;
  std::chrono::steady_clock::time_point t0;
};

namespace {

template <typename T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) RET_ERR(FTC_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return FTC_OK;
}

bool use_tc(const ftc_layer* L) { return g_engine == 0 && L->tc != nullptr; }

int run_conv(ftc_layer* L, const float* D, const float* W, float* O, bool faults, bool sums,
             const uint32_t* plane_mask, int img_lo, int img_hi, cudaStream_t s,
             const FusedDetect* fd = nullptr, bool dt_ready = false) {
  ConvArgs a{};
  a.fd = fd;
  a.dt_ready = dt_ready;
  a.D = D;
  a.W = W;
  a.bias = L->d.bias_enabled ? L->bias : nullptr;
  a.O = O;
  a.N = L->d.N;
  a.C = L->d.C;
  a.H = L->d.H;
  a.M = L->d.M;
  a.R = L->d.R;
  a.U = L->d.stride;
  a.pad = L->d.pad;
  a.groups = L->d.groups;
  a.E = L->E;
  a.Ckw = L->Ckw;
  a.faults = faults ? L->faults_dev : nullptr;
  a.nfaults = faults ? L->nfaults : 0;
  a.scale_tab = L->scale_tab;
  a.rowsum = sums ? L->rowsum : nullptr;
  a.rowsum_m = sums ? L->rowsum_m : nullptr;
  a.plane_mask = plane_mask;
  a.img_lo = img_lo;
  a.img_hi = img_hi;
  // The tensor-core engine packs the golden W once; a corrupted working W (kernel
  // fault injection) runs through the SIMT engine.
  if (use_tc(L) && W == L->W) {
    if (sums) L->rs_parts = tc_rowsum_parts(L->tc);
    // a producer staged the NHWC copy of exactly this D (whole batch only)
    if (L->nhwc_ready && D == L->D_staged && img_lo == 0 && img_hi == L->d.N) a.dt_ready = true;
    L->nhwc_ready = false;
    return conv_tc_launch(L->tc, a, s);
  }
  L->nhwc_ready = false;
  if (sums) L->rs_parts = 1;
  return conv_simt_launch(a, s);
}

// conv with optional event bracketing (bench.py's per-kernel roofline timing)
int timed_conv(ftc_layer* L, const float* D, const float* W, float* O, bool faults, bool sums,
               cudaStream_t s, const FusedDetect* fd = nullptr, bool dt_ready = false) {
  if (L->timing) {
    if (L->conv_timed_pending) {  // harvest the previous bracket first
      FTC_CUDA_CHECK(cudaEventSynchronize(L->ev_c1));
      float ms = 0.f;
      FTC_CUDA_CHECK(cudaEventElapsedTime(&ms, L->ev_c0, L->ev_c1));
      L->conv_ms += ms;
      L->conv_launches += 1;
      L->conv_timed_pending = false;
    }
    FTC_CUDA_CHECK(cudaEventRecord(L->ev_c0, s));
  }
  int st = run_conv(L, D, W, O, faults, sums, nullptr, 0, L->d.N, s, fd, dt_ready);
  if (L->timing && st == FTC_OK) {
    FTC_CUDA_CHECK(cudaEventRecord(L->ev_c1, s));
    L->conv_timed_pending = true;
  }
  return st;
}

int harvest_timing(ftc_layer* L) {
  if (L->conv_timed_pending) {
    FTC_CUDA_CHECK(cudaEventSynchronize(L->ev_c1));
    float ms = 0.f;
    FTC_CUDA_CHECK(cudaEventElapsedTime(&ms, L->ev_c0, L->ev_c1));
    L->conv_ms += ms;
    L->conv_launches += 1;
    L->conv_timed_pending = false;
  }
  return FTC_OK;
}

int alloc_error_path(ftc_layer* L) {
  if (L->ep_alloc) return FTC_OK;
  const int N = L->d.N, M = L->d.M, E2 = L->E2;
  const size_t fam[7] = {(size_t)M * E2, (size_t)N * E2, (size_t)M * E2, (size_t)N * E2,
                         (size_t)E2,     (size_t)E2,     (size_t)E2};
  for (int k = 0; k < 7; ++k) {
    CK(dalloc(&L->cs[k], fam[k]));
    CK(dalloc(&L->s[k], fam[k]));
  }
  CK(dalloc(&L->tmp_c, (size_t)M * E2));
  CK(dalloc(&L->tmp_s, (size_t)M * E2));
  CK(dalloc(&L->tmp_cw1, L->nCw));
  CK(dalloc(&L->tmp_cw2, L->nCw));
  CK(dalloc(&L->ov, L->nO));
  CK(dalloc(&L->present, L->nO));
  CK(dalloc(&L->touched5, E2));
  CK(dalloc(&L->touched1, (size_t)M * E2));
  CK(dalloc(&L->fresh567, 3 * (size_t)E2));
  CK(dalloc(&L->tlist, E2));
  CK(dalloc(&L->tcount, 1));
  FTC_CUDA_CHECK(cudaMemset(L->present, 0, L->nO));
  FTC_CUDA_CHECK(cudaMemset(L->touched5, 0, E2));
  FTC_CUDA_CHECK(cudaMemset(L->touched1, 0, (size_t)M * E2));
  const int cap = (int)((size_t)std::max(M, N) * E2 + E2);
  L->patches.cap = cap;
  CK(dalloc(&L->patches.n, cap));
  CK(dalloc(&L->patches.m, cap));
  CK(dalloc(&L->patches.f, cap));
  CK(dalloc(&L->patches.d, cap));
  CK(dalloc(&L->res, 1));
  FTC_CUDA_CHECK(cudaMallocHost((void**)&L->res_h, sizeof(SchemeResult)));
  CK(dalloc(&L->colmask, (size_t)M * E2));
  CK(dalloc(&L->rowmask, (size_t)N * E2));
  CK(dalloc(&L->colany, M));
  CK(dalloc(&L->rowany, N));
  const size_t words = ((size_t)N * M + 31) / 32;
  CK(dalloc(&L->plane_mask, words));
  L->plane_mask_h.resize(words);
  CK(dalloc(&L->iscratch, 16));
  FTC_CUDA_CHECK(cudaMallocHost((void**)&L->iscratch_h, 16 * sizeof(int32_t)));
  L->ep_alloc = true;
  return FTC_OK;
}

void free_layer(ftc_layer* L) {
  auto F = [](void* p) {
    if (p) cudaFree(p);
  };
  F(L->W); F(L->W_work); F(L->bias); F(L->agg); F(L->cw1g); F(L->cw2g); F(L->cw1w); F(L->cw2w);
  F(L->cd1); F(L->cd2); F(L->co5f); F(L->so5acc); F(L->co5tab); F(L->cd1ws); F(L->rowsum); F(L->rowsum_m); F(L->stats); F(L->faults_dev);
  F(L->D_work); F(L->D_host_buf); F(L->O_host_buf);
  for (int k = 0; k < 7; ++k) {
    F(L->cs[k]);
    F(L->s[k]);
  }
  F(L->tmp_c); F(L->tmp_s); F(L->tmp_cw1); F(L->tmp_cw2); F(L->ov); F(L->present); F(L->touched5);
  F(L->touched1); F(L->fresh567); F(L->tlist); F(L->tcount); F(L->patches.n); F(L->patches.m); F(L->patches.f); F(L->patches.d); F(L->res);
  F(L->colmask); F(L->rowmask); F(L->colany); F(L->rowany); F(L->plane_mask); F(L->iscratch);
  if (L->stats_h) cudaFreeHost(L->stats_h);
  if (L->fstats_h) cudaFreeHost(L->fstats_h);
  F(L->fstats);
  F(L->fticket);
  F(L->scale_tab);
  if (L->faults_h) cudaFreeHost(L->faults_h);
  if (L->res_h) cudaFreeHost(L->res_h);
  if (L->iscratch_h) cudaFreeHost(L->iscratch_h);
  if (L->side) cudaStreamDestroy(L->side);
  if (L->ev_start) cudaEventDestroy(L->ev_start);
  if (L->ev_ck) cudaEventDestroy(L->ev_ck);
  if (L->ev_done) cudaEventDestroy(L->ev_done);
  if (L->ev_c0) cudaEventDestroy(L->ev_c0);
  if (L->ev_c1) cudaEventDestroy(L->ev_c1);
  if (L->tc) tc_plan_destroy(L->tc);
  delete L;
}

int validate(const ftc_conv_desc* d, int* E) {
  if (!d) RET_ERR(FTC_INVALID_ARGUMENT, "null descriptor");
  if (d->N <= 0 || d->C <= 0 || d->H <= 0 || d->M <= 0 || d->R <= 0 || d->pad < 0)
    RET_ERR(FTC_SHAPE_ERROR, "tensor dimensions must be positive");
  // check_conv_shapes (conv.hpp:16-26)
  if (d->groups <= 0) RET_ERR(FTC_CONFIG_ERROR, "groups must be positive");
  if (d->C % d->groups != 0 || d->M % d->groups != 0)
    RET_ERR(FTC_CONFIG_ERROR, "groups must divide Ch and M");
  // output_extent (tensor.hpp:100-107)
  if (d->stride <= 0) RET_ERR(FTC_CONFIG_ERROR, "stride must be positive");
  const long long Hp = (long long)d->H + 2LL * d->pad;
  if (Hp < d->R) RET_ERR(FTC_CONFIG_ERROR, "kernel larger than padded input");
  if ((Hp - d->R) % d->stride != 0)
    RET_ERR(FTC_CONFIG_ERROR, "output extent (H+2p-R+U)/U is not an integer");
  *E = (int)((Hp - d->R) / d->stride + 1);
  return FTC_OK;
}

// ------------------------------------------------------------------ error path pieces
bool getenv_flag(const char* name);  // defined below

struct EP {
  ftc_layer* L;
  cudaStream_t s;
  unsigned cs_have = 0, s_have = 0;
  bool ov_dirty = false;
  // families the verifier may trust (further restricted to what was computed): the
  // workflow's {O1,O3,O5,O6,O7}; {O5} for one scheme in isolation (acceptance.cpp:247-251)
  unsigned trust_mask = FTC_CK_O1 | FTC_CK_O3 | FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7;
};

VirtualO vobj(EP& e) {
  VirtualO v;
  v.O = e.L->O;
  v.ov = e.ov_dirty ? e.L->ov : nullptr;
  v.present = e.ov_dirty ? e.L->present : nullptr;
  return v;
}

// workflow.hpp:168-180 (ensure_cs) at T=double on device
int ensure_cs(EP& e, unsigned want) {
  ftc_layer* L = e.L;
  const unsigned need = want & ~e.cs_have;
  if (!need) return FTC_OK;
  const ftc_conv_desc& d = L->d;
  const int U = d.stride, p = d.pad, E = L->E;
  // the weighted family of a pair (Co3 beside Co1 for RC, Co4 beside Co2 for ClC) goes to
  // the layer's side stream: two independent exact-order FP64 convs of equal length
  static const bool ep_serial = getenv_flag("FTC_EP_SERIAL");
  const bool pair = ((need & FTC_CK_O1) && (need & FTC_CK_O3)) || ((need & FTC_CK_O2) && (need & FTC_CK_O4));
  const bool fork = pair && !ep_serial && L->side && L->ev_start && L->ev_ck;
  cudaStream_t s2 = e.s;
  if (fork) {
    FTC_CUDA_CHECK(cudaEventRecord(L->ev_start, e.s));
    FTC_CUDA_CHECK(cudaStreamWaitEvent(L->side, L->ev_start, 0));
    s2 = L->side;
  }
  if (need & FTC_CK_O1)
    CK(launch_conv_f64_exact(L->cd1, true, L->Wcur, false, L->cs[0], 1, d.C, d.H, d.M, L->Ckw, d.R,
                             U, p, d.groups, E, e.s));
  if (need & FTC_CK_O2)
    CK(launch_conv_f64_exact(L->Dconv, false, L->cw1, true, L->cs[1], d.N, d.C, d.H, 1, d.C, d.R,
                             U, p, 1, E, e.s));
  if (need & FTC_CK_O3)
    CK(launch_conv_f64_exact(L->cd2, true, L->Wcur, false, L->cs[2], 1, d.C, d.H, d.M, L->Ckw, d.R,
                             U, p, d.groups, E, s2));
  if (need & FTC_CK_O4)
    CK(launch_conv_f64_exact(L->Dconv, false, L->cw2, true, L->cs[3], d.N, d.C, d.H, 1, d.C, d.R,
                             U, p, 1, E, s2));
  if (fork) {
    FTC_CUDA_CHECK(cudaEventRecord(L->ev_ck, L->side));
    FTC_CUDA_CHECK(cudaStreamWaitEvent(e.s, L->ev_ck, 0));
  }
  {  // Co5 / Co6 / Co7: the conv_blocks of (Cd1, Cw1), (Cd1, Cw2), (Cd2, Cw1) in one launch
    const double* ins[3];
    const double* ws[3];
    double* outs[3];
    int nj = 0;
    const double* pin[3] = {L->cd1, L->cd1, L->cd2};
    const double* pw[3] = {L->cw1, L->cw2, L->cw1};
    for (int k = 0; k < 3; ++k)
      if (need & (FTC_CK_O5 << k)) {
        ins[nj] = pin[k];
        ws[nj] = pw[k];
        outs[nj] = L->cs[4 + k];
        ++nj;
      }
    if (nj) CK(launch_conv_block3(ins, ws, outs, nj, d.C, d.H, d.R, U, p, E, e.s));
  }
  e.cs_have |= need;
  return FTC_OK;
}

// workflow.hpp:183-196 (ensure_s)
int ensure_s(EP& e, unsigned want) {
  ftc_layer* L = e.L;
  const unsigned need = want & ~e.s_have;
  if (!need) return FTC_OK;
  double* so[7];
  for (int k = 0; k < 7; ++k) so[k] = L->s[k];
  CK(launch_output_summations(vobj(e), L->d.N, L->d.M, L->E, need,
                              L->d.bias_enabled ? L->bias : nullptr, L->agg, so, e.s));
  e.s_have |= need;
  return FTC_OK;
}

Fam fam(EP& e) {
  Fam F;
  for (int k = 0; k < 7; ++k) {
    F.c[k] = (e.cs_have & (1u << k)) ? e.L->cs[k] : nullptr;
    F.s[k] = (e.s_have & (1u << k)) ? e.L->s[k] : nullptr;
  }
  return F;
}

int sync_result(EP& e) {
  FTC_CUDA_CHECK(cudaMemcpyAsync(e.L->res_h, e.L->res, sizeof(SchemeResult), cudaMemcpyDeviceToHost, e.s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(e.s));
  return FTC_OK;
}

int detect_exact_clean(EP& e, bool* clean, double* mrd) {
  ftc_layer* L = e.L;
  FTC_CUDA_CHECK(cudaMemsetAsync(L->stats, 0, sizeof(DetectStats), e.s));
  CK(launch_detect_exact(L->cs[4], L->s[4], L->E2, L->plan.tau, nullptr, L->stats, e.s));
  FTC_CUDA_CHECK(cudaMemcpyAsync(L->stats_h, L->stats, sizeof(DetectStats), cudaMemcpyDeviceToHost, e.s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(e.s));
  *clean = L->stats_h->flagged == 0;
  if (mrd) {
    unsigned long long b = L->stats_h->max_rel_dev_bits;
    double v;
    std::memcpy(&v, &b, sizeof v);
    *mrd = v;
  }
  return FTC_OK;
}

int count_differ_sync(EP& e, const double* c, const double* s_, long long n, int* count) {
  ftc_layer* L = e.L;
  FTC_CUDA_CHECK(cudaMemsetAsync(L->iscratch, 0, sizeof(int32_t), e.s));
  CK(launch_count_differ(c, s_, n, L->plan.tau, L->iscratch, e.s));
  FTC_CUDA_CHECK(cudaMemcpyAsync(L->iscratch_h, L->iscratch, sizeof(int32_t), cudaMemcpyDeviceToHost, e.s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(e.s));
  *count = L->iscratch_h[0];
  return FTC_OK;
}

// CocProbes (workflow.hpp:247-270)
int probe(EP& e, bool row0, bool* consistent) {
  ftc_layer* L = e.L;
  const ftc_conv_desc& d = L->d;
  double* so[7] = {};
  if (row0) {
    // conv_block(D.block(0), ic.cw1, p) vs sum_m O[0,m] - sum_b
    CK(launch_conv_f64_exact(L->Dconv, false, L->cw1, true, L->tmp_c, 1, d.C, d.H, 1, d.C, d.R,
                             d.stride, d.pad, 1, L->E, e.s));
    so[1] = L->tmp_s;
    CK(launch_output_summations(vobj(e), 1, d.M, L->E, FTC_CK_O2,
                                d.bias_enabled ? L->bias : nullptr, L->agg, so, e.s));
  } else {
    // conv_block(Cd1[group 0], W.block(0), p) vs sum_n O[n,0] - N*B[0]
    CK(launch_conv_f64_exact(L->cd1, true, L->Wcur, false, L->tmp_c, 1, L->Ckw, d.H, 1, L->Ckw,
                             d.R, d.stride, d.pad, 1, L->E, e.s));
    so[0] = L->tmp_s;  // column 0 is the first E2 entries of So1
    CK(launch_output_summations(vobj(e), d.N, d.M, L->E, FTC_CK_O1,
                                d.bias_enabled ? L->bias : nullptr, L->agg, so, e.s));
  }
  int cnt = 0;
  CK(count_differ_sync(e, L->tmp_c, L->tmp_s, L->E2, &cnt));
  *consistent = cnt == 0;
  return FTC_OK;
}

// workflow.hpp:205-219 over the current patch list; on failure roll back.
int verify_patches(EP& e, int np, bool* pass) {
  ftc_layer* L = e.L;
  const unsigned trusted = e.cs_have & e.trust_mask;
  VerifyWS ws{L->ov, L->present, L->touched5, L->touched1, L->fresh567, L->tlist, L->tcount};
  CK(run_verify(fam(e), trusted, L->O, L->d.N, L->d.M, L->E2, L->d.bias_enabled, L->bias, L->agg,
                L->plan.tau, L->patches, L->res, np, ws, L->iscratch, e.s));
  e.ov_dirty = true;
  FTC_CUDA_CHECK(cudaMemcpyAsync(L->iscratch_h, L->iscratch, sizeof(int32_t), cudaMemcpyDeviceToHost, e.s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(e.s));
  *pass = L->iscratch_h[0] == 0;
  if (!*pass) CK(run_rollback(L->patches, np, L->d.M, L->E2, ws, e.s));
  return FTC_OK;
}

// Data repair: recompute the (n,m) planes named by the patch list from the
// caller's input (ftc_abi.h: "corrected (n,m) planes recomputed on device").
int repair_planes(EP& e, int np, ftc_layer_report* rep) {
  ftc_layer* L = e.L;
  const int N = L->d.N, M = L->d.M;
  const size_t words = ((size_t)N * M + 31) / 32;
  FTC_CUDA_CHECK(cudaMemsetAsync(L->plane_mask, 0, words * sizeof(uint32_t), e.s));
  CK(run_patch_planes(L->patches, np, M, L->plane_mask, e.s));
  FTC_CUDA_CHECK(cudaMemcpyAsync(L->plane_mask_h.data(), L->plane_mask, words * sizeof(uint32_t),
                                 cudaMemcpyDeviceToHost, e.s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(e.s));
  int lo = N, hi = -1, nb = 0;
  for (int n = 0; n < N; ++n)
    for (int m = 0; m < M; ++m) {
      const size_t pl = (size_t)n * M + m;
      if (!((L->plane_mask_h[pl >> 5] >> (pl & 31)) & 1u)) continue;
      if (nb < FTC_MAX_BLOCKS) {
        rep->blocks[nb][0] = n;
        rep->blocks[nb][1] = m;
      }
      ++nb;
      lo = std::min(lo, n);
      hi = std::max(hi, n);
    }
  rep->n_blocks = nb;
  rep->repaired_planes = nb;
  if (nb > 0)
    CK(run_conv(L, L->D, L->Wcur, L->O, false, false, L->plane_mask, lo, hi + 1, e.s));
  return FTC_OK;
}

void add_stage(ftc_layer_report* rep, int st) {
  if (rep->n_stages < FTC_MAX_STAGES) rep->stages[rep->n_stages++] = st;
}

// Outcome of one correcting scheme: 1 = settled, 0 = escalate
int finish_valid(EP& e, int stage, ftc_layer_report* rep, int* settled) {
  ftc_layer* L = e.L;
  const int np = std::min(L->res_h->n_patches, L->patches.cap);
  bool pass = false;
  CK(verify_patches(e, np, &pass));
  if (pass) {
    rep->stage = stage;
    CK(repair_planes(e, np, rep));
    *settled = 1;
  } else {
    *settled = 0;
  }
  return FTC_OK;
}

int clear_overrides(EP& e) {
  ftc_layer* L = e.L;
  if (e.ov_dirty) {
    FTC_CUDA_CHECK(cudaMemsetAsync(L->present, 0, L->nO, e.s));
    FTC_CUDA_CHECK(cudaMemsetAsync(L->touched5, 0, L->E2, e.s));
    FTC_CUDA_CHECK(cudaMemsetAsync(L->touched1, 0, (size_t)L->d.M * L->E2, e.s));
  }
  return FTC_OK;
}

// workflow.hpp:221-245: exact-order input checksums, CoC-D on exact-order Co5/So5, and
// verify_kernel / reload.  *resolved = 1 when the layer is settled here (clean on the
// exact re-detection, or clean after the reload).
int detect_and_reload(EP& e, ftc_layer_report* rep, int* resolved) {
  ftc_layer* L = e.L;
  const ftc_conv_desc& d = L->d;
  *resolved = 0;

  // The clean path may have produced only a fast Cd1: take the exact-order input
  // checksums of the caller's (pre-fault) D, re-applying injected checksum faults.
  if (L->cd_ext1) {
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->cd1, L->cd_ext1, L->nCd * sizeof(double), cudaMemcpyDeviceToDevice, e.s));
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->cd2, L->cd_ext2, L->nCd * sizeof(double), cudaMemcpyDeviceToDevice, e.s));
    L->cd_ext1 = L->cd_ext2 = nullptr;
  }
  if (!L->ck_exact) {
    CK(launch_input_checksums(L->D, d.N, L->nCd, L->cd1, L->cd2, e.s));
    if (L->has_cd_faults) {
      CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_CD1, L->cd1, true, L->scale_tab, d.C, d.H, d.H, L->nCd, e.s));
      CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_CD2, L->cd2, true, L->scale_tab, d.C, d.H, d.H, L->nCd, e.s));
    }
    L->ck_exact = true;
  }
  // Re-establish the CoC-D verdict on exact-order Co5/So5 (bitwise the reference's).  So6
  // and So7 come with So5: the three chains run side by side in one launch whose time is
  // the chain length, and CoC needs them next (values identical whenever computed: O is
  // unchanged until a scheme patches it)
  // The chain-bound So5-7 launch runs on the layer's side stream beside Co5 -- and, ahead
  // of their use, Co6/Co7 and the kernel checksums of verify_kernel -- on the main one:
  // all read only D, W, the input checksums and the unpatched O (this path is entered
  // after the clean-path screen fired, so the exact re-detection nearly always confirms)
  static const bool ep_serial = getenv_flag("FTC_EP_SERIAL");
  const bool fork = !ep_serial && L->side && L->ev_start && L->ev_ck;
  if (fork) {
    FTC_CUDA_CHECK(cudaEventRecord(L->ev_start, e.s));
    FTC_CUDA_CHECK(cudaStreamWaitEvent(L->side, L->ev_start, 0));
    cudaStream_t main_s = e.s;
    e.s = L->side;
    const int st_s = ensure_s(e, FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7);
    e.s = main_s;
    if (st_s != FTC_OK) return st_s;
    CK(ensure_cs(e, FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
    CK(launch_kernel_checksums(L->Wcur, d.M, L->Ckw, d.R, d.groups, L->tmp_cw1, L->tmp_cw2, e.s));
    FTC_CUDA_CHECK(cudaEventRecord(L->ev_ck, L->side));
    FTC_CUDA_CHECK(cudaStreamWaitEvent(e.s, L->ev_ck, 0));
  } else {
    CK(ensure_cs(e, FTC_CK_O5));
    CK(ensure_s(e, FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
  }
  bool clean = false;
  double mrd = 0.0;
  CK(detect_exact_clean(e, &clean, &mrd));
  rep->max_rel_dev = mrd;
  rep->n_flagged = L->stats_h->flagged;
  rep->detected = !clean;
  if (clean) {
    rep->stage = FTC_STAGE_NONE;
    *resolved = 1;
    return FTC_OK;
  }

  // verify_kernel (checksums.hpp:250-259) / reload (workflow.hpp:232-245)
  if (!fork) CK(launch_kernel_checksums(L->Wcur, d.M, L->Ckw, d.R, d.groups, L->tmp_cw1, L->tmp_cw2, e.s));
  int kbad = 0;
  CK(count_differ_sync(e, L->tmp_cw1, L->cw1, L->nCw, &kbad));
  if (kbad) {
    L->Wcur = L->W;
    L->cw1 = L->cw1g;
    L->cw2 = L->cw2g;
    e.cs_have = 0;
    rep->weights_reloaded = 1;
    CK(ensure_cs(e, FTC_CK_O5));
    CK(detect_exact_clean(e, &clean, nullptr));
    if (clean) {
      rep->stage = FTC_STAGE_RELOAD;
      *resolved = 1;
    }
  }
  return FTC_OK;
}

int error_path(ftc_layer* L, ftc_layer_report* rep) {
  CK(alloc_error_path(L));
  EP e{L, L->stream};
  const ftc_conv_desc& d = L->d;
  int ret = FTC_OK;
  auto cleanup = [&]() -> int { return clear_overrides(e); };
  bool clean = false;
  int resolved = 0;
  CK(detect_and_reload(e, rep, &resolved));
  if (resolved) return cleanup();

  // CoC (workflow.hpp:277-288)
  CK(ensure_cs(e, FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
  CK(ensure_s(e, FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
  add_stage(rep, FTC_STAGE_COC);
  CK(run_coc_analyze(fam(e), d.N, d.M, L->E2, L->plan.tau, L->res, L->patches, e.s));
  CK(sync_result(e));
  int settled = 0;
  switch (L->res_h->status) {
    case SCH_EMPTY:
      rep->stage = FTC_STAGE_COC;
      return cleanup();
    case SCH_VALID:
      CK(finish_valid(e, FTC_STAGE_COC, rep, &settled));
      if (settled) return cleanup();
      break;
    case SCH_PROBE_ROW0:
    case SCH_PROBE_COL0: {
      bool ok = false;
      CK(probe(e, L->res_h->status == SCH_PROBE_ROW0, &ok));
      if (ok) {
        rep->stage = FTC_STAGE_DISCARD;
        return cleanup();
      }
      break;
    }
    default:
      break;
  }

  // RC / ClC (workflow.hpp:290-309)
  for (int pass_ = 0; pass_ < 2; ++pass_) {
    const bool rc = pass_ == 0;
    if (rc ? !L->plan.rc_enabled : !L->plan.clc_enabled) continue;
    const unsigned fams = rc ? (FTC_CK_O1 | FTC_CK_O3) : (FTC_CK_O2 | FTC_CK_O4);
    CK(ensure_cs(e, fams));
    CK(ensure_s(e, fams));
    add_stage(rep, rc ? FTC_STAGE_RC : FTC_STAGE_CLC);
    CK(run_line_analyze(fam(e), rc, d.N, d.M, L->E2, L->plan.tau, L->res, L->patches, e.s));
    CK(sync_result(e));
    if (L->res_h->status == SCH_EMPTY) {
      rep->stage = rc ? FTC_STAGE_RC : FTC_STAGE_CLC;
      return cleanup();
    }
    if (L->res_h->status == SCH_VALID) {
      CK(finish_valid(e, rc ? FTC_STAGE_RC : FTC_STAGE_CLC, rep, &settled));
      if (settled) return cleanup();
    }
  }

  // FC (workflow.hpp:310-321)
  CK(ensure_cs(e, FTC_CK_O1 | FTC_CK_O2));
  CK(ensure_s(e, FTC_CK_O1 | FTC_CK_O2));
  add_stage(rep, FTC_STAGE_FC);
  CK(run_fc_analyze(fam(e), d.N, d.M, L->E2, L->plan.tau, L->res, L->patches, L->colmask,
                    L->rowmask, L->colany, L->rowany, e.s));
  CK(sync_result(e));
  if (L->res_h->status == SCH_DISCARD) {
    rep->stage = FTC_STAGE_DISCARD;
    return cleanup();
  }
  if (L->res_h->status == SCH_VALID) {
    CK(finish_valid(e, FTC_STAGE_FC, rep, &settled));
    if (settled) return cleanup();
  }

  // recompute (workflow.hpp:325-338): fresh conv (no hooks), fresh input
  // checksums, Co5/So5 only
  add_stage(rep, FTC_STAGE_RECOMPUTE);
  CK(cleanup());
  e.ov_dirty = false;
  for (int attempt = 0; attempt < 2; ++attempt) {
    CK(run_conv(L, L->Dconv, L->Wcur, L->O, false, false, nullptr, 0, d.N, e.s));
    CK(launch_input_checksums(L->Dconv, d.N, L->nCd, L->cd1, L->cd2, e.s));
    CK(launch_kernel_checksums(L->Wcur, d.M, L->Ckw, d.R, d.groups, L->tmp_cw1, L->tmp_cw2, e.s));
    L->cw1 = L->tmp_cw1;
    L->cw2 = L->tmp_cw2;
    e.cs_have = 0;
    e.s_have = 0;
    CK(ensure_cs(e, FTC_CK_O5));
    CK(ensure_s(e, FTC_CK_O5));
    CK(detect_exact_clean(e, &clean, nullptr));
    if (clean) {
      rep->stage = FTC_STAGE_RECOMPUTE;
      rep->recomputed = 1;
      return FTC_OK;
    }
  }
  ret = FTC_INTEGRITY_ERROR;
  set_error(ret, "layer recomputation failed verification twice");
  return ret;
}

// acceptance.cpp:207-292 (isolation_succeeds): the detection + reload preamble, then ONE
// scheme on its own with a Co5-only verifier and no CoC probes (an index-0 pattern is a
// discard).  *status: -1 settled by the preamble (clean / reload), 0 corrected (planes
// repaired), 1 discard, 2 escalate (patches rolled back, O untouched).
int isolated_path(ftc_layer* L, int scheme, int* status, ftc_layer_report* rep) {
  CK(alloc_error_path(L));
  EP e{L, L->stream};
  e.trust_mask = FTC_CK_O5;
  const ftc_conv_desc& d = L->d;
  auto cleanup = [&]() -> int { return clear_overrides(e); };
  int resolved = 0;
  *status = -1;
  CK(detect_and_reload(e, rep, &resolved));
  if (resolved) return cleanup();
  int settled = 0;
  *status = 2;
  if (scheme == 1) {
    CK(ensure_cs(e, FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
    CK(ensure_s(e, FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
    add_stage(rep, FTC_STAGE_COC);
    CK(run_coc_analyze(fam(e), d.N, d.M, L->E2, L->plan.tau, L->res, L->patches, e.s));
    CK(sync_result(e));
    switch (L->res_h->status) {
      case SCH_EMPTY: *status = 0; break;
      case SCH_VALID:
        CK(finish_valid(e, FTC_STAGE_COC, rep, &settled));
        *status = settled ? 0 : 2;
        break;
      case SCH_PROBE_ROW0:
      case SCH_PROBE_COL0: *status = 1; break;
      default: break;
    }
  } else if (scheme == 2 || scheme == 3) {
    const bool rc = scheme == 2;
    const unsigned fams = rc ? (FTC_CK_O1 | FTC_CK_O3) : (FTC_CK_O2 | FTC_CK_O4);
    CK(ensure_cs(e, fams));
    CK(ensure_s(e, fams));
    add_stage(rep, rc ? FTC_STAGE_RC : FTC_STAGE_CLC);
    CK(run_line_analyze(fam(e), rc, d.N, d.M, L->E2, L->plan.tau, L->res, L->patches, e.s));
    CK(sync_result(e));
    if (L->res_h->status == SCH_EMPTY) {
      *status = 0;
    } else if (L->res_h->status == SCH_VALID) {
      CK(finish_valid(e, rc ? FTC_STAGE_RC : FTC_STAGE_CLC, rep, &settled));
      *status = settled ? 0 : 2;
    }
  } else {
    CK(ensure_cs(e, FTC_CK_O1 | FTC_CK_O2 | FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
    CK(ensure_s(e, FTC_CK_O1 | FTC_CK_O2 | FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7));
    add_stage(rep, FTC_STAGE_FC);
    CK(run_fc_analyze(fam(e), d.N, d.M, L->E2, L->plan.tau, L->res, L->patches, L->colmask,
                      L->rowmask, L->colany, L->rowany, e.s));
    CK(sync_result(e));
    if (L->res_h->status == SCH_DISCARD) {
      *status = 1;
    } else if (L->res_h->status == SCH_VALID) {
      CK(finish_valid(e, FTC_STAGE_FC, rep, &settled));
      *status = settled ? 0 : 2;
    }
  }
  if (*status == 1) rep->stage = FTC_STAGE_DISCARD;
  return cleanup();
}

int stage_faults(ftc_layer* L, const ftc_fault* faults, int n, cudaStream_t s) {
  L->nfaults = 0;
  L->n_out_faults = 0;
  if (n <= 0 || !faults) return FTC_OK;
  if (n > L->faults_cap) {
    if (L->faults_dev) cudaFree(L->faults_dev);
    if (L->faults_h) cudaFreeHost(L->faults_h);
    L->faults_cap = std::max(n, 16);
    CK(dalloc(&L->faults_dev, L->faults_cap));
    FTC_CUDA_CHECK(cudaMallocHost((void**)&L->faults_h, L->faults_cap * sizeof(ftc_fault)));
  }
  // the pinned staging buffer may still feed an earlier async copy
  FTC_CUDA_CHECK(cudaStreamSynchronize(s));
  std::memcpy(L->faults_h, faults, n * sizeof(ftc_fault));
  // SCALE faults: expand the reference's per-element magnitudes on the host with the
  // same generator and distribution (mt19937_64(seed), uniform_real_distribution
  // <double>(0, 1), mag = 0.5 + 1.5 u, fault.hpp:76-80) in make_hooks' iteration order;
  // the device record's `bit` carries the fault's offset into the table
  {
    std::vector<double> tab;
    const ftc_conv_desc& d = L->d;
    for (int q = 0; q < n; ++q) {
      ftc_fault& f = L->faults_h[q];
      if (f.mode != FTC_FAULT_SCALE) continue;
      long long dims[4];
      switch (f.target) {
        case FTC_FAULT_OUTPUT: dims[0] = d.N; dims[1] = d.M; dims[2] = L->E; dims[3] = L->E; break;
        case FTC_FAULT_FMAP: dims[0] = d.N; dims[1] = d.C; dims[2] = d.H; dims[3] = d.H; break;
        case FTC_FAULT_KERNEL: dims[0] = d.M; dims[1] = L->Ckw; dims[2] = d.R; dims[3] = d.R; break;
        case FTC_FAULT_CD1: case FTC_FAULT_CD2: dims[0] = 1; dims[1] = d.C; dims[2] = d.H; dims[3] = d.H; break;
        default: dims[0] = 1; dims[1] = d.C; dims[2] = d.R; dims[3] = d.R; break;
      }
      const int coord[4] = {f.n, f.m, f.x, f.y};
      long long count = 1;
      for (int a = 0; a < 4; ++a) {
        if (coord[a] >= dims[a]) RET_ERR(FTC_CONFIG_ERROR, "fault coordinates out of range");
        if (coord[a] < 0) count *= dims[a];
      }
      f.bit = (uint32_t)tab.size();
      std::mt19937_64 rng(f.seed);
      std::uniform_real_distribution<double> u(0.0, 1.0);
      for (long long k = 0; k < count; ++k) tab.push_back(0.5 + 1.5 * u(rng));
    }
    if (!tab.empty()) {
      if (tab.size() > L->scale_cap) {
        if (L->scale_tab) cudaFree(L->scale_tab);
        L->scale_cap = tab.size();
        CK(dalloc(&L->scale_tab, L->scale_cap));
      }
      FTC_CUDA_CHECK(cudaMemcpy(L->scale_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
  }
  FTC_CUDA_CHECK(cudaMemcpyAsync(L->faults_dev, L->faults_h, n * sizeof(ftc_fault), cudaMemcpyHostToDevice, s));
  L->nfaults = n;
  for (int q = 0; q < n; ++q)
    if (faults[q].target == FTC_FAULT_OUTPUT) ++L->n_out_faults;
  return FTC_OK;
}

bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && *v != '0';
}

bool has_target(const ftc_fault* f, int n, int t) {
  for (int q = 0; q < n; ++q)
    if (f[q].target == t) return true;
  return false;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int32_t ftc_abi_version(void) { return FTC_ABI_VERSION; }

const char* ftc_last_error(void) { return ftc::g_err.c_str(); }

int ftc_set_conv_engine(int engine) {
  if (engine != 0 && engine != 1) RET_ERR(FTC_INVALID_ARGUMENT, "engine must be 0 (tcgen05) or 1 (simt)");
  g_engine = engine;
  return FTC_OK;
}

int ftc_get_conv_engine(void) { return g_engine; }

int ftc_output_extent(int32_t H, int32_t R, int32_t pad, int32_t stride, int32_t* E) {
  ftc_conv_desc d{1, 1, H, 1, R, stride, pad, 1, 0};
  int e = 0;
  CK(validate(&d, &e));
  if (E) *E = e;
  return FTC_OK;
}

int ftc_layer_create(const ftc_conv_desc* desc, const float* W_host, const float* bias_host,
                     ftc_layer** out) {
  int E = 0;
  CK(validate(desc, &E));
  if (!W_host || !out) RET_ERR(FTC_INVALID_ARGUMENT, "null W or out");
  if (desc->bias_enabled && !bias_host) RET_ERR(FTC_SHAPE_ERROR, "bias length must equal kernel count M");
  ftc_layer* L = new ftc_layer();
  L->d = *desc;
  L->E = E;
  L->E2 = E * E;
  L->Ckw = desc->C / desc->groups;
  L->nD = (long long)desc->N * desc->C * desc->H * desc->H;
  L->nW = (long long)desc->M * L->Ckw * desc->R * desc->R;
  L->nO = (long long)desc->N * desc->M * L->E2;
  L->nCd = (long long)desc->C * desc->H * desc->H;
  L->nCw = (long long)desc->C * desc->R * desc->R;
  auto fail = [&](int st) {
    free_layer(L);
    return st;
  };
  int st;
  if ((st = dalloc(&L->W, L->nW)) || (st = dalloc(&L->agg, 2)) || (st = dalloc(&L->cw1g, L->nCw)) ||
      (st = dalloc(&L->cw2g, L->nCw)) || (st = dalloc(&L->cw1w, L->nCw)) ||
      (st = dalloc(&L->cw2w, L->nCw)) || (st = dalloc(&L->cd1, L->nCd)) ||
      (st = dalloc(&L->cd2, L->nCd)) || (st = dalloc(&L->co5f, L->E2)) ||
      (st = dalloc(&L->so5acc, L->E2)) || (st = dalloc(&L->stats, 1)))
    return fail(st);
  if (cudaMemset(L->so5acc, 0, L->E2 * sizeof(double)) != cudaSuccess ||
      cudaMemset(L->co5f, 0, L->E2 * sizeof(double)) != cudaSuccess)  // Co5 may be scattered into
    return fail(FTC_CUDA_ERROR);
  {
    // Cd1 workspace of the fused clean path when no producer supplies Cd1
    const long long n = cd1_ws_doubles_g(desc->N, desc->C, desc->H, L->nCd);
    if ((st = dalloc(&L->cd1ws, (size_t)n)) || (st = dalloc(&L->co5tab, (size_t)L->nCw))) return fail(st);
    if (cudaMemset(L->cd1ws, 0, (size_t)n * sizeof(double)) != cudaSuccess) return fail(FTC_CUDA_ERROR);
  }
  if (cudaMallocHost((void**)&L->stats_h, sizeof(DetectStats)) != cudaSuccess)
    return fail(FTC_CUDA_ERROR);
  if ((st = dalloc(&L->fstats, 1)) || (st = dalloc(&L->fticket, 1))) return fail(st);
  if (cudaMemset(L->fstats, 0, sizeof(DetectStats)) != cudaSuccess ||
      cudaMemset(L->fticket, 0, sizeof(unsigned int)) != cudaSuccess ||
      cudaHostAlloc((void**)&L->fstats_h, sizeof(DetectStats), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&L->fstats_hd, L->fstats_h, 0) != cudaSuccess)
    return fail(FTC_CUDA_ERROR);
  if (cudaMemcpy(L->W, W_host, L->nW * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(FTC_CUDA_ERROR);
  if (desc->bias_enabled) {
    if ((st = dalloc(&L->bias, desc->M))) return fail(st);
    if (cudaMemcpy(L->bias, bias_host, desc->M * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(FTC_CUDA_ERROR);
    if ((st = launch_bias_aggregates(L->bias, desc->M, L->agg, 0))) return fail(st);
  } else {
    cudaMemset(L->agg, 0, 2 * sizeof(double));
  }
  if ((st = launch_kernel_checksums(L->W, desc->M, L->Ckw, desc->R, desc->groups, L->cw1g, L->cw2g, 0)))
    return fail(st);
  if ((st = launch_co5_taps(L->cw1g, desc->C, desc->H, desc->R, L->co5tab, 0))) return fail(st);
  if (cudaStreamCreateWithFlags(&L->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_start, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_ck, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_done, cudaEventDisableTiming) != cudaSuccess)
    return fail(FTC_CUDA_ERROR);
  if (tc_supported(*desc)) {
    if ((st = tc_plan_create(*desc, L->W, &L->tc, 0))) return fail(st);
  }
  {
    const size_t parts = (size_t)tc_rowsum_parts(L->tc);
    if ((st = dalloc(&L->rowsum, parts * desc->N * L->E2)) ||
        (st = dalloc(&L->rowsum_m, parts * desc->N * L->E2)))
      return fail(st);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(FTC_CUDA_ERROR, "layer setup kernels failed");
    return fail(FTC_CUDA_ERROR);
  }
  *out = L;
  return FTC_OK;
}

int ftc_layer_destroy(ftc_layer* L) {
  if (!L) return FTC_OK;
  cudaDeviceSynchronize();
  free_layer(L);
  return FTC_OK;
}

int ftc_layer_extent(const ftc_layer* L, int32_t* E) {
  if (!L || !E) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  *E = L->E;
  return FTC_OK;
}

int ftc_conv_forward(ftc_layer* L, const float* D, float* O, void* stream) {
  if (!L || !D || !O) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  L->nfaults = 0;
  return timed_conv(L, D, L->W, O, false, false, (cudaStream_t)stream);
}

int ftc_layer_desc(const ftc_layer* L, ftc_conv_desc* desc) {
  if (!L || !desc) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  *desc = L->d;
  return FTC_OK;
}

int ftc_conv_forward_faulted(ftc_layer* L, const float* D, float* O, const ftc_fault* faults, int32_t n_faults,
                             void* stream) {
  if (!L || !D || !O) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (L->inflight) RET_ERR(FTC_INVALID_ARGUMENT, "a protected call is in flight on this layer");
  cudaStream_t s = (cudaStream_t)stream;
  CK(stage_faults(L, faults, n_faults, s));
  const ftc_conv_desc& d = L->d;
  const float* Dc = D;
  const float* Wc = L->W;
  if (L->nfaults && has_target(faults, n_faults, FTC_FAULT_FMAP)) {
    if (!L->D_work) CK(dalloc(&L->D_work, L->nD));
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->D_work, D, L->nD * sizeof(float), cudaMemcpyDeviceToDevice, s));
    CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_FMAP, L->D_work, false, L->scale_tab, d.C, d.H, d.H,
                        L->nD, s));
    Dc = L->D_work;
  }
  if (L->nfaults && has_target(faults, n_faults, FTC_FAULT_KERNEL)) {
    if (!L->W_work) CK(dalloc(&L->W_work, L->nW));
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->W_work, L->W, L->nW * sizeof(float), cudaMemcpyDeviceToDevice, s));
    CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_KERNEL, L->W_work, false, L->scale_tab, L->Ckw, d.R,
                        d.R, L->nW, s));
    Wc = L->W_work;
  }
  const int st = run_conv(L, Dc, Wc, O, L->n_out_faults > 0, false, nullptr, 0, d.N, s);
  L->nfaults = 0;
  L->n_out_faults = 0;
  return st;
}

int ftc_conv_forward_host(ftc_layer* L, const float* D_host, float* O_host, void* stream) {
  if (!L || !D_host || !O_host) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (!L->D_host_buf) CK(dalloc(&L->D_host_buf, L->nD));
  if (!L->O_host_buf) CK(dalloc(&L->O_host_buf, L->nO));
  FTC_CUDA_CHECK(cudaMemcpyAsync(L->D_host_buf, D_host, L->nD * sizeof(float), cudaMemcpyHostToDevice, s));
  CK(ftc_conv_forward(L, L->D_host_buf, L->O_host_buf, stream));
  FTC_CUDA_CHECK(cudaMemcpyAsync(O_host, L->O_host_buf, L->nO * sizeof(float), cudaMemcpyDeviceToHost, s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(s));
  return FTC_OK;
}

int ftc_layer_input_nhwc(ftc_layer* L, float** nhwc) {
  if (!L || !nhwc) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  *nhwc = (use_tc(L) && tc_im2col(L->tc)) ? tc_nhwc_buffer(L->tc) : nullptr;
  return FTC_OK;
}

int ftc_layer_input_nhwc_ready(ftc_layer* L, const float* D) {
  if (!L || !D) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (!(use_tc(L) && tc_im2col(L->tc))) RET_ERR(FTC_INVALID_ARGUMENT, "layer does not stage an NHWC input");
  L->nhwc_ready = true;
  L->D_staged = D;
  return FTC_OK;
}

int ftc_layer_set_timing(ftc_layer* L, int32_t enable) {
  if (!L) RET_ERR(FTC_INVALID_ARGUMENT, "null layer");
  if (enable && !L->ev_c0) {
    FTC_CUDA_CHECK(cudaEventCreate(&L->ev_c0));
    FTC_CUDA_CHECK(cudaEventCreate(&L->ev_c1));
  }
  CK(harvest_timing(L));
  L->timing = enable != 0;
  return FTC_OK;
}

int ftc_layer_kernel_time(ftc_layer* L, double* conv_ms, int32_t* conv_launches, int32_t reset) {
  if (!L) RET_ERR(FTC_INVALID_ARGUMENT, "null layer");
  CK(harvest_timing(L));
  if (conv_ms) *conv_ms = L->conv_ms;
  if (conv_launches) *conv_launches = L->conv_launches;
  if (reset) {
    L->conv_ms = 0.0;
    L->conv_launches = 0;
  }
  return FTC_OK;
}

uint64_t ftc_kernel_launches(void) { return g_launches.load(); }

static int launch_impl(ftc_layer* L, const ftc_plan* plan, const float* D, float* O,
                       const double* cd1_in, const double* cd2_in, const ftc_fault* faults,
                       int32_t n_faults, void* stream) {
  if (!L || !plan || !D || !O) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (L->inflight) RET_ERR(FTC_INVALID_ARGUMENT, "a protected call is already in flight on this layer");
  cudaStream_t s = (cudaStream_t)stream;
  L->t0 = std::chrono::steady_clock::now();
  L->plan = *plan;
  L->D = D;
  L->O = O;
  L->stream = s;
  CK(stage_faults(L, faults, n_faults, s));
  const ftc_conv_desc& d = L->d;
  // working copies for pre_conv faults (the reference copies D and W, workflow.hpp:151-152)
  L->Dconv = D;
  L->Wcur = L->W;
  L->cw1 = L->cw1g;
  L->cw2 = L->cw2g;
  if (L->nfaults && has_target(faults, n_faults, FTC_FAULT_FMAP)) {
    if (!L->D_work) CK(dalloc(&L->D_work, L->nD));
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->D_work, D, L->nD * sizeof(float), cudaMemcpyDeviceToDevice, s));
    CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_FMAP, L->D_work, false, L->scale_tab, d.C, d.H, d.H,
                        L->nD, s));
    L->Dconv = L->D_work;
  }
  if (L->nfaults && has_target(faults, n_faults, FTC_FAULT_KERNEL)) {
    if (!L->W_work) CK(dalloc(&L->W_work, L->nW));
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->W_work, L->W, L->nW * sizeof(float), cudaMemcpyDeviceToDevice, s));
    CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_KERNEL, L->W_work, false, L->scale_tab, L->Ckw, d.R,
                        d.R, L->nW, s));
    L->Wcur = L->W_work;
  }
  const bool cwf = L->nfaults && (has_target(faults, n_faults, FTC_FAULT_CW1) ||
                                  has_target(faults, n_faults, FTC_FAULT_CW2));
  if (cwf) {
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->cw1w, L->cw1g, L->nCw * sizeof(double), cudaMemcpyDeviceToDevice, s));
    FTC_CUDA_CHECK(cudaMemcpyAsync(L->cw2w, L->cw2g, L->nCw * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_CW1, L->cw1w, true, L->scale_tab, d.C, d.R, d.R, L->nCw, s));
    CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_CW2, L->cw2w, true, L->scale_tab, d.C, d.R, d.R, L->nCw, s));
    L->cw1 = L->cw1w;
    L->cw2 = L->cw2w;
  }
  // side stream: input checksums of the caller's (pre-fault) D, then Co5.  When the
  // producer of D already reduced it (glue kernels of a net), the exact Cd1/Cd2 are
  // taken as given; otherwise a fast Cd1-only pass feeds CoC-D.
  L->has_cd_faults = L->nfaults && (has_target(faults, n_faults, FTC_FAULT_CD1) ||
                                    has_target(faults, n_faults, FTC_FAULT_CD2));
  const double* cd1_use = L->cd1;
  L->cd_ext1 = L->cd_ext2 = nullptr;
  const bool pre_faults = L->Dconv != D || L->Wcur != L->W || cwf || L->has_cd_faults;
  // Fused clean path (tcgen05 engine, golden operands): Cd1 comes from the producer
  // (glue kernels) or one streaming pass over D (small batches: the same pass stages the
  // NHWC copy for the TMA im2col engine); the conv computes Co5 in its checksum warp and
  // accumulates So5 from its row sums; one small kernel then runs CoC-D.
  static const bool fused_off = getenv("FTC_NO_FUSED") != nullptr;
  if (!fused_off && use_tc(L) && !pre_faults) {
    bool dt_ready = false, co5_ready = false;
    if (cd1_in) {
      cd1_use = cd1_in;
      if (cd2_in) {  // exact-order checksums: kept for the error path
        L->cd_ext1 = cd1_in;
        L->cd_ext2 = cd2_in;
        L->ck_exact = true;
      } else {
        L->ck_exact = false;
      }
    } else {
      const bool stage = tc_im2col(L->tc) && !(L->nhwc_ready && L->D_staged == D);
      if (stage && d.N <= 32) {
        // small batch: one pass writes the NHWC copy, the exact-order Cd1/Cd2 and, by
        // linearity, Co5 (each block scatters its Cd1 elements' share) -- unless Co5 fits
        // in the conv's checksum warp (FTC_CO5_IN=1 forces that: experiments)
        static const bool co5_force = getenv_flag("FTC_CO5_IN");
        const Co5Job job{L->co5f, L->cw1, d.H, d.R, d.stride, d.pad, L->E};
        CK(launch_nhwc_cd(D, tc_nhwc_buffer(L->tc), d.C, d.H * d.H, 0, d.N, L->cd1, L->cd2, s,
                          co5_force ? nullptr : &job));
        co5_ready = !co5_force;
        dt_ready = true;
        cd1_use = L->cd1;
        L->ck_exact = true;
      } else if (stage) {
        // larger batches: one pass parallel over image groups stages the NHWC copy and
        // reduces the any-order Cd1 (the exact-order checksums wait for the error path)
        CK(launch_act_pool_nhwc_cd1(D, nullptr, tc_nhwc_buffer(L->tc), d.N, d.C, d.H, 0, 1, 1, 0, L->cd1ws, s));
        dt_ready = true;
        cd1_use = L->cd1ws;
        L->ck_exact = false;
      } else {
        CK(launch_cd1_parts(D, d.N, L->nCd, L->cd1ws, s));
        cd1_use = L->cd1ws;
        L->ck_exact = false;
      }
    }
    // Co5 in the conv's checksum warp when it fits in the conv's shadow, else in the
    // CoC-D kernel after the conv (one launch either way)
    const bool co5_in = !co5_ready && (tc_co5_in_kernel(L->tc, d.N, L->E) || getenv_flag("FTC_CO5_IN"));
    FusedDetect fd{L->co5f, L->so5acc, L->agg, plan->tau, d.bias_enabled ? 1 : 0, L->fstats, L->fticket,
                   L->fstats_hd, co5_in ? cd1_use : nullptr, L->co5tab};
    // the staging pass / conv scatter into the Co5 and So5 accumulators, which only
    // the detect kernels re-zero: on a failed launch clear them here, or every later
    // call on this layer would read stale partial sums as a CoC-D mismatch
    int st = timed_conv(L, D, L->Wcur, O, L->n_out_faults > 0, false, s, &fd, dt_ready);
    // CoC-D on the layer's side stream (forked after the conv, so the caller's next
    // kernels do not wait for the compare) is an experiment, FTC_DETECT_SIDE=1: it saved
    // ~0.8% on VGG-19 and cost config 1 ~4 us of fork/join, so the compare stays in line
    cudaStream_t ds = s;
    static const bool detect_side = getenv_flag("FTC_DETECT_SIDE");
    if (st == FTC_OK && detect_side) {
      if (cudaEventRecord(L->ev_start, s) == cudaSuccess && cudaStreamWaitEvent(L->side, L->ev_start, 0) == cudaSuccess)
        ds = L->side;
    }
    if (st == FTC_OK) {
      if (co5_in || co5_ready)
        st = launch_detect_fused(L->co5f, L->so5acc, d.N, L->E2, d.bias_enabled ? 1 : 0, L->agg, plan->tau,
                                 L->fstats, L->fticket, L->fstats_hd, ds);
      else
        st = launch_co5_detect(cd1_use, L->cw1, L->co5f, L->so5acc, d.N, d.C, d.H, d.R, d.stride, d.pad, L->E,
                               d.bias_enabled ? 1 : 0, L->agg, plan->tau, L->fstats, L->fticket, L->fstats_hd, ds);
    }
    if (st != FTC_OK) {
      cudaStreamSynchronize(ds);
      cudaMemsetAsync(L->co5f, 0, L->E2 * sizeof(double), s);
      cudaMemsetAsync(L->so5acc, 0, L->E2 * sizeof(double), s);
      return st;
    }
    FTC_CUDA_CHECK(cudaEventRecord(L->ev_done, ds));
    L->inflight = true;
    return FTC_OK;
  }
  // The conv is enqueued first so its persistent CTAs are dispatched before the
  // side-stream checksum work, which then fills the SM resources they leave free.
  FTC_CUDA_CHECK(cudaEventRecord(L->ev_start, s));
  CK(timed_conv(L, L->Dconv, L->Wcur, O, L->n_out_faults > 0, true, s));
  FTC_CUDA_CHECK(cudaStreamWaitEvent(L->side, L->ev_start, 0));
  if (cd1_in && !cd2_in) {  // producer Cd1 in any order (ftc_protected_conv_launch_cd1)
    if (L->has_cd_faults) cd1_in = nullptr;  // checksum faults: reduce D here instead
  }
  if (cd1_in && !cd2_in) {
    cd1_use = cd1_in;
    L->ck_exact = false;
  } else if (cd1_in && !L->has_cd_faults) {
    // read the producer's checksums in place; copied into the layer only if the
    // error path runs
    cd1_use = cd1_in;
    L->cd_ext1 = cd1_in;
    L->cd_ext2 = cd2_in;
    L->ck_exact = true;
  } else {
    if (cd1_in) {
      FTC_CUDA_CHECK(cudaMemcpyAsync(L->cd1, cd1_in, L->nCd * sizeof(double), cudaMemcpyDeviceToDevice, L->side));
      FTC_CUDA_CHECK(cudaMemcpyAsync(L->cd2, cd2_in, L->nCd * sizeof(double), cudaMemcpyDeviceToDevice, L->side));
      L->ck_exact = true;
    } else if (launch_cd1_fast(D, d.N, L->nCd, L->cd1, L->side) == FTC_OK) {
      L->ck_exact = false;
    } else {
      CK(launch_input_checksums(D, d.N, L->nCd, L->cd1, L->cd2, L->side));
      L->ck_exact = true;
    }
    if (L->has_cd_faults) {
      CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_CD1, L->cd1, true, L->scale_tab, d.C, d.H, d.H, L->nCd, L->side));
      if (L->ck_exact)
        CK(run_apply_faults(L->faults_dev, L->nfaults, FTC_FAULT_CD2, L->cd2, true, L->scale_tab, d.C, d.H, d.H, L->nCd, L->side));
    }
  }
  CK(launch_co5_sliced(cd1_use, L->cw1, L->co5f, d.C, d.H, d.R, d.stride, d.pad, L->E, L->side));
  FTC_CUDA_CHECK(cudaEventRecord(L->ev_ck, L->side));
  FTC_CUDA_CHECK(cudaStreamWaitEvent(s, L->ev_ck, 0));
  CK(launch_detect_so5(L->co5f, L->rowsum, L->rs_parts, d.N, L->E2, d.bias_enabled, L->agg, plan->tau,
                       L->fstats, L->fticket, L->fstats_hd, s));
  FTC_CUDA_CHECK(cudaEventRecord(L->ev_done, s));
  L->inflight = true;
  return FTC_OK;
}

int ftc_protected_conv_launch(ftc_layer* L, const ftc_plan* plan, const float* D, float* O,
                              const ftc_fault* faults, int32_t n_faults, void* stream) {
  return launch_impl(L, plan, D, O, nullptr, nullptr, faults, n_faults, stream);
}

int ftc_protected_conv_launch_cd1(ftc_layer* L, const ftc_plan* plan, const float* D, float* O,
                                  const double* cd1, const ftc_fault* faults, int32_t n_faults, void* stream) {
  if (!cd1) RET_ERR(FTC_INVALID_ARGUMENT, "null input checksum");
  return launch_impl(L, plan, D, O, cd1, nullptr, faults, n_faults, stream);
}

int ftc_protected_conv_launch_ck(ftc_layer* L, const ftc_plan* plan, const float* D, float* O,
                                 const double* cd1, const double* cd2, const ftc_fault* faults,
                                 int32_t n_faults, void* stream) {
  if (!cd1 || !cd2) RET_ERR(FTC_INVALID_ARGUMENT, "null input checksums");
  return launch_impl(L, plan, D, O, cd1, cd2, faults, n_faults, stream);
}

int ftc_protected_conv_finish(ftc_layer* L, ftc_layer_report* rep) {
  if (!L || !rep) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (!L->inflight) RET_ERR(FTC_INVALID_ARGUMENT, "no protected call in flight");
  L->inflight = false;
  std::memset(rep, 0, sizeof *rep);
  FTC_CUDA_CHECK(cudaEventSynchronize(L->ev_done));
  FTC_CUDA_CHECK(cudaGetLastError());
  const auto t1 = std::chrono::steady_clock::now();
  rep->t_detect_ms = std::chrono::duration<double, std::milli>(t1 - L->t0).count();
  {
    unsigned long long b = ((volatile DetectStats*)L->fstats_h)->max_rel_dev_bits;
    std::memcpy(&rep->max_rel_dev, &b, sizeof(double));
  }
  const int flagged = ((volatile DetectStats*)L->fstats_h)->flagged;
  rep->n_flagged = flagged;
  int st = FTC_OK;
  if (flagged == 0) {
    rep->detected = 0;
    rep->stage = FTC_STAGE_NONE;
  } else {
    st = error_path(L, rep);
  }
  rep->t_total_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - L->t0).count();
  return st;
}

int ftc_protected_conv_peek(ftc_layer* L, int32_t* flagged) {
  if (!L || !flagged) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (!L->inflight) RET_ERR(FTC_INVALID_ARGUMENT, "no protected call in flight");
  FTC_CUDA_CHECK(cudaEventSynchronize(L->ev_done));
  *flagged = ((volatile DetectStats*)L->fstats_h)->flagged;
  return FTC_OK;
}

int ftc_protected_check(ftc_layer* L, const ftc_plan* plan, const float* D, float* O,
                        ftc_layer_report* rep, void* stream) {
  if (!L || !plan || !D || !O || !rep) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (L->inflight) RET_ERR(FTC_INVALID_ARGUMENT, "a protected call is already in flight on this layer");
  cudaStream_t s = (cudaStream_t)stream;
  L->t0 = std::chrono::steady_clock::now();
  L->plan = *plan;
  L->D = D;
  L->Dconv = D;
  L->O = O;
  L->stream = s;
  L->Wcur = L->W;
  L->cw1 = L->cw1g;
  L->cw2 = L->cw2g;
  L->nfaults = 0;
  L->n_out_faults = 0;
  L->has_cd_faults = false;
  L->cd_ext1 = L->cd_ext2 = nullptr;
  std::memset(rep, 0, sizeof *rep);
  // exact input checksums; detection is the error path's exact CoC-D
  CK(launch_input_checksums(D, L->d.N, L->nCd, L->cd1, L->cd2, s));
  L->ck_exact = true;
  int st = error_path(L, rep);
  rep->t_total_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - L->t0).count();
  return st;
}

int ftc_protected_conv(ftc_layer* L, const ftc_plan* plan, const float* D, float* O,
                       const ftc_fault* faults, int32_t n_faults, ftc_layer_report* rep,
                       void* stream) {
  CK(ftc_protected_conv_launch(L, plan, D, O, faults, n_faults, stream));
  return ftc_protected_conv_finish(L, rep);
}

int ftc_layer_detect_record(ftc_layer* L, void* dst, void* stream) {
  if (!L || !dst) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (!L->inflight) RET_ERR(FTC_INVALID_ARGUMENT, "no protected call in flight");
  // stream-ordered after the detect kernel (side stream: ev_done), which published
  // {flagged, max_rel_dev} into the mapped record (device alias) before its grid completed
  FTC_CUDA_CHECK(cudaStreamWaitEvent((cudaStream_t)stream, L->ev_done, 0));
  FTC_CUDA_CHECK(cudaMemcpyAsync(dst, L->fstats_hd, sizeof(DetectStats), cudaMemcpyDeviceToDevice,
                                 (cudaStream_t)stream));
  return FTC_OK;
}

int ftc_protected_conv_cancel(ftc_layer* L) {
  if (!L) RET_ERR(FTC_INVALID_ARGUMENT, "null layer");
  if (!L->inflight) return FTC_OK;
  L->inflight = false;
  // the clean path re-arms its accumulators itself; only wait for it to drain
  FTC_CUDA_CHECK(cudaEventSynchronize(L->ev_done));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int ftc_isolated_scheme(ftc_layer* L, const ftc_plan* plan, const float* D, float* O, const ftc_fault* faults,
                        int32_t n_faults, int32_t scheme, int32_t* status, ftc_layer_report* rep, void* stream) {
  if (!L || !rep || !status) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  if (scheme < FTC_SCHEME_COC || scheme > FTC_SCHEME_FC) RET_ERR(FTC_CONFIG_ERROR, "scheme must be 1..4");
  CK(ftc_protected_conv_launch(L, plan, D, O, faults, n_faults, stream));
  L->inflight = false;
  std::memset(rep, 0, sizeof *rep);
  FTC_CUDA_CHECK(cudaEventSynchronize(L->ev_done));
  FTC_CUDA_CHECK(cudaGetLastError());
  const int flagged = ((volatile DetectStats*)L->fstats_h)->flagged;
  rep->n_flagged = flagged;
  *status = -1;
  if (flagged == 0) {
    rep->stage = FTC_STAGE_NONE;
    return FTC_OK;
  }
  return isolated_path(L, scheme, status, rep);
}

int ftc_protected_conv_host(ftc_layer* L, const ftc_plan* plan, const float* D_host, float* O_host,
                            const ftc_fault* faults, int32_t n_faults, ftc_layer_report* rep,
                            void* stream) {
  if (!L || !D_host || !O_host) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (!L->D_host_buf) CK(dalloc(&L->D_host_buf, L->nD));
  if (!L->O_host_buf) CK(dalloc(&L->O_host_buf, L->nO));
  FTC_CUDA_CHECK(cudaMemcpyAsync(L->D_host_buf, D_host, L->nD * sizeof(float), cudaMemcpyHostToDevice, s));
  int st = ftc_protected_conv(L, plan, L->D_host_buf, L->O_host_buf, faults, n_faults, rep, stream);
  if (st != FTC_OK && st != FTC_INTEGRITY_ERROR) return st;
  FTC_CUDA_CHECK(cudaMemcpyAsync(O_host, L->O_host_buf, L->nO * sizeof(float), cudaMemcpyDeviceToHost, s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(s));
  return st;
}

// ------------------------------------------------------------------ device memory
int ftc_device_alloc(size_t bytes, void** ptr) {
  if (!ptr) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  *ptr = nullptr;
  if (bytes == 0) return FTC_OK;
  FTC_CUDA_CHECK(cudaMalloc(ptr, bytes));
  return FTC_OK;
}

int ftc_device_free(void* ptr) {
  if (ptr) FTC_CUDA_CHECK(cudaFree(ptr));
  return FTC_OK;
}

int ftc_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream) {
  if (bytes == 0) return FTC_OK;
  if (!dst || !src) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  static const cudaMemcpyKind kinds[3] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                                          cudaMemcpyDeviceToDevice};
  if (kind < 0 || kind > 2) RET_ERR(FTC_INVALID_ARGUMENT, "kind must be 0 (h2d), 1 (d2h) or 2 (d2d)");
  cudaStream_t s = (cudaStream_t)stream;
  FTC_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, kinds[kind], s));
  FTC_CUDA_CHECK(cudaStreamSynchronize(s));
  return FTC_OK;
}

int ftc_memset_zero(void* dst, size_t bytes, void* stream) {
  if (bytes == 0) return FTC_OK;
  if (!dst) RET_ERR(FTC_INVALID_ARGUMENT, "null argument");
  FTC_CUDA_CHECK(cudaMemsetAsync(dst, 0, bytes, (cudaStream_t)stream));
  return FTC_OK;
}

// ------------------------------------------------------------------ building blocks
int ftc_input_checksums(const ftc_conv_desc* d, const float* D, double* cd1, double* cd2,
                        void* stream) {
  int E;
  CK(validate(d, &E));
  return launch_input_checksums(D, d->N, (long long)d->C * d->H * d->H, cd1, cd2,
                                (cudaStream_t)stream);
}

int ftc_kernel_checksums(const ftc_conv_desc* d, const float* W, double* cw1, double* cw2,
                         void* stream) {
  int E;
  CK(validate(d, &E));
  return launch_kernel_checksums(W, d->M, d->C / d->groups, d->R, d->groups, cw1, cw2,
                                 (cudaStream_t)stream);
}

int ftc_output_checksums(const ftc_conv_desc* d, uint32_t which, const float* D, const float* W,
                         const double* cd1, const double* cd2, const double* cw1,
                         const double* cw2, double* const co[7], void* stream) {
  int E;
  CK(validate(d, &E));
  if ((which & (FTC_CK_O3 | FTC_CK_O7)) && !cd2)
    RET_ERR(FTC_CONFIG_ERROR, "requested checksum needs Cd2 which is absent");
  if ((which & (FTC_CK_O4 | FTC_CK_O6)) && !cw2)
    RET_ERR(FTC_CONFIG_ERROR, "requested checksum needs Cw2 which is absent");
  cudaStream_t s = (cudaStream_t)stream;
  const int Ckw = d->C / d->groups, U = d->stride, p = d->pad;
  if (which & FTC_CK_O1) CK(launch_conv_f64_exact(cd1, true, W, false, co[0], 1, d->C, d->H, d->M, Ckw, d->R, U, p, d->groups, E, s));
  if (which & FTC_CK_O2) CK(launch_conv_f64_exact(D, false, cw1, true, co[1], d->N, d->C, d->H, 1, d->C, d->R, U, p, 1, E, s));
  if (which & FTC_CK_O3) CK(launch_conv_f64_exact(cd2, true, W, false, co[2], 1, d->C, d->H, d->M, Ckw, d->R, U, p, d->groups, E, s));
  if (which & FTC_CK_O4) CK(launch_conv_f64_exact(D, false, cw2, true, co[3], d->N, d->C, d->H, 1, d->C, d->R, U, p, 1, E, s));
  if (which & FTC_CK_O5) CK(launch_conv_f64_exact(cd1, true, cw1, true, co[4], 1, d->C, d->H, 1, d->C, d->R, U, p, 1, E, s));
  if (which & FTC_CK_O6) CK(launch_conv_f64_exact(cd1, true, cw2, true, co[5], 1, d->C, d->H, 1, d->C, d->R, U, p, 1, E, s));
  if (which & FTC_CK_O7) CK(launch_conv_f64_exact(cd2, true, cw1, true, co[6], 1, d->C, d->H, 1, d->C, d->R, U, p, 1, E, s));
  return FTC_OK;
}

int ftc_output_summations(int32_t N, int32_t M, int32_t E, const float* O, uint32_t which,
                          const float* bias, double* const so[7], void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* agg = nullptr;
  if (bias) {
    CK(dalloc(&agg, 2));
    CK(launch_bias_aggregates(bias, M, agg, s));
  }
  VirtualO v{O, nullptr, nullptr};
  int st = launch_output_summations(v, N, M, E, which, bias, agg, so, s);
  if (agg) {
    cudaStreamSynchronize(s);
    cudaFree(agg);
  }
  return st;
}

int ftc_detect_coc_d(const double* co5, const double* so5, int32_t E2, double tau, uint8_t* mask,
                     int32_t* clean, double* max_rel_dev, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  DetectStats* st = nullptr;
  CK(dalloc(&st, 1));
  cudaMemsetAsync(st, 0, sizeof(DetectStats), s);
  int r = launch_detect_exact(co5, so5, E2, tau, mask, st, s);
  DetectStats h{};
  if (r == FTC_OK) {
    cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  }
  cudaFree(st);
  if (r != FTC_OK) return r;
  if (clean) *clean = h.flagged == 0;
  if (max_rel_dev) std::memcpy(max_rel_dev, &h.max_rel_dev_bits, sizeof(double));
  return FTC_OK;
}

int ftc_verify_kernel(const ftc_conv_desc* d, const float* W, const double* cw1_ref, double tau,
                      int32_t* ok, void* stream) {
  int E;
  CK(validate(d, &E));
  cudaStream_t s = (cudaStream_t)stream;
  const long long nCw = (long long)d->C * d->R * d->R;
  double *cw1 = nullptr, *cw2 = nullptr;
  int32_t* cnt = nullptr;
  CK(dalloc(&cw1, nCw));
  CK(dalloc(&cw2, nCw));
  CK(dalloc(&cnt, 1));
  cudaMemsetAsync(cnt, 0, sizeof(int32_t), s);
  int r = launch_kernel_checksums(W, d->M, d->C / d->groups, d->R, d->groups, cw1, cw2, s);
  if (r == FTC_OK) r = launch_count_differ(cw1, cw1_ref, nCw, tau, cnt, s);
  int32_t h = 0;
  if (r == FTC_OK) {
    cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  }
  cudaFree(cw1);
  cudaFree(cw2);
  cudaFree(cnt);
  if (r != FTC_OK) return r;
  if (ok) *ok = h == 0;
  return FTC_OK;
}

}  // extern "C"
