// ftc_common.cuh -- shared device helpers and internal kernel interfaces of the
// B200-native ABFT-protected convolution.  Reference paths are relative to
// /root/reference/proj/core/include/ftconv/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/ftc_abi.h"

namespace ftc {

// ------------------------------------------------------------------ errors
struct Error {
  int code;
  std::string msg;
};
void set_error(int code, const std::string& msg);
#define FTC_CUDA_CHECK(expr)                                                        \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::ftc::set_error(FTC_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
      return FTC_CUDA_ERROR;                                                        \
    }                                                                               \
  } while (0)

// every kernel launch of the library goes through FTC_LAUNCH so the launch
// counter (ftc_kernel_launches) sees it
void count_launch();
#define FTC_LAUNCH(...)     \
  do {                      \
    __VA_ARGS__;            \
    ::ftc::count_launch();  \
  } while (0)

// Programmatic dependent launch (sm_90+): the kernel may be scheduled while the previous
// kernel on the stream drains; it runs griddepcontrol.wait before touching memory the
// previous kernel produced.  Off with FTC_NO_PDL=1 (A/B experiments).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
#define FTC_LAUNCH_PDL(kernel, grid, block, smem, stream, ...)                        \
  do {                                                                                 \
    FTC_CUDA_CHECK(::ftc::launch_pdl(kernel, grid, block, smem, stream, __VA_ARGS__)); \
    ::ftc::count_launch();                                                             \
  } while (0)

// device side of PDL: wait for the previous grid's completion (and memory), and let the
// next grid launch (no-ops without the launch attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------ device helpers
// FP64 arithmetic of the checksum path goes through the _rn intrinsics so nvcc can
// never contract a*b+c into an FMA: the association order AND the rounding of
// every product match the reference at T=double (x86-64 SSE2, no FMA).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// values_differ (checksums.hpp:54-60): |c-s| > tau*max(|c|,|s|,1) in double.
// Any NaN -> false; inf vs anything -> inf > tau*inf -> false.
__device__ __forceinline__ bool values_differ(double c, double s, double tau) {
  const double cc = fabs(c), ss = fabs(s);
  double m = cc;
  if (m < ss) m = ss;
  if (m < 1.0) m = 1.0;
  return fabs(dsub(c, s)) > dmul(tau, m);
}

// Clean-path CoC-D on any-order FP64 sums (fused Co5 / atomics-summed So5) flags with a
// guard band: |c-s| > (1 - kGuard)*tau*max(|c|,|s|,1).  Their deviation from the exact-
// order sums is bounded by ~n*2^-53*sum|x| (n <= 2^17 terms on the BASELINE layers),
// orders of magnitude below kGuard*tau*max(..); a position the reference would flag is
// therefore never read as clean, and anything inside the band goes to the error path,
// whose exact-order re-detection (detect_exact_clean) makes the verdict.  NaN/Inf
// behave as in values_differ.
constexpr double kGuard = 1e-3;
__device__ __forceinline__ bool values_differ_guarded(double c, double s, double tau) {
  const double cc = fabs(c), ss = fabs(s);
  double m = cc;
  if (m < ss) m = ss;
  if (m < 1.0) m = 1.0;
  return fabs(c - s) > (tau * (1.0 - kGuard)) * m;
}

// locate_index (schemes.hpp:57-62).  llround of non-finite/huge values is
// "integer indefinite" on x86 (-> rejected), reproduced by the range guard.
__device__ __forceinline__ bool locate_index(double r, int n, int* out) {
  if (!(fabs(r) < 4.0e18)) return false;
  const long long i = llround(r);
  if (fabs(dsub(r, (double)i)) > 0.01) return false;
  if (i < 0 || i >= (long long)n) return false;
  *out = (int)i;
  return true;
}

// flip_bit (fault.hpp:82-93): sign bit excluded
__device__ __forceinline__ float flip_bit_f32(float v, unsigned bit) {
  return __uint_as_float(__float_as_uint(v) ^ (1u << (bit % 31u)));
}

// Row-major index of element (a0..a3) over the fault's "all" (negative) axes, the
// iteration order of the reference's make_hooks loops (fault.hpp:111-172).
__device__ __forceinline__ long long fault_elem_index(const ftc_fault& f, int a0, int a1, int a2, int a3, int d1,
                                                      int d2, int d3) {
  long long k = 0;
  if (f.n < 0) k = a0;
  if (f.m < 0) k = k * d1 + a1;
  if (f.x < 0) k = k * d2 + a2;
  if (f.y < 0) k = k * d3 + a3;
  return k;
}

// the reference's perturb: v += T(mag * max(1, |v|)) (fault.hpp:76-80), exact roundings
__device__ __forceinline__ float scale_f32(float v, double mag) {
  return __fadd_rn(v, (float)__dmul_rn(mag, fmax(1.0, fabs((double)v))));
}
__device__ __forceinline__ double scale_f64(double v, double mag) {
  return __dadd_rn(v, __dmul_rn(mag, fmax(1.0, fabs(v))));
}

// post_conv fault applied to one output element (inside conv epilogues); tab holds the
// SCALE magnitudes (the device record's `bit` is its offset into tab)
__device__ __forceinline__ float apply_output_faults(float v, int n, int m, int x, int y, int M, int E,
                                                     const ftc_fault* f, int nf, const double* tab) {
  for (int q = 0; q < nf; ++q) {
    const ftc_fault& a = f[q];
    if (a.target != FTC_FAULT_OUTPUT) continue;
    if ((a.n >= 0 && a.n != n) || (a.m >= 0 && a.m != m) || (a.x >= 0 && a.x != x) ||
        (a.y >= 0 && a.y != y))
      continue;
    if (a.mode == FTC_FAULT_BITFLIP)
      v = flip_bit_f32(v, a.bit);
    else if (a.mode == FTC_FAULT_ADD)
      v = v + (a.value + a.n_coef * (float)n + a.m_coef * (float)m);
    else if (a.mode == FTC_FAULT_SCALE)
      v = scale_f32(v, tab[a.bit + fault_elem_index(a, n, m, x, y, M, E, E)]);
    else
      v = a.value;
  }
  return v;
}

// ------------------------------------------------------------------ conv engine
struct DetectStats {
  int32_t flagged;
  int32_t pad_;
  unsigned long long max_rel_dev_bits;
};

struct Co5Tap {  // one (c, i, j) term of Co5 = Cd1 (*) Cw1
  int off;         // c*H*H + i*H + j
  short i, j;
  double w;        // Cw1[c][i][j]
};

struct FusedDetect {
  double* co5;            // [E2]: written by the conv's checksum warp when cdp != null,
                          // else computed before the conv
  double* so5;            // [E2] accumulator: zero on entry, re-zeroed by the last CTA
  const double* agg;      // bias aggregates (agg[0] = sum_m B[m])
  double tau;
  int bias;
  DetectStats* st;        // device counters, zero on entry, re-zeroed
  unsigned int* ticket;   // zero on entry, re-zeroed
  DetectStats* host_out;  // mapped host record
  // in-kernel Co5 = Cd1 (*) Cw1 (tcgen05 engine, checksum warps), or null when co5 is
  // precomputed
  const double* cd1;      // [C][H][H]
  const Co5Tap* taps;     // [C*R*R] per-tap offsets and Cw1 values
};

struct ConvArgs {
  const float* D;  // N x C x H x H
  const float* W;  // M x Ckw x R x R (reference layout)
  const float* bias;  // M or null
  float* O;           // N x M x E x E
  int N, C, H, M, R, U, pad, groups, E, Ckw;
  const ftc_fault* faults;  // device list (post_conv OUTPUT faults), may be null
  int nfaults;
  const double* scale_tab;  // SCALE fault magnitudes (see apply_output_faults)
  double* rowsum;    // [N][E2] sum_m O (So2 before bias adjust), may be null
  double* rowsum_m;  // [N][E2] sum_m m*O (So4 before bias adjust), may be null
  const uint32_t* plane_mask;  // N*M bits: store only these planes (repair); null = all
  int img_lo, img_hi;          // images to compute
  const FusedDetect* fd;       // tcgen05 im2col engine only; null = detection runs outside
  bool dt_ready;               // tcgen05 im2col/NHWC engine: the NHWC copy is already filled
};

int conv_simt_launch(const ConvArgs& a, cudaStream_t s);

// tcgen05 engine: per-layer packed operands + launch
struct TcPlan;
int tc_plan_create(const ftc_conv_desc& d, const float* W_dev, TcPlan** out, cudaStream_t s);
void tc_plan_destroy(TcPlan* p);
bool tc_supported(const ftc_conv_desc& d);
int conv_tc_launch(const TcPlan* p, const ConvArgs& a, cudaStream_t s);
int tc_rowsum_parts(const TcPlan* p);
bool tc_im2col(const TcPlan* p);           // TMA im2col engine (fused detection available)
bool tc_co5_in_kernel(const TcPlan* p, int N, int E);  // fused path: Co5 by the conv's checksum warp
float* tc_nhwc_buffer(const TcPlan* p);    // its NHWC input copy
// D (NCHW) -> Dt (NHWC) for images [n_lo, n_lo + nimg); with cd1 != null also the exact
// input checksums Cd1/Cd2 (n ascending, FP64; whole batch only: n_lo = 0, nimg = N)
struct Co5Job {  // have the staging pass also produce Co5 = Cd1 (*) Cw1 (co5 zero on entry)
  double* co5;
  const double* cw1;
  int H, R, U, pad, E;
};
int launch_nhwc_cd(const float* D, float* Dt, int C, int HW, int n_lo, int nimg, double* cd1, double* cd2,
                   cudaStream_t s, const Co5Job* co5 = nullptr);  // N-tiles = row-sum partial slabs of N*E2

// ------------------------------------------------------------------ checksum kernels
// input_checksums (exact order)
int launch_input_checksums(const float* D, int N, long long per, double* cd1, double* cd2,
                           cudaStream_t s);
// kernel_checksums (exact order)
int launch_kernel_checksums(const float* W, int M, int Ckw, int R, int groups, double* cw1,
                            double* cw2, cudaStream_t s);
// exact-order FP64 conv: out[b][mo][x][y] = sum_{k,i,j} in[b][kbase+k] * w[mo][k][i][j]
//  in: float (D) or double (checksums); w: float (W) or double (Cw)
int launch_conv_f64_exact(const void* in, bool in_f64, const void* w, bool w_f64, double* out,
                          int B, int Cin, int H, int Mo, int Ckw, int R, int U, int pad,
                          int groups, int E, cudaStream_t s);
// conv_block (conv.hpp:135-145) of up to three (Cd, Cw) pairs at once (Co5 = Cd1*Cw1,
// Co6 = Cd1*Cw2, Co7 = Cd2*Cw1): one launch, the jobs side by side
int launch_conv_block3(const double* const in[3], const double* const w[3], double* const out[3], int nj, int Cin,
                       int H, int R, int U, int pad, int E, cudaStream_t s);
// bias aggregates: agg[0]=sum_b, agg[1]=sum_mb (BiasAdjuster ctor, checksums.hpp:199-208)
int launch_bias_aggregates(const float* bias, int M, double* agg, cudaStream_t s);

struct VirtualO {  // FP32 O plus FP64 overrides left by the verifier's rollbacks
  const float* O;
  const double* ov;        // N*M*E2 or null
  const uint8_t* present;  // N*M*E2 or null
};
// So5/So6/So7 in the reference's (n, m) order for the positions in list[0 : *count]
// (list == null: all E2 positions), written at their positions; agg: bias aggregates or null
int launch_seq_sums567(const VirtualO& v, int N, int M, int E2, const int* list, const int* count, const double* agg,
                       double* so5, double* so6, double* so7, cudaStream_t s);
// output_summations + BiasAdjuster (exact order)
int launch_output_summations(const VirtualO& v, int N, int M, int E, uint32_t which,
                             const float* bias, const double* agg, double* const so[7],
                             cudaStream_t s);
// clean path: Cd1 only, parallel over positions (FTC_CONFIG_ERROR when the plane size
// is odd -> caller uses the exact kernel)
int launch_cd1_fast(const float* D, int N, long long per, double* cd1, cudaStream_t s);
// clean path: Cd1 = sum_n D_n in FP64, any order, through a workspace [Cd1][tickets]
// [partial slabs over image groups] (zero-filled once; the kernels re-arm the tickets).
// The act+pool glue kernels write the next layer's Cd1 the same way.
int launch_detect_fused(double* co5, double* so5, int N, int E2, int bias, const double* agg, double tau,
                        DetectStats* st, unsigned int* ticket, DetectStats* host_out, cudaStream_t s);
int launch_co5_detect(const double* cd1, const double* cw1, double* co5, double* so5, int N, int C, int H, int R,
                      int U, int pad, int E, int bias, const double* agg, double tau, DetectStats* st,
                      unsigned int* ticket, DetectStats* host_out, cudaStream_t s);
int launch_co5_taps(const double* cw1, int C, int H, int R, Co5Tap* taps, cudaStream_t s);
long long cd1_ws_doubles(int N, long long per);
long long cd1_ws_doubles_g(int N, int C, int Ho, long long per);  // also covers the glue kernels' layout
// act + pool (k x k, stride s, pad p) with NHWC staging (out_t) and the consumer's Cd1 in
// ws; out (NCHW) may be NULL (staging pass of a caller-supplied D: act 0, k = s = 1)
int launch_act_pool_nhwc_cd1(const float* in, float* out, float* out_t, int N, int C, int H, int act, int k,
                             int s, int p, double* ws, cudaStream_t st);
// C, Ho: the pooling producer's shape when the workspace is shared with it (0, 0: none)
int launch_cd1_parts(const float* D, int N, long long per, double* ws, cudaStream_t s, int C = 0, int Ho = 0);
int launch_act_pool_nhwc(const float* in, float* out, float* out_t, int N, int C, int H, int act, int k, int s,
                         int p, cudaStream_t st);
// clean path: Co5 (adaptive positions x channel slices), then So5 from the fused row
// sums + compare; the last block publishes the record into mapped host memory
// (host_out) and re-zeroes st/ticket for the next call
int launch_co5_sliced(const double* cd1, const double* cw1, double* co5, int C, int H, int R, int U,
                      int pad, int E, cudaStream_t s);
int launch_detect_so5(double* co5, const double* rowsum, int parts, int N, int E2, int bias,
                      const double* agg, double tau, DetectStats* st, unsigned int* ticket,
                      DetectStats* host_out, cudaStream_t s);
int launch_detect_exact(const double* co5, const double* so5, int E2, double tau, uint8_t* mask,
                        DetectStats* st, cudaStream_t s);
int launch_count_differ(const double* c, const double* s_, long long n, double tau, int* count,
                        cudaStream_t s);

// ------------------------------------------------------------------ scheme kernels
struct SchemeResult {
  int32_t status;     // see SchemeStatus
  int32_t n_patches;
  int32_t line;       // located row/column/index
  int32_t invalid;
  int32_t lmin, lmax; // located-index range among flags
  int32_t any;
  int32_t fail;       // verifier failure flag
  int32_t nr, nc;     // FC: flagged row/column counts
  int32_t r0, c0;     // FC: the single flagged row/column
  int32_t m6, m7;     // CoC pattern flags
  int32_t c5bad;      // FC: Co5 inconsistent somewhere
  int32_t mode;       // patch source: 0 = column flags (row = line), 1 = row flags (col = line)
};
enum SchemeStatus {
  SCH_VALID = 0,      // patches emitted, verifier pending
  SCH_DISCARD = 1,
  SCH_ESCALATE = 2,
  SCH_EMPTY = 3,      // corrected with no blocks
  SCH_PROBE_ROW0 = 4, // CoC pattern m6 && !m7
  SCH_PROBE_COL0 = 5, // CoC pattern m7 && !m6
};
struct Patches {
  int32_t* n;
  int32_t* m;
  int32_t* f;
  double* d;
  int32_t cap;
};
struct Fam {  // the 7 families (checksums c, summations s); null if absent
  const double* c[7];
  const double* s[7];
};
int run_coc_analyze(const Fam& F, int N, int M, int E2, double tau, SchemeResult* r,
                    const Patches& p, cudaStream_t s);
int run_line_analyze(const Fam& F, bool rc, int N, int M, int E2, double tau, SchemeResult* r,
                     const Patches& p, cudaStream_t s);
int run_fc_analyze(const Fam& F, int N, int M, int E2, double tau, SchemeResult* r,
                   const Patches& p, uint8_t* colmask, uint8_t* rowmask, int32_t* colany,
                   int32_t* rowany, cudaStream_t s);

struct VerifyWS {
  double* ov;
  uint8_t* present;
  uint8_t* touched5;  // E2
  uint8_t* touched1;  // M*E2
  double* fresh;      // 3*E2: fresh So5/So6/So7 of the touched positions
  int* tlist;         // E2: the touched positions
  int* tcount;        // 1
};
// workflow.hpp:205-219 verifier emulated over the patch list (see ftc_schemes.cu)
int run_verify(const Fam& F, unsigned trusted, const float* O, int N, int M, int E2, int bias,
               const float* bias_dev, const double* agg, double tau, const Patches& p,
               const SchemeResult* r_dev, int np_host, const VerifyWS& ws, int32_t* fail,
               cudaStream_t s);
// rollback (schemes.hpp:71-74) in the FP64 override map, then clear the touch marks
int run_rollback(const Patches& p, int np_host, int M, int E2, const VerifyWS& ws, cudaStream_t s);
// plane mask (N*M bits) from the patch list
int run_patch_planes(const Patches& p, int np_host, int M, uint32_t* mask, cudaStream_t s);
// pre_conv faults on a float or double target
int run_apply_faults(const ftc_fault* f_dev, int nf, int target, void* t, bool is_f64, const double* tab, int d1,
                     int d2, int d3, long long count, cudaStream_t s);

}  // namespace ftc
