/*
 * ftc_abi.h -- C ABI of the B200-native ABFT-protected convolution
 * (FT-CNN, arXiv 2003.12203).  Implemented by paper_2003_12203_b200/libftconv_b200.so.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference is a
 * header-only C++20 library (proj/core/include/ftconv/); its API works on host
 * Tensor4<T> objects and throws C++ exceptions.  Each entry point below replaces
 * one reference interface (cited file:line, relative to proj/core/include/ftconv/)
 * with plain pointers/sizes and a status code.  The C++ host API in
 * include/ftconv_b200/ftconv.hpp restores the reference's names, Tensor4 values
 * and exception semantics on top of this ABI.
 *
 * Memory: unless a function name ends in `_host`, every tensor pointer is a
 * DEVICE pointer owned by the caller.  Tensors are dense NCHW, last dimension
 * fastest (tensor.hpp:17-33): D is N x C x H x H, W is M x (C/groups) x R x R,
 * O is N x M x E x E with E = (H + 2*pad - R)/stride + 1 (tensor.hpp:100-107).
 * Checksums/summations are FP64 (the reference workflow at T=double).
 *
 * Streams: `stream` is a cudaStream_t passed as void*; NULL = legacy default stream.
 * One protected layer may be in flight per layer handle.
 *
 * Errors: status codes map 1:1 to the reference exceptions (errors.hpp:9-27);
 * ftc_last_error() returns the message of the calling thread's last failure.
 */
#ifndef FTC_ABI_H
#define FTC_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTC_ABI_VERSION 1
#define FTC_MAX_BLOCKS 4096
#define FTC_MAX_STAGES 8

/* errors.hpp:9-27 */
typedef enum ftc_status {
  FTC_OK = 0,
  FTC_SHAPE_ERROR = 1,     /* ShapeError */
  FTC_CONFIG_ERROR = 2,    /* ConfigError */
  FTC_IO_ERROR = 3,        /* IoError */
  FTC_INTEGRITY_ERROR = 4, /* IntegrityError: recompute failed twice (workflow.hpp:338) */
  FTC_CUDA_ERROR = 5,      /* device/runtime failure (no reference counterpart) */
  FTC_INVALID_ARGUMENT = 6
} ftc_status;

/* CkSel, checksums.hpp:14-23 */
enum {
  FTC_CK_O1 = 1u << 0, FTC_CK_O2 = 1u << 1, FTC_CK_O3 = 1u << 2, FTC_CK_O4 = 1u << 3,
  FTC_CK_O5 = 1u << 4, FTC_CK_O6 = 1u << 5, FTC_CK_O7 = 1u << 6, FTC_CK_ALL = 0x7f
};

/* ResolveStage, report.hpp:12-21 */
typedef enum ftc_stage {
  FTC_STAGE_NONE = 0, FTC_STAGE_RELOAD, FTC_STAGE_COC, FTC_STAGE_RC, FTC_STAGE_CLC,
  FTC_STAGE_FC, FTC_STAGE_DISCARD, FTC_STAGE_RECOMPUTE
} ftc_stage;

/* Layer geometry: Tensor4 shapes + ConvParams (tensor.hpp:92-97). */
typedef struct ftc_conv_desc {
  int32_t N;      /* batch (block rows) */
  int32_t C;      /* input channels Ch */
  int32_t H;      /* input side (square) */
  int32_t M;      /* kernels (block columns) */
  int32_t R;      /* kernel side (square) */
  int32_t stride; /* U */
  int32_t pad;
  int32_t groups;
  int32_t bias_enabled;
} ftc_conv_desc;

/* LayerPlan, workflow.hpp:23-29 */
typedef struct ftc_plan {
  int32_t rc_enabled;
  int32_t clc_enabled;
  double tau;
  double t0, t1, t2, p_r;
} ftc_plan;

/* Fault injection.  std::function FaultHooks (workflow.hpp:117-121) cannot cross
 * an ABI or run on a device; they become a POD list (fault.hpp:42-53, 111-172):
 *   target OUTPUT  = post_conv: applied inside the conv epilogue, before O is
 *                    stored and before the fused summations read it;
 *   target FMAP/KERNEL/CD1/CD2/CW1/CW2 = pre_conv: applied to the layer's working
 *                    copies after the input checksums were taken.
 * Coordinates: OUTPUT (n, m, x, y); FMAP (n, c=m, x, y); KERNEL (m=n, c=m, i=x, j=y)
 * i.e. index = ((n*d1 + m)*d2 + x)*d3 + y of the target tensor; the CD1/CD2/CW1/CW2
 * targets use n = 0.
 * A negative coordinate means "all" along that axis (output_block/row/column).
 * Modes: BITFLIP flips bit (bit % 31) of the FP32 word (fault.hpp:82-87; on the
 * FP64 checksums bit % 63); ADD adds value + n_coef*n + m_coef*m; SET stores value;
 * SCALE is the reference's `perturb` (fault.hpp:72-80): v += T(mag_k * max(1, |v|)),
 * mag_k = 0.5 + 1.5 * u_k with u_k the k-th uniform_real_distribution<double>(0, 1)
 * draw of mt19937_64(seed), k = the element's row-major index over the fault's "all"
 * (negative) axes -- make_hooks' iteration order (fault.hpp:111-172). */
typedef enum ftc_fault_target {
  FTC_FAULT_OUTPUT = 0, FTC_FAULT_FMAP = 1, FTC_FAULT_KERNEL = 2,
  FTC_FAULT_CD1 = 3, FTC_FAULT_CD2 = 4, FTC_FAULT_CW1 = 5, FTC_FAULT_CW2 = 6
} ftc_fault_target;
typedef enum ftc_fault_mode {
  FTC_FAULT_BITFLIP = 0, FTC_FAULT_ADD = 1, FTC_FAULT_SET = 2, FTC_FAULT_SCALE = 3
} ftc_fault_mode;
typedef struct ftc_fault {
  int32_t target;
  int32_t mode;
  int32_t n, m, x, y;
  uint32_t bit;
  float value;
  float n_coef, m_coef;
  uint64_t seed;  /* SCALE: the FaultSpec seed (fault.hpp:53) */
} ftc_fault;

/* LayerReport, report.hpp:38-47, as POD (fixed-capacity vectors). */
typedef struct ftc_layer_report {
  int32_t detected;
  int32_t stage;            /* ftc_stage */
  int32_t weights_reloaded;
  int32_t recomputed;
  int32_t n_blocks;         /* total corrected blocks; first FTC_MAX_BLOCKS listed */
  int32_t blocks[FTC_MAX_BLOCKS][2]; /* (i, j) = (n, m), ascending */
  int32_t n_stages;
  int32_t stages[FTC_MAX_STAGES];    /* stages_attempted */
  double max_rel_dev;       /* DetectionResult::max_rel_dev (schemes.hpp:21) of CoC-D */
  int32_t n_flagged;        /* CoC-D mismatching positions */
  int32_t repaired_planes;  /* (n,m) planes recomputed on device */
  double t_detect_ms;       /* host-measured wall time of the clean path */
  double t_total_ms;        /* host-measured wall time including the error path */
} ftc_layer_report;

typedef struct ftc_layer ftc_layer;

/* ---------------------------------------------------------------- library */
int32_t ftc_abi_version(void);
const char* ftc_last_error(void);
/* Device conv engine: 0 = tcgen05 3xTF32 implicit GEMM (default), 1 = FP32 SIMT
 * direct conv.  Both are hand-written sm_100a kernels; there is no CPU path. */
int ftc_set_conv_engine(int engine);
int ftc_get_conv_engine(void);

/* output_extent, tensor.hpp:100-107 (ConfigError unless integral) */
int ftc_output_extent(int32_t H, int32_t R, int32_t pad, int32_t stride, int32_t* E);

/* ---------------------------------------------------------------- layer */
/* build_model's per-layer work (model.hpp:77-108): validates shapes
 * (conv.hpp:16-26), uploads the golden W and bias, precomputes the golden kernel
 * checksums Cw1/Cw2 on device (model.hpp:104, checksums.hpp:70-88) and the packed
 * tensor-core operands.  W_host/bias_host are HOST pointers (bias may be NULL). */
int ftc_layer_create(const ftc_conv_desc* desc, const float* W_host, const float* bias_host,
                     ftc_layer** out);
int ftc_layer_destroy(ftc_layer* layer);
int ftc_layer_extent(const ftc_layer* layer, int32_t* E);
/* the geometry the layer was created with */
int ftc_layer_desc(const ftc_layer* layer, ftc_conv_desc* desc);

/* conv_forward(D, W, bias, p) (conv.hpp:114-131) with the layer's golden W. */
int ftc_conv_forward(ftc_layer* layer, const float* D, float* O, void* stream);

/* conv_forward with HOST D and O (copies on `stream`, blocking). */
int ftc_conv_forward_host(ftc_layer* layer, const float* D_host, float* O_host, void* stream);

/* run_protected_layer (workflow.hpp:141-339): CoC-D detection; on a mismatch
 * kernel verify/reload, CoC -> [RC] -> [ClC] -> FC -> recompute, all evaluated on
 * device, and the corrected (n,m) planes recomputed on device.  Blocks until the
 * report is final.  Returns FTC_INTEGRITY_ERROR when recompute fails twice. */
int ftc_protected_conv(ftc_layer* layer, const ftc_plan* plan, const float* D, float* O,
                       const ftc_fault* faults, int32_t n_faults, ftc_layer_report* report,
                       void* stream);

/* run_protected_layer for an output computed elsewhere: O (device, N x M x E x E)
 * plays the role of the post_conv hook's output (workflow.hpp:158-160); detection,
 * the escalation chain and the repair run exactly as in ftc_protected_conv (repair
 * rewrites the corrected planes of O from D; recompute rewrites all of O). */
int ftc_protected_check(ftc_layer* layer, const ftc_plan* plan, const float* D, float* O,
                        ftc_layer_report* report, void* stream);

/* Same as ftc_protected_conv with HOST input/output buffers (the reference's own
 * calling convention: run_protected_layer takes and returns host tensors).  The
 * host<->device copies run on `stream`. */
int ftc_protected_conv_host(ftc_layer* layer, const ftc_plan* plan, const float* D_host,
                            float* O_host, const ftc_fault* faults, int32_t n_faults,
                            ftc_layer_report* report, void* stream);

/* Split form for pipelines: _launch enqueues the clean path (checksums, conv with
 * fused summations, CoC-D) without blocking; _finish waits for it, runs the error
 * path if CoC-D fired and fills the report.  Between the two calls D and O must
 * stay valid. */
int ftc_protected_conv_launch(ftc_layer* layer, const ftc_plan* plan, const float* D, float* O,
                              const ftc_fault* faults, int32_t n_faults, void* stream);
int ftc_protected_conv_finish(ftc_layer* layer, ftc_layer_report* report);
/* Waits for the clean path of the call in flight and returns its CoC-D screen count
 * (*flagged > 0: _finish will run the error path, which reads D in NCHW) without ending
 * the call: a pipeline that skipped the NCHW copy of D (ftc_glue_nchw_optional)
 * materialises it first. */
int ftc_protected_conv_peek(ftc_layer* layer, int32_t* flagged);
/* Abandon the call in flight (a pipeline replays it on repaired input): waits for the
 * clean path to drain and drops its verdict without running the error path. */
int ftc_protected_conv_cancel(ftc_layer* layer);
/* Stream-ordered copy of the in-flight call's clean-path CoC-D record into device
 * memory `dst` (16 bytes: int32 flagged positions, int32 pad, float64 max_rel_dev):
 * lets a multi-GPU pipeline all-gather the per-layer detection records on the device
 * (NCCL) without a host round trip; the full LayerReport still comes from _finish. */
int ftc_layer_detect_record(ftc_layer* layer, void* dst, void* stream);

/* One correcting scheme in isolation -- the reference's acceptance criterion C4
 * (proj/tests/acceptance.cpp:207-292, isolation_succeeds): the clean path and the
 * detection + verify_kernel/reload preamble of run_protected_layer, then ONLY `scheme`
 * (FTC_SCHEME_COC/RC/CLC/FC) with a Co5-only verifier (:247-251) and no CoC probes.
 * *status: -1 settled by the preamble (clean, or clean after a reload), 0 corrected
 * (the corrected (n,m) planes are recomputed in O; report->corrected_blocks lists them),
 * 1 discard (checksum corruption), 2 escalate (O holds the unrepaired output). */
enum { FTC_SCHEME_COC = 1, FTC_SCHEME_RC = 2, FTC_SCHEME_CLC = 3, FTC_SCHEME_FC = 4 };
int ftc_isolated_scheme(ftc_layer* layer, const ftc_plan* plan, const float* D, float* O,
                        const ftc_fault* faults, int32_t n_faults, int32_t scheme, int32_t* status,
                        ftc_layer_report* report, void* stream);

/* _launch with the input checksums supplied by the producer of D: cd1/cd2 are
 * device FP64 C*H*H tensors holding sum_n D_n and sum_n n*D_n in ascending n
 * (checksums.hpp:100-107), e.g. fused into the previous layer's glue kernel
 * (ftc_glue_act_pool_ck).  Saves the input-checksum pass over D. */
int ftc_protected_conv_launch_ck(ftc_layer* layer, const ftc_plan* plan, const float* D, float* O,
                                 const double* cd1, const double* cd2, const ftc_fault* faults,
                                 int32_t n_faults, void* stream);
/* _launch with only the clean-path input checksum supplied by the producer of D:
 * cd1 = sum_n D_n in FP64 in any order (ftc_glue_act_pool_cd1 writes it at the
 * start of its workspace).  CoC-D needs nothing else; the exact-order Cd1/Cd2
 * (checksums.hpp:100-107) are recomputed from D only if CoC-D fires. */
int ftc_protected_conv_launch_cd1(ftc_layer* layer, const ftc_plan* plan, const float* D, float* O,
                                  const double* cd1, const ftc_fault* faults, int32_t n_faults,
                                  void* stream);

/* ---- Fault campaigns (fault.hpp:42-291, replay.hpp) -------------------------------
 * FaultSpec as POD.  target: 0 output_block, 1 output_row, 2 output_column, 3 fmap,
 * 4 kernel, 5 checksum; checksum: 0 none, 1 cd1, 2 cd2, 3 cw1, 4 cw2; x/y = -1: all;
 * mode: 0 scale (additive perturbation from `seed`), 1 bitflip (`bit`). */
typedef struct ftc_fault_spec {
  int32_t layer_index;
  int32_t target;
  int32_t checksum;
  int32_t mode;
  int64_t i, j;
  int64_t x, y;
  uint32_t bit;
  uint32_t pad_;
  uint64_t seed;
} ftc_fault_spec;
typedef struct ftc_ground_truth {
  int32_t benign;
  int32_t expected_stage; /* ftc_stage */
  int32_t output_diverges;
} ftc_ground_truth;
typedef struct ftc_layer_grid {
  int64_t N, M, Ch, H, R; /* LayerGrid (fault.hpp:191-193) */
} ftc_layer_grid;

/* campaign(layers, n_runs, weights, seed) (fault.hpp:195-271): the reproducible corpus,
 * bit-identical to the reference's (same generator and distributions); weights over
 * {output_block, output_row, output_column, fmap, kernel, checksum}. */
int ftc_campaign(const ftc_layer_grid* layers, int32_t n_layers, int64_t n_runs, const double* weights6,
                 uint64_t seed, ftc_fault_spec* specs, ftc_ground_truth* truths);
/* ground_truth(f, N, M) (fault.hpp:174-211) */
int ftc_ground_truth_of(const ftc_fault_spec* spec, int64_t N, int64_t M, ftc_ground_truth* out);
/* make_hooks(f) (fault.hpp:111-172) as device fault records (at most 1) */
int ftc_spec_faults(const ftc_fault_spec* spec, ftc_fault* out, int32_t* n_out);
/* conv_forward of a run the faults hit (pre_conv + post_conv), no ABFT: what a fault
 * does to an unprotected run (replay_entry's above-threshold test, replay.hpp:84-101) */
int ftc_conv_forward_faulted(ftc_layer* layer, const float* D, float* O, const ftc_fault* faults,
                             int32_t n_faults, void* stream);

/* ---- Layer plans (workflow.hpp:19-112, 428-501) ------------------------------------ */
typedef struct ftc_layer_dims {
  int64_t N, M, Ch, H, R, E; /* LayerDims (workflow.hpp:38-40) */
} ftc_layer_dims;
typedef struct ftc_plan_info {  /* LayerPlan with its profiled runtimes (workflow.hpp:22-28) */
  int32_t rc_enabled, clc_enabled;
  double tau;
  double t0, t1, t2; /* CoC+FC, CoC+RC, CoC+RC+FC */
  double p_r;
} ftc_plan_info;
typedef struct ftc_profile_result {  /* ProfileResult (workflow.hpp:423-427) */
  double rc_t0, rc_t1, rc_t2;
  double clc_t0, clc_t1, clc_t2;
  int32_t used_cost_model;
} ftc_profile_result;
/* scheme: 0 coc_d, 1 coc, 2 rc, 3 clc, 4 fc (schemes.hpp:15) */
double ftc_cost_model(int32_t scheme, const ftc_layer_dims* dims, double alpha, double beta);
int32_t ftc_decide_rc(double t0, double t1, double t2, double p_r, double p_c);
int32_t ftc_decide_clc(double t0, double t1, double t2, double p_r, double p_c);
void ftc_estimate_error_probs(const ftc_layer_dims* dims, double* p_r, double* p_c);
/* make_default_plan(dims, tau, {alpha, beta}) (workflow.hpp:99-112) */
int ftc_make_default_plan(const ftc_layer_dims* dims, double tau, double alpha, double beta, ftc_plan_info* out);
/* profile_layer (workflow.hpp:428-501) on the device path: the protected layer timed
 * (host wall clock, median of `reps`) under the six forced-fault variants -- a row fault
 * O(1,m,.,.) += 3 + m and a column fault O(n,1,.,.) += 3 + n -- falling back to the
 * cost model for degenerate layers (N < 2 or M < 2) or non-positive times. */
int ftc_profile_layer(ftc_layer* layer, const float* D, double tau, int32_t reps, ftc_profile_result* out,
                      void* stream);

/* ---------------------------------------------------------------- back-propagation
 * conv_backward (conv.hpp:150-185) and run_protected_backward (workflow.hpp:340-417).
 * D (N,C,H,H), W (M,C,R,R), dO (N,M,E,E) device FP32; dW (M,C,R,R), dD (N,C,H,H)
 * device FP32 outputs.  Gradients accumulate in FP64; the protection checks the FP64
 * gradients (sum_m dW vs conv_backward(D, 0, sum_m dO).dW, sum_n dD vs
 * conv_backward(0, W, sum_n dO).dD, values_differ(tau)), recomputes once on a
 * mismatch and returns FTC_INTEGRITY_ERROR if the recompute fails too; outputs are the
 * checked gradients rounded to FP32.  groups != 1 or bias -> FTC_CONFIG_ERROR. */
typedef struct ftc_grad_fault {  /* the reference's post_hook as a substitution */
  int32_t target;                /* 0 dW, 1 dD */
  int32_t mode;                  /* 0 set, 1 add */
  int64_t index;                 /* flat NCHW index */
  double value;
} ftc_grad_fault;
typedef struct ftc_backward_report {  /* BackwardReport (workflow.hpp:343-347) */
  int32_t dw_detected, dd_detected, recomputed;
} ftc_backward_report;
int ftc_conv_backward(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO, float* dW,
                      float* dD, void* stream);
/* hook faults apply to the first pass only, like the reference's post_hook */
int ftc_protected_backward(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO, double tau,
                           const ftc_grad_fault* hook, int32_t n_hook, float* dW, float* dD,
                           ftc_backward_report* report, void* stream);

/* host-buffer forms of the two (copies in, device pass, copies out; synchronous) */
int ftc_conv_backward_host(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO, float* dW,
                           float* dD, void* stream);
int ftc_protected_backward_host(const ftc_conv_desc* desc, const float* D, const float* W, const float* dO,
                                double tau, const ftc_grad_fault* hook, int32_t n_hook, float* dW, float* dD,
                                ftc_backward_report* report, void* stream);

/* Seeded uniform draws exactly as Tensor4<T>::random (tensor.hpp:57-66) and
 * random_weights (model_io.cpp:176-192): std::mt19937_64(seed) through
 * std::uniform_real_distribution<double>(lo, hi), n values into out (host memory). */
int ftc_mt64_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out);

/* Channel-last input staging for the TMA im2col engine (C % 32 == 0 layers): the layer
 * keeps an NHWC copy of its input that every launch refreshes from D.  A producer that
 * already wrote D in NHWC form into that buffer (ftc_glue_act_pool_nhwc) calls
 * _input_nhwc_ready so the next launch (protected or not) skips the refresh; D itself
 * must still hold the same values in NCHW (checksums, error path).  *nhwc = NULL when
 * the layer's engine does not stage its input. */
int ftc_layer_input_nhwc(ftc_layer* layer, float** nhwc);
int ftc_layer_input_nhwc_ready(ftc_layer* layer, const float* D);

/* Instrumentation for bench.py: when enabled, CUDA events bracket the conv kernel
 * of every protected/unprotected call on its launching stream; _kernel_time
 * returns the accumulated device time (ms) and launch count (reset if `reset`).
 * ftc_kernel_launches counts every kernel this library has launched. */
int ftc_layer_set_timing(ftc_layer* layer, int32_t enable);
int ftc_layer_kernel_time(ftc_layer* layer, double* conv_ms, int32_t* conv_launches,
                          int32_t reset);
uint64_t ftc_kernel_launches(void);

/* ---------------------------------------------------------------- device memory
 * For hosts that do not link the CUDA runtime themselves (the C++ wrappers in
 * include/ftconv_b200/, a cgo/JNI/ctypes binding): device allocations and copies
 * through the library's own runtime.  kind: 0 host->device, 1 device->host,
 * 2 device->device; the copy is ordered on `stream` and complete on return. */
int ftc_device_alloc(size_t bytes, void** ptr);
int ftc_device_free(void* ptr);
int ftc_memcpy(void* dst, const void* src, size_t bytes, int32_t kind, void* stream);
int ftc_memset_zero(void* dst, size_t bytes, void* stream);

/* ---------------------------------------------------------------- building blocks
 * Device implementations of checksums.hpp / schemes.hpp primitives, FP64,
 * summed in the reference's association order (bitwise equal to the reference at
 * T=double on the same FP32 data).  All pointers are device pointers. */

/* input_checksums (checksums.hpp:91-113): Cd1 = sum_n D_n, Cd2 = sum_n n*D_n, C*H*H each */
int ftc_input_checksums(const ftc_conv_desc* desc, const float* D, double* cd1, double* cd2,
                        void* stream);
/* kernel_checksums (checksums.hpp:70-88): C*R*R each (groups concatenated) */
int ftc_kernel_checksums(const ftc_conv_desc* desc, const float* W, double* cw1, double* cw2,
                         void* stream);
/* output_checksums (checksums.hpp:134-161).  co[k] receives Co(k+1) when bit k of
 * `which` is set: Co1,Co3 are M grids, Co2,Co4 N grids, Co5..7 one E x E grid. */
int ftc_output_checksums(const ftc_conv_desc* desc, uint32_t which, const float* D, const float* W,
                         const double* cd1, const double* cd2, const double* cw1,
                         const double* cw2, double* const co[7], void* stream);
/* output_summations (checksums.hpp:165-190) + BiasAdjuster (:195-245) if bias != NULL */
int ftc_output_summations(int32_t N, int32_t M, int32_t E, const float* O, uint32_t which,
                          const float* bias, double* const so[7], void* stream);
/* detect_coc_d (schemes.hpp:79-94): writes the E2-byte mismatch mask (may be NULL) and
 * returns clean / max_rel_dev through HOST pointers (synchronises `stream`). */
int ftc_detect_coc_d(const double* co5, const double* so5, int32_t E2, double tau, uint8_t* mask,
                     int32_t* clean, double* max_rel_dev, void* stream);
/* verify_kernel (checksums.hpp:250-259); result through a HOST pointer. */
int ftc_verify_kernel(const ftc_conv_desc* desc, const float* W, const double* cw1_ref, double tau,
                      int32_t* ok, void* stream);

/* ---------------------------------------------------------------- net glue
 * Not reference interfaces: the reference chains convs directly (replay.hpp:14-25)
 * and has no activation/pooling/residual ops; the BASELINE conv stacks need them
 * between protected layers.  act: 0 none, 1 ReLU, 2 leaky-ReLU(0.1). */
/* out = maxpool_{k,s,p}(act(in)); k = s = 1, p = 0 is a plain activation.  With
 * in == out == NULL only the output side is returned in *Ho. */
int ftc_glue_act_pool(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t act,
                      int32_t k, int32_t s, int32_t p, int32_t* Ho, void* stream);
/* ftc_glue_act_pool that also reduces its output over the batch for the NEXT
 * protected layer: cd1 = sum_n out_n, cd2 = sum_n n*out_n (FP64, ascending n, i.e.
 * input_checksums of `out` exactly, checksums.hpp:100-107). */
int ftc_glue_act_pool_ck(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t act,
                         int32_t k, int32_t s, int32_t p, double* cd1, double* cd2, void* stream);
/* ftc_glue_act_pool(_ck) that also writes its output channel-last into out_nhwc
 * (N, Ho*Ho, C) for the next layer's TMA im2col staging (C % 32 == 0); cd1/cd2 may
 * be NULL (no checksums). */
int ftc_glue_act_pool_nhwc(const float* in, float* out, float* out_nhwc, int32_t N, int32_t C, int32_t H,
                           int32_t act, int32_t k, int32_t s, int32_t p, double* cd1, double* cd2,
                           void* stream);
/* ftc_glue_act_pool(_nhwc) that also writes, with ws != NULL, the next protected
 * layer's clean-path Cd1 = sum_n out_n (FP64, any order) into ws[0 : C*Ho*Ho] -- pass
 * ws to ftc_protected_conv_launch_cd1.  ws holds ftc_glue_ws_doubles(...) doubles
 * (Cd1, per-image-group partial slabs, tickets) and must be zero-filled once before
 * first use; the kernels leave it re-armed.  out_nhwc may be NULL. */
int64_t ftc_glue_ws_doubles(int32_t N, int32_t C, int32_t H, int32_t k, int32_t s, int32_t p);
int ftc_glue_act_pool_cd1(const float* in, float* out, float* out_nhwc, int32_t N, int32_t C, int32_t H,
                          int32_t act, int32_t k, int32_t s, int32_t p, double* ws, void* stream);
/* 1 when ftc_glue_act_pool_cd1 accepts out == NULL for this shape: the pass then writes
 * only the channel-last copy (and Cd1) -- the consumer's clean path reads nothing else,
 * saving 4 of the 12 bytes per element an activation pass moves.  The NCHW tensor is
 * needed again only by the consumer's error path (see ftc_protected_conv_peek). */
int32_t ftc_glue_nchw_optional(const float* in, int32_t C, int32_t H, int32_t k, int32_t s, int32_t p);
/* out = act(a + b) elementwise over n values (b may be NULL) */
int ftc_glue_add_act(const float* a, const float* b, float* out, int64_t n, int32_t act,
                     void* stream);
/* explicit zero pad of `lo` rows/cols at top/left and `hi` at bottom/right (hi < 0
 * crops): expresses floor-mode strided convs through the exact extent rule */
int ftc_glue_pad_crop(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t lo,
                      int32_t hi, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FTC_ABI_H */
