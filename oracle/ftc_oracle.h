/*
 * ftc_oracle.h -- CPU restatement of the reference's ABFT-protected convolution
 * path (FT-CNN, arXiv 2003.12203; reference at proj/core/include/ftconv/).
 *
 * TEST INFRASTRUCTURE ONLY.  This oracle is the checker the GPU path is judged
 * against.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it.  It is never linked into, called by, or used as a fallback for the
 * product library (paper_2003_12203_b200/libftconv_b200.so).
 *
 * Parity pin: every function here is checked bitwise against the reference
 * itself (oracle/_ref/libftref.so, compiled from the reference headers by
 * oracle/Makefile) and against the golden vectors in tests/golden/, see
 * tests/test_oracle_pin.py.
 *
 * Conventions follow the reference exactly:
 *   - tensors are dense NCHW, last dimension fastest (tensor.hpp:17-33);
 *   - the conv accumulates in (k,i,j) order with a T accumulator
 *     (conv.hpp:39-62), no FMA contraction (build with -ffp-contract=off);
 *   - checksum arithmetic of the verdict engine is T=double, i.e. the
 *     reference workflow instantiated at double.
 */
#ifndef FTC_ORACLE_H
#define FTC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Layer geometry.  D is (N, C, H, H); W is (M, C/groups, R, R); O is (N, M, E, E). */
typedef struct or_dims {
  int N, C, H, M, R;
  int stride, pad, groups;
  int bias; /* ConvParams::bias_enabled */
} or_dims;

/* status codes (errors.hpp:9-27) */
enum { OR_OK = 0, OR_SHAPE_ERROR = 1, OR_CONFIG_ERROR = 2, OR_IO_ERROR = 3, OR_INTEGRITY_ERROR = 4 };

/* CkSel (checksums.hpp:14-23) */
enum { OR_CK_O1 = 1, OR_CK_O2 = 2, OR_CK_O3 = 4, OR_CK_O4 = 8, OR_CK_O5 = 16, OR_CK_O6 = 32, OR_CK_O7 = 64, OR_CK_ALL = 127 };

/* ResolveStage (report.hpp:12-21) */
enum { OR_ST_NONE = 0, OR_ST_RELOAD, OR_ST_COC, OR_ST_RC, OR_ST_CLC, OR_ST_FC, OR_ST_DISCARD, OR_ST_RECOMPUTE };

/* CorrectionStatus (schemes.hpp:24) */
enum { OR_CORRECTED = 0, OR_DISCARD = 1, OR_ESCALATE = 2 };

#define OR_MAX_BLOCKS 4096

/* LayerReport (report.hpp:38-47) as POD */
typedef struct or_report {
  int detected, stage, weights_reloaded, recomputed;
  int n_blocks;                  /* total number of corrected blocks */
  int blocks[OR_MAX_BLOCKS][2];  /* (i, j) = (n, m), sorted */
  int n_stages;
  int stages[8];
  double max_rel_dev;            /* DetectionResult::max_rel_dev of the first CoC-D */
} or_report;

/* LayerPlan (workflow.hpp:23-29) subset that drives the verdict */
typedef struct or_plan {
  int rc_enabled, clc_enabled;
  double tau;
} or_plan;

/* pre_conv fault (FaultHooks::pre_conv, workflow.hpp:117-121, fault.hpp:138-168),
 * restated as a substitution: element `index` of `target` is set to `value`
 * (mode 0) or incremented by `value` (mode 1) after the input checksums were taken. */
enum { OR_T_D = 0, OR_T_W = 1, OR_T_CD1 = 2, OR_T_CD2 = 3, OR_T_CW1 = 4, OR_T_CW2 = 5 };
typedef struct or_pre_fault {
  int target;
  long long index;
  int mode;
  double value;
} or_pre_fault;

/* ---- generators shared with the reference (tensor.hpp:57-66) ---- */
void or_mt64_uniform(uint64_t seed, double lo, double hi, size_t n, double* out);
void or_mt64_uniform_f32(uint64_t seed, double lo, double hi, size_t n, float* out);

/* ---- extent rule (tensor.hpp:100-107) ---- */
int or_output_extent(int H, int R, int pad, int stride, int* E);
int or_check_dims(const or_dims* d, int* E);

/* ---- convolution (conv.hpp:39-62, 114-131) ---- */
int or_conv_forward_f32(const or_dims* d, const float* D, const float* W, const float* bias, float* O);
int or_conv_forward_f64(const or_dims* d, const double* D, const double* W, const double* bias, double* O);

/* ---- checksums (checksums.hpp) at T=double ---- */
int or_values_differ(double c, double s, double tau);                                   /* :54-60 */
void or_kernel_checksums(const or_dims* d, const double* W, double* cw1, double* cw2);   /* :70-88 */
void or_input_checksums(const or_dims* d, const double* D, double* cd1, double* cd2);    /* :91-107 */
/* co[k] for k=0..6 receives Co(k+1) when bit k of `which` is set:
 * Co1,Co3: M grids; Co2,Co4: N grids; Co5..7: 1 grid (checksums.hpp:134-161) */
int or_output_checksums(const or_dims* d, unsigned which, const double* D, const double* W,
                        const double* cd1, const double* cd2, const double* cw1, const double* cw2,
                        double* co[7]);
/* so[k] likewise (checksums.hpp:165-190); if bias != NULL the BiasAdjuster rows are applied (:195-236) */
int or_output_summations(int N, int M, int E, const double* O, unsigned which, const double* bias,
                         double* so[7]);
int or_verify_kernel(const or_dims* d, const double* W, const double* cw1_ref, double tau); /* :250-259 */
int or_detect_coc_d(const double* co5, const double* so5, int E2, double tau, uint8_t* mask,
                    double* max_rel_dev); /* schemes.hpp:79-94; returns clean */
int or_locate_index(double r, int n, int* out); /* schemes.hpp:57-62 */

/* ---- run_protected_layer<double> (workflow.hpp:141-339) ----
 * O_conv: if non-NULL, the post_conv hook's output (the contract's substitution of
 *         the GPU's FP32 output, widened, with flips applied); otherwise the
 *         oracle computes conv_forward<double>(D, W) itself.
 * pre/n_pre: pre_conv faults (applied after input checksums).
 * O_out: final output (N*M*E*E doubles), may be NULL.
 * isolation: -1 = full workflow; 2..5 = one scheme in isolation (Scheme::coc=1.. as in
 *            acceptance.cpp:207-292 with a Co5-only verifier): 1=coc 2=rc 3=clc 4=fc.
 * Returns OR_OK, or OR_INTEGRITY_ERROR when recompute fails twice (workflow.hpp:338). */
int or_protected_layer(const or_dims* d, const double* D, const double* W_golden, const double* bias,
                       const or_plan* plan, const double* O_conv, const or_pre_fault* pre, int n_pre,
                       or_report* rep, double* O_out);

/* The same with a second seam for BASELINE-scale parity runs: O_recompute, if non-NULL,
 * stands in for the recompute stage's fresh conv_forward<double> (workflow.hpp:327) --
 * the GPU's own fault-free FP32 output, widened.  The stage still re-takes the input
 * checksums, Co5 and So5 and judges them at tau exactly as :325-338; only the O the
 * check runs on differs (a double conv is consistent to ~1e-15 and always passes, so the
 * seam can only make the check stricter).  NULL = the reference behaviour. */
int or_protected_layer_seam(const or_dims* d, const double* D, const double* W_golden, const double* bias,
                            const or_plan* plan, const double* O_conv, const double* O_recompute,
                            const or_pre_fault* pre, int n_pre, or_report* rep, double* O_out);

/* One scheme in isolation with the detection + reload preamble and a Co5-only
 * verifier (acceptance.cpp:207-292).  scheme: 1=coc 2=rc 3=clc 4=fc.
 * Returns the CorrectionStatus (or -1 if detection was clean / reload resolved it). */
int or_isolated_scheme(const or_dims* d, const double* D, const double* W_golden, const double* bias,
                       double tau, const double* O_conv, int scheme, double* O_out, int* n_blocks,
                       int* blocks /* 2*OR_MAX_BLOCKS */);

/* fault.hpp:82-87 -- u ^= 1u << (bit % 31) on the FP32 word */
float or_flip_bit_f32(float v, unsigned bit);

/* ---- back-propagation (conv.hpp:150-185, workflow.hpp:340-417), T=double ---- */
int or_conv_backward_f64(const or_dims* d, const double* D, const double* W, const double* dO, double* dW,
                         double* dD);
/* hook: post_hook restated as substitutions on the first pass (target 0 dW, 1 dD;
 * mode 0 set, 1 add) */
int or_protected_backward(const or_dims* d, const double* D, const double* W, const double* dO, double tau,
                          const or_pre_fault* hook, int n_hook, double* dW, double* dD, int* dw_detected,
                          int* dd_detected, int* recomputed);

/* workflow.hpp:55-112 plan helpers */
double or_cost_model(int scheme, int N, int M, int Ch, int H, int R, int E, double alpha, double beta);
int or_decide_rc(double t0, double t1, double t2, double p_r, double p_c);
int or_decide_clc(double t0, double t1, double t2, double p_r, double p_c);
void or_make_default_plan(int N, int M, int Ch, int H, int R, int E, double tau, int* rc, int* clc,
                          double* t0, double* t1, double* t2, double* p_r);

#ifdef __cplusplus
}
#endif
#endif
