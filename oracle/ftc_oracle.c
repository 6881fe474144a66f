/*
 * ftc_oracle.c -- CPU restatement of the reference's ABFT-protected convolution
 * (see ftc_oracle.h).  TEST INFRASTRUCTURE ONLY: never part of the product path.
 *
 * Each function cites the reference file:line it restates; paths are relative to
 * /root/reference/proj/core/include/ftconv/.  Loops that the reference runs
 * sequentially are parallelised here only across independent outputs, so every
 * individual sum keeps the reference's association order and the results are
 * bitwise identical to the reference (pinned in tests/test_oracle_pin.py).
 *
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off -fopenmp).
 */
#include "ftc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG */
/* std::mt19937_64 (the engine behind Tensor4::random, tensor.hpp:57-66). */
typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* std::uniform_real_distribution<double>(lo,hi) over libstdc++'s
 * generate_canonical<double,53>: one 64-bit draw / 2^64, clamped below 1. */
static double mt64_uniform(mt64* s, double lo, double hi) {
  double c = (double)mt64_next(s) / 18446744073709551616.0;
  if (c >= 1.0) c = nextafter(1.0, 0.0);
  return c * (hi - lo) + lo;
}

void or_mt64_uniform(uint64_t seed, double lo, double hi, size_t n, double* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (size_t i = 0; i < n; ++i) out[i] = mt64_uniform(&s, lo, hi);
}

void or_mt64_uniform_f32(uint64_t seed, double lo, double hi, size_t n, float* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (size_t i = 0; i < n; ++i) out[i] = (float)mt64_uniform(&s, lo, hi);
}

/* ------------------------------------------------------------------ shapes */
/* output_extent, tensor.hpp:100-107 */
int or_output_extent(int H, int R, int pad, int stride, int* E) {
  const long Hp = (long)H + 2L * pad;
  if (stride <= 0) return OR_CONFIG_ERROR;
  if (Hp < R) return OR_CONFIG_ERROR;
  if ((Hp - R) % stride != 0) return OR_CONFIG_ERROR;
  *E = (int)((Hp - R) / stride + 1);
  return OR_OK;
}

/* check_conv_shapes, conv.hpp:16-26 (square D and W are implied by or_dims) */
int or_check_dims(const or_dims* d, int* E) {
  if (d->groups <= 0) return OR_CONFIG_ERROR;
  if (d->C % d->groups != 0 || d->M % d->groups != 0) return OR_CONFIG_ERROR;
  return or_output_extent(d->H, d->R, d->pad, d->stride, E);
}

/* ------------------------------------------------------------------ conv */
/* conv_direct, conv.hpp:39-62, plus the bias broadcast of conv_forward :118-129.
 * padded_at (:28-37) is the bounds test returning T(0). */
#define DEFINE_CONV(NAME, T)                                                                 \
  static void NAME(int N, int C, int H, int M, int Ckw, int R, int U, int pad, int groups,    \
                   int E, const T* D, const T* W, const T* bias, T* O) {                      \
    const int mpg = M / groups;                                                              \
    _Pragma("omp parallel for collapse(2) schedule(static)")                                 \
    for (int n = 0; n < N; ++n)                                                              \
      for (int m = 0; m < M; ++m) {                                                          \
        const int kbase = (m / mpg) * Ckw;                                                   \
        for (int x = 0; x < E; ++x)                                                          \
          for (int y = 0; y < E; ++y) {                                                      \
            T acc = (T)0;                                                                    \
            for (int k = 0; k < Ckw; ++k)                                                    \
              for (int i = 0; i < R; ++i)                                                    \
                for (int j = 0; j < R; ++j) {                                                \
                  const long hh = (long)U * x + i - pad, ww = (long)U * y + j - pad;         \
                  T v = (T)0;                                                                \
                  if (hh >= 0 && ww >= 0 && hh < H && ww < H)                                \
                    v = D[(((size_t)n * C + kbase + k) * H + hh) * H + ww];                  \
                  acc += v * W[(((size_t)m * Ckw + k) * R + i) * R + j];                     \
                }                                                                            \
            T o = acc;                                                                       \
            if (bias) o += bias[m];                                                          \
            O[(((size_t)n * M + m) * E + x) * E + y] = o;                                    \
          }                                                                                  \
      }                                                                                      \
  }

DEFINE_CONV(conv_f32, float)
DEFINE_CONV(conv_f64, double)

int or_conv_forward_f32(const or_dims* d, const float* D, const float* W, const float* bias, float* O) {
  int E, st = or_check_dims(d, &E);
  if (st) return st;
  if (d->bias && !bias) return OR_SHAPE_ERROR;
  conv_f32(d->N, d->C, d->H, d->M, d->C / d->groups, d->R, d->stride, d->pad, d->groups, E, D, W,
           d->bias ? bias : NULL, O);
  return OR_OK;
}

int or_conv_forward_f64(const or_dims* d, const double* D, const double* W, const double* bias, double* O) {
  int E, st = or_check_dims(d, &E);
  if (st) return st;
  if (d->bias && !bias) return OR_SHAPE_ERROR;
  conv_f64(d->N, d->C, d->H, d->M, d->C / d->groups, d->R, d->stride, d->pad, d->groups, E, D, W,
           d->bias ? bias : NULL, O);
  return OR_OK;
}

/* ------------------------------------------------------------------ checksums */
/* values_differ, checksums.hpp:54-60.  Any NaN makes the comparison false; an
 * infinite operand gives inf > tau*inf == false (SURVEY 8(a') step 9). */
int or_values_differ(double c, double s, double tau) {
  const double cc = fabs(c), ss = fabs(s);
  double m = cc;          /* std::max({cc,ss,1.0}) keeps the first of equal/NaN */
  if (m < ss) m = ss;
  if (m < 1.0) m = 1.0;
  return fabs(c - s) > tau * m;
}

/* kernel_checksums, checksums.hpp:70-88: global m index weights, groups concat. */
void or_kernel_checksums(const or_dims* d, const double* W, double* cw1, double* cw2) {
  const int M = d->M, Ckw = d->C / d->groups, R = d->R, G = d->groups, mpg = M / G;
  const size_t per = (size_t)Ckw * R * R;
  memset(cw1, 0, sizeof(double) * per * G);
  memset(cw2, 0, sizeof(double) * per * G);
  for (int g = 0; g < G; ++g)
    for (int mg = 0; mg < mpg; ++mg) {
      const int m = g * mpg + mg;
      for (size_t e = 0; e < per; ++e) {
        cw1[g * per + e] += W[m * per + e];
        cw2[g * per + e] += (double)m * W[m * per + e];
      }
    }
}

/* input_checksums, checksums.hpp:91-107: ascending-n accumulation. */
void or_input_checksums(const or_dims* d, const double* D, double* cd1, double* cd2) {
  const size_t per = (size_t)d->C * d->H * d->H;
  memset(cd1, 0, sizeof(double) * per);
  memset(cd2, 0, sizeof(double) * per);
  for (int n = 0; n < d->N; ++n)
    for (size_t e = 0; e < per; ++e) {
      const double v = D[n * per + e];
      cd1[e] += v;
      cd2[e] += (double)n * v;
    }
}

/* output_checksums, checksums.hpp:134-161.  Co1/Co3 use the real (grouped) W;
 * everything against Cw runs ungrouped (`flat`); Co5..7 are conv_block
 * (conv.hpp:135-145), i.e. a plain ungrouped conv of one block. */
int or_output_checksums(const or_dims* d, unsigned which, const double* D, const double* W,
                        const double* cd1, const double* cd2, const double* cw1, const double* cw2,
                        double* co[7]) {
  int E, st = or_check_dims(d, &E);
  if (st) return st;
  if ((which & (OR_CK_O3 | OR_CK_O7)) && !cd2) return OR_CONFIG_ERROR;
  if ((which & (OR_CK_O4 | OR_CK_O6)) && !cw2) return OR_CONFIG_ERROR;
  const int C = d->C, H = d->H, M = d->M, R = d->R, U = d->stride, p = d->pad, G = d->groups;
  const int Ckw = C / G;
  if (which & OR_CK_O1) conv_f64(1, C, H, M, Ckw, R, U, p, G, E, cd1, W, NULL, co[0]);
  if (which & OR_CK_O2) conv_f64(d->N, C, H, 1, C, R, U, p, 1, E, D, cw1, NULL, co[1]);
  if (which & OR_CK_O3) conv_f64(1, C, H, M, Ckw, R, U, p, G, E, cd2, W, NULL, co[2]);
  if (which & OR_CK_O4) conv_f64(d->N, C, H, 1, C, R, U, p, 1, E, D, cw2, NULL, co[3]);
  if (which & OR_CK_O5) conv_f64(1, C, H, 1, C, R, U, p, 1, E, cd1, cw1, NULL, co[4]);
  if (which & OR_CK_O6) conv_f64(1, C, H, 1, C, R, U, p, 1, E, cd1, cw2, NULL, co[5]);
  if (which & OR_CK_O7) conv_f64(1, C, H, 1, C, R, U, p, 1, E, cd2, cw1, NULL, co[6]);
  return OR_OK;
}

/* BiasAdjuster, checksums.hpp:195-236 (0-based weights, wn = N(N-1)/2). */
static void bias_apply(int N, int M, int E, const double* b, unsigned which, double* so[7]) {
  double sum_b = 0.0, sum_mb = 0.0;
  for (int m = 0; m < M; ++m) {
    sum_b += b[m];
    sum_mb += (double)m * b[m];
  }
  const double wn = (double)((size_t)N * (size_t)(N - 1) / 2);
  const double nN = (double)N;
  const size_t E2 = (size_t)E * E;
  if (which & OR_CK_O1)
    for (int m = 0; m < M; ++m)
      for (size_t f = 0; f < E2; ++f) so[0][m * E2 + f] -= nN * b[m];
  if (which & OR_CK_O2)
    for (size_t f = 0; f < (size_t)N * E2; ++f) so[1][f] -= sum_b;
  if (which & OR_CK_O3)
    for (int m = 0; m < M; ++m)
      for (size_t f = 0; f < E2; ++f) so[2][m * E2 + f] -= wn * b[m];
  if (which & OR_CK_O4)
    for (size_t f = 0; f < (size_t)N * E2; ++f) so[3][f] -= sum_mb;
  if (which & OR_CK_O5)
    for (size_t f = 0; f < E2; ++f) so[4][f] -= nN * sum_b;
  if (which & OR_CK_O6)
    for (size_t f = 0; f < E2; ++f) so[5][f] -= nN * sum_mb;
  if (which & OR_CK_O7)
    for (size_t f = 0; f < E2; ++f) so[6][f] -= wn * sum_b;
}

/* output_summations, checksums.hpp:165-190 (loop order n, m, x, y; every
 * per-position sum runs in ascending (n, m) order). */
int or_output_summations(int N, int M, int E, const double* O, unsigned which, const double* bias,
                         double* so[7]) {
  const size_t E2 = (size_t)E * E;
  if (which & (OR_CK_O1 | OR_CK_O3)) {
#pragma omp parallel for schedule(static)
    for (long q = 0; q < (long)(M * E2); ++q) {
      const int m = (int)(q / E2);
      const size_t f = q % E2;
      double s1 = 0.0, s3 = 0.0;
      for (int n = 0; n < N; ++n) {
        const double v = O[((size_t)n * M + m) * E2 + f];
        s1 += v;
        s3 += (double)n * v;
      }
      if (which & OR_CK_O1) so[0][q] = s1;
      if (which & OR_CK_O3) so[2][q] = s3;
    }
  }
  if (which & (OR_CK_O2 | OR_CK_O4)) {
#pragma omp parallel for schedule(static)
    for (long q = 0; q < (long)(N * E2); ++q) {
      const int n = (int)(q / E2);
      const size_t f = q % E2;
      double s2 = 0.0, s4 = 0.0;
      for (int m = 0; m < M; ++m) {
        const double v = O[((size_t)n * M + m) * E2 + f];
        s2 += v;
        s4 += (double)m * v;
      }
      if (which & OR_CK_O2) so[1][q] = s2;
      if (which & OR_CK_O4) so[3][q] = s4;
    }
  }
  if (which & (OR_CK_O5 | OR_CK_O6 | OR_CK_O7)) {
#pragma omp parallel for schedule(static)
    for (long f = 0; f < (long)E2; ++f) {
      double s5 = 0.0, s6 = 0.0, s7 = 0.0;
      for (int n = 0; n < N; ++n)
        for (int m = 0; m < M; ++m) {
          const double v = O[((size_t)n * M + m) * E2 + f];
          s5 += v;
          s6 += (double)m * v;
          s7 += (double)n * v;
        }
      if (which & OR_CK_O5) so[4][f] = s5;
      if (which & OR_CK_O6) so[5][f] = s6;
      if (which & OR_CK_O7) so[6][f] = s7;
    }
  }
  if (bias) bias_apply(N, M, E, bias, which, so);
  return OR_OK;
}

/* verify_kernel, checksums.hpp:250-259 */
int or_verify_kernel(const or_dims* d, const double* W, const double* cw1_ref, double tau) {
  const size_t per = (size_t)d->C * d->R * d->R;
  double* cw1 = malloc(sizeof(double) * per);
  double* cw2 = malloc(sizeof(double) * per);
  or_kernel_checksums(d, W, cw1, cw2);
  int ok = 1;
  for (size_t i = 0; i < per && ok; ++i)
    if (or_values_differ(cw1[i], cw1_ref[i], tau)) ok = 0;
  free(cw1);
  free(cw2);
  return ok;
}

/* ------------------------------------------------------------------ schemes */
/* detect_coc_d, schemes.hpp:79-94 */
int or_detect_coc_d(const double* co5, const double* so5, int E2, double tau, uint8_t* mask,
                    double* max_rel_dev) {
  int clean = 1;
  double mrd = 0.0;
  for (int i = 0; i < E2; ++i) {
    const double c = co5[i], s = so5[i];
    double den = fabs(c);
    if (den < fabs(s)) den = fabs(s);
    if (den < 1.0) den = 1.0;
    const double dev = fabs(c - s) / den;
    if (mrd < dev) mrd = dev; /* std::max(a, b): a < b ? b : a -- NaN devs never win */
    const int bad = or_values_differ(c, s, tau);
    if (mask) mask[i] = (uint8_t)bad;
    if (bad) clean = 0;
  }
  if (max_rel_dev) *max_rel_dev = mrd;
  return clean;
}

/* locate_index, schemes.hpp:57-62 */
int or_locate_index(double r, int n, int* out) {
  const long long i = llround(r);
  if (fabs(r - (double)i) > 0.01) return 0;
  if (i < 0 || i >= (long long)n) return 0;
  *out = (int)i;
  return 1;
}

float or_flip_bit_f32(float v, unsigned bit) {
  uint32_t u;
  memcpy(&u, &v, 4);
  u ^= (1u << (bit % 31u));
  memcpy(&v, &u, 4);
  return v;
}

/* ------------------------------------------------------------------ workflow state */
typedef struct patch { int i, j; size_t f; double delta; } patch;

typedef struct layer_state {
  or_dims d;
  int E;
  size_t E2;
  double tau;
  double* D;        /* working copy */
  double* W;        /* working copy */
  const double* W_golden;
  const double* bias;
  double *cd1, *cd2, *cw1, *cw2;
  double *cw1_ref, *cw2_ref;
  double* O;
  double* cs[7];
  double* s[7];
  unsigned cs_have, s_have;
  int verifier_mode; /* 0: workflow verifier (workflow.hpp:205-219); 1: Co5-only (acceptance) */
} layer_state;

static size_t fam_len(const layer_state* L, int k) {
  if (k == 0 || k == 2) return (size_t)L->d.M * L->E2;
  if (k == 1 || k == 3) return (size_t)L->d.N * L->E2;
  return L->E2;
}

/* workflow.hpp:168-180 */
static void ensure_cs(layer_state* L, unsigned want) {
  const unsigned need = want & ~L->cs_have;
  if (!need) return;
  double* co[7] = {0};
  for (int k = 0; k < 7; ++k)
    if (need & (1u << k)) {
      if (!L->cs[k]) L->cs[k] = malloc(sizeof(double) * fam_len(L, k));
      co[k] = L->cs[k];
    }
  or_output_checksums(&L->d, need, L->D, L->W, L->cd1, L->cd2, L->cw1, L->cw2, co);
  L->cs_have |= need;
}

/* workflow.hpp:183-196 */
static void ensure_s(layer_state* L, unsigned want) {
  const unsigned need = want & ~L->s_have;
  if (!need) return;
  double* so[7] = {0};
  for (int k = 0; k < 7; ++k)
    if (need & (1u << k)) {
      if (!L->s[k]) L->s[k] = malloc(sizeof(double) * fam_len(L, k));
      so[k] = L->s[k];
    }
  or_output_summations(L->d.N, L->d.M, L->E, L->O, need, L->d.bias ? L->bias : NULL, so);
  L->s_have |= need;
}

static int grids_consistent(const double* c, const double* s, size_t n, double tau) {
  for (size_t i = 0; i < n; ++i)
    if (or_values_differ(c[i], s[i], tau)) return 0;
  return 1;
}

/* The workflow verifier, workflow.hpp:205-219: fresh (bias-adjusted) sums of the
 * whole output against every trusted family computed so far. */
static int verifier(layer_state* L) {
  unsigned trusted = L->cs_have & (OR_CK_O1 | OR_CK_O3 | OR_CK_O5 | OR_CK_O6 | OR_CK_O7);
  if (L->verifier_mode == 1) trusted = OR_CK_O5; /* acceptance.cpp:247-251 */
  double* fresh[7] = {0};
  for (int k = 0; k < 7; ++k)
    if (trusted & (1u << k)) fresh[k] = malloc(sizeof(double) * fam_len(L, k));
  or_output_summations(L->d.N, L->d.M, L->E, L->O, trusted, L->d.bias ? L->bias : NULL, fresh);
  int ok = 1;
  const int order[5] = {4, 5, 6, 0, 2};
  for (int q = 0; q < 5 && ok; ++q) {
    const int k = order[q];
    if (trusted & (1u << k)) ok = grids_consistent(L->cs[k], fresh[k], fam_len(L, k), L->tau);
  }
  for (int k = 0; k < 7; ++k) free(fresh[k]);
  return ok;
}

static size_t oidx(const layer_state* L, int n, int m, size_t f) {
  return ((size_t)n * L->d.M + m) * L->E2 + f;
}

static void apply_patches(layer_state* L, const patch* p, size_t np) {
  for (size_t q = 0; q < np; ++q) L->O[oidx(L, p[q].i, p[q].j, p[q].f)] += p[q].delta;
}

static void rollback(layer_state* L, const patch* p, size_t np) { /* schemes.hpp:71-74 */
  for (size_t q = 0; q < np; ++q) L->O[oidx(L, p[q].i, p[q].j, p[q].f)] -= p[q].delta;
}

typedef struct outcome {
  int status;
  int n_blocks;
  int* blocks; /* 2*n_blocks, sorted (std::set<BlockCoord>) */
} outcome;

static int cmp_block(const void* a, const void* b) {
  const int* x = a;
  const int* y = b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
  return 0;
}

/* set of (i,j) from the patch list, sorted and unique (std::set<BlockCoord>) */
static void blocks_from_patches(outcome* oc, const patch* p, size_t np) {
  int* b = malloc(sizeof(int) * 2 * (np ? np : 1));
  for (size_t q = 0; q < np; ++q) {
    b[2 * q] = p[q].i;
    b[2 * q + 1] = p[q].j;
  }
  qsort(b, np, 2 * sizeof(int), cmp_block);
  size_t u = 0;
  for (size_t q = 0; q < np; ++q)
    if (u == 0 || cmp_block(&b[2 * (u - 1)], &b[2 * q]) != 0) {
      b[2 * u] = b[2 * q];
      b[2 * u + 1] = b[2 * q + 1];
      ++u;
    }
  oc->blocks = b;
  oc->n_blocks = (int)u;
}

/* commit lambda of correct_fc (schemes.hpp:337-351); same shape in rc/clc/coc */
static void commit(layer_state* L, patch* p, size_t np, outcome* oc) {
  apply_patches(L, p, np);
  if (verifier(L)) {
    oc->status = OR_CORRECTED;
    blocks_from_patches(oc, p, np);
  } else {
    rollback(L, p, np);
    oc->status = OR_ESCALATE;
  }
}

/* probes, workflow.hpp:247-270 */
static int probe_row0(layer_state* L) {
  /* conv_block(D.block(0), ic.cw1, p) vs sum_m O[0,m] - sum_b */
  const or_dims* d = &L->d;
  double* c = malloc(sizeof(double) * L->E2);
  conv_f64(1, d->C, d->H, 1, d->C, d->R, d->stride, d->pad, 1, L->E, L->D, L->cw1, NULL, c);
  double* sum = calloc(L->E2, sizeof(double));
  for (int m = 0; m < d->M; ++m)
    for (size_t i = 0; i < L->E2; ++i) sum[i] += L->O[oidx(L, 0, m, i)];
  if (d->bias) {
    double sb = 0.0;
    for (int m = 0; m < d->M; ++m) sb += L->bias[m];
    for (size_t i = 0; i < L->E2; ++i) sum[i] -= sb;
  }
  const int ok = grids_consistent(c, sum, L->E2, L->tau);
  free(c);
  free(sum);
  return ok;
}

static int probe_col0(layer_state* L) {
  /* conv_block(Cd1[group 0], W.block(0), p) vs sum_n O[n,0] - N*B[0] */
  const or_dims* d = &L->d;
  const int Ckw = d->C / d->groups;
  double* c = malloc(sizeof(double) * L->E2);
  /* channel_slice(cd1, 0, Ckw) is the leading Ckw channels: a prefix of cd1 */
  conv_f64(1, Ckw, d->H, 1, Ckw, d->R, d->stride, d->pad, 1, L->E, L->cd1, L->W, NULL, c);
  double* sum = calloc(L->E2, sizeof(double));
  for (int n = 0; n < d->N; ++n)
    for (size_t i = 0; i < L->E2; ++i) sum[i] += L->O[oidx(L, n, 0, i)];
  if (d->bias)
    for (size_t i = 0; i < L->E2; ++i) sum[i] -= (double)d->N * L->bias[0];
  const int ok = grids_consistent(c, sum, L->E2, L->tau);
  free(c);
  free(sum);
  return ok;
}

/* correct_coc, schemes.hpp:99-183 */
static void correct_coc(layer_state* L, int use_probes, outcome* oc) {
  const double *c5 = L->cs[4], *c6 = L->cs[5], *c7 = L->cs[6];
  const double *s5 = L->s[4], *s6 = L->s[5], *s7 = L->s[6];
  const size_t E2 = L->E2;
  const double tau = L->tau;
  oc->n_blocks = 0;
  oc->blocks = NULL;

  size_t nflag = 0;
  size_t* flagged = malloc(sizeof(size_t) * E2);
  for (size_t i = 0; i < E2; ++i)
    if (or_values_differ(c5[i], s5[i], tau)) flagged[nflag++] = i;
  if (nflag == 0) {
    oc->status = OR_CORRECTED;
    free(flagged);
    return;
  }
  int valid = 1, have = 0, li = 0, lj = 0;
  for (size_t q = 0; q < nflag; ++q) {
    const size_t f = flagged[q];
    const double delta = c5[f] - s5[f];
    if (fabs(delta) < tau) {
      valid = 0;
      break;
    }
    const double ri = (c7[f] - s7[f]) / delta;
    const double rj = (c6[f] - s6[f]) / delta;
    int i, j;
    const int oki = or_locate_index(ri, L->d.N, &i);
    const int okj = or_locate_index(rj, L->d.M, &j);
    if (!oki || !okj || (have && !(li == i && lj == j))) {
      valid = 0;
      break;
    }
    have = 1;
    li = i;
    lj = j;
  }
  if (valid && have) {
    patch* p = malloc(sizeof(patch) * nflag);
    for (size_t q = 0; q < nflag; ++q) {
      const size_t f = flagged[q];
      p[q].i = li;
      p[q].j = lj;
      p[q].f = f;
      p[q].delta = c5[f] - s5[f];
    }
    apply_patches(L, p, nflag);
    if (verifier(L)) {
      oc->status = OR_CORRECTED;
      oc->blocks = malloc(sizeof(int) * 2);
      oc->blocks[0] = li;
      oc->blocks[1] = lj;
      oc->n_blocks = 1;
    } else {
      rollback(L, p, nflag);
      oc->status = OR_ESCALATE;
    }
    free(p);
    free(flagged);
    return;
  }
  free(flagged);
  /* pattern analysis (:161-182) */
  const int m6 = !grids_consistent(c6, s6, E2, tau);
  const int m7 = !grids_consistent(c7, s7, E2, tau);
  if (m6 && !m7) {
    oc->status = use_probes ? (probe_row0(L) ? OR_DISCARD : OR_ESCALATE) : OR_DISCARD;
    return;
  }
  if (m7 && !m6) {
    oc->status = use_probes ? (probe_col0(L) ? OR_DISCARD : OR_ESCALATE) : OR_DISCARD;
    return;
  }
  oc->status = OR_ESCALATE;
}

/* correct_rc (schemes.hpp:187-241) and, mirrored, correct_clc (:244-298).
 * rc=1: flags from Co1/So1 per column j, row from (Co3-So3)/delta.
 * rc=0: flags from Co2/So2 per row n, column from (Co4-So4)/delta. */
static void correct_line(layer_state* L, int rc, outcome* oc) {
  const double* c1 = rc ? L->cs[0] : L->cs[1];
  const double* c3 = rc ? L->cs[2] : L->cs[3];
  const double* s1 = rc ? L->s[0] : L->s[1];
  const double* s3 = rc ? L->s[2] : L->s[3];
  const int outer = rc ? L->d.M : L->d.N;
  const int range = rc ? L->d.N : L->d.M;
  const size_t E2 = L->E2;
  const double tau = L->tau;
  oc->n_blocks = 0;
  oc->blocks = NULL;
  size_t cap = 1024, np = 0;
  patch* p = malloc(sizeof(patch) * cap);
  int have = 0, line = 0;
  for (int j = 0; j < outer; ++j)
    for (size_t f = 0; f < E2; ++f) {
      const size_t q = (size_t)j * E2 + f;
      if (!or_values_differ(c1[q], s1[q], tau)) continue;
      const double delta = c1[q] - s1[q];
      if (fabs(delta) < tau) {
        oc->status = OR_ESCALATE;
        free(p);
        return;
      }
      const double r = (c3[q] - s3[q]) / delta;
      int i;
      if (!or_locate_index(r, range, &i) || (have && line != i)) {
        oc->status = OR_ESCALATE;
        free(p);
        return;
      }
      have = 1;
      line = i;
      if (np == cap) p = realloc(p, sizeof(patch) * (cap *= 2));
      p[np].i = rc ? i : j;
      p[np].j = rc ? j : i;
      p[np].f = f;
      p[np].delta = c1[q] - s1[q];
      ++np;
    }
  if (np == 0) {
    oc->status = OR_CORRECTED;
    free(p);
    return;
  }
  commit(L, p, np, oc);
  free(p);
}

/* locate_via_coc lambda, schemes.hpp:355-372 */
static int locate_via_coc(layer_state* L, const double* w, const double* sw, int range, int* idx_out) {
  const double *c5 = L->cs[4], *s5 = L->s[4];
  int have = 0, idx = 0, any = 0;
  for (size_t f = 0; f < L->E2; ++f) {
    if (!or_values_differ(c5[f], s5[f], L->tau)) continue;
    any = 1;
    const double d = c5[f] - s5[f];
    if (fabs(d) < L->tau) return 0;
    const double r = (w[f] - sw[f]) / d;
    int k;
    if (!or_locate_index(r, range, &k) || (have && idx != k)) return 0;
    have = 1;
    idx = k;
  }
  if (!any) return 0;
  *idx_out = idx;
  return 1;
}

/* correct_fc, schemes.hpp:305-447 */
static void correct_fc(layer_state* L, outcome* oc) {
  const int N = L->d.N, M = L->d.M;
  const size_t E2 = L->E2;
  const double tau = L->tau;
  const double *c1 = L->cs[0], *c2 = L->cs[1], *s1 = L->s[0], *s2 = L->s[1];
  oc->n_blocks = 0;
  oc->blocks = NULL;
  uint8_t* colmask = calloc((size_t)M * E2, 1);
  uint8_t* rowmask = calloc((size_t)N * E2, 1);
  int* cset = malloc(sizeof(int) * M);
  int* rset = malloc(sizeof(int) * N);
  int nc = 0, nr = 0;
  for (int j = 0; j < M; ++j) {
    int any = 0;
    for (size_t f = 0; f < E2; ++f)
      if (or_values_differ(c1[(size_t)j * E2 + f], s1[(size_t)j * E2 + f], tau)) {
        colmask[(size_t)j * E2 + f] = 1;
        any = 1;
      }
    if (any) cset[nc++] = j;
  }
  for (int n = 0; n < N; ++n) {
    int any = 0;
    for (size_t f = 0; f < E2; ++f)
      if (or_values_differ(c2[(size_t)n * E2 + f], s2[(size_t)n * E2 + f], tau)) {
        rowmask[(size_t)n * E2 + f] = 1;
        any = 1;
      }
    if (any) rset[nr++] = n;
  }
  patch* p = NULL;
  size_t np = 0;
  if (nr == 0 && nc == 0) {
    oc->status = OR_DISCARD;
    goto done;
  }
  if (nr == 0 || nc == 0) {
    if (grids_consistent(L->cs[4], L->s[4], E2, tau)) {
      oc->status = OR_DISCARD;
      goto done;
    }
    int k;
    const int ok = (nr == 0) ? locate_via_coc(L, L->cs[6], L->s[6], N, &k)
                             : locate_via_coc(L, L->cs[5], L->s[5], M, &k);
    if (!ok) {
      oc->status = OR_ESCALATE;
      goto done;
    }
    if (k == 0) {
      oc->status = OR_DISCARD;
      goto done;
    }
    if (nr == 0) { /* columns flagged: row k, Co1 deltas */
      p = malloc(sizeof(patch) * ((size_t)M * E2));
      for (int a = 0; a < nc; ++a) {
        const int j = cset[a];
        for (size_t f = 0; f < E2; ++f)
          if (colmask[(size_t)j * E2 + f])
            p[np++] = (patch){k, j, f, c1[(size_t)j * E2 + f] - s1[(size_t)j * E2 + f]};
      }
    } else { /* rows flagged: column k, Co2 deltas */
      p = malloc(sizeof(patch) * ((size_t)N * E2));
      for (int a = 0; a < nr; ++a) {
        const int n = rset[a];
        for (size_t f = 0; f < E2; ++f)
          if (rowmask[(size_t)n * E2 + f])
            p[np++] = (patch){n, k, f, c2[(size_t)n * E2 + f] - s2[(size_t)n * E2 + f]};
      }
    }
    commit(L, p, np, oc);
    goto done;
  }
  if (nr == 1) {
    const int i = rset[0];
    p = malloc(sizeof(patch) * ((size_t)M * E2));
    for (int a = 0; a < nc; ++a) {
      const int j = cset[a];
      for (size_t f = 0; f < E2; ++f)
        if (colmask[(size_t)j * E2 + f])
          p[np++] = (patch){i, j, f, c1[(size_t)j * E2 + f] - s1[(size_t)j * E2 + f]};
    }
    commit(L, p, np, oc);
    goto done;
  }
  if (nc == 1) {
    const int j = cset[0];
    p = malloc(sizeof(patch) * ((size_t)N * E2));
    for (int a = 0; a < nr; ++a) {
      const int n = rset[a];
      for (size_t f = 0; f < E2; ++f)
        if (rowmask[(size_t)n * E2 + f])
          p[np++] = (patch){n, j, f, c2[(size_t)n * E2 + f] - s2[(size_t)n * E2 + f]};
    }
    commit(L, p, np, oc);
    goto done;
  }
  oc->status = OR_ESCALATE;
done:
  free(p);
  free(colmask);
  free(rowmask);
  free(cset);
  free(rset);
}

/* ------------------------------------------------------------------ driver */
static int state_init(layer_state* L, const or_dims* d, const double* D, const double* Wg,
                      const double* bias, double tau) {
  memset(L, 0, sizeof *L);
  L->d = *d;
  int st = or_check_dims(d, &L->E);
  if (st) return st;
  if (d->bias && !bias) return OR_SHAPE_ERROR;
  L->E2 = (size_t)L->E * L->E;
  L->tau = tau;
  const size_t nD = (size_t)d->N * d->C * d->H * d->H;
  const size_t nW = (size_t)d->M * (d->C / d->groups) * d->R * d->R;
  const size_t nCd = (size_t)d->C * d->H * d->H, nCw = (size_t)d->C * d->R * d->R;
  L->D = malloc(sizeof(double) * nD);
  memcpy(L->D, D, sizeof(double) * nD);
  L->W = malloc(sizeof(double) * nW);
  memcpy(L->W, Wg, sizeof(double) * nW);
  L->W_golden = Wg;
  L->bias = bias;
  L->cd1 = malloc(sizeof(double) * nCd);
  L->cd2 = malloc(sizeof(double) * nCd);
  L->cw1 = malloc(sizeof(double) * nCw);
  L->cw2 = malloc(sizeof(double) * nCw);
  L->cw1_ref = malloc(sizeof(double) * nCw);
  L->cw2_ref = malloc(sizeof(double) * nCw);
  or_input_checksums(d, L->D, L->cd1, L->cd2);
  or_kernel_checksums(d, L->W, L->cw1, L->cw2);
  memcpy(L->cw1_ref, L->cw1, sizeof(double) * nCw);
  memcpy(L->cw2_ref, L->cw2, sizeof(double) * nCw);
  L->O = malloc(sizeof(double) * (size_t)d->N * d->M * L->E2);
  return OR_OK;
}

static void state_free(layer_state* L) {
  free(L->D);
  free(L->W);
  free(L->cd1);
  free(L->cd2);
  free(L->cw1);
  free(L->cw2);
  free(L->cw1_ref);
  free(L->cw2_ref);
  free(L->O);
  for (int k = 0; k < 7; ++k) {
    free(L->cs[k]);
    free(L->s[k]);
  }
}

static void apply_pre(layer_state* L, const or_pre_fault* pre, int n_pre) {
  for (int q = 0; q < n_pre; ++q) {
    double* t = NULL;
    switch (pre[q].target) {
      case OR_T_D: t = L->D; break;
      case OR_T_W: t = L->W; break;
      case OR_T_CD1: t = L->cd1; break;
      case OR_T_CD2: t = L->cd2; break;
      case OR_T_CW1: t = L->cw1; break;
      case OR_T_CW2: t = L->cw2; break;
      default: continue;
    }
    if (pre[q].mode == 0)
      t[pre[q].index] = pre[q].value;
    else
      t[pre[q].index] += pre[q].value;
  }
}

static void clear_cs(layer_state* L) { L->cs_have = 0; }

static void report_add_stage(or_report* rep, int st) {
  if (rep->n_stages < 8) rep->stages[rep->n_stages++] = st;
}

static void report_finish(or_report* rep, const outcome* oc, int stage) {
  rep->stage = stage;
  rep->n_blocks = oc->n_blocks;
  for (int b = 0; b < oc->n_blocks && b < OR_MAX_BLOCKS; ++b) {
    rep->blocks[b][0] = oc->blocks[2 * b];
    rep->blocks[b][1] = oc->blocks[2 * b + 1];
  }
}

/* run_protected_layer, workflow.hpp:141-339 */
int or_protected_layer(const or_dims* d, const double* D, const double* W_golden, const double* bias,
                       const or_plan* plan, const double* O_conv, const or_pre_fault* pre, int n_pre,
                       or_report* rep, double* O_out) {
  return or_protected_layer_seam(d, D, W_golden, bias, plan, O_conv, NULL, pre, n_pre, rep, O_out);
}

int or_protected_layer_seam(const or_dims* d, const double* D, const double* W_golden, const double* bias,
                            const or_plan* plan, const double* O_conv, const double* O_recompute,
                            const or_pre_fault* pre, int n_pre, or_report* rep, double* O_out) {
  memset(rep, 0, sizeof *rep);
  layer_state L;
  int st = state_init(&L, d, D, W_golden, bias, plan->tau);
  if (st) {
    state_free(&L);
    return st;
  }
  const size_t nO = (size_t)d->N * d->M * L.E2;
  apply_pre(&L, pre, n_pre);
  if (O_conv)
    memcpy(L.O, O_conv, sizeof(double) * nO);
  else
    conv_f64(d->N, d->C, d->H, d->M, d->C / d->groups, d->R, d->stride, d->pad, d->groups, L.E, L.D,
             L.W, d->bias ? bias : NULL, L.O);
  const double tau = plan->tau;
  int ret = OR_OK;
  outcome oc = {0, 0, NULL};

  ensure_cs(&L, OR_CK_O5);
  ensure_s(&L, OR_CK_O5);
  const int clean = or_detect_coc_d(L.cs[4], L.s[4], (int)L.E2, tau, NULL, &rep->max_rel_dev);
  rep->detected = !clean;
  if (clean) {
    rep->stage = OR_ST_NONE;
    goto out;
  }
  if (!or_verify_kernel(d, L.W, L.cw1, tau)) { /* :232-245 */
    const size_t nW = (size_t)d->M * (d->C / d->groups) * d->R * d->R;
    const size_t nCw = (size_t)d->C * d->R * d->R;
    memcpy(L.W, W_golden, sizeof(double) * nW);
    memcpy(L.cw1, L.cw1_ref, sizeof(double) * nCw);
    memcpy(L.cw2, L.cw2_ref, sizeof(double) * nCw);
    clear_cs(&L);
    rep->weights_reloaded = 1;
    ensure_cs(&L, OR_CK_O5);
    if (or_detect_coc_d(L.cs[4], L.s[4], (int)L.E2, tau, NULL, NULL)) {
      rep->stage = OR_ST_RELOAD;
      goto out;
    }
  }
  ensure_cs(&L, OR_CK_O5 | OR_CK_O6 | OR_CK_O7); /* :277-288 */
  ensure_s(&L, OR_CK_O5 | OR_CK_O6 | OR_CK_O7);
  report_add_stage(rep, OR_ST_COC);
  correct_coc(&L, 1, &oc);
  if (oc.status == OR_CORRECTED) {
    report_finish(rep, &oc, OR_ST_COC);
    goto out;
  }
  if (oc.status == OR_DISCARD) {
    rep->stage = OR_ST_DISCARD;
    goto out;
  }
  if (plan->rc_enabled) { /* :290-299 */
    ensure_cs(&L, OR_CK_O1 | OR_CK_O3);
    ensure_s(&L, OR_CK_O1 | OR_CK_O3);
    report_add_stage(rep, OR_ST_RC);
    free(oc.blocks);
    oc.blocks = NULL;
    correct_line(&L, 1, &oc);
    if (oc.status == OR_CORRECTED) {
      report_finish(rep, &oc, OR_ST_RC);
      goto out;
    }
  }
  if (plan->clc_enabled) { /* :300-309 */
    ensure_cs(&L, OR_CK_O2 | OR_CK_O4);
    ensure_s(&L, OR_CK_O2 | OR_CK_O4);
    report_add_stage(rep, OR_ST_CLC);
    free(oc.blocks);
    oc.blocks = NULL;
    correct_line(&L, 0, &oc);
    if (oc.status == OR_CORRECTED) {
      report_finish(rep, &oc, OR_ST_CLC);
      goto out;
    }
  }
  ensure_cs(&L, OR_CK_O1 | OR_CK_O2); /* :310-321 */
  ensure_s(&L, OR_CK_O1 | OR_CK_O2);
  report_add_stage(rep, OR_ST_FC);
  free(oc.blocks);
  oc.blocks = NULL;
  correct_fc(&L, &oc);
  if (oc.status == OR_CORRECTED) {
    report_finish(rep, &oc, OR_ST_FC);
    goto out;
  }
  if (oc.status == OR_DISCARD) {
    rep->stage = OR_ST_DISCARD;
    goto out;
  }
  /* recompute, :325-338 */
  report_add_stage(rep, OR_ST_RECOMPUTE);
  {
    ret = OR_INTEGRITY_ERROR;
    const size_t nCd = (size_t)d->C * d->H * d->H;
    double* co5 = malloc(sizeof(double) * L.E2);
    double* so5 = malloc(sizeof(double) * L.E2);
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (O_recompute)
        memcpy(L.O, O_recompute, sizeof(double) * nO);
      else
        conv_f64(d->N, d->C, d->H, d->M, d->C / d->groups, d->R, d->stride, d->pad, d->groups, L.E,
                 L.D, L.W, d->bias ? bias : NULL, L.O);
      or_input_checksums(d, L.D, L.cd1, L.cd2);
      or_kernel_checksums(d, L.W, L.cw1, L.cw2);
      double* co[7] = {0, 0, 0, 0, co5, 0, 0};
      double* so[7] = {0, 0, 0, 0, so5, 0, 0};
      or_output_checksums(d, OR_CK_O5, L.D, L.W, L.cd1, L.cd2, L.cw1, L.cw2, co);
      or_output_summations(d->N, d->M, L.E, L.O, OR_CK_O5, d->bias ? bias : NULL, so);
      if (or_detect_coc_d(co5, so5, (int)L.E2, tau, NULL, NULL)) {
        rep->stage = OR_ST_RECOMPUTE;
        rep->recomputed = 1;
        ret = OR_OK;
        break;
      }
    }
    (void)nCd;
    free(co5);
    free(so5);
  }
out:
  if (O_out) memcpy(O_out, L.O, sizeof(double) * nO);
  free(oc.blocks);
  state_free(&L);
  return ret;
}

/* acceptance.cpp:207-292 isolation_succeeds, minus the output comparison */
int or_isolated_scheme(const or_dims* d, const double* D, const double* W_golden, const double* bias,
                       double tau, const double* O_conv, int scheme, double* O_out, int* n_blocks,
                       int* blocks) {
  layer_state L;
  int st = state_init(&L, d, D, W_golden, bias, tau);
  if (st) {
    state_free(&L);
    return -100 - st;
  }
  const size_t nO = (size_t)d->N * d->M * L.E2;
  memcpy(L.O, O_conv, sizeof(double) * nO);
  L.verifier_mode = 1;
  int ret = -1;
  outcome oc = {0, 0, NULL};
  ensure_cs(&L, OR_CK_O5);
  ensure_s(&L, OR_CK_O5);
  if (or_detect_coc_d(L.cs[4], L.s[4], (int)L.E2, tau, NULL, NULL)) goto out;
  if (!or_verify_kernel(d, L.W, L.cw1, tau)) {
    const size_t nW = (size_t)d->M * (d->C / d->groups) * d->R * d->R;
    const size_t nCw = (size_t)d->C * d->R * d->R;
    memcpy(L.W, W_golden, sizeof(double) * nW);
    memcpy(L.cw1, L.cw1_ref, sizeof(double) * nCw);
    memcpy(L.cw2, L.cw2_ref, sizeof(double) * nCw);
    clear_cs(&L);
    ensure_cs(&L, OR_CK_O5);
    if (or_detect_coc_d(L.cs[4], L.s[4], (int)L.E2, tau, NULL, NULL)) goto out;
  }
  switch (scheme) {
    case 1:
      ensure_cs(&L, OR_CK_O6 | OR_CK_O7);
      ensure_s(&L, OR_CK_O5 | OR_CK_O6 | OR_CK_O7);
      correct_coc(&L, 0, &oc);
      break;
    case 2:
      ensure_cs(&L, OR_CK_O1 | OR_CK_O3);
      ensure_s(&L, OR_CK_O1 | OR_CK_O3);
      correct_line(&L, 1, &oc);
      break;
    case 3:
      ensure_cs(&L, OR_CK_O2 | OR_CK_O4);
      ensure_s(&L, OR_CK_O2 | OR_CK_O4);
      correct_line(&L, 0, &oc);
      break;
    default:
      ensure_cs(&L, OR_CK_O1 | OR_CK_O2 | OR_CK_O6 | OR_CK_O7);
      ensure_s(&L, OR_CK_O1 | OR_CK_O2 | OR_CK_O5 | OR_CK_O6 | OR_CK_O7);
      correct_fc(&L, &oc);
      break;
  }
  ret = oc.status;
  if (n_blocks) *n_blocks = oc.n_blocks;
  if (blocks)
    for (int b = 0; b < oc.n_blocks && b < OR_MAX_BLOCKS; ++b) {
      blocks[2 * b] = oc.blocks[2 * b];
      blocks[2 * b + 1] = oc.blocks[2 * b + 1];
    }
out:
  if (O_out) memcpy(O_out, L.O, sizeof(double) * nO);
  free(oc.blocks);
  state_free(&L);
  return ret;
}

/* ------------------------------------------------------------------ plan helpers */
/* cost_model, workflow.hpp:55-75; scheme: 0=coc_d 1=coc 2=rc 3=clc 4=fc (schemes.hpp:15) */
double or_cost_model(int scheme, int N_, int M_, int Ch_, int H_, int R_, int E_, double a, double b) {
  const double N = N_, M = M_, Ch = Ch_;
  const double H2 = (double)H_ * H_, R2 = (double)R_ * R_, E2 = (double)E_ * E_;
  switch (scheme) {
    case 4: return a * (N + M) * Ch * R2 * E2 + b * (N * Ch * H2 + 2 * N * M * E2);
    case 2: return 2 * a * M * Ch * R2 * E2 + 2 * b * (N * Ch * H2 + N * M * E2);
    case 3: return 2 * a * N * Ch * R2 * E2 + 2 * b * N * M * E2;
    case 1: return 3 * a * Ch * R2 * E2 + b * (2 * N * Ch * H2 + 3 * N * M * E2);
    case 0: return a * Ch * R2 * E2 + b * (2 * N * Ch * H2 + N * M * E2);
  }
  return -1.0;
}

int or_decide_rc(double t0, double t1, double t2, double p_r, double p_c) {
  return p_r * (t0 - t1) > p_c * (t2 - t0); /* workflow.hpp:79-81 */
}

int or_decide_clc(double t0, double t1, double t2, double p_r, double p_c) {
  return p_c * (t0 - t1) > p_r * (t2 - t0); /* workflow.hpp:84-86 */
}

/* make_default_plan, workflow.hpp:99-112 with estimate_error_probs :90-95 */
void or_make_default_plan(int N, int M, int Ch, int H, int R, int E, double tau, int* rc, int* clc,
                          double* t0, double* t1, double* t2, double* p_r) {
  const double coc = or_cost_model(1, N, M, Ch, H, R, E, 1.0, 1.0);
  *t0 = coc + or_cost_model(4, N, M, Ch, H, R, E, 1.0, 1.0);
  *t1 = coc + or_cost_model(2, N, M, Ch, H, R, E, 1.0, 1.0);
  *t2 = *t1 + or_cost_model(4, N, M, Ch, H, R, E, 1.0, 1.0);
  const double nd = (double)((size_t)N * Ch * H * H);
  const double nw = (double)((size_t)M * Ch * R * R);
  *p_r = nd / (nd + nw);
  *rc = or_decide_rc(*t0, *t1, *t2, *p_r, 1.0 - *p_r);
  *clc = 0;
}

/* ------------------------------------------------------------------ back-propagation
 * conv_backward (conv.hpp:150-185) at T=double: one pass over (n, m, x, y) ascending,
 * each upstream gradient value scattered into dW and dD over (k, i, j) ascending;
 * padded taps skipped.  groups != 1 -> ConfigError; dO must be N x M x E x E. */
int or_conv_backward_f64(const or_dims* d, const double* D, const double* W, const double* dO, double* dW,
                         double* dD) {
  int E;
  if (d->groups != 1) return OR_CONFIG_ERROR;
  int st = or_check_dims(d, &E);
  if (st) return st;
  const int N = d->N, M = d->M, Ch = d->C, R = d->R, H = d->H, U = d->stride, p = d->pad;
  memset(dW, 0, sizeof(double) * (size_t)M * Ch * R * R);
  memset(dD, 0, sizeof(double) * (size_t)N * Ch * H * H);
  for (int n = 0; n < N; ++n)
    for (int m = 0; m < M; ++m)
      for (int x = 0; x < E; ++x)
        for (int y = 0; y < E; ++y) {
          const double g = dO[(((size_t)n * M + m) * E + x) * E + y];
          for (int k = 0; k < Ch; ++k)
            for (int i = 0; i < R; ++i)
              for (int j = 0; j < R; ++j) {
                const long long h = (long long)U * x + i - p, w = (long long)U * y + j - p;
                if (h < 0 || w < 0 || h >= H || w >= H) continue;
                dW[(((size_t)m * Ch + k) * R + i) * R + j] += D[(((size_t)n * Ch + k) * H + h) * H + w] * g;
                dD[(((size_t)n * Ch + k) * H + h) * H + w] += W[(((size_t)m * Ch + k) * R + i) * R + j] * g;
              }
        }
  return OR_OK;
}

/* run_protected_backward (workflow.hpp:350-417) at T=double.  The post_hook is
 * restated as a substitution list applied to the first pass only: element `index`
 * of dW (target 0) or dD (target 1) set to `value` (mode 0) or incremented (mode 1).
 * Returns OR_INTEGRITY_ERROR when the recompute fails verification. */
static void bwd_check(const or_dims* d, const double* dW, const double* dD, const double* cdw, const double* cdd,
                      double tau, int* bad_w, int* bad_d) {
  const int N = d->N, M = d->M, Ch = d->C, R = d->R, H = d->H;
  *bad_w = *bad_d = 0;
  for (int k = 0; k < Ch && !*bad_w; ++k)
    for (int i = 0; i < R && !*bad_w; ++i)
      for (int j = 0; j < R; ++j) {
        double s = 0.0;
        for (int m = 0; m < M; ++m) s += dW[(((size_t)m * Ch + k) * R + i) * R + j];
        if (or_values_differ(cdw[((size_t)k * R + i) * R + j], s, tau)) {
          *bad_w = 1;
          break;
        }
      }
  for (int k = 0; k < Ch && !*bad_d; ++k)
    for (int a = 0; a < H && !*bad_d; ++a)
      for (int b = 0; b < H; ++b) {
        double s = 0.0;
        for (int n = 0; n < N; ++n) s += dD[(((size_t)n * Ch + k) * H + a) * H + b];
        if (or_values_differ(cdd[((size_t)k * H + a) * H + b], s, tau)) {
          *bad_d = 1;
          break;
        }
      }
}

int or_protected_backward(const or_dims* d, const double* D, const double* W, const double* dO, double tau,
                          const or_pre_fault* hook, int n_hook, double* dW, double* dD, int* dw_detected,
                          int* dd_detected, int* recomputed) {
  int E;
  if (d->groups != 1) return OR_CONFIG_ERROR;
  int st = or_check_dims(d, &E);
  if (st) return st;
  const int N = d->N, M = d->M, Ch = d->C, R = d->R, H = d->H;
  *dw_detected = *dd_detected = *recomputed = 0;
  /* upstream-gradient block sums (workflow.hpp:358-367) */
  double* rows = calloc((size_t)N * E * E, sizeof(double));
  double* cols = calloc((size_t)M * E * E, sizeof(double));
  for (int n = 0; n < N; ++n)
    for (int m = 0; m < M; ++m)
      for (int x = 0; x < E; ++x)
        for (int y = 0; y < E; ++y) {
          const double g = dO[(((size_t)n * M + m) * E + x) * E + y];
          rows[((size_t)n * E + x) * E + y] += g;
          cols[((size_t)m * E + x) * E + y] += g;
        }
  /* cdw = conv_backward(D, w1, rows).dW, cdd = conv_backward(d1, W, cols).dD (:369-374) */
  or_dims dw = *d, dd = *d;
  dw.M = 1;
  dd.N = 1;
  double* w1 = calloc((size_t)Ch * R * R, sizeof(double));
  double* d1 = calloc((size_t)Ch * H * H, sizeof(double));
  double* cdw = malloc(sizeof(double) * (size_t)Ch * R * R);
  double* cdd = malloc(sizeof(double) * (size_t)Ch * H * H);
  double* junk_d = malloc(sizeof(double) * (size_t)N * Ch * H * H);
  double* junk_w = malloc(sizeof(double) * (size_t)M * Ch * R * R);
  or_conv_backward_f64(&dw, D, w1, rows, cdw, junk_d);
  or_conv_backward_f64(&dd, d1, W, cols, junk_w, cdd);
  or_conv_backward_f64(d, D, W, dO, dW, dD);
  for (int h = 0; h < n_hook; ++h) {
    double* t = hook[h].target == 0 ? dW : dD;
    if (hook[h].mode == 0)
      t[hook[h].index] = hook[h].value;
    else
      t[hook[h].index] += hook[h].value;
  }
  int bw, bd;
  bwd_check(d, dW, dD, cdw, cdd, tau, &bw, &bd);
  *dw_detected = bw;
  *dd_detected = bd;
  int ret = OR_OK;
  if (bw || bd) {
    or_conv_backward_f64(d, D, W, dO, dW, dD);
    *recomputed = 1;
    bwd_check(d, dW, dD, cdw, cdd, tau, &bw, &bd);
    if (bw || bd) ret = OR_INTEGRITY_ERROR;
  }
  free(rows); free(cols); free(w1); free(d1); free(cdw); free(cdd); free(junk_d); free(junk_w);
  return ret;
}
