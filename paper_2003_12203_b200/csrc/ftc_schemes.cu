// ftc_schemes.cu -- device verdict engine: CoC / RC / ClC / FC analysis
// (schemes.hpp:99-447) and the workflow's mandatory verifier (workflow.hpp:205-219).
//
// Each scheme runs as scan -> decide -> emit on device.  The reference walks the
// flagged positions sequentially and stops at the first inconsistency; every
// outcome it can reach is a function of the whole flag set ("all flags locatable,
// |delta| >= tau, and located to one index"), which the scan computes with
// order-independent min/max/or reductions, so the verdict is the same.
//
// The reference repairs O by delta-adding in T=double and re-summing the whole
// output to verify.  Here the FP32 output is never touched by a candidate patch:
// patched values live in an FP64 override map (the "virtual O"), the verifier
// re-sums only the positions a patch touched (in reference order, from the virtual
// O) and reuses the cached sums elsewhere -- bitwise the reference's fresh sums --
// and rollback (schemes.hpp:71-74) is applied in the override map, so later
// stages see exactly the O the reference would.  The data repair itself is a
// plane recompute (ftc_layer.cu).
#include <cuda_runtime.h>
#include <limits.h>

#include "ftc_common.cuh"

namespace ftc {
namespace {

constexpr int kT = 256;

inline int grid_for(long long n) {
  long long b = (n + kT - 1) / kT;
  if (b < 1) b = 1;
  if (b > 4096) b = 4096;
  return (int)b;
}

__global__ void k_result_init(SchemeResult* r) {
  SchemeResult z = {};
  z.lmin = INT_MAX;
  z.lmax = -1;
  z.r0 = INT_MAX;
  z.c0 = INT_MAX;
  *r = z;
}

__device__ __forceinline__ double vo(const float* O, const double* ov, const uint8_t* present,
                                     long long i) {
  if (present && present[i]) return ov[i];
  return (double)O[i];
}

// ------------------------------------------------------------------ CoC (schemes.hpp:99-183)
__global__ void k_coc_scan(Fam F, int N, int M, int E2, double tau, SchemeResult* r) {
  const double *c5 = F.c[4], *c6 = F.c[5], *c7 = F.c[6];
  const double *s5 = F.s[4], *s6 = F.s[5], *s7 = F.s[6];
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < E2; f += gridDim.x * blockDim.x) {
    if (values_differ(c6[f], s6[f], tau)) r->m6 = 1;
    if (values_differ(c7[f], s7[f], tau)) r->m7 = 1;
    if (!values_differ(c5[f], s5[f], tau)) continue;
    r->any = 1;
    const double delta = c5[f] - s5[f];
    if (fabs(delta) < tau) {
      r->invalid = 1;
      continue;
    }
    const double ri = (c7[f] - s7[f]) / delta;
    const double rj = (c6[f] - s6[f]) / delta;
    int i, j;
    if (!locate_index(ri, N, &i) || !locate_index(rj, M, &j)) {
      r->invalid = 1;
      continue;
    }
    const int code = i * M + j;
    atomicMin(&r->lmin, code);
    atomicMax(&r->lmax, code);
  }
}

__global__ void k_coc_decide(SchemeResult* r) {
  if (!r->any) {
    r->status = SCH_EMPTY;  // no flagged position: "corrected", no blocks (:116-119)
  } else if (!r->invalid && r->lmin == r->lmax) {
    r->status = SCH_VALID;
    r->line = r->lmin;
  } else if (r->m6 && !r->m7) {
    r->status = SCH_PROBE_ROW0;  // (:163-171)
  } else if (r->m7 && !r->m6) {
    r->status = SCH_PROBE_COL0;  // (:172-180)
  } else {
    r->status = SCH_ESCALATE;
  }
}

__global__ void k_coc_emit(Fam F, int M, int E2, double tau, SchemeResult* r, Patches p) {
  if (r->status != SCH_VALID) return;
  const int i = r->line / M, j = r->line % M;
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < E2; f += gridDim.x * blockDim.x) {
    const double c5 = F.c[4][f], s5 = F.s[4][f];
    if (!values_differ(c5, s5, tau)) continue;
    const int q = atomicAdd(&r->n_patches, 1);
    if (q < p.cap) {
      p.n[q] = i;
      p.m[q] = j;
      p.f[q] = f;
      p.d[q] = c5 - s5;
    }
  }
}

// ------------------------------------------------------------------ RC / ClC (:187-298)
// rc: flags over (j, f) of Co1/So1, row = locate((Co3-So3)/delta, N)
// clc: flags over (n, f) of Co2/So2, col = locate((Co4-So4)/delta, M)
__global__ void k_line_scan(const double* c1, const double* s1, const double* c3,
                            const double* s3, long long total, int range, double tau,
                            SchemeResult* r) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    if (!values_differ(c1[q], s1[q], tau)) continue;
    r->any = 1;
    const double delta = c1[q] - s1[q];
    if (fabs(delta) < tau) {
      r->invalid = 1;
      continue;
    }
    int i;
    if (!locate_index((c3[q] - s3[q]) / delta, range, &i)) {
      r->invalid = 1;
      continue;
    }
    atomicMin(&r->lmin, i);
    atomicMax(&r->lmax, i);
  }
}

__global__ void k_line_decide(SchemeResult* r) {
  if (r->invalid)
    r->status = SCH_ESCALATE;
  else if (!r->any)
    r->status = SCH_EMPTY;  // (:224-227)
  else if (r->lmin != r->lmax)
    r->status = SCH_ESCALATE;
  else {
    r->status = SCH_VALID;
    r->line = r->lmin;
  }
}

__global__ void k_line_emit(const double* c1, const double* s1, long long total, int E2, bool rc,
                            double tau, SchemeResult* r, Patches p) {
  if (r->status != SCH_VALID) return;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    if (!values_differ(c1[q], s1[q], tau)) continue;
    const int outer = (int)(q / E2), f = (int)(q % E2);
    const int k = atomicAdd(&r->n_patches, 1);
    if (k < p.cap) {
      p.n[k] = rc ? r->line : outer;
      p.m[k] = rc ? outer : r->line;
      p.f[k] = f;
      p.d[k] = c1[q] - s1[q];
    }
  }
}

// ------------------------------------------------------------------ FC (:305-447)
__global__ void k_fc_scan(Fam F, int N, int M, int E2, double tau, uint8_t* colmask,
                          uint8_t* rowmask, int32_t* colany, int32_t* rowany, SchemeResult* r) {
  const long long tc = (long long)M * E2, tr = (long long)N * E2;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < tc + tr + E2;
       q += (long long)gridDim.x * blockDim.x) {
    if (q < tc) {
      const bool b = values_differ(F.c[0][q], F.s[0][q], tau);
      colmask[q] = b;
      if (b) colany[q / E2] = 1;
    } else if (q < tc + tr) {
      const long long t = q - tc;
      const bool b = values_differ(F.c[1][t], F.s[1][t], tau);
      rowmask[t] = b;
      if (b) rowany[t / E2] = 1;
    } else {
      const long long f = q - tc - tr;
      if (values_differ(F.c[4][f], F.s[4][f], tau)) r->c5bad = 1;
    }
  }
}

// one block: counts, the single row/column, and locate_via_coc (:355-372)
__global__ void k_fc_decide(Fam F, int N, int M, int E2, double tau, const int32_t* colany,
                            const int32_t* rowany, SchemeResult* r) {
  __shared__ int s_nr, s_nc, s_r0, s_c0, s_fail, s_any, s_min, s_max;
  if (threadIdx.x == 0) {
    s_nr = s_nc = 0;
    s_r0 = s_c0 = INT_MAX;
    s_fail = s_any = 0;
    s_min = INT_MAX;
    s_max = -1;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < M; j += blockDim.x)
    if (colany[j]) {
      atomicAdd(&s_nc, 1);
      atomicMin(&s_c0, j);
    }
  for (int n = threadIdx.x; n < N; n += blockDim.x)
    if (rowany[n]) {
      atomicAdd(&s_nr, 1);
      atomicMin(&s_r0, n);
    }
  __syncthreads();
  const int nr = s_nr, nc = s_nc;
  const bool need_locate = (nr == 0) != (nc == 0) && r->c5bad;
  if (need_locate) {
    const double* w = (nr == 0) ? F.c[6] : F.c[5];
    const double* sw = (nr == 0) ? F.s[6] : F.s[5];
    const int range = (nr == 0) ? N : M;
    for (int f = threadIdx.x; f < E2; f += blockDim.x) {
      const double c5 = F.c[4][f], s5 = F.s[4][f];
      if (!values_differ(c5, s5, tau)) continue;
      s_any = 1;
      const double d = c5 - s5;
      if (fabs(d) < tau) {
        s_fail = 1;
        continue;
      }
      int k;
      if (!locate_index((w[f] - sw[f]) / d, range, &k)) {
        s_fail = 1;
        continue;
      }
      atomicMin(&s_min, k);
      atomicMax(&s_max, k);
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  r->nr = nr;
  r->nc = nc;
  r->r0 = s_r0;
  r->c0 = s_c0;
  if (nr == 0 && nc == 0) {
    r->status = SCH_DISCARD;  // (:374-379)
  } else if (nr == 0 || nc == 0) {
    if (!r->c5bad) {
      r->status = SCH_DISCARD;  // (:385-388)
    } else if (s_fail || !s_any || s_min != s_max) {
      r->status = SCH_ESCALATE;  // locate_via_coc -> nullopt (:389-393)
    } else if (s_min == 0) {
      r->status = SCH_DISCARD;  // index 0 ~ checksum corruption (:394-398)
    } else {
      r->status = SCH_VALID;
      r->line = s_min;
      r->mode = (nr == 0) ? 0 : 1;
    }
  } else if (nr == 1) {
    r->status = SCH_VALID;  // (:427-435)
    r->line = s_r0;
    r->mode = 0;
  } else if (nc == 1) {
    r->status = SCH_VALID;  // (:436-443)
    r->line = s_c0;
    r->mode = 1;
  } else {
    r->status = SCH_ESCALATE;
  }
}

__global__ void k_fc_emit(Fam F, int N, int M, int E2, const uint8_t* colmask,
                          const uint8_t* rowmask, SchemeResult* r, Patches p) {
  if (r->status != SCH_VALID) return;
  const bool cols = r->mode == 0;
  const long long total = (long long)(cols ? M : N) * E2;
  const uint8_t* mask = cols ? colmask : rowmask;
  const double* c = cols ? F.c[0] : F.c[1];
  const double* s = cols ? F.s[0] : F.s[1];
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    if (!mask[q]) continue;
    const int outer = (int)(q / E2), f = (int)(q % E2);
    const int k = atomicAdd(&r->n_patches, 1);
    if (k < p.cap) {
      p.n[k] = cols ? r->line : outer;
      p.m[k] = cols ? outer : r->line;
      p.f[k] = f;
      p.d[k] = c[q] - s[q];
    }
  }
}

// ------------------------------------------------------------------ verifier
__global__ void k_verify_apply(Patches p, int np, int M, int E2, const float* O, VerifyWS ws) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < np; q += gridDim.x * blockDim.x) {
    const long long idx = ((long long)p.n[q] * M + p.m[q]) * E2 + p.f[q];
    const double base = vo(O, ws.ov, ws.present, idx);
    ws.ov[idx] = dadd(base, p.d[q]);  // O(i,j,x,y) += d (schemes.hpp:144, 230, 340)
    ws.present[idx] = 1;
    ws.touched5[p.f[q]] = 1;
    ws.touched1[(long long)p.m[q] * E2 + p.f[q]] = 1;
  }
}

// the positions a patch touched (their So5/So6/So7 are re-summed fresh)
__global__ void k_touched_list(const uint8_t* __restrict__ touched5, int E2, int* list, int* count) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < E2 && touched5[f]) list[atomicAdd(count, 1)] = f;
}

// fresh So5/So6/So7 where touched (launch_seq_sums567 over the touched list, reference
// order), cached elsewhere; compare (workflow.hpp:209-211)
__global__ void k_verify_pos(Fam F, unsigned trusted, int E2, double tau, VerifyWS ws, int32_t* fail) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= E2) return;
  const bool t = ws.touched5[f];
  bool bad = false;
  for (int k = 0; k < 3; ++k) {
    const unsigned bit = FTC_CK_O5 << k;
    if (!(trusted & bit)) continue;
    const double sv = t ? ws.fresh[(long long)k * E2 + f] : F.s[4 + k][f];
    if (values_differ(F.c[4 + k][f], sv, tau)) bad = true;
  }
  if (bad) *fail = 1;
}

// fresh So1/So3 per (m, f) where touched, cached elsewhere (workflow.hpp:212-217)
__global__ void k_verify_col(Fam F, unsigned trusted, const float* O, const float* bias_dev,
                             int N, int M, int E2, double tau, VerifyWS ws, int32_t* fail) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)M * E2) return;
  double s1, s3;
  if (ws.touched1[q]) {
    const int m = (int)(q / E2), f = (int)(q % E2);
    s1 = s3 = 0.0;
    for (int n0 = 0; n0 < N; n0 += 8) {  // 8 loads in flight, then the ordered adds
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = n0 + u < N ? vo(O, ws.ov, ws.present, ((long long)(n0 + u) * M + m) * E2 + f) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (n0 + u < N) {
          s1 = dadd(s1, x[u]);
          s3 = dadd(s3, dmul((double)(n0 + u), x[u]));
        }
      }
    }
    if (bias_dev) {
      const double b = bias_dev[m];
      s1 = dsub(s1, dmul((double)N, b));
      s3 = dsub(s3, dmul((double)((long long)N * (N - 1) / 2), b));
    }
  } else {
    s1 = (trusted & FTC_CK_O1) ? F.s[0][q] : 0.0;
    s3 = (trusted & FTC_CK_O3) ? F.s[2][q] : 0.0;
  }
  bool bad = false;
  if ((trusted & FTC_CK_O1) && values_differ(F.c[0][q], s1, tau)) bad = true;
  if ((trusted & FTC_CK_O3) && values_differ(F.c[2][q], s3, tau)) bad = true;
  if (bad) *fail = 1;
}

// Rollback of a rejected patch set.  The touch marks stay set for the rest of the
// layer: a rolled-back element can differ from the original by the rounding of
// (O + d) - d, so later verifications must re-sum those positions rather than
// reuse cached sums (fresh sums of an unchanged position equal the cached ones
// bitwise, so over-marking is always safe).
__global__ void k_rollback(Patches p, int np, int M, int E2, VerifyWS ws) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < np; q += gridDim.x * blockDim.x) {
    const long long idx = ((long long)p.n[q] * M + p.m[q]) * E2 + p.f[q];
    ws.ov[idx] = dsub(ws.ov[idx], p.d[q]);  // O -= delta (schemes.hpp:73)
  }
}

__global__ void k_patch_planes(Patches p, int np, int M, uint32_t* mask) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < np; q += gridDim.x * blockDim.x) {
    const long long pl = (long long)p.n[q] * M + p.m[q];
    atomicOr(&mask[pl >> 5], 1u << (pl & 31));
  }
}

// pre_conv faults on a 4-D target (d0 implied) -- fault.hpp:138-168 semantics
template <typename T>
__global__ void k_apply_faults(const ftc_fault* fl, int nf, int target, T* t, int d1, int d2,
                               int d3, long long count, const double* tab) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % d3), b = (int)((e / d3) % d2), a1 = (int)((e / ((long long)d3 * d2)) % d1);
    const int a0 = (int)(e / ((long long)d3 * d2 * d1));
    T v = t[e];
    bool hit = false;
    for (int q = 0; q < nf; ++q) {
      const ftc_fault& f = fl[q];
      if (f.target != target) continue;
      if ((f.n >= 0 && f.n != a0) || (f.m >= 0 && f.m != a1) || (f.x >= 0 && f.x != b) ||
          (f.y >= 0 && f.y != c))
        continue;
      hit = true;
      if (f.mode == FTC_FAULT_BITFLIP) {
        if (sizeof(T) == 4) {
          v = (T)__uint_as_float(__float_as_uint((float)v) ^ (1u << (f.bit % 31u)));
        } else {
          v = (T)__longlong_as_double(__double_as_longlong((double)v) ^ (1ll << (f.bit % 63u)));
        }
      } else if (f.mode == FTC_FAULT_ADD) {
        v = v + (T)(f.value + f.n_coef * (float)a0 + f.m_coef * (float)a1);
      } else if (f.mode == FTC_FAULT_SCALE) {
        const double mag = tab[f.bit + fault_elem_index(f, a0, a1, b, c, d1, d2, d3)];
        if (sizeof(T) == 4)
          v = (T)scale_f32((float)v, mag);
        else
          v = (T)scale_f64((double)v, mag);
      } else {
        v = (T)f.value;
      }
    }
    if (hit) t[e] = v;
  }
}

}  // namespace

// ------------------------------------------------------------------ launchers
int run_coc_analyze(const Fam& F, int N, int M, int E2, double tau, SchemeResult* r,
                    const Patches& p, cudaStream_t s) {
  FTC_LAUNCH(k_result_init<<<1, 1, 0, s>>>(r));
  FTC_LAUNCH(k_coc_scan<<<grid_for(E2), kT, 0, s>>>(F, N, M, E2, tau, r));
  FTC_LAUNCH(k_coc_decide<<<1, 1, 0, s>>>(r));
  FTC_LAUNCH(k_coc_emit<<<grid_for(E2), kT, 0, s>>>(F, M, E2, tau, r, p));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int run_line_analyze(const Fam& F, bool rc, int N, int M, int E2, double tau, SchemeResult* r,
                     const Patches& p, cudaStream_t s) {
  const double* c1 = rc ? F.c[0] : F.c[1];
  const double* s1 = rc ? F.s[0] : F.s[1];
  const double* c3 = rc ? F.c[2] : F.c[3];
  const double* s3 = rc ? F.s[2] : F.s[3];
  const long long total = (long long)(rc ? M : N) * E2;
  FTC_LAUNCH(k_result_init<<<1, 1, 0, s>>>(r));
  FTC_LAUNCH(k_line_scan<<<grid_for(total), kT, 0, s>>>(c1, s1, c3, s3, total, rc ? N : M, tau, r));
  FTC_LAUNCH(k_line_decide<<<1, 1, 0, s>>>(r));
  FTC_LAUNCH(k_line_emit<<<grid_for(total), kT, 0, s>>>(c1, s1, total, E2, rc, tau, r, p));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int run_fc_analyze(const Fam& F, int N, int M, int E2, double tau, SchemeResult* r,
                   const Patches& p, uint8_t* colmask, uint8_t* rowmask, int32_t* colany,
                   int32_t* rowany, cudaStream_t s) {
  FTC_LAUNCH(k_result_init<<<1, 1, 0, s>>>(r));
  FTC_CUDA_CHECK(cudaMemsetAsync(colany, 0, sizeof(int32_t) * M, s));
  FTC_CUDA_CHECK(cudaMemsetAsync(rowany, 0, sizeof(int32_t) * N, s));
  const long long total = (long long)(M + N + 1) * E2;
  FTC_LAUNCH(k_fc_scan<<<grid_for(total), kT, 0, s>>>(F, N, M, E2, tau, colmask, rowmask, colany, rowany, r));
  FTC_LAUNCH(k_fc_decide<<<1, 1024, 0, s>>>(F, N, M, E2, tau, colany, rowany, r));
  FTC_LAUNCH(k_fc_emit<<<grid_for((long long)(M > N ? M : N) * E2), kT, 0, s>>>(F, N, M, E2, colmask, rowmask,
                                                                      r, p));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int run_verify(const Fam& F, unsigned trusted, const float* O, int N, int M, int E2, int bias,
               const float* bias_dev, const double* agg, double tau, const Patches& p,
               const SchemeResult* r_dev, int np, const VerifyWS& ws, int32_t* fail,
               cudaStream_t s) {
  (void)r_dev;
  FTC_CUDA_CHECK(cudaMemsetAsync(fail, 0, sizeof(int32_t), s));
  if (np > 0) {
    k_verify_apply<<<grid_for(np), kT, 0, s>>>(p, np, M, E2, O, ws);
    count_launch();
  }
  if (trusted & (FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7)) {
    FTC_CUDA_CHECK(cudaMemsetAsync(ws.tcount, 0, sizeof(int), s));
    FTC_LAUNCH(k_touched_list<<<grid_for(E2), kT, 0, s>>>(ws.touched5, E2, ws.tlist, ws.tcount));
    const VirtualO v{O, ws.ov, ws.present};
    if (const int st_ = launch_seq_sums567(v, N, M, E2, ws.tlist, ws.tcount, bias ? agg : nullptr,
                          (trusted & FTC_CK_O5) ? ws.fresh : nullptr,
                          (trusted & FTC_CK_O6) ? ws.fresh + E2 : nullptr,
                          (trusted & FTC_CK_O7) ? ws.fresh + 2 * (long long)E2 : nullptr, s))
      return st_;
    FTC_LAUNCH(k_verify_pos<<<grid_for(E2), kT, 0, s>>>(F, trusted, E2, tau, ws, fail));
  }
  if (trusted & (FTC_CK_O1 | FTC_CK_O3))
    FTC_LAUNCH(k_verify_col<<<(int)(((long long)M * E2 + kT - 1) / kT), kT, 0, s>>>(
        F, trusted, O, bias ? bias_dev : nullptr, N, M, E2, tau, ws, fail));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int run_rollback(const Patches& p, int np, int M, int E2, const VerifyWS& ws, cudaStream_t s) {
  if (np > 0) {
    k_rollback<<<grid_for(np), kT, 0, s>>>(p, np, M, E2, ws);
    count_launch();
  }
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int run_patch_planes(const Patches& p, int np, int M, uint32_t* mask, cudaStream_t s) {
  if (np > 0) {
    k_patch_planes<<<grid_for(np), kT, 0, s>>>(p, np, M, mask);
    count_launch();
  }
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int run_apply_faults(const ftc_fault* f_dev, int nf, int target, void* t, bool is_f64, const double* tab, int d1,
                     int d2, int d3, long long count, cudaStream_t s) {
  if (is_f64)
    FTC_LAUNCH(k_apply_faults<double><<<grid_for(count), kT, 0, s>>>(f_dev, nf, target, (double*)t, d1, d2,
                                                          d3, count, tab));
  else
    FTC_LAUNCH(k_apply_faults<float><<<grid_for(count), kT, 0, s>>>(f_dev, nf, target, (float*)t, d1, d2, d3,
                                                         count, tab));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // namespace ftc
