// ftc_checksums.cu -- FP64 checksum, summation and CoC-D kernels.
//
// Everything the error path consumes is computed in the reference's association
// order (one thread owns one output and walks the reduced index ascending), so at
// T=double the results are bitwise equal to checksums.hpp on the same FP32 data;
// the clean-path detection (Co5 fast, fused So5) trades that for parallelism.
#include <cuda_runtime.h>
#include <stdlib.h>

#include "ftc_common.cuh"

namespace ftc {

namespace {

constexpr int kThreads = 256;

inline int blocks_for(long long n, int threads = kThreads) {
  long long b = (n + threads - 1) / threads;
  return (int)(b < 1 ? 1 : b);
}

// ------------------------------------------------------------------ K2: input_checksums
// checksums.hpp:100-107.  Thread = 4 consecutive (k,a,b) positions; the batch loop
// is fully independent across n (loads in flight) and accumulates n ascending.
// HBM-bound: reads |D|, writes 2 x C*H*H doubles.
__global__ void __launch_bounds__(kThreads) k_input_checksums_v4(const float* __restrict__ D, int N,
                                                                 long long per4,
                                                                 double* __restrict__ cd1,
                                                                 double* __restrict__ cd2) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per4) return;
  const float4* src = reinterpret_cast<const float4*>(D) + e;
  double s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0};
  int n = 0;
  for (; n + 4 <= N; n += 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(src + (long long)(n + u) * per4);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double w = (double)(n + u);
      const double a[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s1[q] = dadd(s1[q], a[q]);
        s2[q] = dadd(s2[q], dmul(w, a[q]));
      }
    }
  }
  for (; n < N; ++n) {
    const float4 v = __ldg(src + (long long)n * per4);
    const double w = (double)n;
    const double a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      s1[q] = dadd(s1[q], a[q]);
      s2[q] = dadd(s2[q], dmul(w, a[q]));
    }
  }
  double2* o1 = reinterpret_cast<double2*>(cd1) + 2 * e;
  double2* o2 = reinterpret_cast<double2*>(cd2) + 2 * e;
  o1[0] = make_double2(s1[0], s1[1]);
  o1[1] = make_double2(s1[2], s1[3]);
  o2[0] = make_double2(s2[0], s2[1]);
  o2[1] = make_double2(s2[2], s2[3]);
}

__global__ void k_input_checksums_scalar(const float* __restrict__ D, int N, long long per,
                                         double* __restrict__ cd1, double* __restrict__ cd2) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per) return;
  double s1 = 0.0, s2 = 0.0;
  int n = 0;
  for (; n + 16 <= N; n += 16) {  // 16 loads in flight, then the ordered adds
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(D + (long long)(n + u) * per + e);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      s1 = dadd(s1, (double)v[u]);
      s2 = dadd(s2, dmul((double)(n + u), (double)v[u]));
    }
  }
  for (; n < N; ++n) {
    const double v = __ldg(D + (long long)n * per + e);
    s1 = dadd(s1, v);
    s2 = dadd(s2, dmul((double)n, v));
  }
  cd1[e] = s1;
  cd2[e] = s2;
}

// ------------------------------------------------------------------ K3: kernel_checksums
// checksums.hpp:78-87: position (g*Ckw + k, i, j) sums kernels m of group g ascending
// with the GLOBAL index m as weight.
__global__ void k_kernel_checksums(const float* __restrict__ W, int M, int Ckw, int R, int groups,
                                   double* __restrict__ cw1, double* __restrict__ cw2) {
  const int per = Ckw * R * R;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per * groups) return;
  const int g = e / per, r = e % per, mpg = M / groups;
  double s1 = 0.0, s2 = 0.0;
  for (int mg0 = 0; mg0 < mpg; mg0 += 8) {  // 8 loads in flight, then the ordered adds
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = mg0 + u < mpg ? (double)W[(long long)(g * mpg + mg0 + u) * per + r] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (mg0 + u < mpg) {
        s1 = dadd(s1, v[u]);
        s2 = dadd(s2, dmul((double)(g * mpg + mg0 + u), v[u]));
      }
    }
  }
  cw1[e] = s1;
  cw2[e] = s2;
}

// ------------------------------------------------------------------ K4: exact FP64 conv
// conv_direct (conv.hpp:39-62) at T=double: one thread per output, (k,i,j) ascending,
// padded taps contribute 0*w exactly like padded_at (:28-37).
template <typename TI, typename TW>
struct ExactJobs {  // up to three independent convolutions in one launch (blockIdx.y)
  const TI* in[3];
  const TW* w[3];
  double* out[3];
};
template <typename TI, typename TW, int RT>
__global__ void k_conv_f64_exact(ExactJobs<TI, TW> jobs, int B, int Cin, int H, int Mo, int Ckw, int Rrt, int U,
                                 int pad, int groups, int E) {
  const TI* __restrict__ in = jobs.in[blockIdx.y];
  const TW* __restrict__ w = jobs.w[blockIdx.y];
  double* __restrict__ out = jobs.out[blockIdx.y];
  const int R = RT > 0 ? RT : Rrt;
  const long long total = (long long)B * Mo * E * E;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int y = (int)(idx % E);
  const int x = (int)((idx / E) % E);
  const int mo = (int)((idx / ((long long)E * E)) % Mo);
  const int b = (int)(idx / ((long long)E * E * Mo));
  const int mpg = Mo / groups;
  const int kbase = (mo / mpg) * Ckw;
  const TI* src = in + ((long long)b * Cin + kbase) * H * H;
  const TW* ker = w + (long long)mo * Ckw * R * R;
  double acc = 0.0;
  if constexpr (RT > 0) {
    // the k x R x R window's loads issue together; the products are added in (k, i, j) order
    uint32_t vmask = 0;
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int j = 0; j < RT; ++j) {
        const int hh = U * x + i - pad, ww = U * y + j - pad;
        if (hh >= 0 && hh < H && ww >= 0 && ww < H) vmask |= 1u << (i * RT + j);
      }
    const long long o0 = (long long)(U * x - pad) * H + (U * y - pad);
    for (int k = 0; k < Ckw; ++k) {
      double v[RT * RT], wv[RT * RT];
#pragma unroll
      for (int t = 0; t < RT * RT; ++t) {
        v[t] = ((vmask >> t) & 1u) ? (double)src[(long long)k * H * H + o0 + (t / RT) * H + (t % RT)] : 0.0;
        wv[t] = (double)ker[k * RT * RT + t];
      }
#pragma unroll
      for (int t = 0; t < RT * RT; ++t) acc = dadd(acc, dmul(v[t], wv[t]));
    }
  } else {
    for (int k = 0; k < Ckw; ++k)
      for (int i = 0; i < R; ++i) {
        const int hh = U * x + i - pad;
        const bool rok = hh >= 0 && hh < H;
        for (int j = 0; j < R; ++j) {
          const int ww = U * y + j - pad;
          double v = 0.0;
          if (rok && ww >= 0 && ww < H) v = (double)src[((long long)k * H + hh) * H + ww];
          acc = dadd(acc, dmul(v, (double)ker[(k * R + i) * R + j]));
        }
      }
  }
  out[idx] = acc;
}

// BiasAdjuster ctor (checksums.hpp:199-208) at T=double
__global__ void k_bias_aggregates(const float* __restrict__ b, int M, double* agg) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double sb = 0.0, smb = 0.0;
  for (int m = 0; m < M; ++m) {
    const double v = b[m];
    sb = dadd(sb, v);
    smb = dadd(smb, dmul((double)m, v));
  }
  agg[0] = sb;
  agg[1] = smb;
}

// ------------------------------------------------------------------ K5: output_summations
__device__ __forceinline__ double vo(const VirtualO& v, long long i) {
  if (v.present && v.present[i]) return v.ov[i];
  return (double)v.O[i];
}

// So1/So3 (per column m, n ascending) + bias rows (checksums.hpp:212-220)
__global__ void k_sum_cols(VirtualO v, int N, int M, int E2, uint32_t which, const float* bias,
                           double* so1, double* so3) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)M * E2) return;
  const int m = (int)(q / E2), f = (int)(q % E2);
  double s1 = 0.0, s3 = 0.0;
  for (int n0 = 0; n0 < N; n0 += 8) {  // 8 loads in flight, then the ordered adds
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = n0 + u < N ? vo(v, ((long long)(n0 + u) * M + m) * E2 + f) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (n0 + u < N) {
        s1 = dadd(s1, x[u]);
        s3 = dadd(s3, dmul((double)(n0 + u), x[u]));
      }
    }
  }
  if (bias) {
    const double b = bias[m];
    s1 = dsub(s1, dmul((double)N, b));
    s3 = dsub(s3, dmul((double)((long long)N * (N - 1) / 2), b));
  }
  if (which & FTC_CK_O1) so1[q] = s1;
  if (which & FTC_CK_O3) so3[q] = s3;
}

// So2/So4 (per row n, m ascending) (checksums.hpp:215-223)
__global__ void k_sum_rows(VirtualO v, int N, int M, int E2, uint32_t which, const double* agg,
                           double* so2, double* so4) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)N * E2) return;
  const int n = (int)(q / E2), f = (int)(q % E2);
  double s2 = 0.0, s4 = 0.0;
  for (int m0 = 0; m0 < M; m0 += 8) {  // 8 loads in flight, then the ordered adds
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = m0 + u < M ? vo(v, ((long long)n * M + m0 + u) * E2 + f) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (m0 + u < M) {
        s2 = dadd(s2, x[u]);
        s4 = dadd(s4, dmul((double)(m0 + u), x[u]));
      }
    }
  }
  if (agg) {
    s2 = dsub(s2, agg[0]);
    s4 = dsub(s4, agg[1]);
  }
  if (which & FTC_CK_O2) so2[q] = s2;
  if (which & FTC_CK_O4) so4[q] = s4;
}

// So5/So6/So7 (checksums.hpp:176-189): for every position the (n, m) sequence, n outer,
// m inner, summed strictly in order -- one chain of N*M dependent FP64 adds per position
// and family (32768 at AlexNet conv2), so the kernel is bound by how fast a chain steps
// (DADD latency 8.2 cycles on B200, tools/ubench_fp64.cu).  A warp owns one (position,
// family): lane l loads term q = 32b + l of batch b and forms its product
// y = w(q) * x(q) (exact: w = 1, m or n), and the chain walks the batch with shuffles,
// s = dadd(s, y of lane u) for u = 0..31 -- two SHFL and one DADD per term, the shuffles
// independent of s, so the chain runs at the add latency.  Batches are loaded three
// ahead (registers).  The three families of a position are adjacent warps of one block
// and share the position's sectors in L1.  (A warp per position with lane 0 adding from
// shared memory took ~1 ms per call at conv2; a lane per position with a cp.async ring,
// ~2 ms: the per-lane copy instructions, not the adds, set the pace,
// tools/ubench_seq.cu.)
constexpr int kSeqWarps = 3;  // warps per block: the three families of one position
#ifndef FTC_SEQ_AHEAD
#define FTC_SEQ_AHEAD 4
#endif
constexpr int kSeqAhead = FTC_SEQ_AHEAD;  // 32-term batches loaded ahead of the chain
template <bool VIRT>
__global__ void __launch_bounds__(32 * kSeqWarps) k_seq_sums567(VirtualO v, int N, int M, int E2,
                                                                const int* __restrict__ list,
                                                                const int* __restrict__ count, const double* agg,
                                                                double* __restrict__ so5, double* __restrict__ so6,
                                                                double* __restrict__ so7, int dbg) {
  (void)dbg;
  const int lane = threadIdx.x & 31, fam = threadIdx.x >> 5;
  const int p = blockIdx.x;
  const int npos = list ? *count : E2;
  if (p >= npos) return;
  double* out = fam == 0 ? so5 : fam == 1 ? so6 : so7;
  if (!out) return;  // whole warp
  const int f = list ? list[p] : p;
  const long long NM = (long long)N * M;
  const long long nb = (NM + 31) / 32;
  // this lane's term of batch b, weighted (exact product); terms past the end are +0.0,
  // which leaves a sum that started at +0.0 unchanged
  auto term = [&](long long b) -> double {
    const long long q = b * 32 + lane;
    if (q >= NM) return 0.0;
    const long long idx = q * E2 + f;
    double x = (double)__ldg(v.O + idx);
    if (VIRT && __ldg(v.present + idx)) x = __ldg(v.ov + idx);
    if (fam == 0) return x;
    const int n = (int)(q / M), m = (int)(q - (long long)n * M);
    return dmul((double)(fam == 1 ? m : n), x);
  };
  double s = 0.0;
  auto walk = [&](double y) {
    double t[32];  // all of the batch's shuffles first, then the 32 dependent adds
#pragma unroll
    for (int u = 0; u < 32; ++u) t[u] = __shfl_sync(0xffffffffu, y, u);
#pragma unroll
    for (int u = 0; u < 32; ++u) s = dadd(s, t[u]);
  };
  // kSeqAhead batches in flight (registers, rotated by a fully unrolled inner loop)
  double y[kSeqAhead];
#pragma unroll
  for (int k = 0; k < kSeqAhead; ++k) y[k] = term(k);
  for (long long b = 0; b < nb; b += kSeqAhead) {
#pragma unroll
    for (int k = 0; k < kSeqAhead; ++k) {
      if (b + k < nb) {
        const double cur = y[k];
        y[k] = term(b + k + kSeqAhead);
        walk(cur);
      }
    }
  }
  if (lane != 0) return;
  if (agg) {  // BiasAdjuster (checksums.hpp:226-235)
    const double nN = (double)N, wnn = (double)((long long)N * (N - 1) / 2);
    s = dsub(s, fam == 0 ? dmul(nN, agg[0]) : fam == 1 ? dmul(nN, agg[1]) : dmul(wnn, agg[0]));
  }
  out[f] = s;
}

// So5/So6/So7, staged form: a block owns 32 positions.  Warp 0 is the chain warp, a lane
// per position running its three chains (s5, s6, s7: three independent DADDs per term, so
// the add latency is covered); the 12 warps on the other three sub-partitions stage the
// terms ahead of it: coalesced loads of O (lane = position), the verifier's FP64
// overrides, the exact products m*x and n*x, written as FP64 rows [family][term][32
// positions] into a double-buffered shared-memory tile.  The loaders hold the next two
// tiles in registers, so a load has two chain tiles (~3K cycles each) to land.  Same
// operations in the same order as k_seq_sums567 (n outer, m inner; x, m*x, n*x exact
// products, one DADD each), hence bitwise the same sums, at ~23 cycles per term instead
// of ~50 (one chain per warp fed by shuffles): AlexNet conv2 So5-7 877 -> 393 us.
constexpr int kStT = 128;        // terms per staged tile
constexpr int kStLW = 12;            // loader warps: warps 1-15 of the block except 4, 8, 12, so the chain warp's
                                     // scheduler (sub-partition 0) issues for nobody else (7, 15 and 12 loader warps
                                     // measured alike: the chain warp's load -> add order set the pace)
constexpr int kStLoad = kStLW * 32;  // loader threads
constexpr int kStPer = (kStT * 32 + kStLoad - 1) / kStLoad;  // elements per loader thread and tile
template <bool VIRT>
__global__ void __launch_bounds__(512) k_seq_sums567_staged(VirtualO v, int N, int M, int E2,
                                                          const int* __restrict__ list,
                                                          const int* __restrict__ count, const double* agg,
                                                          double* __restrict__ so5, double* __restrict__ so6,
                                                          double* __restrict__ so7) {
  extern __shared__ double st_tile[];  // [2][3][kStT][32]
  const int npos = list ? *count : E2;
  const int p0 = blockIdx.x * 32;
  if (p0 >= npos) return;  // whole block
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long NM = (long long)N * M;
  const int ntile = (int)((NM + kStT - 1) / kStT);
  const int pl = p0 + lane;
  const bool pok = pl < npos;
  const int f = pok ? (list ? list[pl] : pl) : 0;
  // loader state: element e = li + kStLoad * j of a tile is (term e / 32, position e % 32);
  // a warp's lanes share the term and cover the 32 positions.  Two tiles of loads are in
  // flight in registers (fetched two barriers before they are stashed), and the weights
  // (double)m, (double)n advance incrementally (a term step of kStLW per element): no integer
  // division or int -> FP64 conversion per element.
  const bool loader = (warp & 3) != 0;
  const int li = ((warp >> 2) * 3 + (warp & 3) - 1) * 32 + lane;  // loaders: 0 .. kStLoad - 1
  float xr[2][kStPer];
  uint8_t pr[2][kStPer];
  // element j of a tile: term row tr + kStLW j (tr = li / 32), valid rows < kStT -- only
  // j = kStPer - 1 can fall off the tile (rows 126, 127 exist for tr < 2)
  const int tr = li >> 5;
  const long long step = (long long)kStLW * E2;
  // loads are unconditional: lanes without a position read lane 0's (f = 0 region is
  // valid memory; their sums are never written), and rows past N*M in the last tile are
  // clamped to the last term (the chain never reads those rows)
  auto fetch = [&](int tile, int rs) {
    const long long q0 = (long long)tile * kStT + tr;
    if ((long long)(tile + 1) * kStT <= NM) {
      const float* src = v.O + q0 * E2 + f;
      const uint8_t* psrc = VIRT ? v.present + q0 * E2 + f : nullptr;
#pragma unroll
      for (int j = 0; j < kStPer - 1; ++j) {
        xr[rs][j] = __ldg(src);
        if (VIRT) pr[rs][j] = __ldg(psrc);
        src += step;
        if (VIRT) psrc += step;
      }
      if (tr < kStT - kStLW * (kStPer - 1)) {
        xr[rs][kStPer - 1] = __ldg(src);
        if (VIRT) pr[rs][kStPer - 1] = __ldg(psrc);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kStPer; ++j) {
        const long long q = min(q0 + kStLW * j, NM - 1);
        xr[rs][j] = __ldg(v.O + q * E2 + f);
        if (VIRT) pr[rs][j] = __ldg(v.present + q * E2 + f);
      }
    }
  };
  const double dM = (double)M;
  auto stash = [&](int tile, int b, int rs) {
    double* t5 = st_tile + (size_t)b * 3 * kStT * 32 + li;
    const unsigned q0 = (unsigned)tile * kStT + (unsigned)tr;
    const unsigned n0 = q0 / (unsigned)M;
    double dn = (double)n0, dm = (double)(q0 - n0 * (unsigned)M);
#pragma unroll
    for (int j = 0; j < kStPer; ++j) {
      if (j < kStPer - 1 || tr < kStT - kStLW * (kStPer - 1)) {
        double x = (double)xr[rs][j];
        if (VIRT && pr[rs][j]) x = __ldg(v.ov + min((long long)q0 + kStLW * j, NM - 1) * E2 + f);
        t5[kStLoad * j] = x;  // rows past N*M hold values the chain never reads
        t5[kStLoad * j + kStT * 32] = dmul(dm, x);
        t5[kStLoad * j + 2 * kStT * 32] = dmul(dn, x);
      }
      dm += (double)kStLW;  // exact small integers in FP64; M >= kStLW (launcher), so one wrap at most
      if (dm >= dM) {
        dm -= dM;
        dn += 1.0;
      }
    }
  };
  if (loader) {
    fetch(0, 0);
    if (ntile > 1) fetch(1, 1);
    stash(0, 0, 0);
    if (ntile > 2) fetch(2, 0);
  }
  __syncthreads();
  double s5 = 0.0, s6 = 0.0, s7 = 0.0;
  for (int k = 0; k < ntile; ++k) {
    if (loader) {
      // tile k+1 sits in register set (k+1)&1 (fetched an iteration ago); once stashed,
      // that set takes tile k+3
      if (k + 1 < ntile) {
        if ((k + 1) & 1) {
          stash(k + 1, 1, 1);
          if (k + 3 < ntile) fetch(k + 3, 1);
        } else {
          stash(k + 1, 0, 0);
          if (k + 3 < ntile) fetch(k + 3, 0);
        }
      }
    } else if (warp == 0) {
      const double* t5 = st_tile + (size_t)(k & 1) * 3 * kStT * 32 + lane;
      const double* t6 = t5 + kStT * 32;
      const double* t7 = t6 + kStT * 32;
      const int nt = (int)min((long long)kStT, NM - (long long)k * kStT);
      int t = 0;
      // all 24 loads of a batch issue before its adds (volatile asm keeps the order: left
      // to the compiler the loads were interleaved four at a time with the adds and every
      // add waited out a shared-memory latency, ~32 cycles per term; a double-buffered
      // form with the next batch's loads ahead of the current adds measured no faster)
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(t5);
      for (; t + 8 <= nt; t += 8) {
        double a[8], b[8], c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t ad = sa + (uint32_t)(t + u) * 256u;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[u]) : "r"(ad));
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(b[u]) : "r"(ad + (uint32_t)kStT * 256u));
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(c[u]) : "r"(ad + 2u * (uint32_t)kStT * 256u));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(s5) : "d"(a[u]));
          asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(s6) : "d"(b[u]));
          asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(s7) : "d"(c[u]));
        }
      }
      for (; t < nt; ++t) {
        s5 = dadd(s5, t5[t * 32]);
        s6 = dadd(s6, t6[t * 32]);
        s7 = dadd(s7, t7[t * 32]);
      }
    }
    __syncthreads();
  }
  if (warp != 0 || !pok) return;
  if (agg) {  // BiasAdjuster (checksums.hpp:226-235)
    const double nN = (double)N, wnn = (double)((long long)N * (N - 1) / 2);
    s5 = dsub(s5, dmul(nN, agg[0]));
    s6 = dsub(s6, dmul(nN, agg[1]));
    s7 = dsub(s7, dmul(wnn, agg[0]));
  }
  if (so5) so5[f] = s5;
  if (so6) so6[f] = s6;
  if (so7) so7[f] = s7;
}

// ------------------------------------------------------------------ K6: CoC-D
__device__ __forceinline__ void detect_one(double c, double s, double tau, int* flagged,
                                           unsigned long long* mrd_bits, bool* bad) {
  double den = fabs(c);
  if (den < fabs(s)) den = fabs(s);
  if (den < 1.0) den = 1.0;
  const double dev = fabs(c - s) / den;
  // std::max(a,b) = a<b?b:a ignores NaN devs; non-negative doubles order as u64
  if (dev == dev && dev > 0.0) atomicMax(mrd_bits, (unsigned long long)__double_as_longlong(dev));
  *bad = values_differ(c, s, tau);
  if (*bad) atomicAdd(flagged, 1);
}

__global__ void k_detect_exact(const double* __restrict__ co5, const double* __restrict__ so5,
                               int E2, double tau, uint8_t* mask, DetectStats* st) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= E2) return;
  bool bad;
  detect_one(co5[f], so5[f], tau, &st->flagged, &st->max_rel_dev_bits, &bad);
  if (mask) mask[f] = bad ? 1 : 0;
}

__global__ void k_count_differ(const double* __restrict__ c, const double* __restrict__ s,
                               long long n, double tau, int* count) {
  int local = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (values_differ(c[i], s[i], tau)) ++local;
  if (local) atomicAdd(count, local);
}

// Clean-path Cd1 only (CoC-D needs Co5 = Cd1 (*) Cw1; Cd2 feeds only the weighted
// families of the error path, which recomputes both exactly).  Two positions per
// thread, eight images in flight per thread: enough bytes in flight to stream D at
// HBM rate.
__global__ void __launch_bounds__(128) k_cd1_fast(const float* __restrict__ D, int N, long long per4,
                                                  double* __restrict__ cd1) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per4) return;
  const float4* src = reinterpret_cast<const float4*>(D) + e;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int n = 0;
  for (; n + 16 <= N; n += 16) {
    float4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldcs(src + (long long)(n + u) * per4);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 += v[u].x;
      a1 += v[u].y;
      a2 += v[u].z;
      a3 += v[u].w;
    }
  }
  for (; n < N; ++n) {
    const float4 v = __ldg(src + (long long)n * per4);
    a0 += v.x;
    a1 += v.y;
    a2 += v.z;
    a3 += v.w;
  }
  double2* o = reinterpret_cast<double2*>(cd1) + 2 * e;
  o[0] = make_double2(a0, a1);
  o[1] = make_double2(a2, a3);
}

// Adaptive forms for the clean path: a 256-thread block covers P positions x S slices
// (S = 256 / P) so a layer with few positions still fills the GPU and each thread does
// only a few channels (Co5) or batch terms (So5) -- the fixed 32-position blocks left
// 13x13 layers on 6 blocks with 24-48 serial steps per thread.
template <int RT>
__global__ void __launch_bounds__(256) k_co5_adapt(const double* __restrict__ cd1, const double* __restrict__ cw1,
                                                  double* __restrict__ co5, int C, int H, int Rrt, int U, int pad,
                                                  int E, int P) {
  __shared__ double red[256];
  const int R = RT > 0 ? RT : Rrt, RR = R * R, E2 = E * E, S = 256 / P;
  const int t = threadIdx.x, pl = t % P, sl = t / P;
  const int f = blockIdx.x * P + pl;
  double c5 = 0.0;
  if (f < E2) {
    const int x = f / E, y = f - (f / E) * E;
    const int hb = x * U - pad, wb = y * U - pad;
    for (int c = sl; c < C; c += S) {
      const double* src = cd1 + (long long)c * H * H;
      const double* ker = cw1 + c * RR;
      if constexpr (RT > 0) {
        double v[RT * RT];
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
          for (int j = 0; j < RT; ++j) {
            const bool ok = (unsigned)(hb + i) < (unsigned)H && (unsigned)(wb + j) < (unsigned)H;
            v[i * RT + j] = ok ? __ldg(src + (hb + i) * H + wb + j) : 0.0;
          }
#pragma unroll
        for (int q = 0; q < RT * RT; ++q) c5 = fma(v[q], __ldg(ker + q), c5);
      } else {
        for (int i = 0; i < R; ++i) {
          const int hh = hb + i;
          if (hh < 0 || hh >= H) continue;
          for (int j = 0; j < R; ++j) {
            const int ww = wb + j;
            if (ww < 0 || ww >= H) continue;
            c5 = fma(__ldg(src + hh * H + ww), __ldg(ker + i * R + j), c5);
          }
        }
      }
    }
  }
  red[t] = c5;
  __syncthreads();
  if (t < P && f < E2) {
    double cc = 0.0;
    for (int q = 0; q < S; ++q) cc += red[q * P + t];
    co5[f] = cc;
  }
}

__global__ void __launch_bounds__(256) k_detect_adapt(double* __restrict__ co5,
                                                     const double* __restrict__ rowsum, int parts, int N, int E2,
                                                     int bias, const double* agg, double tau, DetectStats* st,
                                                     unsigned int* ticket, DetectStats* host_out, int P) {
  __shared__ double red[256];
  const int S = 256 / P;
  const int t = threadIdx.x, pl = t % P, sl = t / P;
  const int f = blockIdx.x * P + pl;
  double s5 = 0.0;
  if (f < E2) {
    const long long slab = (long long)N * E2;
    const int terms = N * parts;
    for (int q = sl; q < terms; q += S) {
      const int sq = q / N, n = q - sq * N;
      s5 += __ldg(rowsum + sq * slab + (long long)n * E2 + f);
    }
  }
  red[t] = s5;
  __syncthreads();
  if (t < 32) {
    int bad = 0;
    unsigned long long devb = 0ull;
    for (int pp = t; pp < P; pp += 32) {
      const int ff = blockIdx.x * P + pp;
      if (ff >= E2) continue;
      double ss = 0.0;
      for (int q = 0; q < S; ++q) ss += red[q * P + pp];
      if (bias) ss -= (double)N * agg[0];
      const double c = co5[ff];
      co5[ff] = 0.0;  // keep the clean-path Co5 buffer zero between calls
      double den = fabs(c);
      if (den < fabs(ss)) den = fabs(ss);
      if (den < 1.0) den = 1.0;
      const double dev = fabs(c - ss) / den;
      if (dev == dev && dev > 0.0) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(dev);
        devb = b > devb ? b : devb;
      }
      bad += values_differ_guarded(c, ss, tau) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bad += __shfl_xor_sync(0xffffffffu, bad, o);
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, devb, o);
      devb = other > devb ? other : devb;
    }
    if (t == 0) {
      if (bad) atomicAdd(&st->flagged, bad);
      if (devb) atomicMax(&st->max_rel_dev_bits, devb);
      __threadfence();
      const unsigned int done = atomicAdd(ticket, 1u);
      if (done == gridDim.x - 1) {  // last block: publish and reset
        __threadfence();
        const int fl = atomicExch(&st->flagged, 0);
        const unsigned long long mb = atomicExch(&st->max_rel_dev_bits, 0ull);
        volatile DetectStats* h = host_out;
        h->flagged = fl;
        h->max_rel_dev_bits = mb;
        __threadfence_system();
        *ticket = 0u;
      }
    }
  }
}

// Co5 tap table of the fused clean path: k = (c*R + i)*R + j (the conv_block order)
__global__ void k_co5_taps(const double* __restrict__ cw1, int C, int H, int R, Co5Tap* taps) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= C * R * R) return;
  const int c = k / (R * R), ij = k % (R * R), i = ij / R, j = ij % R;
  Co5Tap t;
  t.off = c * H * H + i * H + j;
  t.i = (short)i;
  t.j = (short)j;
  t.w = cw1[k];
  taps[k] = t;
}

// CoC-D of the fused clean path: So5 was accumulated by the conv epilogue (FP64 atomics,
// bias not yet removed), Co5 by its checksum warp.  One thread per position compares
// them (values_differ, checksums.hpp:54-60) and re-zeroes So5; the last block publishes
// {flagged, max_rel_dev} into the mapped host record and re-arms the counters.
// One-block CoC-D for E2 <= kDetect1Max (experiment, FTC_DETECT_1BLOCK=1): a thread
// walks E2 / 1024 positions, the block reduces the count and the max deviation through
// shared memory and thread 0 publishes the record -- no grid-wide fence/ticket/atomics.
// Same 8 us under ncu as the multi-block kernel, and config 1's protected step went from
// 69 to 86 us with it (one SM, behind the persistent conv), so it is off.
constexpr int kDetect1Max = 8192;
__global__ void __launch_bounds__(1024) k_detect_fused1(double* __restrict__ co5, double* __restrict__ so5, int N,
                                                       int E2, int bias, const double* agg, double tau,
                                                       DetectStats* host_out) {
  __shared__ int s_bad[32];
  __shared__ unsigned long long s_dev[32];
  pdl_trigger();
  pdl_wait();
  int bad = 0;
  unsigned long long devb = 0ull;
  const double bsum = bias ? (double)N * agg[0] : 0.0;
  for (int f = threadIdx.x; f < E2; f += blockDim.x) {
    double ss = __ldcg(so5 + f);
    so5[f] = 0.0;
    if (bias) ss -= bsum;
    const double c = __ldcg(co5 + f);
    co5[f] = 0.0;  // Co5 may have been scattered (staging pass): re-arm it too
    double den = fabs(c);
    if (den < fabs(ss)) den = fabs(ss);
    if (den < 1.0) den = 1.0;
    const double dev = fabs(c - ss) / den;
    if (dev == dev && dev > 0.0) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(dev);
      devb = b > devb ? b : devb;
    }
    bad += values_differ_guarded(c, ss, tau) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, devb, o);
    devb = other > devb ? other : devb;
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_bad[w] = bad;
    s_dev[w] = devb;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int fl = 0;
    unsigned long long mb = 0ull;
    for (int k = 0; k < nw; ++k) {
      fl += s_bad[k];
      mb = s_dev[k] > mb ? s_dev[k] : mb;
    }
    volatile DetectStats* h = host_out;
    h->flagged = fl;
    h->max_rel_dev_bits = mb;
    __threadfence_system();
  }
}

__global__ void __launch_bounds__(256) k_detect_fused(double* __restrict__ co5, double* __restrict__ so5,
                                                     int N, int E2, int bias, const double* agg, double tau,
                                                     DetectStats* st, unsigned int* ticket, DetectStats* host_out) {
  pdl_trigger();
  pdl_wait();
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  int bad = 0;
  unsigned long long devb = 0ull;
  if (f < E2) {
    double ss = __ldcg(so5 + f);
    so5[f] = 0.0;
    if (bias) ss -= (double)N * agg[0];
    const double c = __ldcg(co5 + f);
    co5[f] = 0.0;  // Co5 may have been scattered (staging pass): re-arm it too
    double den = fabs(c);
    if (den < fabs(ss)) den = fabs(ss);
    if (den < 1.0) den = 1.0;
    const double dev = fabs(c - ss) / den;
    if (dev == dev && dev > 0.0) devb = (unsigned long long)__double_as_longlong(dev);
    bad = values_differ_guarded(c, ss, tau) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, devb, o);
    devb = other > devb ? other : devb;
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(&st->flagged, bad);
    if (devb) atomicMax(&st->max_rel_dev_bits, devb);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(ticket, 1u);
    if (done == gridDim.x - 1) {
      __threadfence();
      const int fl = atomicExch(&st->flagged, 0);
      const unsigned long long mb = atomicExch(&st->max_rel_dev_bits, 0ull);
      volatile DetectStats* h = host_out;
      h->flagged = fl;
      h->max_rel_dev_bits = mb;
      __threadfence_system();
      *ticket = 0u;
    }
  }
}

// Fused clean path, small layers: Co5 (as k_co5_adapt) and CoC-D against the So5 the
// conv accumulated, in one launch after the conv -- Co5 need not exist before it.
template <int RT>
__global__ void __launch_bounds__(256) k_co5_detect(const double* __restrict__ cd1, const double* __restrict__ cw1,
                                                   double* __restrict__ co5, double* __restrict__ so5, int N, int C,
                                                   int H, int Rrt, int U, int pad, int E, int P, int bias,
                                                   const double* agg, double tau, DetectStats* st,
                                                   unsigned int* ticket, DetectStats* host_out) {
  __shared__ double red[256];
  pdl_trigger();
  pdl_wait();
  const int R = RT > 0 ? RT : Rrt, RR = R * R, E2 = E * E, S = 256 / P;
  const int t = threadIdx.x, pl = t % P, sl = t / P;
  const int f = blockIdx.x * P + pl;
  double c5 = 0.0;
  if (f < E2) {
    const int x = f / E, y = f - (f / E) * E;
    const int hb = x * U - pad, wb = y * U - pad;
    for (int c = sl; c < C; c += S) {
      const double* src = cd1 + (long long)c * H * H;
      const double* ker = cw1 + c * RR;
      if constexpr (RT > 0) {
        // the window's loads issued together (predicated, no branches between them):
        // after the large layers' conv this kernel is exposed, one L2 round trip per
        // channel instead of one per tap
        double v[RT * RT], w[RT * RT];
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
          for (int j = 0; j < RT; ++j) {
            const bool ok = (unsigned)(hb + i) < (unsigned)H && (unsigned)(wb + j) < (unsigned)H;
            v[i * RT + j] = ok ? __ldg(src + (hb + i) * H + wb + j) : 0.0;
            w[i * RT + j] = __ldg(ker + i * RT + j);
          }
#pragma unroll
        for (int q = 0; q < RT * RT; ++q) c5 = fma(v[q], w[q], c5);
      } else {
        for (int i = 0; i < R; ++i) {
          const int hh = hb + i;
          if (hh < 0 || hh >= H) continue;
          for (int j = 0; j < R; ++j) {
            const int ww = wb + j;
            if (ww < 0 || ww >= H) continue;
            c5 = fma(__ldg(src + hh * H + ww), __ldg(ker + i * R + j), c5);
          }
        }
      }
    }
  }
  red[t] = c5;
  __syncthreads();
  int bad = 0;
  unsigned long long devb = 0ull;
  if (t < P && f < E2) {
    double c = 0.0;
    for (int q = 0; q < S; ++q) c += red[q * P + t];
    co5[f] = 0.0;  // the clean-path Co5 buffer is zero between calls (the staging pass scatters into it)
    double ss = __ldcg(so5 + f);
    so5[f] = 0.0;
    if (bias) ss -= (double)N * agg[0];
    double den = fabs(c);
    if (den < fabs(ss)) den = fabs(ss);
    if (den < 1.0) den = 1.0;
    const double dev = fabs(c - ss) / den;
    if (dev == dev && dev > 0.0) devb = (unsigned long long)__double_as_longlong(dev);
    bad = values_differ_guarded(c, ss, tau) ? 1 : 0;
  }
  if (t < 32) {  // P <= 32: the compares live in warp 0
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bad += __shfl_xor_sync(0xffffffffu, bad, o);
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, devb, o);
      devb = other > devb ? other : devb;
    }
    if (t == 0) {
      if (bad) atomicAdd(&st->flagged, bad);
      if (devb) atomicMax(&st->max_rel_dev_bits, devb);
      __threadfence();
      const unsigned int done = atomicAdd(ticket, 1u);
      if (done == gridDim.x - 1) {
        __threadfence();
        const int fl = atomicExch(&st->flagged, 0);
        const unsigned long long mb = atomicExch(&st->max_rel_dev_bits, 0ull);
        volatile DetectStats* h = host_out;
        h->flagged = fl;
        h->max_rel_dev_bits = mb;
        __threadfence_system();
        *ticket = 0u;
      }
    }
  }
}

inline int pick_positions(int work_per_position) {
  // slices S ~ work/4 (a few serial steps per thread), P = 256 / S positions per block
  int S = 16;
  while (S < 256 && S * 4 < work_per_position) S <<= 1;
  return 256 / S;
}

}  // namespace

// ------------------------------------------------------------------ launchers
int launch_input_checksums(const float* D, int N, long long per, double* cd1, double* cd2,
                           cudaStream_t s) {
  // vector form when there are enough positions to fill the GPU; otherwise one position
  // per thread with 16 batch loads in flight (small planes are latency-bound)
  const bool vec = (per % 4 == 0) && per >= 4 * 148 * 256 && ((uintptr_t)D % 16 == 0) &&
                   ((uintptr_t)cd1 % 16 == 0) && ((uintptr_t)cd2 % 16 == 0);
  if (vec)
    FTC_LAUNCH(k_input_checksums_v4<<<blocks_for(per / 4), kThreads, 0, s>>>(D, N, per / 4, cd1, cd2));
  else
    FTC_LAUNCH(k_input_checksums_scalar<<<blocks_for(per), kThreads, 0, s>>>(D, N, per, cd1, cd2));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_co5_taps(const double* cw1, int C, int H, int R, Co5Tap* taps, cudaStream_t s) {
  if (R > 32767 || (long long)C * H * H >= (1LL << 31)) return FTC_CONFIG_ERROR;
  FTC_LAUNCH(k_co5_taps<<<blocks_for((long long)C * R * R), kThreads, 0, s>>>(cw1, C, H, R, taps));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_kernel_checksums(const float* W, int M, int Ckw, int R, int groups, double* cw1,
                            double* cw2, cudaStream_t s) {
  const int n = Ckw * R * R * groups;
  FTC_LAUNCH(k_kernel_checksums<<<blocks_for(n), kThreads, 0, s>>>(W, M, Ckw, R, groups, cw1, cw2));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

template <typename TI, typename TW>
void conv_f64_exact_dispatch(const ExactJobs<TI, TW>& j, int nj, int B, int Cin, int H, int Mo, int Ckw, int R,
                             int U, int pad, int groups, int E, int g, cudaStream_t s) {
  const dim3 grid((unsigned)g, (unsigned)nj);
  switch (R) {
    case 1: FTC_LAUNCH(k_conv_f64_exact<TI, TW, 1><<<grid, 128, 0, s>>>(j, B, Cin, H, Mo, Ckw, R, U, pad, groups, E)); break;
    case 3: FTC_LAUNCH(k_conv_f64_exact<TI, TW, 3><<<grid, 128, 0, s>>>(j, B, Cin, H, Mo, Ckw, R, U, pad, groups, E)); break;
    case 5: FTC_LAUNCH(k_conv_f64_exact<TI, TW, 5><<<grid, 128, 0, s>>>(j, B, Cin, H, Mo, Ckw, R, U, pad, groups, E)); break;
    default: FTC_LAUNCH(k_conv_f64_exact<TI, TW, 0><<<grid, 128, 0, s>>>(j, B, Cin, H, Mo, Ckw, R, U, pad, groups, E)); break;
  }
}

int launch_conv_f64_exact(const void* in, bool in_f64, const void* w, bool w_f64, double* out,
                          int B, int Cin, int H, int Mo, int Ckw, int R, int U, int pad,
                          int groups, int E, cudaStream_t s) {
  const long long total = (long long)B * Mo * E * E;
  const int g = blocks_for(total, 128);
  if (in_f64 && w_f64)
    conv_f64_exact_dispatch(ExactJobs<double, double>{{(const double*)in}, {(const double*)w}, {out}}, 1, B, Cin, H,
                            Mo, Ckw, R, U, pad, groups, E, g, s);
  else if (in_f64)
    conv_f64_exact_dispatch(ExactJobs<double, float>{{(const double*)in}, {(const float*)w}, {out}}, 1, B, Cin, H, Mo,
                            Ckw, R, U, pad, groups, E, g, s);
  else if (w_f64)
    conv_f64_exact_dispatch(ExactJobs<float, double>{{(const float*)in}, {(const double*)w}, {out}}, 1, B, Cin, H, Mo,
                            Ckw, R, U, pad, groups, E, g, s);
  else
    conv_f64_exact_dispatch(ExactJobs<float, float>{{(const float*)in}, {(const float*)w}, {out}}, 1, B, Cin, H, Mo,
                            Ckw, R, U, pad, groups, E, g, s);
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_conv_block3(const double* const in[3], const double* const w[3], double* const out[3], int nj, int Cin,
                       int H, int R, int U, int pad, int E, cudaStream_t s) {
  ExactJobs<double, double> j{};
  for (int k = 0; k < nj; ++k) {
    j.in[k] = in[k];
    j.w[k] = w[k];
    j.out[k] = out[k];
  }
  conv_f64_exact_dispatch(j, nj, 1, Cin, H, 1, Cin, R, U, pad, 1, E, blocks_for((long long)E * E, 128), s);
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_bias_aggregates(const float* bias, int M, double* agg, cudaStream_t s) {
  FTC_LAUNCH(k_bias_aggregates<<<1, 32, 0, s>>>(bias, M, agg));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_seq_sums567(const VirtualO& v, int N, int M, int E2, const int* list, const int* count, const double* agg,
                       double* so5, double* so6, double* so7, cudaStream_t s) {
  // long chains (the error path at batch scale): the staged form, a lane per position fed
  // by loader warps; short ones keep the warp-per-chain form (more chains in flight)
  static const bool staged_off = getenv("FTC_SEQ_STAGED") && atoi(getenv("FTC_SEQ_STAGED")) == 0;
  if (!staged_off && M >= kStLW && (long long)N * M >= 1024 && (long long)N * M < (1LL << 31)) {
    const size_t smem = (size_t)2 * 3 * kStT * 32 * sizeof(double);
    // per-device function attribute; the error path is rare, so it is set on every call
    FTC_CUDA_CHECK(cudaFuncSetAttribute(k_seq_sums567_staged<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FTC_CUDA_CHECK(cudaFuncSetAttribute(k_seq_sums567_staged<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const dim3 gs((unsigned)((E2 + 31) / 32));
    if (v.present)
      FTC_LAUNCH(k_seq_sums567_staged<true><<<gs, 512, smem, s>>>(v, N, M, E2, list, count, agg, so5, so6, so7));
    else
      FTC_LAUNCH(k_seq_sums567_staged<false><<<gs, 512, smem, s>>>(v, N, M, E2, list, count, agg, so5, so6, so7));
    FTC_CUDA_CHECK(cudaGetLastError());
    return FTC_OK;
  }
  const dim3 g((unsigned)E2);
  if (v.present)
    FTC_LAUNCH(k_seq_sums567<true><<<g, 32 * kSeqWarps, 0, s>>>(v, N, M, E2, list, count, agg, so5, so6, so7, 0));
  else
    FTC_LAUNCH(k_seq_sums567<false><<<g, 32 * kSeqWarps, 0, s>>>(v, N, M, E2, list, count, agg, so5, so6, so7, 0));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_output_summations(const VirtualO& v, int N, int M, int E, uint32_t which,
                             const float* bias, const double* agg, double* const so[7],
                             cudaStream_t s) {
  const int E2 = E * E;
  if (which & (FTC_CK_O1 | FTC_CK_O3))
    FTC_LAUNCH(k_sum_cols<<<blocks_for((long long)M * E2), kThreads, 0, s>>>(v, N, M, E2, which, bias, so[0],
                                                                   so[2]));
  if (which & (FTC_CK_O2 | FTC_CK_O4))
    FTC_LAUNCH(k_sum_rows<<<blocks_for((long long)N * E2), kThreads, 0, s>>>(v, N, M, E2, which,
                                                                   bias ? agg : nullptr, so[1],
                                                                   so[3]));
  if (which & (FTC_CK_O5 | FTC_CK_O6 | FTC_CK_O7))
    if (const int st_ = launch_seq_sums567(v, N, M, E2, nullptr, nullptr, bias ? agg : nullptr, (which & FTC_CK_O5) ? so[4] : nullptr,
                          (which & FTC_CK_O6) ? so[5] : nullptr, (which & FTC_CK_O7) ? so[6] : nullptr, s))
      return st_;
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_cd1_fast(const float* D, int N, long long per, double* cd1, cudaStream_t s) {
  if (per % 4 != 0 || ((uintptr_t)D % 16) != 0 || ((uintptr_t)cd1 % 16) != 0) {
    // plane size not a multiple of 4: the exact kernel produces Cd1 (and Cd2)
    return FTC_CONFIG_ERROR;
  }
  FTC_LAUNCH(k_cd1_fast<<<blocks_for(per / 4, 128), 128, 0, s>>>(D, N, per / 4, cd1));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_co5_sliced(const double* cd1, const double* cw1, double* co5, int C, int H, int R, int U,
                      int pad, int E, cudaStream_t s) {
  const int P = pick_positions(C);
  const int g = (E * E + P - 1) / P;
  switch (R) {
    case 1: FTC_LAUNCH(k_co5_adapt<1><<<g, 256, 0, s>>>(cd1, cw1, co5, C, H, R, U, pad, E, P)); break;
    case 3: FTC_LAUNCH(k_co5_adapt<3><<<g, 256, 0, s>>>(cd1, cw1, co5, C, H, R, U, pad, E, P)); break;
    case 5: FTC_LAUNCH(k_co5_adapt<5><<<g, 256, 0, s>>>(cd1, cw1, co5, C, H, R, U, pad, E, P)); break;
    default: FTC_LAUNCH(k_co5_adapt<0><<<g, 256, 0, s>>>(cd1, cw1, co5, C, H, R, U, pad, E, P)); break;
  }
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_detect_so5(double* co5, const double* rowsum, int parts, int N, int E2, int bias,
                      const double* agg, double tau, DetectStats* st, unsigned int* ticket,
                      DetectStats* host_out, cudaStream_t s) {
  const int P = pick_positions(N * parts);
  FTC_LAUNCH(k_detect_adapt<<<(E2 + P - 1) / P, 256, 0, s>>>(co5, rowsum, parts, N, E2, bias, agg, tau, st, ticket,
                                                             host_out, P));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_co5_detect(const double* cd1, const double* cw1, double* co5, double* so5, int N, int C, int H, int R,
                      int U, int pad, int E, int bias, const double* agg, double tau, DetectStats* st,
                      unsigned int* ticket, DetectStats* host_out, cudaStream_t s) {
  // positions per block: as many slices as fill ~2 waves of 256-thread blocks, P <= 32
  const int E2 = E * E;
  int P = 32;
  while (P > 1 && (E2 + P - 1) / P < 2 * 148 * 4 && 256 / P < C) P >>= 1;
  const int g = (E2 + P - 1) / P;
#define FTC_C5D(RT)                                                                                                  \
  FTC_LAUNCH_PDL(k_co5_detect<RT>, dim3(g), dim3(256), 0, s, cd1, cw1, co5, so5, N, C, H, R, U, pad, E, P, bias, agg, \
                 tau, st, ticket, host_out)
  switch (R) {
    case 1: FTC_C5D(1); break;
    case 3: FTC_C5D(3); break;
    case 5: FTC_C5D(5); break;
    default: FTC_C5D(0); break;
  }
#undef FTC_C5D
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_detect_fused(double* co5, double* so5, int N, int E2, int bias, const double* agg, double tau,
                        DetectStats* st, unsigned int* ticket, DetectStats* host_out, cudaStream_t s) {
  static const bool one_block = getenv("FTC_DETECT_1BLOCK") != nullptr;  // experiment: slower (see above)
  if (one_block && E2 <= kDetect1Max) {
    FTC_LAUNCH_PDL(k_detect_fused1, dim3(1), dim3(1024), 0, s, co5, so5, N, E2, bias, agg, tau, host_out);
    FTC_CUDA_CHECK(cudaGetLastError());
    return FTC_OK;
  }
  FTC_LAUNCH_PDL(k_detect_fused, dim3(blocks_for(E2)), dim3(kThreads), 0, s, co5, so5, N, E2, bias, agg, tau, st, ticket,
                 host_out);
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_detect_exact(const double* co5, const double* so5, int E2, double tau, uint8_t* mask,
                        DetectStats* st, cudaStream_t s) {
  FTC_LAUNCH(k_detect_exact<<<blocks_for(E2), kThreads, 0, s>>>(co5, so5, E2, tau, mask, st));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_count_differ(const double* c, const double* s_, long long n, double tau, int* count,
                        cudaStream_t s) {
  int g = blocks_for(n);
  if (g > 1184) g = 1184;
  FTC_LAUNCH(k_count_differ<<<g, kThreads, 0, s>>>(c, s_, n, tau, count));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // namespace ftc
