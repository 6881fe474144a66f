// ftc_conv_tc.cu -- tcgen05 implicit-GEMM convolution, 3xTF32 (engine 0).
//
// conv_forward (conv.hpp:114-131) as a GEMM: rows = output pixels p = (n, x, y)
// (128 per tile = UMMA M), columns = kernels m (BN per N-tile), K = (c, i, j) in the
// reference's accumulation order, chunked by 32 (one 128-byte SW128 row of TF32).
//
// FP32 accuracy on TF32 tensor cores: every operand is split v = hi + lo with
// hi = RN_tf32(v) (low 13 mantissa bits zero, read exactly by the tensor core) and
// lo = RN_tf32(v - hi); each K step issues lo*Bhi + hi*Blo + hi*Bhi into one FP32
// TMEM accumulator (the dropped lo*lo term is 2^-22 relative).
//
// Warp roles (persistent CTA per SM, 448 threads):
//   warps 0-3  A producers: gather the im2col row of their pixel straight from D
//              (L1/L2-resident halo), split hi/lo and tcgen05.st it into a TMEM
//              stage (A operand of the TS-form MMA; no shared-memory round trip);
//   warp 4     B loader: one cp.async.bulk per stage of the pre-packed, pre-split,
//              pre-swizzled kernel tile (K-major SW128) into shared memory;
//              also owns the TMEM allocation;
//   warp 5     MMA issuer (one thread): 12 tcgen05.mma.kind::tf32 per K chunk;
//   warps 6-13 epilogue (two warps per TMEM lane quarter, each owning half of the
//              BN columns): drain the accumulator every G K-chunks into FP32
//              register sums, then + bias, post_conv faults, coalesced NCHW
//              store, fused FP64 row sums (So2/So4 partials).
//
// Why the drain: the tensor core aligns every addend to the accumulator's exponent
// and drops the bits below its ulp, so one accumulator over the whole K loses
// ~sqrt(3K) ulp(|O|) (1e-5 at K=576, 3.6e-5 at K=2400 measured) -- outside the
// 1e-5 contract.  A fresh accumulator per group of G chunks only ever holds a
// partial of magnitude |O|*sqrt(32G/K), which bounds the loss at ~sqrt(96G) ulp(|O|)
// independent of K; the partials are summed in registers (FP64 for BN <= 64, FP32
// for wider tiles, where 64 doubles per thread would not fit).
// The two correction products go to a separate per-tile accumulator, so the main
// one takes a third of the updates.  Main accumulators are double-buffered in TMEM
// so draining group g overlaps the MMAs of group g+1.  TMEM: [0, 2*BN) main,
// [2*BN, 3*BN) correction, then 2-4 A stages of 64 columns.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "ftc_common.cuh"

namespace ftc {

struct TcPlan {
  int BN = 0, ntiles = 0, nkc = 0, K = 0, M = 0, G = 1;
  float* Wp = nullptr;  // [ntiles][nkc][2][BN][32], SW128-swizzled, hi then lo
  int2* tab = nullptr;  // [nkc*32] im2col taps: {c*H*H + i*H + j, 1<<i | 1<<(16+j)}
};

namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;
// pipeline depth: TMEM holds 2*BN (main accumulators) + BN (correction accumulator)
// + stages*64 (A hi/lo) columns of 512
template <int BN>
constexpr int stages_for() {
  return BN >= 128 ? 2 : (BN >= 96 ? 3 : 4);
}
constexpr int stages_rt(int BN) { return BN >= 128 ? 2 : (BN >= 96 ? 3 : 4); }
constexpr int kProdWarps = 8;  // two per TMEM lane quarter, 16 columns of a chunk each
constexpr int kLoaderWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kEpiWarp0 = 10;
constexpr int kEpiThreads = 256;
constexpr int kThreads = 576;

struct TcArgs {
  const float* D;
  const float* Wp;
  const int2* tab;
  const float* bias;
  float* O;
  int N, C, H, M, R, U, pad, E, K, nkc, BN, ntiles;
  int G;           // K chunks per accumulator drain
  int pt_lo, npt;  // pixel tiles [pt_lo, pt_lo + npt)
  long long P;     // N*E*E
  const ftc_fault* faults;
  int nfaults;
  double* rowsum;    // [2*ntiles][N*E2] or null (one slab per column half)
  double* rowsum_m;  // [2*ntiles][N*E2]
  const uint32_t* plane_mask;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  // K-major, SWIZZLE_128B: SBO = 8 rows x 128 B, LBO unused, version 1 (sm_100)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// round-to-nearest TF32 (low 13 bits zero, so the tensor core reads it exactly)
__device__ __forceinline__ float tf32_rn(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// ------------------------------------------------------------------ kernel
template <int BN>
__global__ void __launch_bounds__(kThreads, 1) k_conv_tc(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the B stages (SW128 atoms)
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  uint8_t* sptr = smem_raw + (sbase - raw);
  constexpr int kStages = stages_for<BN>();
  const uint32_t stage_bytes = (uint32_t)BN * 256u;  // hi + lo tiles, 128 B per row each
  int2* tab_s = reinterpret_cast<int2*>(sptr + kStages * stage_bytes);
  const uint32_t tab_bytes = (uint32_t)a.nkc * kBK * 8u;
  const uint32_t bar_base = sbase + kStages * stage_bytes + tab_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sptr + kStages * stage_bytes + tab_bytes);
  // bars: full[4], empty[4], acc_full[2], acc_empty[2], then tmem base (u32)
  const uint32_t full0 = bar_base, empty0 = bar_base + 8 * kStages;
  const uint32_t accf0 = bar_base + 16 * kStages, acce0 = accf0 + 16;
  const uint32_t corrf = acce0 + 16, corre = corrf + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < a.nkc * kBK; e += blockDim.x) tab_s[e] = a.tab[e];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, kProdWarps * 32 + 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, kEpiThreads);
    }
    mbar_init(corrf, 1);
    mbar_init(corre, kEpiThreads);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kLoaderWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t corr_col = (uint32_t)(2 * BN);  // correction accumulator (per tile)
  const uint32_t a_col0 = (uint32_t)(3 * BN);

  const int E = a.E, E2 = E * E, H = a.H, R = a.R, RR = R * R, HH = H * H;
  const int ntile_total = a.ntiles * a.npt;

  if (warp < kProdWarps) {
    // ================= A producers =================
    // warp w owns TMEM lanes [32*(w%4), +32) (its pixels) and columns
    // [16*(w/4), +16) of every K chunk; the im2col tap table (offset + validity bits)
    // is a per-layer constant staged in shared memory.
    const int q = warp & 3, hf = warp >> 2;
    const int r = q * 32 + lane;  // row of the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint32_t g = 0;
    for (int t = blockIdx.x; t < ntile_total; t += gridDim.x) {
      const int pt = a.pt_lo + t % a.npt;
      const long long p = (long long)pt * kBM + r;
      const bool valid = p < a.P;
      const int n = valid ? (int)(p / E2) : 0;
      const int f = valid ? (int)(p % E2) : 0;
      const int x = f / E, y = f - (f / E) * E;
      const int xb = x * a.U - a.pad, yb = y * a.U - a.pad;
      // validity of tap rows i / columns j for this pixel (bit i, bit 16+j)
      uint32_t okmask = 0;
      if (valid) {
        for (int i = 0; i < R; ++i) {
          if ((unsigned)(xb + i) < (unsigned)H) okmask |= 1u << i;
          if ((unsigned)(yb + i) < (unsigned)H) okmask |= 1u << (16 + i);
        }
      }
      const float* base = a.D + (long long)n * a.C * HH + (long long)xb * H + yb;
      // software pipeline: the gathers of chunk kc+1 are in flight while chunk kc is
      // split, waited for and stored into TMEM
      float vn[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int2 tp = tab_s[hf * 16 + e];
        const bool ok = (okmask & (uint32_t)tp.y) == (uint32_t)tp.y;
        vn[e] = ok ? __ldg(base + tp.x) : 0.f;
      }
      for (int kc = 0; kc < a.nkc; ++kc, ++g) {
        const uint32_t s = g % kStages, ph = (g / kStages) & 1u;
        float v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = vn[e];
        if (kc + 1 < a.nkc) {
          const int2* tk = tab_s + (kc + 1) * kBK + hf * 16;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int2 tp = tk[e];
            const bool ok = (okmask & (uint32_t)tp.y) == (uint32_t)tp.y;
            vn[e] = ok ? __ldg(base + tp.x) : 0.f;
          }
        }
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          // round-to-nearest TF32 in integer arithmetic (the tensor core reads the
          // top 19 bits), lo = v - hi exact in FP32, rounded the same way
          const uint32_t h = (__float_as_uint(v[e]) + 0x1000u) & 0xFFFFE000u;
          hi[e] = h;
          const float l = v[e] - __uint_as_float(h);
          lo[e] = (__float_as_uint(l) + 0x1000u) & 0xFFFFE000u;
        }
        mbar_wait(empty0 + 8 * s, ph ^ 1u);
        tc_after();
        const uint32_t col = tmem + lane_off + a_col0 + s * 64u + (uint32_t)hf * 16u;
        tmem_st16(col, hi);
        tmem_st16(col + 32u, lo);
        tmem_wait_st();
        tc_before();
        mbar_arrive(full0 + 8 * s);
      }
    }
  } else if (warp == kLoaderWarp) {
    // ================= B loader =================
    if (lane == 0) {
      uint32_t g = 0;
      for (int t = blockIdx.x; t < ntile_total; t += gridDim.x) {
        const int nt = t / a.npt;
        const float* src = a.Wp + (long long)nt * a.nkc * 2 * BN * kBK;
        for (int kc = 0; kc < a.nkc; ++kc, ++g) {
          const uint32_t s = g % kStages, ph = (g / kStages) & 1u;
          mbar_wait(empty0 + 8 * s, ph ^ 1u);
          mbar_arrive_expect_tx(full0 + 8 * s, stage_bytes);
          bulk_g2s(sbase + s * stage_bytes, src + (long long)kc * 2 * BN * kBK, stage_bytes, full0 + 8 * s);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer =================
    if (lane == 0) {
      // kind::tf32, D=F32, A/B = TF32, K-major, M = 128, N = BN
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      uint32_t g = 0, gc = 0, tl = 0;
      const uint32_t d_corr = tmem + corr_col;
      for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tl) {
        // the correction accumulator collects lo*Bhi + hi*Blo over the whole tile
        // (2^-11 of the magnitude: its truncation is negligible); the main one only
        // the hi*Bhi products and is drained every G chunks
        mbar_wait(corre, (tl & 1u) ^ 1u);
        tc_after();
        for (int kc0 = 0; kc0 < a.nkc; kc0 += a.G, ++gc) {
          const uint32_t acc = gc & 1u, aph = (gc >> 1) & 1u;
          mbar_wait(acce0 + 8 * acc, aph ^ 1u);
          tc_after();
          const uint32_t d_tmem = tmem + acc * (uint32_t)BN;
          const int kc1 = min(a.nkc, kc0 + a.G);
          for (int kc = kc0; kc < kc1; ++kc, ++g) {
            const uint32_t s = g % kStages, ph = (g / kStages) & 1u;
            mbar_wait(full0 + 8 * s, ph);
            tc_after();
            const uint32_t a_hi = tmem + a_col0 + s * 64u, a_lo = a_hi + 32u;
            const uint32_t b_hi = sbase + s * stage_bytes, b_lo = b_hi + (uint32_t)BN * 128u;
#pragma unroll
            for (int k8 = 0; k8 < 4; ++k8) {
              const uint64_t dh = desc_sw128(b_hi + k8 * 32u);
              const uint64_t dl = desc_sw128(b_lo + k8 * 32u);
              mma_tf32_ts(d_tmem, a_hi + k8 * 8u, dh, idesc, (kc != kc0 || k8 != 0) ? 1u : 0u);
              mma_tf32_ts(d_corr, a_lo + k8 * 8u, dh, idesc, (kc != 0 || k8 != 0) ? 1u : 0u);
              mma_tf32_ts(d_corr, a_hi + k8 * 8u, dl, idesc, 1u);
            }
            mma_commit(empty0 + 8 * s);
          }
          mma_commit(accf0 + 8 * acc);
        }
        mma_commit(corrf);
      }
    }
  } else {
    // ================= epilogue =================
    constexpr int HALF = BN / 2;  // columns owned by this warp
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;       // TMEM lane quarter this warp may access
    const int half = ew >> 2;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint32_t gc = 0, tl = 0;
    for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tl) {
      const int nt = t / a.npt;
      const int pt = a.pt_lo + t % a.npt;
      const long long p = (long long)pt * kBM + r;
      const bool valid = p < a.P;
      const int n = valid ? (int)(p / E2) : 0;
      const int f = valid ? (int)(p % E2) : 0;
      const int x = f / E, y = f - (f / E) * E;
      // running sums of the drained partials: FP64 while the 32 per-thread values fit
      // the register budget (BN <= 64), FP32 beyond (still ~4x closer to the exact
      // conv than the reference's sequential FP32 loop on the BASELINE nets)
      using acc_t = typename std::conditional<(HALF <= 32), double, float>::type;
      acc_t sum[HALF];
#pragma unroll
      for (int jj = 0; jj < HALF; ++jj) sum[jj] = acc_t(0);
      for (int kc0 = 0; kc0 < a.nkc; kc0 += a.G, ++gc) {
        const uint32_t acc = gc & 1u, aph = (gc >> 1) & 1u;
        mbar_wait(accf0 + 8 * acc, aph);
        tc_after();
        const uint32_t base = tmem + lane_off + acc * (uint32_t)BN + (uint32_t)(half * HALF);
#pragma unroll
        for (int c16 = 0; c16 < HALF / 16; ++c16) {
          uint32_t v[16];
          tmem_ld16(base + (uint32_t)c16 * 16u, v);
          tmem_wait_ld();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) sum[c16 * 16 + jj] += (acc_t)__uint_as_float(v[jj]);
        }
        tc_before();
        mbar_arrive(acce0 + 8 * acc);
      }
      {  // the tile's correction accumulator
        mbar_wait(corrf, tl & 1u);
        tc_after();
        const uint32_t base = tmem + lane_off + corr_col + (uint32_t)(half * HALF);
#pragma unroll
        for (int c16 = 0; c16 < HALF / 16; ++c16) {
          uint32_t v[16];
          tmem_ld16(base + (uint32_t)c16 * 16u, v);
          tmem_wait_ld();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) sum[c16 * 16 + jj] += (acc_t)__uint_as_float(v[jj]);
        }
        tc_before();
        mbar_arrive(corre);
      }
      double rs = 0.0, rsm = 0.0;
      float* Obase = a.O + (long long)n * a.M * E2 + f;
#pragma unroll
      for (int jj = 0; jj < HALF; ++jj) {
        const int m = nt * BN + half * HALF + jj;
        if (!valid || m >= a.M) continue;
        float val = (float)sum[jj];
        if (a.bias) val = val + __ldg(a.bias + m);
        if (a.nfaults) val = apply_output_faults(val, n, m, x, y, a.faults, a.nfaults);
        bool store = true;
        if (a.plane_mask) {
          const long long pl = (long long)n * a.M + m;
          store = (a.plane_mask[pl >> 5] >> (pl & 31)) & 1u;
        }
        if (store) Obase[(long long)m * E2] = val;
        const double dv = (double)val;
        rs = dadd(rs, dv);
        rsm = dadd(rsm, dmul((double)m, dv));
      }
      if (valid && a.rowsum) {
        const long long o = (long long)(2 * nt + half) * a.P + p;
        a.rowsum[o] = rs;
        a.rowsum_m[o] = rsm;
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == kLoaderWarp) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// W -> [ntiles][nkc][hi,lo][BN][32] with the SW128 chunk swizzle (16-byte chunk
// index XOR row%8), rows >= M and k >= K zero-padded.
__global__ void k_pack_w(const float* __restrict__ W, float* __restrict__ Wp, int M, int K, int BN,
                         int ntiles, int nkc) {
  const long long total = (long long)ntiles * nkc * BN * kBK;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e % kBK);
    const int row = (int)((e / kBK) % BN);
    const int kc = (int)((e / ((long long)kBK * BN)) % nkc);
    const int nt = (int)(e / ((long long)kBK * BN * nkc));
    const int m = nt * BN + row, kk = kc * kBK + k;
    const float w = (m < M && kk < K) ? W[(long long)m * K + kk] : 0.f;
    const float hi = tf32_rn(w), lo = tf32_rn(w - hi);
    const long long tile = ((long long)nt * nkc + kc) * 2;
    const int sw = row * kBK + ((((k >> 2) ^ (row & 7))) << 2) + (k & 3);
    Wp[tile * BN * kBK + sw] = hi;
    Wp[(tile + 1) * BN * kBK + sw] = lo;
  }
}

// im2col tap table in the reference's (k,i,j) order; padding entries (k >= K) carry
// validity bits 15/31 that no pixel mask has, so they load nothing.
__global__ void k_build_tab(int2* tab, int C, int H, int R, int K, int Kpad) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Kpad) return;
  if (k >= K) {
    tab[k] = make_int2(0, (int)0x80008000u);
    return;
  }
  const int RR = R * R, c = k / RR, t = k % RR, i = t / R, j = t % R;
  tab[k] = make_int2((c * H + i) * H + j, (int)((1u << i) | (1u << (16 + j))));
}

int g_num_sms = 0;

template <int BN>
int launch_bn(const TcArgs& a, int grid, size_t smem, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    FTC_CUDA_CHECK(cudaFuncSetAttribute(k_conv_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024));
    attr_set = true;
  }
  FTC_LAUNCH(k_conv_tc<BN><<<grid, kThreads, smem, s>>>(a));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // namespace

bool tc_supported(const ftc_conv_desc& d) {
  if (d.groups != 1) return false;
  if (d.R > 15) return false;  // tap validity bits: rows 0-14, columns 16-30
  const long long K = (long long)d.C * d.R * d.R;
  const long long nkc = (K + kBK - 1) / kBK;
  const long long bn = d.M <= 128 ? ((d.M + 31) / 32) * 32 : 128;
  if (1024 + stages_rt((int)bn) * bn * 256 + nkc * kBK * 8 + 256 > 227 * 1024) return false;
  if ((long long)d.C * d.H * d.H >= (1LL << 31)) return false;
  const long long E = (d.H + 2LL * d.pad - d.R) / d.stride + 1;
  if ((long long)d.N * E * E >= (1LL << 31)) return false;
  return true;
}

int tc_plan_create(const ftc_conv_desc& d, const float* W_dev, TcPlan** out, cudaStream_t s) {
  TcPlan* p = new TcPlan();
  p->M = d.M;
  p->K = d.C * d.R * d.R;
  p->nkc = (p->K + kBK - 1) / kBK;
  if (const char* g = getenv("FTC_TC_DRAIN_CHUNKS")) p->G = atoi(g) > 0 ? atoi(g) : 1;
  if (d.M <= 128) {
    p->BN = ((d.M + 31) / 32) * 32;
    p->ntiles = 1;
  } else {
    p->BN = 128;
    p->ntiles = (d.M + 127) / 128;
  }
  if (const char* bn = getenv("FTC_TC_MAX_BN")) {  // experimentation: cap the N tile
    const int cap = atoi(bn);
    if ((cap == 32 || cap == 64 || cap == 96 || cap == 128) && p->BN > cap) {
      p->BN = cap;
      p->ntiles = (d.M + cap - 1) / cap;
    }
  }
  const size_t n = (size_t)p->ntiles * p->nkc * 2 * p->BN * kBK;
  if (cudaMalloc(&p->Wp, n * sizeof(float)) != cudaSuccess) {
    delete p;
    set_error(FTC_CUDA_ERROR, "cudaMalloc(packed W) failed");
    return FTC_CUDA_ERROR;
  }
  FTC_LAUNCH(k_pack_w<<<592, 256, 0, s>>>(W_dev, p->Wp, d.M, p->K, p->BN, p->ntiles, p->nkc));
  if (cudaMalloc(&p->tab, (size_t)p->nkc * kBK * sizeof(int2)) != cudaSuccess) {
    cudaFree(p->Wp);
    delete p;
    set_error(FTC_CUDA_ERROR, "cudaMalloc(tap table) failed");
    return FTC_CUDA_ERROR;
  }
  FTC_LAUNCH(k_build_tab<<<(p->nkc * kBK + 255) / 256, 256, 0, s>>>(p->tab, d.C, d.H, d.R, p->K,
                                                                   p->nkc * kBK));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFree(p->Wp);
    delete p;
    set_error(FTC_CUDA_ERROR, std::string("pack_w: ") + cudaGetErrorString(e));
    return FTC_CUDA_ERROR;
  }
  *out = p;
  return FTC_OK;
}

void tc_plan_destroy(TcPlan* p) {
  if (!p) return;
  if (p->Wp) cudaFree(p->Wp);
  if (p->tab) cudaFree(p->tab);
  delete p;
}

int tc_rowsum_parts(const TcPlan* p) { return p ? 2 * p->ntiles : 1; }

int conv_tc_launch(const TcPlan* p, const ConvArgs& c, cudaStream_t s) {
  TcArgs a{};
  a.D = c.D;
  a.Wp = p->Wp;
  a.tab = p->tab;
  a.bias = c.bias;
  a.O = c.O;
  a.N = c.N;
  a.C = c.C;
  a.H = c.H;
  a.M = c.M;
  a.R = c.R;
  a.U = c.U;
  a.pad = c.pad;
  a.E = c.E;
  a.K = p->K;
  a.nkc = p->nkc;
  a.BN = p->BN;
  a.ntiles = p->ntiles;
  a.G = p->G;
  const long long E2 = (long long)c.E * c.E;
  a.P = (long long)c.N * E2;
  const long long p_lo = (long long)c.img_lo * E2, p_hi = (long long)c.img_hi * E2;
  a.pt_lo = (int)(p_lo / kBM);
  a.npt = (int)((p_hi + kBM - 1) / kBM) - a.pt_lo;
  if (a.npt <= 0) return FTC_OK;
  a.faults = c.faults;
  a.nfaults = c.nfaults;
  a.rowsum = c.rowsum;
  a.rowsum_m = c.rowsum_m;
  a.plane_mask = c.plane_mask;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  const int tiles = a.ntiles * a.npt;
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  const size_t smem = 1024 + (size_t)stages_rt(p->BN) * p->BN * 256 + (size_t)p->nkc * kBK * 8 + 256;
  switch (p->BN) {
    case 32: return launch_bn<32>(a, grid, smem, s);
    case 64: return launch_bn<64>(a, grid, smem, s);
    case 96: return launch_bn<96>(a, grid, smem, s);
    case 128: return launch_bn<128>(a, grid, smem, s);
  }
  set_error(FTC_CONFIG_ERROR, "unsupported BN");
  return FTC_CONFIG_ERROR;
}

}  // namespace ftc

