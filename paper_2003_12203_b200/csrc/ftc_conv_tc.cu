// ftc_conv_tc.cu -- tcgen05 implicit-GEMM convolution, 3xTF32 (engine 0).
//
// conv_forward (conv.hpp:114-131) as a GEMM: rows = output pixels p = (n, x, y)
// (128 per tile = UMMA M), columns = kernels m (BN per N-tile), K = (c, i, j) in the
// reference's accumulation order, chunked by 32 (one 128-byte SW128 row of TF32).
//
// FP32 accuracy on TF32 tensor cores: every operand is split v = hi + lo with
// hi = RN_tf32(v) (low 13 mantissa bits zero, read exactly by the tensor core) and
// lo = RN_tf32(v - hi); each K step adds lo*Bhi + hi*Blo + hi*Bhi (the dropped lo*lo
// term is 2^-22 relative).
//
// Warp roles (persistent CTA per SM, 640 threads):
//   warps 0-7   A producers (two per TMEM lane quarter): take the im2col row of their
//               pixel (TMA im2col stage in shared memory, or a gather straight from D),
//               split hi/lo and tcgen05.st it into a TMEM half-stage (warps 0-3: K
//               columns 0-15 of a chunk, 4-7: 16-31) -- the A operand of the TS-form MMA;
//   warp 8      loader: the TMA im2col A stages and one cp.async.bulk per stage of the
//               pre-packed, pre-split, pre-swizzled kernel tile (K-major SW128); owns the
//               TMEM allocation;
//   warps 9-10  MMA issuers: the K chunks of a tile form groups of kG = 2; issuer w
//               takes every other group (12 tcgen05.mma.kind::tf32 per chunk) into its
//               own accumulator X_w;
//   warps 11-18 epilogue (two per TMEM lane quarter, each owning half of the BN
//               columns): drain X after every group into register sums (group order),
//               then + bias, post_conv faults, coalesced NCHW store, fused FP64 row sums
//               (So2/So4 partials);
//   warp 19     (FUSE) checksum warp: Co5 = Cd1 (*) Cw1 at this CTA's share of the
//               output positions, in the shadow of the MMAs; the epilogue adds its row
//               sums into So5 (FP64 atomics); a small kernel after the conv runs CoC-D.
//
// Determinism: each accumulator is written by one thread only (the pipe does not order
// MMAs of different issuing threads into one accumulator), and the epilogue adds the
// group partials in group order, so every output is bitwise reproducible and a
// recomputed plane equals the clean one.
//
// Why the per-group drain: the tensor core aligns every addend to the accumulator's
// exponent and drops the bits below its ulp, so one accumulator over the whole K loses
// ~sqrt(3K) ulp(|O|) (1e-5 at K=576, 3.6e-5 at K=2400 measured) -- outside the 1e-5
// contract.  A fresh accumulator per group of 2 K chunks only holds a partial of
// magnitude |O|*sqrt(64/K); within a group the 16 small correction products go in first
// (while the partial is small: they lose nothing) and the 8 main products last, so a
// group costs 8 truncations of the partial, independent of K.  The partials are summed in registers
// (FP32).
// TMEM: [0, BN) X_0, [BN, 2*BN) X_1, then up to 8 A half-stages of 32 columns
// (16 hi + 16 lo).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <type_traits>

#include "ftc_common.cuh"

namespace ftc {

struct TcPlan {
  // grouped convs: groups x ntg N-tiles, tile nt belongs to group nt / ntg and covers its
  // kernels [nt % ntg * BN, +BN) of Mg; K = Ckw * R * R per group
  int BN = 0, ntiles = 0, nkc = 0, K = 0, M = 0;
  int groups = 1, Mg = 0, ntg = 0, Ckw = 0, Ctot = 0;
  // channel-last gather (C % 32 == 0): the input is transposed to NHWC per launch and
  // K runs tap-major (k = (i*R + j)*C + c), so a K chunk is 32 consecutive channels of
  // one tap: one bounds test and four 16-byte loads per producer thread per chunk
  bool nhwc = false;
  float* Wp = nullptr;  // [ntiles][nkc][2][BN][32], SW128-swizzled, hi then lo
  int2* tab = nullptr;  // NCHW: [nkc*32] per-column taps {c*H*H + i*H + j, 1<<i | 1<<(16+j)}
                        // NHWC: [nkc] per-chunk taps {(i*H + j)*C + c0, same bits}
  float* Dt = nullptr;  // NHWC copy of the input (N*H*H*C), nhwc / im2col only
  // TMA im2col A operand (C % 32 == 0): the tensor engine gathers each K chunk (one
  // tap, 32 channels, 128 consecutive output pixels, zero-filled padding) from the NHWC
  // copy straight into a swizzled shared-memory stage
  bool im2col = false;
  alignas(64) CUtensorMap tmA;
};

namespace {

constexpr int kBM = 128;
constexpr int kBK = 32;
// TMEM budget (512 columns): kNX accumulator buffers of BN columns (issuers rotate over
// them group by group, so an issuer finds its next buffer drained kNX - 1 groups after
// it filled it) + kSA A chunk slots of 64 columns (two half-stages of 16 hi + 16 lo)
template <int BN>
constexpr int acc_bufs() {
  return BN >= 128 ? 3 : 4;
}
template <int BN>
constexpr int stages_for() {
  return (512 - acc_bufs<BN>() * BN) / 64 >= 4 ? 4 : (512 - acc_bufs<BN>() * BN) / 64;
}
constexpr int stages_host(long long) { return 2; }  // minimum B ring depth
// K chunks per accumulator group (one drain each; an issuer holds a group's operands):
// one for BN >= 96, two for the narrower tiles, whose MMAs are short (N = 64: ~47 cycles)
// so a drain per chunk would cost more than the chunk
#ifndef FTC_GROUP_NARROW
#define FTC_GROUP_NARROW 2
#endif
template <int BN>
constexpr int group_chunks() {
  return BN >= 96 ? 1 : FTC_GROUP_NARROW;
}
// one tcgen05.commit per accumulator group (a ring of 8 "group done" barriers that the
// producers, the B loader and the epilogue all wait on) instead of four per chunk --
// same speed (the commits were not the limiter), fewer instructions on the issuers
#ifndef FTC_ONE_COMMIT
#define FTC_ONE_COMMIT 1
#endif
constexpr bool kOneCommit = FTC_ONE_COMMIT;
// epilogue running sums of the group partials in FP32 for every tile width (FP64 for
// BN <= 64 put the narrow layers' drain on the issuers' critical path: VGG c2 traces)
#ifndef FTC_EPI_F32
#define FTC_EPI_F32 1
#endif
#ifndef FTC_SPLIT_LOADER
#define FTC_SPLIT_LOADER 0
#endif
constexpr bool kSplitLoader = FTC_SPLIT_LOADER;
#ifndef FTC_KAS
#define FTC_KAS 4
#endif
constexpr int kAS = FTC_KAS;                 // MODE 2 shared-memory A stages
constexpr uint32_t kAStageBytes = 128u * 128u;  // 128 pixels x 32 FP32 channels
constexpr int kProdWarps = 8;  // two per TMEM lane quarter, 16 columns of a chunk each
constexpr int kLoaderWarp = 8;
constexpr int kMmaWarp = 9;  // and 10: two issuers alternating K chunks
constexpr int kEpiWarp0 = 11;
constexpr int kEpiThreads = 256;
// fused clean path: one checksum warp computes Co5 = Cd1 (*) Cw1 at this CTA's positions
// (a 21st warp would put 6 warps on one SM sub-partition and cap registers at 80)
constexpr int kCkWarp0 = 19;
constexpr int kCkWarps = 1;
#ifndef FTC_CK_UNROLL
#define FTC_CK_UNROLL 8
#endif
constexpr int kCkUnroll = FTC_CK_UNROLL;  // taps in flight per lane
constexpr int kThreads = 640;

struct TcArgs {
  const float* D;
  const float* Wp;
  const int2* tab;
  const float* bias;
  float* O;
  int N, C, H, M, R, U, pad, E, K, nkc, BN, ntiles;
  int Ckw, Mg, ntg;  // grouped convs: channels / kernels per group, N-tiles per group
  int SB;          // B (shared-memory) pipeline stages
  int dbg;         // FTC_TC_DEBUG bits (profiling experiments only; 0 in production)
  int pt_lo, npt;  // pixel tiles [pt_lo, pt_lo + npt)
  long long P;     // N*E*E
  const ftc_fault* faults;
  int nfaults;
  const double* scale_tab;
  double* rowsum;    // [2*ntiles][N*E2] or null (one slab per column half)
  double* rowsum_m;  // [2*ntiles][N*E2]
  const uint32_t* plane_mask;
  FusedDetect fd;  // valid for FUSE instantiations
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
// Critical-path waits (producers, MMA issuers).  FTC_SPIN_NS > 0 backs off between failed
// polls: when the pipeline stalls at a tile boundary ten warps spin here at once and
// take issue slots from the epilogue warps that everyone is waiting for.
#ifndef FTC_SPIN_NS
#define FTC_SPIN_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
    if (FTC_SPIN_NS > 0) __nanosleep(FTC_SPIN_NS);
  }
}
// off the MMA-critical path (epilogue, B loader): back off between polls so the spinning
// warps leave issue slots to the producers and the MMA issuers
#ifndef FTC_WAIT_NS
#define FTC_WAIT_NS 64
#endif
__device__ __forceinline__ void mbar_wait_lazy(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
    if (FTC_WAIT_NS > 0) __nanosleep(FTC_WAIT_NS);
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// CTA-pair B multicast (CL = 2): one half of a B stage lands in both CTAs of the cluster
// at the same shared-memory offset and signals the same barrier offset in each
__device__ __forceinline__ void bulk_g2s_mc2(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_arrive_peer(uint32_t bar, uint32_t peer) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(bar), "r"(peer));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster_lazy(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// im2col TMA: 128 consecutive output pixels (starting at input position (n, h, w) of the
// bounding-box traversal) x channels [c, c+32) at filter tap (oh, ow)
__device__ __forceinline__ void tma_im2col_4d(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                              uint16_t ow, uint16_t oh, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(bar), "h"(ow), "h"(oh)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}\n"
      : "=r"(p));
  return p != 0;
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

__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// wait until accumulator group j of this CTA has completed (kOneCommit ring of 8)
__device__ __forceinline__ void gdone_wait(uint32_t gdone0, uint32_t j, bool lazy) {
  const uint32_t bar = gdone0 + 8 * (j & 7u), ph = (j >> 3) & 1u;
  if (lazy) {
    while (!mbar_try_wait(bar, ph)) __nanosleep(64);
  } else {
    while (!mbar_try_wait(bar, ph)) {
      if (FTC_SPIN_NS > 0) __nanosleep(FTC_SPIN_NS);
    }
  }
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

// v = hi + lo: hi = RN_tf32(v) in integer arithmetic (the tensor core reads the top 19
// bits), lo = v - hi exact in FP32, rounded the same way.  FTC_SPLIT_MODE 1 (experiment):
// lo handed over unrounded (the tensor core ignores the low 13 bits: a truncation of lo,
// 2^-22 |v|, the size of the dropped lo*lo term); 2: cvt.rna.tf32 for both roundings.
#ifndef FTC_SPLIT_MODE
#define FTC_SPLIT_MODE 0
#endif
__device__ __forceinline__ void split_tf32(uint32_t v, uint32_t& hi, uint32_t& lo) {
#if FTC_SPLIT_MODE == 2
  const float h = tf32_rn(__uint_as_float(v));
  hi = __float_as_uint(h);
  lo = __float_as_uint(tf32_rn(__uint_as_float(v) - h));
#else
  const uint32_t h = (v + 0x1000u) & 0xFFFFE000u;
  hi = h;
  const float l = __uint_as_float(v) - __uint_as_float(h);
#if FTC_SPLIT_MODE == 1
  lo = __float_as_uint(l);
#else
  lo = (__float_as_uint(l) + 0x1000u) & 0xFFFFE000u;
#endif
#endif
}

// ------------------------------------------------------------------ kernel
// Out of line: the store loop is unrolled over every column of the tile and an inlined
// fault loop + mask lookup per column made the epilogue ~200 KB of SASS (instruction-
// cache bound, ~40K cycles per tile).  Faults and repair masks are rare; a call is fine.
// profiling aid (FTC_TC_DEBUG bit 64, block 0 only): per-chunk event clocks
__device__ long long g_tc_trace[16][1024];
#define TC_TRACE(on, slot, idx)                                  \
  do {                                                           \
    if ((on) && (idx) < 1024u) g_tc_trace[slot][idx] = clock64(); \
  } while (0)

struct HookOut {
  float v;
  int store;
};
__device__ __noinline__ HookOut epilogue_hooks(float v, int n, int m, int x, int y, const ftc_fault* f, int nf,
                                               const uint32_t* plane_mask, int M, int E, const double* tab) {
  HookOut h;
  h.v = nf ? apply_output_faults(v, n, m, x, y, M, E, f, nf, tab) : v;
  h.store = 1;
  if (plane_mask) {
    const long long pl = (long long)n * M + m;
    h.store = (int)((plane_mask[pl >> 5] >> (pl & 31)) & 1u);
  }
  return h;
}

// MODE 0: NCHW im2col gather by the producers; 1: NHWC gather (4 x 16-byte loads per
// chunk); 2: TMA im2col into shared memory, producers only split and store to TMEM.
// FUSE: clean-path CoC-D operands inside the kernel: the checksum warp computes Co5, the
// epilogue adds its row sums into So5; launch_detect_fused compares them afterwards.
// CL = 2: CTA pairs (cluster of 2) take the two pixel tiles (2k, 2k+1) of one N-tile in
// lockstep and share the B stream: each loader fetches half of every B stage and
// multicasts it into both CTAs (L2 -> SM traffic per chunk 48 -> 32 KB at BN = 128; the
// long-K layers ran at ~85% of the L2 throughput cap).  MODE 2, full pixel range only;
// an odd tile count gives the last pair a phantom tile (p >= P: computed, never stored).
template <int BN, int MODE, bool FUSE, bool GROUPED, int CL = 1>
__global__ void __launch_bounds__(kThreads, 1) k_conv_tc(TcArgs a, const __grid_constant__ CUtensorMap tmA) {
  static_assert(CL == 1 || (CL == 2 && MODE == 2 && !GROUPED && kOneCommit), "CTA-pair mode: TMA im2col layers");
  constexpr bool NHWC = MODE == 1;
  constexpr bool TMAA = MODE >= 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the B stages (SW128 atoms)
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  uint8_t* sptr = smem_raw + (sbase - raw);
  // A ring (TMEM, depth kSA) and B ring (shared memory, depth SB) advance together
  // per K chunk but are sized independently: TMEM bounds A, shared memory bounds B.
  constexpr int kMaxSB = 8;
  const int SB = a.SB;
  constexpr int kSA = stages_for<BN>();
  constexpr int kNX = acc_bufs<BN>();
  constexpr int kG = group_chunks<BN>();
  const uint32_t stage_bytes = (uint32_t)BN * 256u;  // hi + lo tiles, 128 B per row each
  // MODE 2: kAS shared-memory A stages (128 pixels x 32 channels, SW128) follow the B ring
  const uint32_t as_base = sbase + SB * stage_bytes;
  const uint32_t as_bytes = TMAA ? (uint32_t)kAS * kAStageBytes : 0u;
  int2* tab_s = reinterpret_cast<int2*>(sptr + SB * stage_bytes + as_bytes);
  const uint32_t tab_bytes = TMAA ? 0u : (uint32_t)a.nkc * kBK * 8u;
  const uint32_t bar_base = sbase + SB * stage_bytes + as_bytes + tab_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sptr + SB * stage_bytes + as_bytes + tab_bytes);
  // A ring of half-stages: a K chunk's first 16 columns (hf = 0) and last 16 (hf = 1)
  // are separate stages of 32 TMEM columns (16 hi + 16 lo), filled by their own producer
  // warps and released after their own 6 MMAs -- the refill of a stage overlaps 3 half
  // chunks of MMAs instead of 1 whole chunk
  constexpr int kHS = 2 * kSA;
  // bars: fullA[8] emptyA[8] fullB[8] emptyB[8] accf[2] acce[2] (3 spare) fullAs[kAS]
  // emptyAs[kAS], tmem base
  const uint32_t fullA0 = bar_base, emptyA0 = bar_base + 8 * 8;
  const uint32_t fullB0 = bar_base + 8 * 16, emptyB0 = fullB0 + 8 * kMaxSB;
  const uint32_t accf0 = emptyB0 + 8 * kMaxSB, acce0 = accf0 + 8 * 4;
  const uint32_t gdone0 = acce0 + 8 * 4;  // kOneCommit: group j done = gdone[j % 8]
  const uint32_t fullAs0 = gdone0 + 8 * 8, emptyAs0 = fullAs0 + 8 * kAS;  // MODE 2 A ring
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16 + 2 * kMaxSB + 8 + 8 + 2 * kAS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!TMAA)
    for (int e = threadIdx.x; e < a.nkc * kBK; e += blockDim.x) tab_s[e] = a.tab[e];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kHS; ++s) {
      mbar_init(fullA0 + 8 * s, kProdWarps / 2);
      mbar_init(emptyA0 + 8 * s, 1);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(fullB0 + 8 * s, 1);
      mbar_init(emptyB0 + 8 * s, 1);
    }
    for (int b = 0; b < 8; ++b) mbar_init(gdone0 + 8 * b, 1);
    for (int b = 0; b < kNX; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, kEpiThreads / 32);
    }
    if (TMAA) {  // shared-memory A ring: filled by the TMA, released by the producers
      for (int s = 0; s < kAS; ++s) {
        mbar_init(fullAs0 + 8 * s, 1);
        mbar_init(emptyAs0 + 8 * s, kProdWarps);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kLoaderWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  if (CL == 2) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive / multicast
  tc_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the prologue above overlapped the previous kernel's tail; the next kernel (the
  // CoC-D compare or glue) may be scheduled now -- it cannot share an SM with this CTA
  // and waits for this grid before reading anything
  pdl_trigger();
  pdl_wait();
  const uint32_t a_col0 = (uint32_t)(kNX * BN);  // A chunk slots follow the accumulators

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
    uint32_t g = 0, hs = (uint32_t)hf, hph = 0;  // this warp's half-stage slot / phase
    if constexpr (TMAA) {
      // the chunk is already gathered (and zero-padded) by the TMA: read this row's 16
      // values (4 x 16-byte chunks of the SW128 row, conflict-free), release the stage,
      // split hi/lo and store them to the TMEM half-stage like the gather paths
      uint32_t sa = 0, pha = 0;
      const bool pprof2 = (a.dbg & 64) && blockIdx.x == 0 && lane == 0 && (warp == 0 || warp == kProdWarps - 1);
      const uint32_t ngt = (uint32_t)(a.nkc + kG - 1) / (uint32_t)kG;
      uint32_t jh[4] = {0, 0, 0, 0}, tlp = 0;  // groups of the last 4 chunks (kOneCommit)
      for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tlp) {
        for (int kc = 0; kc < a.nkc; ++kc, ++g) {
          const uint32_t s = hs, ph = hph;
          const uint32_t jprev = jh[kSA - 1];  // group of this slot's previous chunk
          jh[3] = jh[2];
          jh[2] = jh[1];
          jh[1] = jh[0];
          jh[0] = tlp * ngt + (uint32_t)kc / (uint32_t)kG;
          hs += 2;
          if (hs >= (uint32_t)kHS) { hs -= (uint32_t)kHS; hph ^= 1u; }
          const uint32_t sa_c = sa, pha_c = pha;
          if (++sa == (uint32_t)kAS) { sa = 0; pha ^= 1u; }
          mbar_wait(fullAs0 + 8 * sa_c, pha_c);
          if (warp == 0) TC_TRACE(pprof2, 0, g);
          const uint32_t row = as_base + sa_c * kAStageBytes + (uint32_t)r * 128u;
          uint32_t v[16];
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const uint32_t c = (uint32_t)(hf * 4 + q4);
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v[4 * q4]), "=r"(v[4 * q4 + 1]), "=r"(v[4 * q4 + 2]), "=r"(v[4 * q4 + 3])
                         : "r"(row + ((c ^ (uint32_t)(r & 7)) << 4))
                         : "memory");
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(emptyAs0 + 8 * sa_c);
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) split_tf32(v[e], hi[e], lo[e]);
          if (!kOneCommit) mbar_wait(emptyA0 + 8 * s, ph ^ 1u);
          else if (g >= (uint32_t)kSA) gdone_wait(gdone0, jprev, false);
          if (warp == 0) TC_TRACE(pprof2, 1, g);
          tc_after();
          const uint32_t col = tmem + lane_off + a_col0 + s * 32u;
          tmem_st16(col, hi);
          tmem_st16(col + 16u, lo);
          tmem_wait_st();
          tc_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(fullA0 + 8 * s);
          TC_TRACE(pprof2, warp == 0 ? 2 : 3, g);
        }
      }
    } else {
    const bool pprof = (a.dbg & 64) && blockIdx.x == 0 && lane == 0 && (warp == 0 || warp == kProdWarps - 1);
    // per-tile gather state: validity of tap rows i / columns j for this pixel (bit i,
    // bit 16+j) and the pixel's window origin
    uint32_t okmask = 0;
    const float* base = a.D;
    auto setup = [&](int t) {
      const int pt = a.pt_lo + t % a.npt;
      const long long p = (long long)pt * kBM + r;
      const bool valid = p < a.P;
      const int n = valid ? (int)(p / E2) : 0;
      const int f = valid ? (int)(p % E2) : 0;
      const int x = f / E, y = f - (f / E) * E;
      const int xb = x * a.U - a.pad, yb = y * a.U - a.pad;
      okmask = 0;
      if (valid) {
        for (int i = 0; i < R; ++i) {
          if ((unsigned)(xb + i) < (unsigned)H) okmask |= 1u << i;
          if ((unsigned)(yb + i) < (unsigned)H) okmask |= 1u << (16 + i);
        }
      }
      // grouped convs: the tile's group's first channel (compile-time 0 otherwise -- any
      // extra live value in this kernel costs the ungrouped hot loops registers)
      const int cg = GROUPED ? (t / a.npt) / a.ntg * a.Ckw : 0;
      base = NHWC ? a.D + (((long long)n * H + xb) * H + yb) * a.C + cg + hf * 16
                  : a.D + ((long long)n * a.C + cg) * HH + (long long)xb * H + yb;
    };
    // software pipeline: the gathers of chunk kc+1 are in flight while chunk kc is split,
    // waited for and stored into TMEM -- across tiles too (the last chunk of a tile
    // prefetches the next tile's first chunk; the tile start used to expose a full
    // gather latency every nkc chunks)
    auto gather = [&](int kc, float (&out)[16]) {
      if constexpr (NHWC) {
        const int2 tp = tab_s[kc];
        const bool ok = (okmask & (uint32_t)tp.y) == (uint32_t)tp.y;
        const float4* src = reinterpret_cast<const float4*>(base + tp.x);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 f = ok ? __ldg(src + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
          out[4 * q4 + 0] = f.x;
          out[4 * q4 + 1] = f.y;
          out[4 * q4 + 2] = f.z;
          out[4 * q4 + 3] = f.w;
        }
      } else {
        const int2* tk = tab_s + kc * kBK + hf * 16;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int2 tp = tk[e];
          const bool ok = (okmask & (uint32_t)tp.y) == (uint32_t)tp.y;
          out[e] = ok ? __ldg(base + tp.x) : 0.f;
        }
      }
    };
    float vn[16];
    if ((int)blockIdx.x < ntile_total) {
      setup(blockIdx.x);
      gather(0, vn);
    }
    const uint32_t ngt0 = (uint32_t)(a.nkc + kG - 1) / (uint32_t)kG;
    uint32_t jh0[4] = {0, 0, 0, 0}, tlp0 = 0;  // groups of the last 4 chunks (kOneCommit)
    for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tlp0) {
      for (int kc = 0; kc < a.nkc; ++kc, ++g) {
        const uint32_t s = hs, ph = hph;
        const uint32_t jprev = jh0[kSA - 1];
        jh0[3] = jh0[2];
        jh0[2] = jh0[1];
        jh0[1] = jh0[0];
        jh0[0] = tlp0 * ngt0 + (uint32_t)kc / (uint32_t)kG;
        hs += 2;
        if (hs >= (uint32_t)kHS) { hs -= (uint32_t)kHS; hph ^= 1u; }
        float v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = vn[e];
        if (!(a.dbg & 1)) {
          if (kc + 1 < a.nkc) {
            gather(kc + 1, vn);
          } else if (t + (int)gridDim.x < ntile_total) {
            setup(t + (int)gridDim.x);
            gather(0, vn);
          }
        }
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) split_tf32(__float_as_uint(v[e]), hi[e], lo[e]);
        if (warp == 0) TC_TRACE(pprof, 0, g);
        if (!kOneCommit) mbar_wait(emptyA0 + 8 * s, ph ^ 1u);
        else if (g >= (uint32_t)kSA) gdone_wait(gdone0, jprev, false);
        if (warp == 0) TC_TRACE(pprof, 1, g);
        tc_after();
        if (!(a.dbg & 2)) {
          const uint32_t col = tmem + lane_off + a_col0 + s * 32u;
          tmem_st16(col, hi);
          tmem_st16(col + 16u, lo);
          tmem_wait_st();
        }
        tc_before();
        __syncwarp();  // one elected arrival per warp: 256 same-address arrivals cost ~500 cycles
        if (lane == 0) mbar_arrive(fullA0 + 8 * s);
        TC_TRACE(pprof, warp == 0 ? 2 : 3, g);
      }
    }
    }
  } else if (warp == kLoaderWarp) {
    // ================= loader =================
    // lane 0 streams the A (TMA im2col) and B stages.  FTC_SPLIT_LOADER=1 moves the A
    // stream to lane 1 (independent thread scheduling); measured 12-20% slower on the
    // BN = 128 layers, so off
    const bool doB = lane == 0;
    const bool doA = TMAA && (kSplitLoader ? lane == 1 : lane == 0);
    if (doA || doB) {
      uint32_t g = 0, sB = 0, phB = 0, sa = 0, pha = 0;
      const uint32_t crank = CL == 2 ? cluster_ctarank() : 0u;
      const int ncb = (GROUPED ? a.Ckw : a.C) / 32;
      const uint32_t ngtl = (uint32_t)(a.nkc + kG - 1) / (uint32_t)kG;
      uint32_t jb[4] = {0, 0, 0, 0}, tll = 0;  // groups of the last 4 chunks (kOneCommit)
      for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tll) {
        const int nt = t / a.npt;
        const int cg = GROUPED ? nt / a.ntg * a.Ckw : 0;  // the tile's group's first channel
        const float* src = a.Wp + (long long)nt * a.nkc * 2 * BN * kBK;
        // MODE 2: the tile's first output pixel, as a TMA im2col traversal start
        long long p0 = (long long)(a.pt_lo + t % a.npt) * kBM;
        if (CL == 2 && p0 >= a.P) p0 = 0;  // phantom tile of an odd pair: any in-range pixels
        const int n0 = (int)(p0 / E2), f0 = (int)(p0 % E2);
        const int cw = (f0 % E) * a.U - a.pad, ch = (f0 / E) * a.U - a.pad;
        if (MODE == 0 && doB) {
          // register-gather layers: L2-prefetch the input rows this CTA's NEXT tile gathers
          // (its window rows of every channel, one bulk prefetch per channel) a tile ahead,
          // so its compulsory misses hit L2 instead of DRAM
          const int tn = t + (int)gridDim.x;
          if (tn < ntile_total && a.C <= 16) {
            const long long q0 = (long long)(a.pt_lo + tn % a.npt) * kBM;
            const long long q1 = min(q0 + kBM, a.P) - 1;
            const int m0 = (int)(q0 / E2), m1 = (int)(q1 / E2);
            for (int nn = m0; nn <= m1; ++nn) {
              const int xa = nn == m0 ? (int)(q0 % E2) / E : 0, xb = nn == m1 ? (int)(q1 % E2) / E : E - 1;
              const int ha = max(0, xa * a.U - a.pad), hb = min(H - 1, xb * a.U - a.pad + R - 1);
              if (ha > hb) continue;
              for (int c = 0; c < a.C; ++c) {
                const float* rb = a.D + ((long long)nn * a.C + c) * HH + (long long)ha * H;
                const uintptr_t lo = reinterpret_cast<uintptr_t>(rb) & ~(uintptr_t)15;
                const uintptr_t hi = (reinterpret_cast<uintptr_t>(rb + (long long)(hb - ha + 1) * H) + 15) &
                                     ~(uintptr_t)15;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo))
                             : "memory");
              }
            }
          }
        }
        int ti = 0, tj = 0, cb = 0;  // K chunk kc = ((ti*R + tj)*ncb + cb)
        for (int kc = 0; kc < a.nkc; ++kc, ++g) {
          if (doA) {
            mbar_wait_lazy(emptyAs0 + 8 * sa, pha ^ 1u);
            TC_TRACE((a.dbg & 64) && blockIdx.x == 0, 12, g);
            if (a.dbg & 1) {  // profiling: skip the A gather
              mbar_arrive(fullAs0 + 8 * sa);
            } else {
              mbar_arrive_expect_tx(fullAs0 + 8 * sa, kAStageBytes);
              tma_im2col_4d(as_base + sa * kAStageBytes, &tmA, cg + cb * 32, cw, ch, n0, (uint16_t)tj, (uint16_t)ti,
                            fullAs0 + 8 * sa);
            }
            if (++sa == (uint32_t)kAS) { sa = 0; pha ^= 1u; }
            if (++cb == ncb) {
              cb = 0;
              if (++tj == R) { tj = 0; ++ti; }
            }
          }
          if (!doB) continue;
          const uint32_t s = sB, ph = phB;
          if (++sB == (uint32_t)SB) { sB = 0; phB ^= 1u; }
          const uint32_t jprev = SB == 2 ? jb[1] : SB == 3 ? jb[2] : jb[3];  // this stage's previous chunk
          jb[3] = jb[2];
          jb[2] = jb[1];
          jb[1] = jb[0];
          jb[0] = tll * ngtl + (uint32_t)kc / (uint32_t)kG;
          if (!kOneCommit) mbar_wait_lazy(emptyB0 + 8 * s, ph ^ 1u);
          else if (g >= (uint32_t)SB) gdone_wait(gdone0, jprev, true);
          if (CL == 2 && g >= (uint32_t)SB) {
            // this CTA has consumed the stage's previous use: tell the peer (its half goes
            // into this CTA's stage too) and wait for the peer's consumption likewise
            mbar_arrive_peer(emptyB0 + 8 * s, crank ^ 1u);
            mbar_wait_cluster_lazy(emptyB0 + 8 * s, ph ^ 1u);
          }
          TC_TRACE((a.dbg & 64) && blockIdx.x == 0, 8, g);
          if (a.dbg & 16) {
            mbar_arrive(fullB0 + 8 * s);
          } else if (CL == 2) {
            // rank 0 fetches the hi tile, rank 1 the lo tile, each into both CTAs
            const uint32_t hb = stage_bytes / 2u;
            mbar_arrive_expect_tx(fullB0 + 8 * s, stage_bytes);
            bulk_g2s_mc2(sbase + s * stage_bytes + crank * hb,
                         reinterpret_cast<const uint8_t*>(src + (long long)kc * 2 * BN * kBK) + crank * hb, hb,
                         fullB0 + 8 * s);
          } else {
            mbar_arrive_expect_tx(fullB0 + 8 * s, stage_bytes);
            bulk_g2s(sbase + s * stage_bytes, src + (long long)kc * 2 * BN * kBK, stage_bytes, fullB0 + 8 * s);
          }
        }
      }
    }
  } else if (warp == kMmaWarp || warp == kMmaWarp + 1) {
    // ================= MMA issuers =================
    // The K chunks of a tile form groups of kG (the last one may be shorter); issuer mw
    // takes every other group of this CTA (groups j = mw, mw + 2, ...) and issues all its
    // MMAs into its own accumulator X_mw: no accumulator is ever written by two threads,
    // so the accumulation order per output is fixed by construction (the pipe does not
    // order MMAs of different issuing threads into one accumulator: with two issuers
    // sharing accumulators under a turn barrier, ~1% of runs differed by a few ulps in
    // single outputs).  The epilogue drains X after every group and adds the partials in
    // group order.  Each issuer has a whole group of the other's MMAs to absorb its
    // commits, waits and its accumulator's drain.
    {
      const uint32_t mw = (uint32_t)(warp - kMmaWarp);
      // kind::tf32, D=F32, A/B = TF32, K-major, M = 128, N = BN
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kBM >> 4) << 24);
      const int my_tiles = (int)blockIdx.x < ntile_total ? (ntile_total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
      const uint32_t ngt = (uint32_t)(a.nkc + kG - 1) / (uint32_t)kG;  // groups per tile
      const uint32_t total = (uint32_t)my_tiles * ngt;
      const bool mprof = (a.dbg & 64) && blockIdx.x == 0;
      for (uint32_t j = mw; j < total; j += 2) {
        const uint32_t tl = j / ngt, jj = j - tl * ngt;
        const uint32_t c0 = tl * (uint32_t)a.nkc + jj * (uint32_t)kG;  // first CTA-local chunk
        const uint32_t nc = min((uint32_t)kG, (uint32_t)a.nkc - jj * (uint32_t)kG);
        // ring positions of chunk c: A chunk slot c % kSA (half-stages 2*slot, +1), B stage c % SB
        uint32_t cs[kG], cph[kG], bs[kG], bph[kG];
#pragma unroll
        for (int u = 0; u < kG; ++u) {
          const uint32_t c = c0 + (uint32_t)u;
          cs[u] = c % (uint32_t)kSA;
          cph[u] = (c / (uint32_t)kSA) & 1u;
          bs[u] = c % (uint32_t)SB;
          bph[u] = (c / (uint32_t)SB) & 1u;
        }
        const uint32_t xbuf = j % (uint32_t)kNX;
        const uint32_t d_tmem = tmem + xbuf * (uint32_t)BN;
        mbar_wait(acce0 + 8 * xbuf, ((j / (uint32_t)kNX) & 1u) ^ 1u);  // drained (group j - kNX)
        TC_TRACE(mprof, 11, c0);
        // all correction products of the group first, while the partial is still small,
        // then the main products: the tensor core truncates each add at the partial's ulp,
        // so the small terms lose nothing and the group costs one truncation per main MMA
        // (4 per chunk), as many as a main-only accumulator.  A chunk's corrections are
        // issued as soon as its operands are in, the mains after the last chunk's.
#pragma unroll
        for (int u = 0; u < kG; ++u)
          if ((uint32_t)u < nc) {
            mbar_wait(fullB0 + 8 * bs[u], bph[u]);
            mbar_wait(fullA0 + 8 * (2u * cs[u]), cph[u]);
            mbar_wait(fullA0 + 8 * (2u * cs[u] + 1u), cph[u]);
            tc_after();
            if (u == 0) TC_TRACE(mprof, 4, c0);
            if (elect_one() && !(a.dbg & 8)) {
#pragma unroll
              for (uint32_t hh = 0; hh < 2; ++hh)
#pragma unroll
                for (uint32_t k = 0; k < 2; ++k) {
                  const uint32_t a_hi = tmem + a_col0 + (2u * cs[u] + hh) * 32u + k * 8u, a_lo = a_hi + 16u;
                  const uint32_t b_hi = sbase + bs[u] * stage_bytes + hh * 64u + k * 32u;
                  const uint32_t b_lo = b_hi + (uint32_t)BN * 128u;
                  mma_tf32_ts(d_tmem, a_lo, desc_sw128(b_hi), idesc, (u | hh | k) ? 1u : 0u);
                  mma_tf32_ts(d_tmem, a_hi, desc_sw128(b_lo), idesc, 1u);
                }
            }
            __syncwarp();
          }
        if (elect_one()) {
          if (!(a.dbg & 8)) {
#pragma unroll
            for (int u = 0; u < kG; ++u)
              if ((uint32_t)u < nc) {
#pragma unroll
                for (uint32_t hh = 0; hh < 2; ++hh)
#pragma unroll
                  for (uint32_t k = 0; k < 2; ++k) {
                    const uint32_t a_hi = tmem + a_col0 + (2u * cs[u] + hh) * 32u + k * 8u;
                    const uint32_t b_hi = sbase + bs[u] * stage_bytes + hh * 64u + k * 32u;
                    mma_tf32_ts(d_tmem, a_hi, desc_sw128(b_hi), idesc, 1u);
                  }
              }
          }
          TC_TRACE(mprof, 5, c0);
          if (kOneCommit) {
            mma_commit(gdone0 + 8 * (j & 7u));  // frees the group's A slots, B stages, accumulator
          } else {
#pragma unroll
            for (int u = 0; u < kG; ++u)
              if ((uint32_t)u < nc) {
                mma_commit(emptyA0 + 8 * (2u * cs[u]));
                mma_commit(emptyA0 + 8 * (2u * cs[u] + 1u));
                mma_commit(emptyB0 + 8 * bs[u]);
              }
            mma_commit(accf0 + 8 * xbuf);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp >= kCkWarp0) {
    // ================= checksum warps (FUSE) =================
    // Co5[f] = sum_{c,i,j} Cd1[c][x*U+i-pad][y*U+j-pad] * Cw1[c][i][j] (conv_block,
    // checksums.hpp:135-145, FP64; zero padding) for f = blockIdx.x + k*gridDim.x: lanes
    // split the taps (kCkUnroll loads in flight each), a shuffle tree sums them.  The
    // compare runs in the next launch on the stream, which sees every store.
    // (The compare used to be the last CTA's job here; its code in the kernel pushed
    // the epilogue's drain loop into register spills: ~12% on the conv.)
    if constexpr (FUSE) {
      if (a.fd.cd1 && !(a.dbg & 8192)) {
        const int Kt = a.C * RR;
        const int cw = warp - kCkWarp0;
        for (int f = blockIdx.x + cw * gridDim.x; f < E2; f += kCkWarps * gridDim.x) {
          const int x = f / E, y = f - (f / E) * E;
          const int hb = x * a.U - a.pad, wb = y * a.U - a.pad;
          const double* cd = a.fd.cd1 + hb * H + wb;
          double acc = 0.0;
          for (int k0 = 0; k0 < Kt; k0 += 32 * kCkUnroll) {
            double v[kCkUnroll], w[kCkUnroll];
#pragma unroll
            for (int u = 0; u < kCkUnroll; ++u) {
              const int k = k0 + u * 32 + lane;
              v[u] = 0.0;
              w[u] = 0.0;
              if (k < Kt) {
                const int4 t = __ldg(reinterpret_cast<const int4*>(a.fd.taps + k));
                const int ti = t.y & 0xFFFF, tj = t.y >> 16;
                if ((unsigned)(hb + ti) < (unsigned)H && (unsigned)(wb + tj) < (unsigned)H) {
                  v[u] = __ldg(cd + t.x);
                  w[u] = __hiloint2double(t.w, t.z);
                }
              }
            }
#pragma unroll
            for (int u = 0; u < kCkUnroll; ++u) acc = fma(v[u], w[u], acc);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) a.fd.co5[f] = acc;
        }
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
    uint32_t gq = 0, tl = 0;  // CTA-local accumulator-group and tile counters
    const bool eprof = (a.dbg & 64) && blockIdx.x == 0 && threadIdx.x == kEpiWarp0 * 32;
    for (int t = blockIdx.x; t < ntile_total; t += gridDim.x, ++tl) {
      const int nt = t / a.npt;
      const int pt = a.pt_lo + t % a.npt;
      const long long p = (long long)pt * kBM + r;
      const bool valid = p < a.P;
      // P < 2^31 (tc_supported): 32-bit divisions (the 64-bit ones sat between a tile's
      // store and the next tile's first drain)
      const unsigned pu = valid ? (unsigned)p : 0u;
      const int n = (int)(pu / (unsigned)E2);
      const int f = (int)(pu - (unsigned)n * (unsigned)E2);
      const int x = f / E, y = f - (f / E) * E;
      // running sums of the group partials, in group order, in FP32 (several times closer
      // to the exact conv than the reference's sequential FP32 loop; FP64 sums for the
      // BN <= 64 tiles made the drain the issuers' bottleneck: VGG c2 2602 -> 2156 us)
      using acc_t = typename std::conditional<(HALF <= 32 && !FTC_EPI_F32), double, float>::type;
      acc_t sum[HALF];
#pragma unroll
      for (int jj = 0; jj < HALF; ++jj) sum[jj] = acc_t(0);
      int m0 = nt * BN + half * HALF, mlim = min(HALF, a.M - m0);
      if constexpr (GROUPED) {
        const int mg0 = nt / a.ntg * a.Mg;  // the group's first kernel
        m0 = mg0 + (nt % a.ntg) * BN + half * HALF;
        mlim = min(HALF, mg0 + a.Mg - m0);
      }
      // hooks (faults / repair mask) and partial column ranges: the sums go back into the
      // tile's last accumulator and a rolled loop with one out-of-line call per column
      // stores them (an unrolled hook body per column is instruction-cache bound); that
      // accumulator is released after the store
      const bool slow = !(mlim == HALF && !a.nfaults && !a.plane_mask);
      uint32_t xb = 0;
      const int ngt = (a.nkc + kG - 1) / kG;  // accumulator groups per tile
      for (int kc = 0; kc < ngt; ++kc, ++gq) {
        const uint32_t b = gq % (uint32_t)kNX;
        xb = tmem + lane_off + b * (uint32_t)BN + (uint32_t)(half * HALF);
        if (kOneCommit)
          gdone_wait(gdone0, gq, true);
        else
          mbar_wait_lazy(accf0 + 8 * b, (gq / (uint32_t)kNX) & 1u);
        TC_TRACE(eprof, 6, tl * (uint32_t)a.nkc + (uint32_t)(kc * kG));
        tc_after();
#pragma unroll
        for (int c16 = 0; c16 < HALF / 16; ++c16) {
          if (a.dbg & 4) break;
          uint32_t v[16];
          tmem_ld16(xb + (uint32_t)c16 * 16u, v);
          tmem_wait_ld();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) sum[c16 * 16 + jj] += (acc_t)__uint_as_float(v[jj]);
        }
        if (!slow || kc + 1 < ngt) {
          tc_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acce0 + 8 * b);
        }
        TC_TRACE(eprof, 7, tl * (uint32_t)a.nkc + (uint32_t)(kc * kG));
      }
      // tile store + fused FP64 row sums (m order, exact roundings)
      double rs = 0.0, rsm = 0.0;
      float* op = a.O + ((long long)n * a.M + m0) * E2 + f;
      const float* bp = a.bias ? a.bias + m0 : nullptr;
      if (!slow) {
        // the FP64 row sums only where someone reads them: So5 (rs) for the fused
        // CoC-D, both sums for the row-sum slabs; the plain conv stores only (3 FP64 ops
        // per output were a third of a 1-chunk tile's epilogue, VGG c1)
        const int sums = a.rowsum ? 2 : (FUSE ? 1 : 0);
        if (valid) {
          // running output pointer (one 64-bit add per column; the opaque asm keeps the
          // compiler from re-deriving op + jj * E2 for every store: that form, with the base
          // re-read from the constant bank, made the plain tile end ~10 instructions per
          // output and 3.3K cycles per tile -- SASS + r02cz no-store experiment)
          float* oq = op;
          if (sums == 0) {
#pragma unroll
            for (int jj = 0; jj < HALF; ++jj) {
              *oq = (float)sum[jj] + (bp ? __ldg(bp + jj) : 0.f);
              oq += E2;
              asm volatile("" : "+l"(oq));
            }
          } else if (sums == 1) {
            // So5 row sum as an error-free FP32 accumulation (TwoSum: s1 + e1 carries the
            // sum to ~2^-46 of the terms' magnitude; the screen's guard band is 1e-3 of
            // tau) and two conversions per thread: a cvt.f64.f32 + DADD per output ran at
            // ~6 conversions per clock per SM, 2.7K cycles of a 6K-cycle tile end that
            // the issuers wait on (r02ce traces)
            float s1 = 0.f, e1 = 0.f;
#pragma unroll
            for (int jj = 0; jj < HALF; ++jj) {
              const float val = (float)sum[jj] + (bp ? __ldg(bp + jj) : 0.f);
              *oq = val;
              oq += E2;
              asm volatile("" : "+l"(oq));
              const float t = __fadd_rn(s1, val);
              const float bb = __fsub_rn(t, s1);
              e1 = __fadd_rn(e1, __fadd_rn(__fsub_rn(s1, __fsub_rn(t, bb)), __fsub_rn(val, bb)));
              s1 = t;
            }
            rs = dadd((double)s1, (double)e1);
          } else {
#pragma unroll
            for (int jj = 0; jj < HALF; ++jj) {
              const float val = (float)sum[jj] + (bp ? __ldg(bp + jj) : 0.f);
              op[jj * E2] = val;
              rs = dadd(rs, (double)val);
              rsm = dadd(rsm, dmul((double)(m0 + jj), (double)val));
            }
          }
        }
      } else {
#pragma unroll
        for (int c16 = 0; c16 < HALF / 16; ++c16) {
          uint32_t v[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) v[jj] = __float_as_uint((float)sum[c16 * 16 + jj]);
          tmem_st16(xb + (uint32_t)c16 * 16u, v);
        }
        tmem_wait_st();
        const bool hooks = a.nfaults || a.plane_mask;
#pragma unroll 1
        for (int c0 = 0; c0 < mlim; c0 += 16) {
          uint32_t v[16];
          tmem_ld16(xb + (uint32_t)c0, v);
          tmem_wait_ld();
          if (valid) {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int j = c0 + jj;
              if (j < mlim) {
                float val = __uint_as_float(v[jj]);
                if (bp) val = val + __ldg(bp + j);
                int st = 1;
                if (hooks) {
                  const HookOut h =
                      epilogue_hooks(val, n, m0 + j, x, y, a.faults, a.nfaults, a.plane_mask, a.M, E, a.scale_tab);
                  val = h.v;
                  st = h.store;
                }
                if (st) op[(long long)j * E2] = val;
                rs = dadd(rs, (double)val);
                rsm = dadd(rsm, dmul((double)(m0 + j), (double)val));
              }
            }
          }
        }
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acce0 + 8 * ((gq - 1u) % (uint32_t)kNX));
      }
      if (valid && a.rowsum) {
        const long long o = (long long)(2 * nt + half) * a.P + p;
        a.rowsum[o] = rs;
        a.rowsum_m[o] = rsm;
      }
      // fused CoC-D: So5 accumulates from the row sums (order-free FP64 atomics; the exact
      // families are recomputed in reference order if anything is flagged)
      if (FUSE && valid && !(a.dbg & 4096)) atomicAdd(a.fd.so5 + f, rs);
      TC_TRACE(eprof, 9, tl);
    }
  }
  tc_before();
  __syncthreads();
  if (CL == 2) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  tc_after();
  if ((a.dbg & 64) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = g_tc_trace[4][0];
    for (int g = 0; g < 600; ++g) {
      printf("TRACE c %d", g);
      for (int k = 0; k < 13; ++k) printf(" %lld", g_tc_trace[k][g] - t0);
      printf("\n");
    }
    for (int g = 0; g < 6; ++g) printf("TRACE tile %d %lld\n", g, g_tc_trace[9][g] - t0);
  }
  if (warp == kLoaderWarp) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// W -> [ntiles][nkc][hi,lo][BN][32] with the SW128 chunk swizzle (16-byte chunk
// index XOR row%8), rows >= M and k >= K zero-padded.
__global__ void k_pack_w(const float* __restrict__ W, float* __restrict__ Wp, int Mg, int ntg, int K, int BN,
                         int ntiles, int nkc, int C, int RR, int tap_major) {
  const long long total = (long long)ntiles * nkc * BN * kBK;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e % kBK);
    const int row = (int)((e / kBK) % BN);
    const int kc = (int)((e / ((long long)kBK * BN)) % nkc);
    const int nt = (int)(e / ((long long)kBK * BN * nkc));
    // tile nt = (group, N-tile within the group); C = channels per group
    const int ml = (nt % ntg) * BN + row, m = nt / ntg * Mg + ml, kk = kc * kBK + k;
    // tap-major K (NHWC gather): kk = t*C + c  <->  reference index c*RR + t
    const long long src = tap_major ? (long long)m * K + (long long)(kk % C) * RR + kk / C : (long long)m * K + kk;
    const float w = (ml < Mg && kk < K) ? W[src] : 0.f;
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

// per-chunk taps for the channel-last gather (C % 32 == 0, so a chunk never straddles taps)
__global__ void k_build_tab_nhwc(int2* tab, int C, int H, int R, int nkc) {
  const int kc = blockIdx.x * blockDim.x + threadIdx.x;
  if (kc >= nkc) return;
  const int k0 = kc * kBK, t = k0 / C, c0 = k0 % C, i = t / R, j = t % R;
  tab[kc] = make_int2((i * H + j) * C + c0, (int)((1u << i) | (1u << (16 + j))));
}

// D[n][c][hw] -> Dt[n][hw][c] for images [n_lo, n_lo + gridDim.z), 32x32 tiles
__global__ void __launch_bounds__(256) k_nchw_to_nhwc(const float* __restrict__ D, float* __restrict__ Dt, int C,
                                                     int HW, int n_lo) {
  __shared__ float t[32][33];
  pdl_wait();
  const long long n = n_lo + blockIdx.z;
  const int hw0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const float* src = D + n * C * HW;
  float* dst = Dt + n * C * HW;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int c = c0 + r, hw = hw0 + threadIdx.x;
    if (c < C && hw < HW) t[r][threadIdx.x] = __ldg(src + (long long)c * HW + hw);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int hw = hw0 + r, c = c0 + threadIdx.x;
    if (c < C && hw < HW) dst[(long long)hw * C + c] = t[threadIdx.x][r];
  }
}

// D (NCHW) -> Dt (NHWC) and, optionally, the exact input checksums: a block owns a
// 32-channel x 8-position tile for every image; each thread accumulates its own (c, hw)
// over n ascending in FP64 (checksums.hpp:100-107 order), 8 images' loads in flight.
__global__ void __launch_bounds__(256) k_nhwc_cd(const float* __restrict__ D, float* __restrict__ Dt, int C,
                                                int HW, int n_lo, int nimg, double* __restrict__ cd1,
                                                double* __restrict__ cd2) {
  __shared__ float t[8][33];
  const int tid = threadIdx.x;
  const int cl = tid >> 3, hl = tid & 7;  // load: a warp reads 4 channel rows x 8 positions
  const int c = blockIdx.y * 32 + cl, hw = blockIdx.x * 8 + hl;
  const bool ok = hw < HW;
  const int wc = tid & 31, wh = tid >> 5;  // store: a warp writes one position's 32 channels
  const int sc = blockIdx.y * 32 + wc, shw = blockIdx.x * 8 + wh;
  double s1 = 0.0, s2 = 0.0;
  for (int b = 0; b < nimg; b += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = (ok && b + u < nimg) ? __ldg(D + ((long long)(n_lo + b + u) * C + c) * HW + hw) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (b + u >= nimg) break;
      if (cd1) {
        s1 = dadd(s1, (double)v[u]);
        s2 = dadd(s2, dmul((double)(n_lo + b + u), (double)v[u]));
      }
      t[hl][cl] = v[u];
      __syncthreads();
      if (shw < HW) Dt[((long long)(n_lo + b + u) * HW + shw) * C + sc] = t[wh][wc];
      __syncthreads();
    }
  }
  if (cd1 && ok) {
    cd1[(long long)c * HW + hw] = s1;
    cd2[(long long)c * HW + hw] = s2;
  }
}

// k_nhwc_cd with 32-channel x 32-position tiles: warp w loads channels w, w+8, w+16,
// w+24 (lane = position, 128-byte rows) for 8 images at a time (32 loads in flight per
// thread), accumulates the exact-order checksums of its 4 (c, position) items over n
// ascending, and writes each image's tile channel-last through shared memory.
struct Co5Scatter {  // optional: the block's share of Co5 = Cd1 (*) Cw1, scattered (FP64 atomics)
  double* co5;         // [E][E], zero on entry (the CoC-D kernel re-zeroes it)
  const double* cw1;   // [C][R][R]
  int H, R, U, pad, E;
};

// Small-batch staging pass (N <= 32): NHWC copy + exact-order Cd1/Cd2 (+ the Co5
// scatter) in one read of D.  A block owns 8 channels x 32 positions; a thread owns one
// (channel, position) and has all of a 16-image chunk's loads in flight (its Cd1/Cd2
// chain is sequential over n, checksums.hpp:100-107), the chunk is transposed through
// shared memory and stored as 32-byte channel runs of the NHWC rows.  Many small blocks
// (784 at config 1) keep load and store phases of different blocks overlapped.
constexpr int kStageImg = 16;
constexpr int kStageCh = 8;
__global__ void __launch_bounds__(256) k_nhwc_cd32(const float* __restrict__ D, float* __restrict__ Dt, int C,
                                                  int HW, int nimg, double* __restrict__ cd1,
                                                  double* __restrict__ cd2, Co5Scatter sc) {
  __shared__ float t[kStageImg][32][kStageCh + 1];
  constexpr int kScTaps = 9;
  __shared__ double red[kScTaps][kStageCh][32];
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hw = blockIdx.x * 32 + lane;
  const bool ok = hw < HW;
  const int c0 = blockIdx.y * kStageCh, c = c0 + warp;
  double s1 = 0.0, s2 = 0.0;
  for (int n0 = 0; n0 < nimg; n0 += kStageImg) {
    const int ni = min(kStageImg, nimg - n0);
    float v[kStageImg];
#pragma unroll
    for (int u = 0; u < kStageImg; ++u)
      v[u] = (ok && u < ni) ? __ldg(D + ((long long)(n0 + u) * C + c) * HW + hw) : 0.f;
#pragma unroll
    for (int u = 0; u < kStageImg; ++u) {
      if (u < ni && cd1) {  // ascending n, FP64, no contraction
        s1 = dadd(s1, (double)v[u]);
        s2 = dadd(s2, dmul((double)(n0 + u), (double)v[u]));
      }
      t[u][lane][warp] = v[u];
    }
    __syncthreads();
    // ni images x 32 positions = rows of 8 channels (32 bytes of an NHWC row); a warp
    // instruction stores 4 rows
    const int r4 = lane >> 3, ch = lane & 7;
    for (int row = warp * 4 + r4; row < ni * 32; row += 32) {
      const int u = row >> 5, pl = row & 31, sp = blockIdx.x * 32 + pl;
      if (sp < HW) Dt[((long long)(n0 + u) * HW + sp) * C + c0 + ch] = t[u][pl][ch];
    }
    __syncthreads();
  }
  pdl_trigger();
  if (cd1 && ok) {
    const long long e = (long long)c * HW + hw;
    cd1[e] = s1;
    cd2[e] = s2;
  }
  if (sc.co5) {
    // Co5 is linear in Cd1: this block's 8 channels x 32 input positions contribute
    // sum_c Cd1[c][h][w] * Cw1[c][i][j] to output (x, y) with x*U + i - pad = h (same for
    // y, j); channels are summed through shared memory, one atomic per (position, tap)
    const int RR = sc.R * sc.R;
    const int h = hw / sc.H, w = hw - (hw / sc.H) * sc.H;
    for (int t0 = 0; t0 < RR; t0 += kScTaps) {  // kScTaps taps per round, one barrier each
      const int nt = min(kScTaps, RR - t0);
      for (int tt = 0; tt < nt; ++tt) red[tt][warp][lane] = s1 * sc.cw1[c * RR + t0 + tt];
      __syncthreads();
      for (int tt = warp; tt < nt; tt += kStageCh) {  // warp per tap: channel sum, one atomic per position
        if (!ok) continue;
        double a = 0.0;
#pragma unroll
        for (int ww = 0; ww < kStageCh; ++ww) a += red[tt][ww][lane];
        const int tap = t0 + tt, i = tap / sc.R, j = tap - (tap / sc.R) * sc.R;
        const int xs = h + sc.pad - i, ys = w + sc.pad - j;
        if (xs >= 0 && ys >= 0 && xs % sc.U == 0 && ys % sc.U == 0) {
          const int x = xs / sc.U, y = ys / sc.U;
          if (x < sc.E && y < sc.E) atomicAdd(sc.co5 + x * sc.E + y, a);
        }
      }
      __syncthreads();
    }
  }
}

// Per-device state: the SM count sizes the persistent grid, and the 227 KB dynamic
// shared-memory opt-in is a per-device function attribute.
constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 || dev >= kMaxDevices ? 0 : dev;
}

int num_sms(int dev) {
  static int sms[kMaxDevices] = {0};
  if (sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = n > 0 ? n : 148;
  }
  return sms[dev];
}

template <int BN, int MODE, bool FUSE, bool GROUPED>
int launch_bn(const TcArgs& a, const CUtensorMap& tm, int grid, size_t smem, cudaStream_t s) {
  static bool attr_set[kMaxDevices] = {false};
  const int dev = current_device();
  if (!attr_set[dev]) {
    FTC_CUDA_CHECK(cudaFuncSetAttribute(k_conv_tc<BN, MODE, FUSE, GROUPED>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_set[dev] = true;
  }
  FTC_LAUNCH_PDL(k_conv_tc<BN, MODE, FUSE, GROUPED>, dim3(grid), dim3(kThreads), smem, s, a, tm);
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

// CTA-pair launch (cluster of 2, B multicast): grid = 2 x the co-resident cluster count
template <int BN, bool FUSE>
int launch_cl2(const TcArgs& a, const CUtensorMap& tm, int tiles, size_t smem, cudaStream_t s) {
  static bool attr_set[kMaxDevices] = {false};
  static int max_clusters[kMaxDevices] = {0};
  const int dev = current_device();
  auto k = k_conv_tc<BN, 2, FUSE, false, 2>;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (!attr_set[dev]) {
    FTC_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    cfg.gridDim = dim3((unsigned)(num_sms(dev) & ~1));
    int nc = 0;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&nc, k, &cfg) != cudaSuccess || nc < 1) nc = num_sms(dev) / 2;
    cfg.numAttrs = 2;
    max_clusters[dev] = nc;
    attr_set[dev] = true;
  }
  const int cap = 2 * max_clusters[dev];
  cfg.gridDim = dim3((unsigned)(tiles < cap ? tiles : cap));
  FTC_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k, a, tm));
  count_launch();
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // namespace

bool tc_supported(const ftc_conv_desc& d) {
  if (d.groups < 1 || d.C % d.groups || d.M % d.groups) return false;
  if (d.R > 15) return false;  // tap validity bits: rows 0-14, columns 16-30
  const long long Ckw = d.C / d.groups, Mg = d.M / d.groups;
  const long long K = Ckw * d.R * d.R;
  const long long nkc = (K + kBK - 1) / kBK;
  const long long bn = Mg <= 128 ? ((Mg + 31) / 32) * 32 : 128;
  if (1024 + stages_host(bn) * bn * 256 + nkc * kBK * 8 + 512 > 227 * 1024) return false;
  if ((long long)d.C * d.H * d.H >= (1LL << 31)) return false;
  const long long E = (d.H + 2LL * d.pad - d.R) / d.stride + 1;
  if ((long long)d.N * E * E >= (1LL << 31)) return false;
  return true;
}

int tc_plan_create(const ftc_conv_desc& d, const float* W_dev, TcPlan** out, cudaStream_t s) {
  TcPlan* p = new TcPlan();
  p->M = d.M;
  p->groups = d.groups;
  p->Ckw = d.C / d.groups;
  p->Mg = d.M / d.groups;
  p->Ctot = d.C;
  p->K = p->Ckw * d.R * d.R;
  p->nkc = (p->K + kBK - 1) / kBK;
  if (p->Mg <= 128) {
    p->BN = ((p->Mg + 31) / 32) * 32;
    p->ntg = 1;
  } else {
    p->BN = 128;
    p->ntg = (p->Mg + 127) / 128;
  }
  // channel-last gather: faster producers, but with the MMA issue chain the bottleneck it
  // does not pay for its transpose pass yet (AlexNet conv2 669 vs 641 us): opt-in
  // K order: tap-major (k = (i*R + j)*C + c) for the channel-last paths
  const bool corners_ok = d.pad <= 127 && d.pad - (d.R - 1) >= -128 && d.stride <= 8;
  p->im2col = p->Ckw % 32 == 0 && corners_ok && !getenv("FTC_TC_NO_TMA") && !getenv("FTC_TC_NHWC");
  p->nhwc = !p->im2col && d.groups == 1 && d.C % 32 == 0 && getenv("FTC_TC_NHWC") != nullptr;
  if (const char* bn = getenv("FTC_TC_MAX_BN")) {  // experimentation: cap the N tile
    const int cap = atoi(bn);
    if ((cap == 32 || cap == 64 || cap == 96 || cap == 128) && p->BN > cap) {
      p->BN = cap;
      p->ntg = (p->Mg + cap - 1) / cap;
    }
  }
  p->ntiles = p->groups * p->ntg;
  const size_t n = (size_t)p->ntiles * p->nkc * 2 * p->BN * kBK;
  if (cudaMalloc(&p->Wp, n * sizeof(float)) != cudaSuccess) {
    delete p;
    set_error(FTC_CUDA_ERROR, "cudaMalloc(packed W) failed");
    return FTC_CUDA_ERROR;
  }
  FTC_LAUNCH(k_pack_w<<<592, 256, 0, s>>>(W_dev, p->Wp, p->Mg, p->ntg, p->K, p->BN, p->ntiles, p->nkc, p->Ckw, d.R * d.R,
                                         (p->nhwc || p->im2col) ? 1 : 0));
  if (cudaMalloc(&p->tab, (size_t)p->nkc * kBK * sizeof(int2)) != cudaSuccess) {
    cudaFree(p->Wp);
    delete p;
    set_error(FTC_CUDA_ERROR, "cudaMalloc(tap table) failed");
    return FTC_CUDA_ERROR;
  }
  if (p->im2col) {
    if (cudaMalloc(&p->Dt, (size_t)d.N * d.C * d.H * d.H * sizeof(float)) != cudaSuccess) {
      cudaFree(p->Wp);
      cudaFree(p->tab);
      delete p;
      set_error(FTC_CUDA_ERROR, "cudaMalloc(NHWC input copy) failed");
      return FTC_CUDA_ERROR;
    }
    // NHWC tensor {C, W, H, N}; the traversal box spans the output positions' window
    // origins (lower corner -pad, upper corner pad - (R-1)) with stride U
    const cuuint64_t dims[4] = {(cuuint64_t)d.C, (cuuint64_t)d.H, (cuuint64_t)d.H, (cuuint64_t)d.N};
    const cuuint64_t strides[3] = {(cuuint64_t)d.C * 4, (cuuint64_t)d.C * d.H * 4,
                                   (cuuint64_t)d.C * d.H * d.H * 4};
    const int lower[2] = {-d.pad, -d.pad};
    const int upper[2] = {d.pad - (d.R - 1), d.pad - (d.R - 1)};
    const cuuint32_t estr[4] = {1, (cuuint32_t)d.stride, (cuuint32_t)d.stride, 1};
    // driver entry point resolved at run time: the library carries no link-time
    // dependency on libcuda (it must load on driverless build hosts)
    static PFN_cuTensorMapEncodeIm2col_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q{};
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                  &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        encode = nullptr;
    }
    const CUresult cr = !encode ? CUDA_ERROR_NOT_FOUND : encode(&p->tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p->Dt, dims, strides,
                                                lower, upper, 32, 128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
      cudaFree(p->Wp);
      cudaFree(p->tab);
      cudaFree(p->Dt);
      delete p;
      set_error(FTC_CUDA_ERROR, "cuTensorMapEncodeIm2col failed (" + std::to_string((int)cr) + ")");
      return FTC_CUDA_ERROR;
    }
  } else if (p->nhwc) {
    cudaMemsetAsync(p->tab, 0, (size_t)p->nkc * kBK * sizeof(int2), s);
    FTC_LAUNCH(k_build_tab_nhwc<<<(p->nkc + 255) / 256, 256, 0, s>>>(p->tab, d.C, d.H, d.R, p->nkc));
    if (cudaMalloc(&p->Dt, (size_t)d.N * d.C * d.H * d.H * sizeof(float)) != cudaSuccess) {
      cudaFree(p->Wp);
      cudaFree(p->tab);
      delete p;
      set_error(FTC_CUDA_ERROR, "cudaMalloc(NHWC input copy) failed");
      return FTC_CUDA_ERROR;
    }
  } else {
    FTC_LAUNCH(k_build_tab<<<(p->nkc * kBK + 255) / 256, 256, 0, s>>>(p->tab, p->Ckw, d.H, d.R, p->K,
                                                                     p->nkc * kBK));
  }
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
  if (p->Dt) cudaFree(p->Dt);
  delete p;
}

int tc_rowsum_parts(const TcPlan* p) { return p ? 2 * p->ntiles : 1; }
bool tc_im2col(const TcPlan* p) { return p && p->im2col; }

// Whether the conv's single checksum warp finishes Co5 well inside the conv: its
// latency rounds (one L2 round trip per kCkUnroll taps per lane, ~700 cycles) against
// the CTA's MMA work (~1000 cycles per K chunk of a tile).  Small convs (config 1: 21
// positions x 576 taps per CTA vs ~3 tiles x 18 chunks) take a separate Co5 kernel.
bool tc_co5_in_kernel(const TcPlan* p, int N, int E) {
  if (!p) return false;
  const long long E2 = (long long)E * E;
  const long long grid = 148;
  const long long pos = (E2 + grid - 1) / grid;
  const long long Kc = (long long)p->K * p->groups;  // Co5 taps run over all channels
  const long long rounds = pos * ((Kc + 32LL * kCkUnroll - 1) / (32LL * kCkUnroll));
  const long long tiles = ((long long)N * E2 + kBM - 1) / kBM * p->ntiles;
  // ~1,000 cycles per K chunk with the TMA im2col A operand, ~1,800 with the register gather
  const long long conv = (tiles + grid - 1) / grid * p->nkc * (p->im2col ? 1000LL : 1800LL);
  // a round is two dependent loads (tap entry, then Cd1) through an L2 the conv keeps
  // ~85% busy: measured ~7,300 cycles (VGG-19 c4: the checksum warp finished 0.55 ms after
  // the MMAs, c3 / c2 75-85 us; r02cc ncu lists).  Layers that do not fit take Co5 in the
  // CoC-D kernel after the conv instead.
  static const long long round_cycles = getenv("FTC_CO5_ROUND") ? atoll(getenv("FTC_CO5_ROUND")) : 8000LL;
  return rounds * round_cycles <= conv;
}
float* tc_nhwc_buffer(const TcPlan* p) { return p ? p->Dt : nullptr; }

int launch_nhwc_cd(const float* D, float* Dt, int C, int HW, int n_lo, int nimg, double* cd1, double* cd2,
                   cudaStream_t s, const Co5Job* co5) {
  if (C % 32) {
    set_error(FTC_CONFIG_ERROR, "launch_nhwc_cd: C % 32 != 0");
    return FTC_CONFIG_ERROR;
  }
  static bool carve = false;
  if (!carve && getenv("FTC_CARVEOUT")) {
    cudaFuncSetAttribute(k_nhwc_cd, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    carve = true;
  }
  if (!cd1) {  // transpose only: parallel over images too
    const dim3 tg((unsigned)((HW + 31) / 32), (unsigned)(C / 32), (unsigned)nimg);
    FTC_LAUNCH_PDL(k_nchw_to_nhwc, tg, dim3(32, 8), 0, s, D, Dt, C, HW, n_lo);
    FTC_CUDA_CHECK(cudaGetLastError());
    return FTC_OK;
  }
  if (n_lo == 0) {
    const dim3 g((unsigned)((HW + 31) / 32), (unsigned)(C / kStageCh));
    Co5Scatter sc{};
    if (co5 && cd1) sc = Co5Scatter{co5->co5, co5->cw1, co5->H, co5->R, co5->U, co5->pad, co5->E};
    FTC_LAUNCH_PDL(k_nhwc_cd32, g, dim3(256), 0, s, D, Dt, C, HW, nimg, cd1, cd2, sc);
    FTC_CUDA_CHECK(cudaGetLastError());
    return FTC_OK;
  }
  const dim3 g((unsigned)((HW + 7) / 8), (unsigned)(C / 32));
  FTC_LAUNCH(k_nhwc_cd<<<g, 256, 0, s>>>(D, Dt, C, HW, n_lo, nimg, cd1, cd2));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

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
  a.Ckw = p->Ckw;
  a.Mg = p->Mg;
  a.ntg = p->ntg;
  const long long E2 = (long long)c.E * c.E;
  a.P = (long long)c.N * E2;
  const long long p_lo = (long long)c.img_lo * E2, p_hi = (long long)c.img_hi * E2;
  a.pt_lo = (int)(p_lo / kBM);
  a.npt = (int)((p_hi + kBM - 1) / kBM) - a.pt_lo;
  if (a.npt <= 0) return FTC_OK;
  a.faults = c.faults;
  a.nfaults = c.nfaults;
  a.scale_tab = c.scale_tab;
  a.rowsum = c.rowsum;
  a.rowsum_m = c.rowsum_m;
  a.plane_mask = c.plane_mask;
  const int n_sms = num_sms(current_device());
  const int tiles = a.ntiles * a.npt;
  const int grid = tiles < n_sms ? tiles : n_sms;
  // as many B stages as shared memory allows (2..8) after the tap table
  const size_t fixed = p->im2col ? 1024 + (size_t)kAS * kAStageBytes + 512 : 1024 + (size_t)p->nkc * kBK * 8 + 512;
  int SB = (int)((227 * 1024 - fixed) / ((size_t)p->BN * 256));
  SB = SB > 4 ? 4 : SB;  // deeper B rings measured no faster and take L1 capacity
  if (SB < stages_host(p->BN)) {
    set_error(FTC_CONFIG_ERROR, "tcgen05 conv: shared memory too small for the B ring");
    return FTC_CONFIG_ERROR;
  }
  if (const char* e = getenv("FTC_TC_B_STAGES")) {  // experimentation
    const int v = atoi(e);
    if (v >= stages_host(p->BN) && v < SB) SB = v;
  }
  a.SB = SB;
  a.dbg = getenv("FTC_TC_DEBUG") ? atoi(getenv("FTC_TC_DEBUG")) : 0;
  const size_t smem = fixed + (size_t)SB * p->BN * 256;
  if (p->nhwc || p->im2col) {
    if (!c.dt_ready) {
      const int st = launch_nhwc_cd(c.D, p->Dt, c.C, c.H * c.H, c.img_lo, c.img_hi - c.img_lo, nullptr, nullptr, s);
      if (st != FTC_OK) return st;
    }
    a.D = p->Dt;
  }
  const bool fuse = c.fd != nullptr;
  if (fuse) {
    if (p->nhwc) {
      set_error(FTC_CONFIG_ERROR, "fused detection: not with the NHWC gather engine");
      return FTC_CONFIG_ERROR;
    }
    a.fd = *c.fd;
  }
  // CTA pairs sharing the B stream (k_conv_tc<..., CL = 2>): TMA im2col layers over the
  // full pixel range with enough tiles for every pair
  static const int cl_mode = getenv("FTC_TC_CL") ? atoi(getenv("FTC_TC_CL")) : 0;
  if (cl_mode == 2 && p->im2col && p->groups == 1 && a.pt_lo == 0 && p_hi == a.P && (p->BN == 64 || p->BN == 128) &&
      tiles >= 2 * n_sms) {
    a.npt = (a.npt + 1) & ~1;
    const int tiles2 = a.ntiles * a.npt;
    if (p->BN == 128)
      return fuse ? launch_cl2<128, true>(a, p->tmA, tiles2, smem, s) : launch_cl2<128, false>(a, p->tmA, tiles2, smem, s);
    return fuse ? launch_cl2<64, true>(a, p->tmA, tiles2, smem, s) : launch_cl2<64, false>(a, p->tmA, tiles2, smem, s);
  }
#define FTC_BN_SWITCH(MODE, FUSE)                                                            \
  switch (p->BN) {                                                                           \
    case 32: return grouped ? launch_bn<32, MODE, FUSE, true>(a, p->tmA, grid, smem, s)       \
                            : launch_bn<32, MODE, FUSE, false>(a, p->tmA, grid, smem, s);     \
    case 64: return grouped ? launch_bn<64, MODE, FUSE, true>(a, p->tmA, grid, smem, s)       \
                            : launch_bn<64, MODE, FUSE, false>(a, p->tmA, grid, smem, s);     \
    case 96: return grouped ? launch_bn<96, MODE, FUSE, true>(a, p->tmA, grid, smem, s)       \
                            : launch_bn<96, MODE, FUSE, false>(a, p->tmA, grid, smem, s);     \
    case 128: return grouped ? launch_bn<128, MODE, FUSE, true>(a, p->tmA, grid, smem, s)     \
                             : launch_bn<128, MODE, FUSE, false>(a, p->tmA, grid, smem, s);   \
  }
  const bool grouped = p->groups > 1;
  if (p->im2col) {
    if (fuse) {
      FTC_BN_SWITCH(2, true)
    } else {
      FTC_BN_SWITCH(2, false)
    }
  } else if (p->nhwc) {
    switch (p->BN) {
      case 32: return launch_bn<32, 1, false, false>(a, p->tmA, grid, smem, s);
      case 64: return launch_bn<64, 1, false, false>(a, p->tmA, grid, smem, s);
      case 96: return launch_bn<96, 1, false, false>(a, p->tmA, grid, smem, s);
      case 128: return launch_bn<128, 1, false, false>(a, p->tmA, grid, smem, s);
    }
  } else if (fuse) {
    FTC_BN_SWITCH(0, true)
  } else {
    FTC_BN_SWITCH(0, false)
  }
#undef FTC_BN_SWITCH
  set_error(FTC_CONFIG_ERROR, "unsupported BN");
  return FTC_CONFIG_ERROR;
}

}  // namespace ftc

