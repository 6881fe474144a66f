// ftc_glue.cu -- inter-layer glue for the BASELINE conv stacks (configs 2-5).
//
// The reference feeds conv -> conv directly (replay.hpp:14-25 clean_chain) and has
// no activation, pooling or residual ops; the BASELINE nets need them between the
// protected convs.  These kernels are the device side of that glue: ReLU /
// leaky-ReLU(0.1) fused with max pooling, residual add + activation, and the
// explicit asymmetric zero-pad / crop that expresses floor-mode strided convs
// through the reference's exact extent rule.  ABFT protects the conv
// outputs themselves (pre-activation), exactly the tensors the checksums cover.
#include <cuda_runtime.h>

#include "ftc_common.cuh"

namespace ftc {
namespace {

__device__ __forceinline__ float act_fn(float v, int act) {
  if (act == 1) return v > 0.f ? v : 0.f;
  if (act == 2) return v > 0.f ? v : 0.1f * v;
  return v;
}

// act + pool, NCHW output only, one thread per output element (flat over (n, c, x, y)
// with 32-bit index math): no idle threads on small planes (a plane-per-block-row grid
// left 86% of the threads of a 6x6-output pool idle).
template <int KT>
__global__ void __launch_bounds__(256) k_act_pool_flat(const float* __restrict__ in, float* __restrict__ out,
                                                      unsigned total, int H, int Ho, int act, int kr, int s, int p) {
  const int k = KT > 0 ? KT : kr;
  const unsigned plane = (unsigned)(Ho * Ho);
  pdl_wait();
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const unsigned pl = e / plane, pos = e - pl * plane;
    const int ox = (int)(pos / (unsigned)Ho), oy = (int)pos - ox * Ho;
    const int x0 = ox * s - p, y0 = oy * s - p;
    const float* src = in + (long long)pl * H * H;
    float m = -INFINITY;
    if constexpr (KT > 0) {
      float v[KT * KT];
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          const int x = x0 + i, y = y0 + j;
          v[i * KT + j] = ((unsigned)x < (unsigned)H && (unsigned)y < (unsigned)H) ? __ldg(src + x * H + y) : 0.f;
        }
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j)
          if ((unsigned)(x0 + i) < (unsigned)H && (unsigned)(y0 + j) < (unsigned)H)
            m = fmaxf(m, act_fn(v[i * KT + j], act));
    } else {
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j)
          if ((unsigned)(x0 + i) < (unsigned)H && (unsigned)(y0 + j) < (unsigned)H)
            m = fmaxf(m, act_fn(__ldg(src + (x0 + i) * H + y0 + j), act));
    }
    out[e] = m;
  }
}

// Workspace layout shared by the Cd1 producers (Cd1Ws): [Cd1: per][tickets][G slabs]
struct Cd1Ws {
  long long per;       // C * H * H
  long long tick_off;  // in doubles
  long long slab_off;  // in doubles
  int tickets;
};

__device__ __forceinline__ unsigned int* ws_tickets(double* ws, long long tick_off) {
  return reinterpret_cast<unsigned int*>(ws + tick_off);
}

// last of the G group blocks of a tile folds the slabs (g ascending) into Cd1 at
// positions [e0, e0 + count) and re-arms the tile's ticket
__device__ __forceinline__ bool ws_arrive(double* ws, long long tick_off, int tile, int G) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ws_tickets(ws, tick_off) + tile, 1u) == (unsigned)(G - 1);
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// Clean-path Cd1 = sum_n D_n (FP64, any order -- CoC-D is tolerance based; the error
// path recomputes the exact-order checksums, checksums.hpp:100-107).  Workspace
// [Cd1][G partial slabs][tickets], zero-filled once: block (x, g) sums image group g at
// 256 positions (one per thread, 32 loads in flight), and the last group block of each x
// folds the slabs into Cd1 (g ascending) and re-arms its ticket.
#ifndef FTC_CD_UNROLL
#define FTC_CD_UNROLL 32
#endif
constexpr int kCdUnroll = FTC_CD_UNROLL;
__global__ void __launch_bounds__(256) k_cd1_parts(const float* __restrict__ D, int N, long long per, int NG,
                                                  double* __restrict__ ws, long long tick_off, long long slab_off) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y, G = gridDim.y;
  const int n_lo = g * NG, n_hi = min(N, n_lo + NG);
  pdl_wait();
  if (e < per) {
    double a = 0.0;
    int n = n_lo;
    for (; n + kCdUnroll <= n_hi; n += kCdUnroll) {  // kCdUnroll loads in flight per thread
      float v[kCdUnroll];
#pragma unroll
      for (int u = 0; u < kCdUnroll; ++u) v[u] = __ldcs(D + (long long)(n + u) * per + e);
#pragma unroll
      for (int u = 0; u < kCdUnroll; ++u) a += (double)v[u];
    }
    for (; n + 4 <= n_hi; n += 4) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(D + (long long)(n + u) * per + e);
#pragma unroll
      for (int u = 0; u < 4; ++u) a += (double)v[u];
    }
    for (; n < n_hi; ++n) a += (double)__ldcs(D + (long long)n * per + e);
    ws[slab_off + per * g + e] = a;
  }
  pdl_trigger();
  if (ws_arrive(ws, tick_off, blockIdx.x, G)) {
    if (e < per) {
      double t = 0.0;
      for (int gg = 0; gg < G; ++gg) t += __ldcg(ws + slab_off + per * gg + e);
      ws[e] = t;
    }
    if (threadIdx.x == 0) ws_tickets(ws, tick_off)[blockIdx.x] = 0u;
  }
}

// k = 1 (activation only) producer of a protected conv's input, positions % 4 == 0:
// act(O) -> D (NCHW, float4 stores) + the TMA engine's NHWC copy + the clean-path Cd1
// slabs, 32 channels x 32 positions per block.  A thread owns one channel x 4 positions
// (one 16-byte load per image) and keeps four images' loads in flight (~128 KB per SM
// at full occupancy: the 8-position variant held 16 KB and sat on memory latency at
// ~3.2 TB/s, r02b ncu); the NHWC rows go out through a shared-memory transpose, one
// barrier pair per four images.
// POOL2: 2x2 stride-2 max-pool after the activation (Ho % 4 == 0, so a thread's 4
// output positions share a row and read two rows of 8 inputs: four 16-byte loads).
#ifndef FTC_V4_PLAIN_IMG
#define FTC_V4_PLAIN_IMG 8
#endif
constexpr int kV4ImgPlain = FTC_V4_PLAIN_IMG;
// images in flight per thread: 8 for the activation-only form (one 16-byte load per image;
// VGG-19 ReLU passes 992 / 957 / 944 us per step at 4 / 2 / 8), 2 for the 2x2-pool form
// (four loads per image: 420 -> 317 us, 4.0 -> 5.3 TB/s; 432 at 1, 408 at 8 -- fewer
// registers, more resident blocks, shorter load / transpose / store phases per barrier)
#ifndef FTC_V4_POOL_IMG
#define FTC_V4_POOL_IMG 2
#endif
// CD1 = false: the same pass without the checksum (the unprotected net's glue, so that the
// ABFT overhead is measured against equally tuned kernels).
template <int ACT, bool POOL2, bool VEC = true, bool CD1 = true>
__global__ void __launch_bounds__(256) k_act_v4_cd1(const float* __restrict__ in, float* __restrict__ out,
                                                   float* __restrict__ out_t, int N, int NG, int C, int HW,
                                                   double* __restrict__ ws, long long tick_off, long long slab_off,
                                                   int Ho) {
  // [image][position][channel], rows of 36 floats (16-byte aligned) with the 4-channel
  // groups of a row XOR-permuted by (position / 8) % 4: the transposing 4-byte writes of a
  // warp (8 positions 4 apart x 4 channels) and the 16-byte row reads are conflict-free
  constexpr int kV4Img = POOL2 ? FTC_V4_POOL_IMG : kV4ImgPlain;
  __shared__ __align__(16) float tile[kV4Img][32][36];
  const int tid = threadIdx.x;
  const int cl = tid >> 3, p4 = (tid & 7) * 4;  // load role: channel row, 4 positions
  const int c = blockIdx.y * 32 + cl, pos = blockIdx.x * 32 + p4;
  const int g4 = tid & 7, prow = tid >> 3;    // store role: 4-channel group (physical), position row
  const int g = blockIdx.z, G = gridDim.z;
  const int n_lo = g * NG, n_hi = min(N, n_lo + NG);
  // VEC: HW % 4 == 0 and 16-byte aligned tensors, so a thread's 4 positions are one
  // float4; otherwise four scalar accesses with per-element bounds (odd extents such as
  // the 57x57 / 55x55 pad and crop outputs of ResNet-18's stride-2 blocks)
  const bool ok = pos < HW;
  const int nq = VEC ? 4 : min(4, HW - pos);
  const long long plane_c = (long long)C * HW;
  // input: HW positions per plane without pooling, (2 Ho)^2 with it
  const int Hi = POOL2 ? 2 * Ho : 0;
  const long long iplane = POOL2 ? (long long)Hi * Hi : HW;
  const long long istep4 = (long long)C * iplane / 4;
  long long ioff = pos;  // element offset of this thread's first input in its plane
  if (POOL2) {
    const int ox = pos / Ho, oy = pos - (pos / Ho) * Ho;
    ioff = (long long)(2 * ox) * Hi + 2 * oy;
  }
  pdl_wait();
  // (with !VEC the pointers are only carriers of the element address: accessed as float)
  const float4* src = reinterpret_cast<const float4*>(in + ((long long)n_lo * C + c) * iplane + ioff);
  float4* op = out ? reinterpret_cast<float4*>(out + ((long long)n_lo * C + c) * HW + pos) : nullptr;
  const long long step4 = plane_c / 4;  // VEC only
  const int row4 = POOL2 ? Hi / 4 : 0;  // one input row in float4s
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int n = n_lo; n < n_hi; n += kV4Img) {
    const int cnt = min(kV4Img, n_hi - n);
    float4 v[kV4Img];
    if (POOL2) {
      float4 r[kV4Img][4];
#pragma unroll
      for (int u = 0; u < kV4Img; ++u)
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4)
          r[u][k4] = (ok && u < cnt) ? __ldcs(src + u * istep4 + (k4 >> 1) * row4 + (k4 & 1))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < kV4Img; ++u) {
        // output j of the 4 takes input columns 2j, 2j+1 of both rows (max of act, the
        // pooling kernels' -inf start)
        const float a0[8] = {r[u][0].x, r[u][0].y, r[u][0].z, r[u][0].w, r[u][1].x, r[u][1].y, r[u][1].z, r[u][1].w};
        const float a1[8] = {r[u][2].x, r[u][2].y, r[u][2].z, r[u][2].w, r[u][3].x, r[u][3].y, r[u][3].z, r[u][3].w};
        float m[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float mm = -INFINITY;
          mm = fmaxf(mm, act_fn(a0[2 * j], ACT));
          mm = fmaxf(mm, act_fn(a0[2 * j + 1], ACT));
          mm = fmaxf(mm, act_fn(a1[2 * j], ACT));
          mm = fmaxf(mm, act_fn(a1[2 * j + 1], ACT));
          m[j] = mm;
        }
        v[u] = make_float4(m[0], m[1], m[2], m[3]);
      }
    } else {
      if (VEC) {
#pragma unroll
        for (int u = 0; u < kV4Img; ++u)
          v[u] = (ok && u < cnt) ? __ldcs(src + u * istep4) : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        const float* sf = in + ((long long)n * C + c) * iplane + ioff;  // element addressing
#pragma unroll
        for (int u = 0; u < kV4Img; ++u) {
          float e4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            e4[q] = (ok && u < cnt && q < nq) ? __ldcs(sf + (long long)u * C * iplane + q) : 0.f;
          v[u] = make_float4(e4[0], e4[1], e4[2], e4[3]);
        }
      }
#pragma unroll
      for (int u = 0; u < kV4Img; ++u) {
        v[u].x = act_fn(v[u].x, ACT);
        v[u].y = act_fn(v[u].y, ACT);
        v[u].z = act_fn(v[u].z, ACT);
        v[u].w = act_fn(v[u].w, ACT);
      }
    }
#pragma unroll
    for (int u = 0; u < kV4Img; ++u) {
      if (ok && u < cnt) {
        if (VEC) {
          if (op) op[u * step4] = v[u];
          if (CD1) {
            acc[0] += (double)v[u].x;
            acc[1] += (double)v[u].y;
            acc[2] += (double)v[u].z;
            acc[3] += (double)v[u].w;
          }
        } else {
          const float e4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
          float* of = out ? out + ((long long)(n + u) * C + c) * HW + pos : nullptr;  // element addressing
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nq) {
              if (of) of[q] = e4[q];
              if (CD1) acc[q] += (double)e4[q];
            }
        }
      }
    }
    if (out_t) {
#pragma unroll
      // a thread's 4 positions p4 .. p4+3 share (position / 8), hence one column
      const int wcol = (((cl >> 2) ^ ((p4 >> 3) & 3)) << 2) | (cl & 3);
#pragma unroll
      for (int u = 0; u < kV4Img; ++u) {
        tile[u][p4 + 0][wcol] = v[u].x;
        tile[u][p4 + 1][wcol] = v[u].y;
        tile[u][p4 + 2][wcol] = v[u].z;
        tile[u][p4 + 3][wcol] = v[u].w;
      }
      __syncthreads();
      // kV4Img images x 32 positions of 32-channel NHWC rows as 16-byte stores: a thread
      // owns (position row, 4-channel group) of every image, a warp 4 whole rows
      {
        const int sp = blockIdx.x * 32 + prow;
        const int lg = g4 ^ ((prow >> 3) & 3);  // logical group of physical group g4
        if (sp < HW) {
          float4* dst = reinterpret_cast<float4*>(out_t + ((long long)n * HW + sp) * C + blockIdx.y * 32 + 4 * lg);
          const long long istep = (long long)HW * C / 4;
#pragma unroll
          for (int u = 0; u < kV4Img; ++u)
            if (u < cnt) dst[u * istep] = *reinterpret_cast<const float4*>(&tile[u][prow][4 * g4]);
        }
      }
      __syncthreads();
    }
    src += kV4Img * istep4;
    if (op) op += kV4Img * step4;
  }
  pdl_trigger();
  if constexpr (!CD1) return;
  const long long per = plane_c;
  const long long e = (long long)c * HW + pos;
  if (ok) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nq) ws[slab_off + per * g + e + q] = acc[q];
  }
  const int tl = blockIdx.y * gridDim.x + blockIdx.x;
  if (ws_arrive(ws, tick_off, tl, G)) {
    if (ok) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q >= nq) continue;
        double t = 0.0;
        for (int gg = 0; gg < G; ++gg) t += __ldcg(ws + slab_off + per * gg + e + q);
        ws[e + q] = t;
      }
    }
    if (tid == 0) ws_tickets(ws, tick_off)[tl] = 0u;
  }
}

// k_act_pool_t over a group of images per block, also summing each thread's (c, position)
// over the group in FP64 into the Cd1 workspace (the consumer conv's clean-path Cd1)
template <int KT, int ACT>
__global__ void __launch_bounds__(256) k_act_pool_t_cd1(const float* __restrict__ in, float* __restrict__ out,
                                                       float* __restrict__ out_t, int N, int NG, int C, int H,
                                                       int kr, int s, int p, int Ho, double* __restrict__ ws,
                                                       long long tick_off, long long slab_off) {
  // images' windows in flight per thread: 1 for 3x3 windows (9 loads each; AlexNet pools
  // 152 -> 136 us, ResNet-18 stem pool 477 -> 414 at 2 -> 1), 4 for activation-only passes
  // of odd planes (351 -> 327 us over ResNet-18's five), 2 otherwise
  constexpr int IMG = KT == 1 ? 4 : (KT == 3 ? 1 : 2);
  __shared__ float tile[IMG][8][33];
  const int k = KT > 0 ? KT : kr;
  const int plane = Ho * Ho;
  const int tid = threadIdx.x;
  const int cl = tid >> 3, pl = tid & 7;
  const int c = blockIdx.y * 32 + cl, pos = blockIdx.x * 8 + pl;
  const int wc = tid & 31, wp = tid >> 5;
  const int spos = blockIdx.x * 8 + wp;
  const int g = blockIdx.z, G = gridDim.z;
  const int n_lo = g * NG, n_hi = min(N, n_lo + NG);
  const bool ok = pos < plane;
  // window origin and its valid rows / columns, fixed across images (no per-tap bounds
  // arithmetic in the image loop)
  int x0 = 0, y0 = 0;
  uint32_t rmask = 0, cmask = 0;
  if (ok) {
    const int ox = pos / Ho, oy = pos - (pos / Ho) * Ho;
    x0 = ox * s - p;
    y0 = oy * s - p;
    for (int i = 0; i < k && i < 32; ++i) {
      if ((unsigned)(x0 + i) < (unsigned)H) rmask |= 1u << i;
      if ((unsigned)(y0 + i) < (unsigned)H) cmask |= 1u << i;
    }
  }
  const long long HH = (long long)H * H;
  pdl_wait();
  const float* src = in + ((long long)n_lo * C + c) * HH + (long long)x0 * H + y0;
  float* op = out ? out + ((long long)n_lo * C + c) * plane + pos : nullptr;
  float* tp = out_t ? out_t + ((long long)n_lo * plane + spos) * C + blockIdx.y * 32 + wc : nullptr;
  const long long istep = (long long)C * HH, ostep = (long long)C * plane;
  auto pool = [&](const float* sp) -> float {
    float m = -INFINITY;
    if constexpr (KT > 0) {
      float v[KT * KT];
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j) v[i * KT + j] = ((rmask >> i) & (cmask >> j) & 1u) ? __ldg(sp + i * H + j) : 0.f;
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j)
          if ((rmask >> i) & (cmask >> j) & 1u) m = fmaxf(m, act_fn(v[i * KT + j], ACT));
    } else {
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j)
          if ((rmask >> i) & (cmask >> j) & 1u) m = fmaxf(m, act_fn(__ldg(sp + i * H + j), ACT));
    }
    return m;
  };
  // IMG images' windows in flight per thread (8 for k = 1 measured slower: VGG-19 relu
  // glue 2.55 vs 2.21 ms per step)
  double acc = 0.0;
  for (int n = n_lo; n < n_hi; n += IMG) {
    const int cnt = min(IMG, n_hi - n);
    float mv[IMG];
#pragma unroll
    for (int u = 0; u < IMG; ++u) mv[u] = (ok && u < cnt) ? pool(src + u * istep) : -INFINITY;
    if (ok) {
#pragma unroll
      for (int u = 0; u < IMG; ++u) {
        if (u < cnt) {
          if (out) op[u * ostep] = mv[u];  // out == NULL: staging pass of a caller-supplied D
          acc += (double)mv[u];
        }
      }
    }
    if (out_t) {
#pragma unroll
      for (int u = 0; u < IMG; ++u) tile[u][pl][cl] = mv[u];
      __syncthreads();
      if (spos < plane) {
#pragma unroll
        for (int u = 0; u < IMG; ++u)
          if (u < cnt) tp[(long long)u * plane * C] = tile[u][wp][wc];
      }
      __syncthreads();
    }
    src += IMG * istep;
    if (op) op += IMG * ostep;
    if (tp) tp += (long long)IMG * plane * C;
  }
  pdl_trigger();
  const long long per = (long long)C * plane;
  const long long e = (long long)c * plane + pos;
  if (ok) ws[slab_off + per * g + e] = acc;
  const int tl = blockIdx.y * gridDim.x + blockIdx.x;
  if (ws_arrive(ws, tick_off, tl, G)) {
    if (ok) {
      double t = 0.0;
      for (int gg = 0; gg < G; ++gg) t += __ldcg(ws + slab_off + per * gg + e);
      ws[e] = t;
    }
    if (tid == 0) ws_tickets(ws, tick_off)[tl] = 0u;
  }
}

// act + pool of a 32-position x 32-channel tile of one image per block (no checksum):
// warp w pools channels w, w+8, w+16, w+24 at the tile's 32 positions (lane = position:
// coalesced NCHW rows), and the tile goes channel-last through shared memory (128-byte
// NHWC rows).  AlexNet pool1 74 us vs 86 us with 8-position tiles.
template <int KT>
__global__ void __launch_bounds__(256) k_act_pool_tile(const float* __restrict__ in, float* __restrict__ out,
                                                      float* __restrict__ out_t, int C, int H, int act, int kr, int s,
                                                      int p, int Ho) {
  __shared__ float tile[32][33];
  const int k = KT > 0 ? KT : kr;
  const int plane = Ho * Ho;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pos = blockIdx.x * 32 + lane;
  const bool ok = pos < plane;
  const int c0 = blockIdx.y * 32;
  const int n = blockIdx.z;
  int x0 = 0, y0 = 0;
  uint32_t rmask = 0, cmask = 0;
  if (ok) {
    const int ox = pos / Ho, oy = pos - (pos / Ho) * Ho;
    x0 = ox * s - p;
    y0 = oy * s - p;
    for (int i = 0; i < k && i < 32; ++i) {
      if ((unsigned)(x0 + i) < (unsigned)H) rmask |= 1u << i;
      if ((unsigned)(y0 + i) < (unsigned)H) cmask |= 1u << i;
    }
  }
  const long long HH = (long long)H * H;
  pdl_wait();
  {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cl = warp + 8 * q, c = c0 + cl;
      float m = -INFINITY;
      if (ok && c < C) {
        const float* src = in + ((long long)n * C + c) * HH + (long long)x0 * H + y0;
        if constexpr (KT > 0) {
          float v[KT * KT];
#pragma unroll
          for (int i = 0; i < KT; ++i)
#pragma unroll
            for (int j = 0; j < KT; ++j)
              v[i * KT + j] = ((rmask >> i) & (cmask >> j) & 1u) ? __ldg(src + i * H + j) : 0.f;
#pragma unroll
          for (int i = 0; i < KT; ++i)
#pragma unroll
            for (int j = 0; j < KT; ++j)
              if ((rmask >> i) & (cmask >> j) & 1u) m = fmaxf(m, act_fn(v[i * KT + j], act));
        } else {
          for (int i = 0; i < k; ++i)
            for (int j = 0; j < k; ++j)
              if ((rmask >> i) & (cmask >> j) & 1u) m = fmaxf(m, act_fn(__ldg(src + i * H + j), act));
        }
        out[((long long)n * C + c) * plane + pos] = m;
      }
      tile[lane][cl] = m;
    }
    if (out_t) {
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int pl = warp + 8 * q, sp = blockIdx.x * 32 + pl;
        if (sp < plane && c0 + lane < C) out_t[((long long)n * plane + sp) * C + c0 + lane] = tile[pl][lane];
      }
    }
  }
}

int launch_act_pool(const float* in, float* out, int NC, int H, int act, int k, int s, int p, int Ho,
                    cudaStream_t st) {
  const long long total = (long long)NC * Ho * Ho;
  // 32-bit flat index per launch; larger tensors go in plane chunks
  const long long plane = (long long)Ho * Ho, chunk_planes = ((1LL << 31) / plane);
  for (long long p0 = 0; p0 < NC; p0 += chunk_planes) {
    const long long np = (NC - p0) < chunk_planes ? (NC - p0) : chunk_planes;
    const unsigned tot = (unsigned)(np * plane);
    long long blocks = ((long long)tot + 255) / 256;
    if (blocks > 148LL * 64) blocks = 148LL * 64;
    const float* ip = in + p0 * H * H;
    float* op = out + p0 * plane;
#define FTC_APF(KT) FTC_LAUNCH_PDL(k_act_pool_flat<KT>, dim3((unsigned)blocks), dim3(256), 0, st, ip, op, tot, H, Ho, act, k, s, p)
    switch (k) {
      case 1: FTC_APF(1); break;
      case 2: FTC_APF(2); break;
      case 3: FTC_APF(3); break;
      default: FTC_APF(0); break;
    }
#undef FTC_APF
  }
  (void)total;
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

__global__ void k_add_act(const float* __restrict__ a, const float* __restrict__ b,
                          float* __restrict__ out, long long n, int act) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = act_fn(a[e] + (b ? b[e] : 0.f), act);
}

// out (N,C,Ho,Ho) = in shifted by (-lo) with zero fill: Ho = H + lo + hi; negative
// hi crops the bottom/right edge.
#ifndef FTC_PAD_PLANES
#define FTC_PAD_PLANES 16
#endif
constexpr int kPadPlanes = FTC_PAD_PLANES;
__global__ void __launch_bounds__(256) k_pad_crop(const float* __restrict__ in, float* __restrict__ out, int NC,
                                                 int H, int lo, int Ho) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Ho * Ho) return;
  const int x = idx / Ho - lo, y = idx - (idx / Ho) * Ho - lo;
  const bool ok = x >= 0 && x < H && y >= 0 && y < H;
  // kPadPlanes planes per step: that many loads in flight per thread (one left the pass at
  // 1.7 TB/s, four at 3.5, eight at 4.0, sixteen at 4.3: ResNet-18 397 -> 321 us per step)
  for (int nc0 = blockIdx.y * kPadPlanes; nc0 < NC; nc0 += gridDim.y * kPadPlanes) {
    float v[kPadPlanes];
#pragma unroll
    for (int u = 0; u < kPadPlanes; ++u)
      v[u] = (ok && nc0 + u < NC) ? __ldg(in + ((long long)(nc0 + u) * H + x) * H + y) : 0.f;
#pragma unroll
    for (int u = 0; u < kPadPlanes; ++u)
      if (nc0 + u < NC) out[(long long)(nc0 + u) * Ho * Ho + idx] = v[u];
  }
}

inline int grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

// Image groups each Cd1 producer reduces separately (enough blocks to cover the SMs a
// few times, at most 16 partial slabs) and the shared workspace layout
int groups_for(int N, long long blocks_per_group) {
  long long G = (16LL * 148 + blocks_per_group - 1) / blocks_per_group;
  if (G > 16) G = 16;
  if (G > N) G = N;
  if (G < 1) G = 1;
  const int NG = (int)((N + G - 1) / G);
  return (N + NG - 1) / NG;  // no empty group
}

int cd1_parts_groups(int N, long long per) { return groups_for(N, (per + 255) / 256); }

int act_pool_groups(int N, int C, int Ho) {
  return groups_for(N, (long long)((Ho * Ho + 7) / 8) * ((C + 31) / 32));
}

// per = C*Ho*Ho; Ho = 0 when there is no pooling producer (k_cd1_parts only)
Cd1Ws cd1_ws_layout(int N, int C, int Ho, long long per) {
  Cd1Ws w{};
  w.per = per;
  long long t = (per + 255) / 256;
  int G = cd1_parts_groups(N, per);
  if (Ho > 0) {
    const long long t2 = (long long)((Ho * Ho + 7) / 8) * ((C + 31) / 32);
    t = t > t2 ? t : t2;
    const int G2 = act_pool_groups(N, C, Ho);
    G = G > G2 ? G : G2;
  }
  w.tickets = (int)t;
  w.tick_off = per;
  w.slab_off = per + (t + 1) / 2;
  (void)G;
  return w;
}

long long cd1_ws_doubles_g(int N, int C, int Ho, long long per) {
  const Cd1Ws w = cd1_ws_layout(N, C, Ho, per);
  int G = cd1_parts_groups(N, per);
  if (Ho > 0) {
    const int G2 = act_pool_groups(N, C, Ho);
    G = G > G2 ? G : G2;
  }
  return w.slab_off + (long long)G * per;
}

long long cd1_ws_doubles(int N, long long per) { return cd1_ws_doubles_g(N, 0, 0, per); }

int launch_act_pool_nhwc(const float* in, float* out, float* out_t, int N, int C, int H, int act, int k, int s,
                         int p, cudaStream_t st) {
  const int Ho = (H + 2 * p - k) / s + 1;
  const dim3 g((unsigned)((Ho * Ho + 31) / 32), (unsigned)((C + 31) / 32), (unsigned)N);
#define FTC_APT(KT) \
  FTC_LAUNCH_PDL(k_act_pool_tile<KT>, g, dim3(256), 0, st, in, out, out_t, C, H, act, k, s, p, Ho)
  switch (k) {
    case 1: FTC_APT(1); break;
    case 2: FTC_APT(2); break;
    case 3: FTC_APT(3); break;
    default: FTC_APT(0); break;
  }
#undef FTC_APT
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int launch_cd1_parts(const float* D, int N, long long per, double* ws, cudaStream_t st, int C, int Ho) {
  const Cd1Ws w = cd1_ws_layout(N, C, Ho, per);
  const int G = cd1_parts_groups(N, per);
  const int NG = (N + G - 1) / G;
  const dim3 g((unsigned)((per + 255) / 256), (unsigned)((N + NG - 1) / NG));
  FTC_LAUNCH_PDL(k_cd1_parts, g, dim3(256), 0, st, D, N, per, NG, ws, w.tick_off, w.slab_off);
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

// Which form of k_act_v4_cd1 (if any) takes a glue pass: the 16-byte form, the 2x2 pool
// form or the scalar-access form; only these run without an NCHW output (out == NULL).
#ifndef FTC_V4_SCALAR_MIN
#define FTC_V4_SCALAR_MIN 64
#endif
struct V4Form {
  bool vec, pool2, any;
};
V4Form v4_form(const float* in, const float* out, int C, int H, int k, int s, int p) {
  static const bool v4_off = getenv("FTC_GLUE_V4") && atoi(getenv("FTC_GLUE_V4")) == 0;
  const int Ho = (H + 2 * p - k) / s + 1;
  const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15) == 0 && (!out || (reinterpret_cast<uintptr_t>(out) & 15) == 0);
  // the scalar-access form for odd planes down to 8x8 (with the 16-byte channel-last stores it
  // wins on AlexNet's 13x13 and ResNet-18's 29x29 / 15x15 too: 82.6K -> 83.5K, 33.2K -> 33.7K
  // images/s; before them it lost on 13x13, 80 vs 75 us)
  V4Form f;
  f.vec = k == 1 && s == 1 && p == 0 && (H * H) % 4 == 0 && aligned;
  const bool plain = f.vec || (k == 1 && s == 1 && p == 0 && H * H >= FTC_V4_SCALAR_MIN);
  f.pool2 = k == 2 && s == 2 && p == 0 && H % 2 == 0 && Ho % 4 == 0 && aligned;
  f.any = (plain || f.pool2) && C % 32 == 0 && !v4_off;
  return f;
}

int launch_act_pool_nhwc_cd1(const float* in, float* out, float* out_t, int N, int C, int H, int act, int k,
                             int s, int p, double* ws, cudaStream_t st) {
  // 8-position x 32-channel tiles looping over image groups: measured faster for the
  // Cd1-producing pass than 32 x 32 tiles (fewer, longer-running blocks were latency
  // bound: AlexNet pool2 59 vs 74 us)
  const int Ho = (H + 2 * p - k) / s + 1;
  const long long per = (long long)C * Ho * Ho;
  const Cd1Ws w = cd1_ws_layout(N, C, Ho, per);
  const int G = act_pool_groups(N, C, Ho);
  const int NG = (N + G - 1) / G;
  const V4Form vf = v4_form(in, out, C, H, k, s, p);
  const bool vec = vf.vec, pool2 = vf.pool2;
  if (vf.any) {
    // 32-position tiles: fewer tiles than the 8-position layout the workspace is sized
    // for, and no more image groups than it holds
    const int HW = Ho * Ho;
    const dim3 gv((unsigned)((HW + 31) / 32), (unsigned)(C / 32), (unsigned)((N + NG - 1) / NG));
#define FTC_V4(A, P)                                                                                           \
  do {                                                                                                         \
    if (ws)                                                                                                    \
      FTC_LAUNCH_PDL((k_act_v4_cd1<A, P>), gv, dim3(256), 0, st, in, out, out_t, N, NG, C, HW, ws, w.tick_off,    \
                     w.slab_off, Ho);                                                                          \
    else                                                                                                       \
      FTC_LAUNCH_PDL((k_act_v4_cd1<A, P, true, false>), gv, dim3(256), 0, st, in, out, out_t, N, NG, C, HW, ws,  \
                     w.tick_off, w.slab_off, Ho);                                                              \
  } while (0)
    if (pool2) {
      if (act == 1) FTC_V4(1, true);
      else if (act == 2) FTC_V4(2, true);
      else FTC_V4(0, true);
    } else if (vec) {
      if (act == 1) FTC_V4(1, false);
      else if (act == 2) FTC_V4(2, false);
      else FTC_V4(0, false);
    } else {
#define FTC_V1(A)                                                                                               \
  do {                                                                                                          \
    if (ws)                                                                                                     \
      FTC_LAUNCH_PDL((k_act_v4_cd1<A, false, false>), gv, dim3(256), 0, st, in, out, out_t, N, NG, C, HW, ws,      \
                     w.tick_off, w.slab_off, Ho);                                                               \
    else                                                                                                        \
      FTC_LAUNCH_PDL((k_act_v4_cd1<A, false, false, false>), gv, dim3(256), 0, st, in, out, out_t, N, NG, C, HW, \
                     ws, w.tick_off, w.slab_off, Ho);                                                           \
  } while (0)
      if (act == 1) FTC_V1(1);
      else if (act == 2) FTC_V1(2);
      else FTC_V1(0);
#undef FTC_V1
    }
#undef FTC_V4
    FTC_CUDA_CHECK(cudaGetLastError());
    return FTC_OK;
  }
  if (!ws)
    return out_t ? launch_act_pool_nhwc(in, out, out_t, N, C, H, act, k, s, p, st)
                 : launch_act_pool(in, out, N * C, H, act, k, s, p, Ho, st);
  const dim3 g((unsigned)((Ho * Ho + 7) / 8), (unsigned)(C / 32), (unsigned)((N + NG - 1) / NG));
#define FTC_APT2(KT, ACT) \
  FTC_LAUNCH_PDL(k_act_pool_t_cd1<KT, ACT>, g, dim3(256), 0, st, in, out, out_t, N, NG, C, H, k, s, p, Ho, ws, \
                 w.tick_off, w.slab_off)
#define FTC_APT(KT)                  \
  if (act == 1) FTC_APT2(KT, 1);      \
  else if (act == 2) FTC_APT2(KT, 2); \
  else FTC_APT2(KT, 0)
  switch (k) {
    case 1: FTC_APT(1); break;
    case 2: FTC_APT(2); break;
    case 3: FTC_APT(3); break;
    default: FTC_APT(0); break;
  }
#undef FTC_APT2
#undef FTC_APT
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // namespace ftc

using namespace ftc;

extern "C" {

int ftc_glue_act_pool(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t act,
                      int32_t k, int32_t s, int32_t p, int32_t* Ho_out, void* stream) {
  if (k <= 0 || s <= 0 || p < 0 || H + 2 * p < k) {
    set_error(FTC_CONFIG_ERROR, "bad pooling window");
    return FTC_CONFIG_ERROR;
  }
  const int Ho = (H + 2 * p - k) / s + 1;
  if (Ho_out) *Ho_out = Ho;
  if (!in || !out) return FTC_OK;  // shape query
  return launch_act_pool(in, out, N * C, H, act, k, s, p, Ho, (cudaStream_t)stream);
}

int ftc_glue_act_pool_ck(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t act,
                         int32_t k, int32_t s, int32_t p, double* cd1, double* cd2, void* stream) {
  if (k <= 0 || s <= 0 || p < 0 || H + 2 * p < k || !in || !out || !cd1 || !cd2) {
    set_error(FTC_CONFIG_ERROR, "bad pooling window or null buffer");
    return FTC_CONFIG_ERROR;
  }
  // act + pool over the whole batch in parallel, then the next layer's input checksums
  // (exact reference order, n ascending) from the pooled tensor while it is L2-hot.
  // (A fused per-(c,x,y) kernel walking n serially had too little parallelism: 25% of
  // the AlexNet step.)
  const int Ho = (H + 2 * p - k) / s + 1;
  const long long per = (long long)C * Ho * Ho;
  {
    const int st = launch_act_pool(in, out, N * C, H, act, k, s, p, Ho, (cudaStream_t)stream);
    if (st != FTC_OK) return st;
  }
  return launch_input_checksums(out, N, per, cd1, cd2, (cudaStream_t)stream);
}

int ftc_glue_act_pool_nhwc(const float* in, float* out, float* out_nhwc, int32_t N, int32_t C, int32_t H,
                           int32_t act, int32_t k, int32_t s, int32_t p, double* cd1, double* cd2,
                           void* stream) {
  if (k <= 0 || s <= 0 || p < 0 || H + 2 * p < k || !in || !out || !out_nhwc || C % 32 || (!cd1) != (!cd2)) {
    set_error(FTC_CONFIG_ERROR, "bad pooling window, null buffer or C % 32 != 0");
    return FTC_CONFIG_ERROR;
  }
  const int Ho = (H + 2 * p - k) / s + 1;
  cudaStream_t st = (cudaStream_t)stream;
  {
    const int rc = launch_act_pool_nhwc(in, out, out_nhwc, N, C, H, act, k, s, p, st);
    if (rc != FTC_OK) return rc;
  }
  if (!cd1) return FTC_OK;
  return launch_input_checksums(out, N, (long long)C * Ho * Ho, cd1, cd2, st);
}

int64_t ftc_glue_ws_doubles(int32_t N, int32_t C, int32_t H, int32_t k, int32_t s, int32_t p) {
  if (N <= 0 || C <= 0 || k <= 0 || s <= 0 || p < 0 || H + 2 * p < k) return 0;
  const int Ho = (H + 2 * p - k) / s + 1;
  return cd1_ws_doubles_g(N, C, Ho, (long long)C * Ho * Ho);
}

int ftc_glue_act_pool_cd1(const float* in, float* out, float* out_nhwc, int32_t N, int32_t C, int32_t H,
                          int32_t act, int32_t k, int32_t s, int32_t p, double* ws, void* stream) {
  if (k <= 0 || s <= 0 || p < 0 || H + 2 * p < k || !in || (!out && !out_nhwc) || (out_nhwc && C % 32)) {
    set_error(FTC_CONFIG_ERROR, "bad pooling window, null buffer or NHWC output with C % 32 != 0");
    return FTC_CONFIG_ERROR;
  }
  // out == NULL: the consumer conv reads only the NHWC copy (ftc_glue_nchw_optional)
  if (!out && !v4_form(in, nullptr, C, H, k, s, p).any) {
    set_error(FTC_CONFIG_ERROR, "this glue shape needs its NCHW output (see ftc_glue_nchw_optional)");
    return FTC_CONFIG_ERROR;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int Ho = (H + 2 * p - k) / s + 1;
  if (!ws) {
    // no checksum (unprotected nets): the same tuned pass without the Cd1 sums when it
    // writes an NHWC copy, else the plain kernels
    return (out_nhwc && C % 32 == 0) ? launch_act_pool_nhwc_cd1(in, out, out_nhwc, N, C, H, act, k, s, p, nullptr, st)
           : out_nhwc                ? launch_act_pool_nhwc(in, out, out_nhwc, N, C, H, act, k, s, p, st)
                                     : launch_act_pool(in, out, N * C, H, act, k, s, p, Ho, st);
  }
  // with the consumer's Cd1: channel-blocked kernel looping over image groups (one
  // pass), or -- C not a multiple of 32 -- act + pool, then Cd1 from the L2-hot output
  if (C % 32 == 0) return launch_act_pool_nhwc_cd1(in, out, out_nhwc, N, C, H, act, k, s, p, ws, st);
  const int rc = launch_act_pool(in, out, N * C, H, act, k, s, p, Ho, st);
  if (rc != FTC_OK) return rc;
  return launch_cd1_parts(out, N, (long long)C * Ho * Ho, ws, st, C, Ho);
}

int32_t ftc_glue_nchw_optional(const float* in, int32_t C, int32_t H, int32_t k, int32_t s, int32_t p) {
  if (k <= 0 || s <= 0 || p < 0 || H + 2 * p < k || !in) return 0;
  return v4_form(in, nullptr, C, H, k, s, p).any ? 1 : 0;
}

int ftc_glue_add_act(const float* a, const float* b, float* out, int64_t n, int32_t act, void* stream) {
  FTC_LAUNCH(k_add_act<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(a, b, out, n, act));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

int ftc_glue_pad_crop(const float* in, float* out, int32_t N, int32_t C, int32_t H, int32_t lo,
                      int32_t hi, void* stream) {
  const int Ho = H + lo + hi;
  if (lo < 0 || Ho <= 0) {
    set_error(FTC_CONFIG_ERROR, "bad pad/crop");
    return FTC_CONFIG_ERROR;
  }
  const int ny = (N * C + kPadPlanes - 1) / kPadPlanes;
  const dim3 g((unsigned)((Ho * Ho + 255) / 256), (unsigned)(ny < 65535 ? ny : 65535));
  FTC_LAUNCH(k_pad_crop<<<g, 256, 0, (cudaStream_t)stream>>>(in, out, N * C, H, lo, Ho));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // extern "C"
