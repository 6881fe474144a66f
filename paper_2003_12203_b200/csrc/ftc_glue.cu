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

// out[n,c,ox,oy] = max over the k x k window (stride s, padding p, -inf padding)
// of act(in[n,c,.,.]); k = 1, s = 1 is a plain activation.  Grid: y = (n, c) plane
// (strided when N*C exceeds the grid limit), x = output positions of the plane; 32-bit
// index math (a 64-bit div/mod per element made this kernel integer-bound).
template <int KT>
__global__ void __launch_bounds__(256) k_act_pool(const float* __restrict__ in, float* __restrict__ out,
                                                 int NC, int H, int act, int kr, int s, int p, int Ho) {
  constexpr int kPlanes = 4;  // planes per thread: their window loads are all in flight
  const int k = KT > 0 ? KT : kr;
  const int plane = Ho * Ho;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= plane) return;
  const int ox = idx / Ho, oy = idx - (idx / Ho) * Ho;
  const int x0 = ox * s - p, y0 = oy * s - p;
  for (int nc0 = blockIdx.y * kPlanes; nc0 < NC; nc0 += gridDim.y * kPlanes) {
    if constexpr (KT > 0) {
      float v[kPlanes][KT * KT];
#pragma unroll
      for (int u = 0; u < kPlanes; ++u) {
        const float* src = in + (long long)(nc0 + u) * H * H;
#pragma unroll
        for (int i = 0; i < KT; ++i)
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            const int x = x0 + i, y = y0 + j;
            const bool ok = nc0 + u < NC && x >= 0 && x < H && y >= 0 && y < H;
            v[u][i * KT + j] = ok ? __ldg(src + x * H + y) : -INFINITY;
          }
      }
#pragma unroll
      for (int u = 0; u < kPlanes; ++u) {
        if (nc0 + u >= NC) break;
        float m = -INFINITY;
#pragma unroll
        for (int i = 0; i < KT; ++i)
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            const int x = x0 + i, y = y0 + j;
            // padding positions are skipped (not act(-inf)) exactly as the generic path
            if (x >= 0 && x < H && y >= 0 && y < H) m = fmaxf(m, act_fn(v[u][i * KT + j], act));
          }
        out[(long long)(nc0 + u) * plane + idx] = m;
      }
    } else {
      for (int u = 0; u < kPlanes && nc0 + u < NC; ++u) {
        const float* src = in + (long long)(nc0 + u) * H * H;
        float m = -INFINITY;
        for (int i = 0; i < k; ++i) {
          const int x = x0 + i;
          if (x < 0 || x >= H) continue;
          for (int j = 0; j < k; ++j) {
            const int y = y0 + j;
            if (y < 0 || y >= H) continue;
            m = fmaxf(m, act_fn(__ldg(src + x * H + y), act));
          }
        }
        out[(long long)(nc0 + u) * plane + idx] = m;
      }
    }
  }
}

// act + pool of one image's 32-channel x 8-position tile, written NCHW and, through
// shared memory, NHWC (the next conv's TMA im2col input): loads by channel rows of 8
// consecutive positions, stores by position rows of 32 channels (128 bytes)
template <int KT>
__global__ void __launch_bounds__(256) k_act_pool_t(const float* __restrict__ in, float* __restrict__ out,
                                                   float* __restrict__ out_t, int C, int H, int act, int kr, int s,
                                                   int p, int Ho) {
  __shared__ float tile[8][33];
  const int k = KT > 0 ? KT : kr;
  const int plane = Ho * Ho;
  const int tid = threadIdx.x;
  const int cl = tid >> 3, pl = tid & 7;
  const int c = blockIdx.y * 32 + cl, pos = blockIdx.x * 8 + pl;
  const long long n = blockIdx.z;
  float m = -INFINITY;
  if (pos < plane) {
    const int ox = pos / Ho, oy = pos - (pos / Ho) * Ho;
    const int x0 = ox * s - p, y0 = oy * s - p;
    const float* src = in + (n * C + c) * H * H;
    if constexpr (KT > 0) {
      float v[KT * KT];
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          const int x = x0 + i, y = y0 + j;
          v[i * KT + j] = (x >= 0 && x < H && y >= 0 && y < H) ? __ldg(src + x * H + y) : 0.f;
        }
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          const int x = x0 + i, y = y0 + j;
          if (x >= 0 && x < H && y >= 0 && y < H) m = fmaxf(m, act_fn(v[i * KT + j], act));
        }
    } else {
      for (int i = 0; i < k; ++i) {
        const int x = x0 + i;
        if (x < 0 || x >= H) continue;
        for (int j = 0; j < k; ++j) {
          const int y = y0 + j;
          if (y < 0 || y >= H) continue;
          m = fmaxf(m, act_fn(__ldg(src + x * H + y), act));
        }
      }
    }
    out[(n * C + c) * plane + pos] = m;
  }
  tile[pl][cl] = m;
  __syncthreads();
  const int wc = tid & 31, wp = tid >> 5;
  const int spos = blockIdx.x * 8 + wp;
  if (spos < plane) out_t[(n * plane + spos) * C + blockIdx.y * 32 + wc] = tile[wp][wc];
}

int launch_act_pool(const float* in, float* out, int NC, int H, int act, int k, int s, int p, int Ho,
                    cudaStream_t st) {
  const int gy = (NC + 3) / 4;
  const dim3 g((unsigned)((Ho * Ho + 255) / 256), (unsigned)(gy < 65535 ? gy : 65535));
  if (k == 3)
    FTC_LAUNCH(k_act_pool<3><<<g, 256, 0, st>>>(in, out, NC, H, act, k, s, p, Ho));
  else if (k == 2)
    FTC_LAUNCH(k_act_pool<2><<<g, 256, 0, st>>>(in, out, NC, H, act, k, s, p, Ho));
  else if (k == 1)
    FTC_LAUNCH(k_act_pool<1><<<g, 256, 0, st>>>(in, out, NC, H, act, k, s, p, Ho));
  else
    FTC_LAUNCH(k_act_pool<0><<<g, 256, 0, st>>>(in, out, NC, H, act, k, s, p, Ho));
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
__global__ void __launch_bounds__(256) k_pad_crop(const float* __restrict__ in, float* __restrict__ out, int NC,
                                                 int H, int lo, int Ho) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Ho * Ho) return;
  const int x = idx / Ho - lo, y = idx - (idx / Ho) * Ho - lo;
  const bool ok = x >= 0 && x < H && y >= 0 && y < H;
  for (int nc = blockIdx.y; nc < NC; nc += gridDim.y)
    out[(long long)nc * Ho * Ho + idx] = ok ? __ldg(in + ((long long)nc * H + x) * H + y) : 0.f;
}

inline int grid_for(long long n) {
  long long b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace
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
  const dim3 g((unsigned)((Ho * Ho + 7) / 8), (unsigned)(C / 32), (unsigned)N);
  cudaStream_t st = (cudaStream_t)stream;
  if (k == 3)
    FTC_LAUNCH(k_act_pool_t<3><<<g, 256, 0, st>>>(in, out, out_nhwc, C, H, act, k, s, p, Ho));
  else if (k == 2)
    FTC_LAUNCH(k_act_pool_t<2><<<g, 256, 0, st>>>(in, out, out_nhwc, C, H, act, k, s, p, Ho));
  else if (k == 1)
    FTC_LAUNCH(k_act_pool_t<1><<<g, 256, 0, st>>>(in, out, out_nhwc, C, H, act, k, s, p, Ho));
  else
    FTC_LAUNCH(k_act_pool_t<0><<<g, 256, 0, st>>>(in, out, out_nhwc, C, H, act, k, s, p, Ho));
  FTC_CUDA_CHECK(cudaGetLastError());
  if (!cd1) return FTC_OK;
  return launch_input_checksums(out, N, (long long)C * Ho * Ho, cd1, cd2, st);
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
  const dim3 g((unsigned)((Ho * Ho + 255) / 256), (unsigned)(N * C < 65535 ? N * C : 65535));
  FTC_LAUNCH(k_pad_crop<<<g, 256, 0, (cudaStream_t)stream>>>(in, out, N * C, H, lo, Ho));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // extern "C"
