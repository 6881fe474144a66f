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
// of act(in[n,c,.,.]); k = 1, s = 1 is a plain activation.
__global__ void k_act_pool(const float* __restrict__ in, float* __restrict__ out, int NC, int H,
                           int act, int k, int s, int p, int Ho) {
  const long long total = (long long)NC * Ho * Ho;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int oy = (int)(e % Ho), ox = (int)((e / Ho) % Ho);
    const long long nc = e / ((long long)Ho * Ho);
    const float* src = in + nc * H * H;
    float m = -INFINITY;
    for (int i = 0; i < k; ++i) {
      const int x = ox * s - p + i;
      if (x < 0 || x >= H) continue;
      for (int j = 0; j < k; ++j) {
        const int y = oy * s - p + j;
        if (y < 0 || y >= H) continue;
        m = fmaxf(m, act_fn(__ldg(src + x * H + y), act));
      }
    }
    out[e] = m;
  }
}

__global__ void k_add_act(const float* __restrict__ a, const float* __restrict__ b,
                          float* __restrict__ out, long long n, int act) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = act_fn(a[e] + (b ? b[e] : 0.f), act);
}

// out (N,C,Ho,Ho) = in shifted by (-lo) with zero fill: Ho = H + lo + hi; negative
// hi crops the bottom/right edge.
__global__ void k_pad_crop(const float* __restrict__ in, float* __restrict__ out, int NC, int H,
                           int lo, int Ho) {
  const long long total = (long long)NC * Ho * Ho;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int y = (int)(e % Ho) - lo, x = (int)((e / Ho) % Ho) - lo;
    const long long nc = e / ((long long)Ho * Ho);
    out[e] = (x >= 0 && x < H && y >= 0 && y < H) ? in[(nc * H + x) * H + y] : 0.f;
  }
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
  FTC_LAUNCH(k_act_pool<<<grid_for((long long)N * C * Ho * Ho), 256, 0, (cudaStream_t)stream>>>(
      in, out, N * C, H, act, k, s, p, Ho));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
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
  FTC_LAUNCH(k_act_pool<<<grid_for((long long)N * per), 256, 0, (cudaStream_t)stream>>>(
      in, out, N * C, H, act, k, s, p, Ho));
  FTC_CUDA_CHECK(cudaGetLastError());
  return launch_input_checksums(out, N, per, cd1, cd2, (cudaStream_t)stream);
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
  FTC_LAUNCH(k_pad_crop<<<grid_for((long long)N * C * Ho * Ho), 256, 0, (cudaStream_t)stream>>>(
      in, out, N * C, H, lo, Ho));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // extern "C"
