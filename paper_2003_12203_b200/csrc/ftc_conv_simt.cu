// ftc_conv_simt.cu -- FP32 SIMT direct convolution (engine 1).
//
// conv_forward (conv.hpp:114-131) as an FFMA kernel: one thread per output pixel
// (n,x,y), MT filters accumulated in registers per pass, W staged through shared
// memory in K-chunks.  It is the bring-up / small-shape engine and the numerical
// cross-check of the tcgen05 engine; its epilogue is the same as the tensor-core
// one: bias, post_conv faults, store, and the fused FP64 row sums
// rowsum[n][x,y] = sum_m O[n,m,x,y] (So2) and rowsum_m = sum_m m*O (So4), taken in
// ascending m exactly as output_summations (checksums.hpp:176-187) does.
#include <cuda_runtime.h>

#include "ftc_common.cuh"

namespace ftc {
namespace {

constexpr int kPix = 128;  // pixels (threads) per block
constexpr int kKC = 32;    // K chunk staged in smem

template <int MT>
__global__ void __launch_bounds__(kPix) k_conv_simt(ConvArgs a) {
  __shared__ float ws[MT][kKC];
  __shared__ int koff[kKC];
  __shared__ int kdi[kKC];
  __shared__ int kdj[kKC];

  const int E = a.E, E2 = E * E, H = a.H, R = a.R, RR = R * R;
  const int Ckw = a.Ckw, K = Ckw * RR, M = a.M, mpg = M / a.groups;
  const long long P = (long long)(a.img_hi - a.img_lo) * E2;
  const long long p = (long long)blockIdx.x * kPix + threadIdx.x;
  const bool valid = p < P;
  const long long pg = (long long)a.img_lo * E2 + (valid ? p : 0);
  const int n = (int)(pg / E2), f = (int)(pg % E2), x = f / E, y = f % E;
  const int xb = x * a.U - a.pad, yb = y * a.U - a.pad;
  const float* Dn = a.D + (long long)n * a.C * H * H;

  double rs = 0.0, rsm = 0.0;
  for (int m0 = 0; m0 < M; m0 += MT) {
    const int kbase = (m0 / mpg) * Ckw;  // MT never straddles a group (host guarantees)
    const float* Dg = Dn + (long long)kbase * H * H;
    float acc[MT];
#pragma unroll
    for (int q = 0; q < MT; ++q) acc[q] = 0.f;
    for (int k0 = 0; k0 < K; k0 += kKC) {
      __syncthreads();
      for (int t = threadIdx.x; t < MT * kKC; t += kPix) {
        const int mm = t / kKC, kk = t % kKC;
        const int m = m0 + mm, k = k0 + kk;
        ws[mm][kk] = (m < M && k < K) ? a.W[(long long)m * K + k] : 0.f;
      }
      if (threadIdx.x < kKC) {
        const int k = k0 + threadIdx.x;
        const int c = k / RR, t = k % RR, i = t / R, j = t % R;
        koff[threadIdx.x] = (k < K) ? (c * H + i) * H + j : 0;
        kdi[threadIdx.x] = (k < K) ? i : -100000;
        kdj[threadIdx.x] = j;
      }
      __syncthreads();
      const int kc = min(kKC, K - k0);
      for (int kk = 0; kk < kc; ++kk) {
        const int hh = xb + kdi[kk], ww = yb + kdj[kk];
        float d = 0.f;
        if (valid && hh >= 0 && hh < H && ww >= 0 && ww < H) d = __ldg(Dg + koff[kk] + xb * H + yb);
#pragma unroll
        for (int q = 0; q < MT; ++q) acc[q] = fmaf(d, ws[q][kk], acc[q]);
      }
    }
    // epilogue
#pragma unroll
    for (int q = 0; q < MT; ++q) {
      const int m = m0 + q;
      if (m >= M || !valid) continue;
      float v = acc[q];
      if (a.bias) v = v + a.bias[m];
      if (a.nfaults) v = apply_output_faults(v, n, m, x, y, a.M, a.E, a.faults, a.nfaults, a.scale_tab);
      const long long oi = ((long long)n * M + m) * E2 + f;
      bool store = true;
      if (a.plane_mask) {
        const long long pl = (long long)n * M + m;
        store = (a.plane_mask[pl >> 5] >> (pl & 31)) & 1u;
      }
      if (store) a.O[oi] = v;
      const double dv = (double)v;
      rs = dadd(rs, dv);
      rsm = dadd(rsm, dmul((double)m, dv));
    }
  }
  if (valid && a.rowsum) {
    a.rowsum[(long long)n * E2 + f] = rs;
    a.rowsum_m[(long long)n * E2 + f] = rsm;
  }
}

}  // namespace

int conv_simt_launch(const ConvArgs& a, cudaStream_t s) {
  const long long P = (long long)(a.img_hi - a.img_lo) * a.E * a.E;
  if (P <= 0) return FTC_OK;
  const int grid = (int)((P + kPix - 1) / kPix);
  const int mpg = a.M / a.groups;
  if (a.groups == 1 || mpg % 16 == 0)
    FTC_LAUNCH(k_conv_simt<16><<<grid, kPix, 0, s>>>(a));
  else
    FTC_LAUNCH(k_conv_simt<1><<<grid, kPix, 0, s>>>(a));
  FTC_CUDA_CHECK(cudaGetLastError());
  return FTC_OK;
}

}  // namespace ftc
