// Exact-order chain sums over a position-major copy T[f][q] of the terms: each lane
// streams its own contiguous row with 16-byte loads P terms ahead.  Cycles per term for
// one chain per lane (family per lane) and three chains per lane.
#include <cstdio>
#include <cuda_runtime.h>
template <int P, int FAMS, int LD = 1>
__global__ void k(const float* T, int npos, int NM, int M, double* out, long long* cyc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int f = FAMS == 3 ? t : t / 3, fam = FAMS == 3 ? 0 : t % 3;
  if (f >= npos) return;
  const float4* row = reinterpret_cast<const float4*>(T + (long long)f * NM);
  float4 buf[P / 4];
#pragma unroll
  for (int u = 0; u < P / 4; ++u) buf[u] = __ldg(row + u);
  double s = 0.0, s6 = 0.0, s7 = 0.0;
  int m = 0, n = 0;
  long long t0 = clock64();
  for (int q0 = 0; q0 < NM; q0 += P) {
#pragma unroll
    for (int u = 0; u < P / 4; ++u) {
      const float4 v = buf[u];
      const int qn = (q0 + P) / 4 + u;
      if (LD == 1) buf[u] = __ldg(row + (qn < NM / 4 ? qn : 0));
      if (LD == 2) buf[u] = __ldg(row + (qn & 15));
      const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double x = (double)xs[e];
        if (FAMS == 3) {
          s = __dadd_rn(s, x);
          s6 = __dadd_rn(s6, __dmul_rn((double)m, x));
          s7 = __dadd_rn(s7, __dmul_rn((double)n, x));
        } else {
          const double w = (double)(fam == 0 ? 1 : fam == 1 ? m : n);
          s = __dadd_rn(s, __dmul_rn(w, x));
        }
        const bool wrap = m + 1 == M;
        m = wrap ? 0 : m + 1;
        n = wrap ? n + 1 : n;
      }
    }
  }
  long long t1 = clock64();
  out[t] = s + s6 + s7;
  if (t == 0) cyc[0] = t1 - t0;
}
int main() {
  const int E2 = 729, NM = 32768, M = 256;
  float* T; double* out; long long* cyc;
  cudaMalloc(&T, (size_t)NM * E2 * 4);
  cudaMemset(T, 0, (size_t)NM * E2 * 4);
  cudaMalloc(&out, 1 << 22);
  cudaMallocManaged(&cyc, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<32, 1><<<(3 * E2 + 63) / 64, 64>>>(T, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long a = cyc[0];
    k<64, 1><<<(3 * E2 + 63) / 64, 64>>>(T, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long b = cyc[0];
    k<32, 3><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long c = cyc[0];
    k<64, 3><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long d = cyc[0];
    k<32, 1><<<(3 * E2 + 15) / 16, 16>>>(T, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long e = cyc[0];
    k<64, 1, 0><<<(3 * E2 + 63) / 64, 64>>>(T, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long g = cyc[0];
    k<64, 1, 2><<<(3 * E2 + 63) / 64, 64>>>(T, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long h = cyc[0];
    printf("no loads %.1f, L1-resident loads %.1f\n", g / (double)NM, h / (double)NM);
    printf("cycles/term: fam/lane P32 %.1f P64 %.1f | 3 fams/lane P32 %.1f P64 %.1f | fam/lane 16 thr/blk %.1f (%s)\n",
           a / (double)NM, b / (double)NM, c / (double)NM, d / (double)NM, e / (double)NM,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
