// Chain sums over a position-major FP64 copy T[f][q]: lane = position, warp-uniform
// family, no conversions on the chain (weights kept as doubles: dm += 1, wrap by compare).
#include <cstdio>
#include <cuda_runtime.h>
template <int FAM, int V = 0, int PF = 0>
__global__ void k(const double* T, int npos, int NM, int M, double* out, long long* cyc, int slot = -1) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= npos) return;
  const double2* row = reinterpret_cast<const double2*>(T + (long long)f * NM);
  constexpr int P = 32;
  double2 buf[P / 2];
#pragma unroll
  for (int u = 0; u < P / 2; ++u) buf[u] = __ldg(row + u);
  double s = 0.0, dm = 0.0, dn = 0.0;
  const double dM = (double)M;
  long long t0 = clock64();
  for (int q0 = 0; q0 < NM; q0 += P) {
#pragma unroll
    for (int u = 0; u < P / 2; ++u) {
      const double2 v = buf[u];
      const int qn = (q0 + P) / 2 + u;
      if (!(V & 1)) buf[u] = __ldg(row + (qn < NM / 2 ? qn : 0));
      if (PF > 0 && (u % 8) == 0) {
        const int qp = qn + PF;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(row + (qp < NM / 2 ? qp : 0)));
      }
      const double xs[2] = {v.x, v.y};
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (FAM == 0) s = __dadd_rn(s, xs[e]);
        if (FAM == 1) s = __dadd_rn(s, __dmul_rn(dm, xs[e]));
        if (FAM == 2) s = __dadd_rn(s, __dmul_rn(dn, xs[e]));
        if (!(V & 2)) {
          dm = __dadd_rn(dm, 1.0);
          if (dm == dM) { dm = 0.0; dn = __dadd_rn(dn, 1.0); }
        }
      }
    }
  }
  long long t1 = clock64();
  out[f] = s;
  if (f == 0) cyc[slot >= 0 ? slot : FAM + 3 * V] = t1 - t0;
}
int main() {
  const int E2 = 729, NM = 32768, M = 256;
  double* T; double* out; long long* cyc;
  cudaMalloc(&T, (size_t)NM * E2 * 8);
  cudaMemset(T, 0, (size_t)NM * E2 * 8);
  cudaMalloc(&out, 1 << 22);
  cudaMallocManaged(&cyc, 256);
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc);
    k<1><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc);
    k<2><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc);
    k<0, 1><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc);
    k<0, 2><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc);
    k<0, 3><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc);
    k<0, 3><<<1, 32>>>(T, E2, NM, M, out, cyc, 12);
    k<0, 0, 64><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc, 15);
    k<0, 0, 128><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc, 18);
    k<0, 0, 256><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc, 21);
    k<1, 0, 128><<<(E2 + 31) / 32, 32>>>(T, E2, NM, M, out, cyc, 25);
    cudaDeviceSynchronize();
    printf("L1 prefetch ahead 64/128/256 double2: %.1f %.1f %.1f; So6 128: %.1f\n", cyc[15] / (double)NM, cyc[18] / (double)NM, cyc[21] / (double)NM, cyc[25] / (double)NM);
    printf("So5 no loads %.1f, no counter %.1f, neither %.1f, neither 1 warp %.1f\n", cyc[3] / (double)NM, cyc[6] / (double)NM, cyc[9] / (double)NM, cyc[12] / (double)NM);
    printf("cycles/term: So5 %.1f So6 %.1f So7 %.1f (%s)\n", cyc[0] / (double)NM, cyc[1] / (double)NM,
           cyc[2] / (double)NM, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
