// Where does the exact-order So5/6/7 kernel spend its time?  Variants of the per-stage
// loop of k_seq_sums567 (16 terms per stage, one FP64 chain per lane), timed with
// clock64 on one warp: cycles per term.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cpa4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
template <int V>
__global__ void k(const float* O, int E2, int NM, double* out, long long* cyc) {
  __shared__ float ring[8][16][32];
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  long long t0 = clock64();
  int m = 0, n = 0;
  const int M = 256;
  for (int st = 0; st < NM / 16; ++st) {
    const int slot = st & 7;
    if (V == 0 || V == 1) {  // issue the stage 7 ahead with cp.async
      for (int u = 0; u < 16; ++u) cpa4(&ring[(st + 7) & 7][u][lane], O + (long long)((st + 7) * 16 + u) * E2 + lane);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 7;" ::: "memory");
      __syncwarp();
    }
    double pr[16];
    for (int u = 0; u < 16; ++u) {
      double x = (double)ring[slot][u][lane];
      const double w = (double)(m + u);
      pr[u] = (V == 1 || V == 3) ? x : __dmul_rn(w, x);
    }
    for (int u = 0; u < 16; ++u) s = __dadd_rn(s, pr[u]);
    m += 16;
    if (m >= M) { m -= M; ++n; }
    __syncwarp();
  }
  long long t1 = clock64();
  out[blockIdx.x * 32 + lane] = s + n;
  if (lane == 0 && blockIdx.x == 0) cyc[V] = t1 - t0;
}
int main() {
  const int E2 = 729, NM = 32768;
  float* O; double* out; long long* cyc;
  cudaMalloc(&O, (size_t)(NM + 256) * E2 * 4);
  cudaMemset(O, 0, (size_t)(NM + 256) * E2 * 4);
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64);
  k<0><<<37, 64>>>(O, E2, NM, out, cyc);
  k<1><<<37, 64>>>(O, E2, NM, out, cyc);
  k<2><<<37, 64>>>(O, E2, NM, out, cyc);
  k<3><<<37, 64>>>(O, E2, NM, out, cyc);
  cudaDeviceSynchronize();
  printf("cycles/term: ring+dmul %.1f  ring,no dmul %.1f  no ring+dmul %.1f  no ring,no dmul %.1f  (%s)\n",
         cyc[0] / (double)NM, cyc[1] / (double)NM, cyc[2] / (double)NM, cyc[3] / (double)NM,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
