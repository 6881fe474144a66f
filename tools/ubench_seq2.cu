// Exact-order chain sums, lane per (position, family): term loads straight into registers
// P terms ahead (volatile ld.global.nc so the compiler keeps them early), one DADD chain
// per lane.  Reports cycles per term for several prefetch depths; O is L2-resident.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ldnc(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
template <int P>
__global__ void k(const float* O, int E2, int NM, int M, double* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 0;  // position (fam 1: w = m)
  const float* base = O + (f % E2);
  float buf[P];
#pragma unroll
  for (int u = 0; u < P; ++u) buf[u] = ldnc(base + (long long)u * E2);
  double s = 0.0;
  int m = 0;
  long long t0 = clock64();
  for (int q0 = 0; q0 < NM; q0 += P) {
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const double x = (double)buf[u];
      const int qn = q0 + P + u;
      buf[u] = ldnc(base + (long long)(qn < NM ? qn : 0) * E2);
      s = __dadd_rn(s, __dmul_rn((double)m, x));
      m = (m + 1 == M) ? 0 : m + 1;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  const int E2 = 729, NM = 32768, M = 256;
  float* O; double* out; long long* cyc;
  cudaMalloc(&O, (size_t)NM * E2 * 4);
  cudaMemset(O, 0, (size_t)NM * E2 * 4);
  cudaMalloc(&out, 1 << 22);
  cudaMallocManaged(&cyc, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<16><<<69, 32>>>(O, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long c16 = cyc[0];
    k<32><<<69, 32>>>(O, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long c32 = cyc[0];
    k<64><<<69, 32>>>(O, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long c64 = cyc[0];
    k<32><<<23, 96>>>(O, E2, NM, M, out, cyc); cudaDeviceSynchronize(); long long c32b = cyc[0];
    printf("cycles/term P=16 %.1f  P=32 %.1f  P=64 %.1f  P=32 3 warps/block %.1f (%s)\n", c16 / (double)NM,
           c32 / (double)NM, c64 / (double)NM, c32b / (double)NM, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
