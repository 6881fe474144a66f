// FP64 issue cost per warp on sm_100a vs active lanes: a warp runs 3 interleaved DADD chains
// (the staged So5/So6/So7 chain warp) with `active` lanes enabled; cycles per step.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain3(double* out, long long* cyc, int iters, double x, int active) {
  double s = threadIdx.x, s2 = 1.0, s3 = 2.0;
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  if (lane < active) {
    for (int i = 0; i < iters; ++i) {
      s = __dadd_rn(s, x);
      s2 = __dadd_rn(s2, x);
      s3 = __dadd_rn(s3, x);
    }
  }
  long long t1 = clock64();
  if (lane < active) {
    for (int i = 0; i < iters; ++i) s = __dadd_rn(s, x);
  }
  long long t2 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = s + s2 + s3;
  if (threadIdx.x == 0 && blockIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64);
  const int iters = 1 << 15;
  for (int warps : {1, 4, 8}) for (int active : {1, 2, 4, 8, 16, 32}) {
    chain3<<<1, 32 * warps>>>(out, cyc, iters, 1.000001, active);
    cudaDeviceSynchronize();
    printf("warps %d active lanes %2d: 3 chains %.1f cyc/step, 1 chain %.1f cyc/step\n", warps, active, (double)cyc[0] / iters, (double)cyc[1] / iters);
  }
  return 0;
}
