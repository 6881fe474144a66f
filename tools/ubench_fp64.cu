// FP64 dependent-chain latency on sm_100a (error-path exact-order sums are one chain of
// N*M FP64 adds per output position): cycles per step of a DADD chain, a DMUL->DADD
// step (s += w*x, no contraction), and three interleaved chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, int iters, double x, double w) {
  double s = threadIdx.x, s2 = 1.0, s3 = 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) s = __dadd_rn(s, x);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) s = __dadd_rn(s, __dmul_rn(w, x));
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) {
    s = __dadd_rn(s, x);
    s2 = __dadd_rn(s2, __dmul_rn(w, x));
    s3 = __dadd_rn(s3, __dmul_rn((double)i, x));
  }
  long long t3 = clock64();
  float f = (float)x;
  double sf = 0.0;
  for (int i = 0; i < iters; ++i) { sf = __dadd_rn(sf, (double)f); f += 1.0f; }
  long long t4 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = s + s2 + s3 + sf;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMallocManaged(&cyc, 64);
  const int iters = 1 << 16;
  for (int threads : {1, 32, 128}) {
    chain<<<1, threads>>>(out, cyc, iters, 1.000001, 1.5);
    cudaDeviceSynchronize();
    printf("threads %3d: dadd chain %.1f cyc/step, dmul+dadd %.1f, 3 chains %.1f, f2f+dadd %.1f\n", threads,
           (double)cyc[0] / iters, (double)cyc[1] / iters, (double)cyc[2] / iters, (double)cyc[3] / iters);
  }
  chain<<<148, 64>>>(out, cyc, iters, 1.000001, 1.5);
  cudaDeviceSynchronize();
  printf("148x64: dadd chain %.1f cyc/step, dmul+dadd %.1f, 3 chains %.1f, f2f+dadd %.1f\n",
         (double)cyc[0] / iters, (double)cyc[1] / iters, (double)cyc[2] / iters, (double)cyc[3] / iters);
  return 0;
}
