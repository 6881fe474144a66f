// Tile-store shape microbenchmark (sm_100a): one 256-thread block per SM writes a 128-pixel x
// 128-channel FP32 tile (64 KB) into an NCHW plane layout (channel stride E2 floats), per
// "tile" iteration, (a) as the conv epilogue does: a thread per pixel and column half, 64
// 4-byte stores, a warp instruction = one 128-byte row; (b) with 16-byte stores: a thread
// holds 4 consecutive pixels of a channel, a warp instruction = 8 pixel groups x 4 channels;
// (c) 16-byte stores where a warp instruction covers one channel's 128 pixels (512 B
// contiguous).  Cycles per tile on block 0 and aggregate GB/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_store(float* O, int E2, int tiles_per_cta, int mode, long long* cyc, int ntile = 6272) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = warp >> 2, q = warp & 3;
  long long t0 = clock64();
  for (int t = 0; t < tiles_per_cta; ++t) {
    const long long tile = ((long long)t * gridDim.x + blockIdx.x) % ntile;
    const long long p0 = tile * 128;                 // pixel base (same image plane for simplicity)
    const long long n = p0 / E2, f0 = p0 % E2;
    float* base = O + n * 128 * (long long)E2 + f0;   // [channel][pixel]
    if (mode == 0) {
      float* op = base + (long long)(half * 64) * E2 + q * 32 + lane;
#pragma unroll
      for (int j = 0; j < 64; ++j) op[(long long)j * E2] = (float)(j + t);
    } else if (mode == 1) {
      // lane: pixel group g = lane / 4 (4 pixels), channel c4 = lane % 4 of a 4-channel block
      const int g = lane >> 2, c = lane & 3;
      float4* op = reinterpret_cast<float4*>(base + (long long)(half * 64 + c) * E2 + q * 32 + g * 4);
#pragma unroll
      for (int j = 0; j < 16; ++j) op[(long long)j * 4 * E2 / 4] = make_float4(j, t, 0.f, 1.f);
    } else {
      // warp instruction = one channel row of 128 pixels (512 B): warp w handles channels w, w+8, ...
      float4* op = reinterpret_cast<float4*>(base + (long long)warp * E2 + lane * 4);
#pragma unroll
      for (int j = 0; j < 16; ++j) op[(long long)j * 8 * E2 / 4] = make_float4(j, t, 0.f, 1.f);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[mode] = t1 - t0;
}
int main() {
  const int E2 = 112 * 112, N = 64;
  float* O; long long* cyc;
  cudaMalloc(&O, (size_t)N * 128 * E2 * 4);
  cudaMallocManaged(&cyc, 64);
  const int tiles = N * E2 / 128, per = tiles / 148;
  for (int grid : {148, 32, 8, 1})
  for (int mode = 0; mode < 3; ++mode) {
    k_store<<<grid, 256>>>(O, E2, per, mode, cyc);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_store<<<grid, 256>>>(O, E2, per, mode, cyc);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("grid %3d mode %d: %.0f cycles per 64 KB tile (block 0), %.1f GB/s aggregate, err %d\n", grid, mode,
           (double)cyc[mode] / per, (double)grid * per * 65536 / ms / 1e6, (int)cudaGetLastError());
  }
  return 0;
}
