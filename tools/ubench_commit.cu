// Microbenchmark (profiling aid, not product): latency of tcgen05.commit -> mbarrier
// wakeup on an idle tensor pipe, and issue->commit-arrival for N back-to-back
// kind::tf32 128xNx8 TS-form MMAs.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
               : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) { while (!try_wait(bar, ph)) {} }
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int BN>
__global__ void __launch_bounds__(128, 1) k(long long* out, int nmma) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t b = smem_u32(&bar);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t sb = (smem_u32(sm) + 1023u) & ~1023u;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t ph = 0;
    long long tc = 0, tm = 0;
    for (int it = 0; it < 64; ++it) {
      long long t0 = clock64();
      commit(b);
      wait(b, ph); ph ^= 1;
      long long t1 = clock64();
      for (int i = 0; i < nmma; ++i) {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem), "r"(tmem + 384u + (uint32_t)(i & 3) * 8u), "l"(desc(sb + (i & 3) * 32u)), "r"(idesc), "r"(1u));
      }
      commit(b);
      wait(b, ph); ph ^= 1;
      long long t2 = clock64();
      if (it >= 8) { tc += t1 - t0; tm += t2 - t1; }
    }
    out[0] = tc / 56; out[1] = tm / 56;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  cudaFuncSetAttribute(k<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  cudaFuncSetAttribute(k<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  for (int n : {0, 1, 3, 12, 24, 48}) {
    k<128><<<1, 128, 64 << 10>>>(d, n); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("BN=128 nmma=%2d  empty-commit %lld cyc  issue->done %lld cyc (%.1f/mma)\n", n, h[0], h[1], n ? (double)h[1] / n : 0.0);
    k<64><<<1, 128, 64 << 10>>>(d, n); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("BN= 64 nmma=%2d  empty-commit %lld cyc  issue->done %lld cyc (%.1f/mma)\n", n, h[0], h[1], n ? (double)h[1] / n : 0.0);
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
