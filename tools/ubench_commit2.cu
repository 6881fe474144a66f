// Microbenchmark (profiling aid, not product): does tcgen05.commit between MMA batches
// serialize the tensor pipe?  NB batches of 12 kind::tf32 128xBNx8 TS MMAs with
// C commits after each batch (C = 0..3), one final commit + wait.
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
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int BN>
__global__ void __launch_bounds__(128, 1) k(long long* out, int nb, int nc, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[5];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 5; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
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
    long long tiss = 0;
    const long long t0 = clock64();
    for (int b = 0; b < nb; ++b) {
      const long long ta = clock64();
      for (int i = 0; i < 12; ++i)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem + (uint32_t)(i % 3 == 0 ? 0 : BN)), "r"(tmem + 384u + (uint32_t)(i & 3) * 8u),
                       "l"(desc(sb + (i & 3) * 32u)), "r"(idesc), "r"(1u));
      tiss += clock64() - ta;
      for (int c = 0; c < nc; ++c) commit(smem_u32(&bars[c + 1]));
      if (mode == 1) {  // also a satisfied-barrier wait per batch, like the kernel's operand waits
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bars[4])) : "memory");
        while (!try_wait(smem_u32(&bars[4]), (uint32_t)(b & 1))) {}
      }
    }
    commit(smem_u32(&bars[0]));
    while (!try_wait(smem_u32(&bars[0]), 0)) {}
    out[0] = clock64() - t0;
    out[1] = tiss;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  cudaFuncSetAttribute(k<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  const int NB = 200;
  for (int mode = 0; mode < 2; ++mode)
    for (int nc = 0; nc <= 3; ++nc) {
      k<128><<<1, 128, 64 << 10>>>(d, NB, nc, mode);
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("BN=128 commits/batch=%d wait/batch=%d : %6.0f cyc/batch (ideal 768), issue %6.0f cyc/batch\n", nc, mode,
             (double)h[0] / NB, (double)h[1] / NB);
    }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
