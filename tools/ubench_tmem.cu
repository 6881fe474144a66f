// Microbenchmark (profiling aid, not product): does tcgen05.ld (epilogue drains) share
// TMEM read bandwidth with TS-form MMAs (A operand read from TMEM)?
// Warp 0 lane 0 issues NMMA kind::tf32 128xBNx8 MMAs; warps 4..11 issue LDTM.x16 over
// a 128-column region NLD times.  Reports cycles of each role alone and together.
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
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
template <int BN, bool SS>
__global__ void __launch_bounds__(384, 1) k(long long* out, int nmma, int nld) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t b = smem_u32(&bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  long long t0 = clock64();
  if (threadIdx.x == 0 && nmma) {
    const uint32_t sb = (smem_u32(sm) + 1023u) & ~1023u;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((128u >> 4) << 24);
    for (int i = 0; i < nmma; ++i) {
      if (SS) {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tmem), "l"(desc(sb + 32768u + (i & 3) * 32u)), "l"(desc(sb + (i & 3) * 32u)), "r"(idesc), "r"(1u));
      } else {
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem), "r"(tmem + 384u + (uint32_t)(i & 3) * 8u), "l"(desc(sb + (i & 3) * 32u)), "r"(idesc), "r"(1u));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
    while (!try_wait(b, 0)) {}
    out[0] = clock64() - t0;
  }
  if (warp >= 4 && warp < 12 && nld) {
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t base = tmem + ((q * 32u) << 16) + 256u + (uint32_t)((warp - 4) >> 2) * 64u;
    float acc = 0.f;
    for (int i = 0; i < nld; ++i) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(base + c * 16u));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += __uint_as_float(v[j]);
      }
    }
    if (lane == 0 && warp == 4) out[1] = clock64() - t0;
    if (acc == 12345.f) out[2] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
template <int BN, bool SS>
void run(long long* d) {
  long long h[3];
  cudaFuncSetAttribute(k<BN, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 << 10);
  const int NM = 1200, NL = 100;  // 1200 MMAs ~ 77K cyc at N=128; 100 x 64 KB LDTM drains
  int cfg[3][2] = {{NM, 0}, {0, NL}, {NM, NL}};
  for (auto& c : cfg) {
    cudaMemset(d, 0, 24);
    k<BN, SS><<<1, 384, 80 << 10>>>(d, c[0], c[1]);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("BN=%3d %s nmma=%4d nld=%3d : mma %7lld cyc (%.1f/mma)  ld %7lld cyc (%.1f B/cyc)\n", BN, SS ? "SS" : "TS",
           c[0], c[1], h[0], c[0] ? (double)h[0] / c[0] : 0.0, h[1], h[1] ? 65536.0 * c[1] / h[1] : 0.0);
  }
}
int main() {
  long long* d; cudaMalloc(&d, 24);
  run<128, false>(d); run<64, false>(d); run<128, true>(d); run<64, true>(d); run<256, true>(d);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
