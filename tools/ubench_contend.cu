// Microbenchmark (profiling aid, not product): tcgen05.mma (kind::tf32, TS, 128x128x8)
// throughput while other warps generate traffic of one kind:
//   0 none | 1 STTM (tcgen05.st x16) | 2 LDTM (tcgen05.ld x16) | 3 LDS.128 |
//   4 LDG.128 (L1-resident) | 5 LDG.128 (L2-resident, 8 MB) | 6 STTM + LDG.128 (L2)
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
__device__ volatile int g_stop;

__global__ void __launch_bounds__(384, 1) k(long long* out, const float4* gsrc, int nmma, int mode, long long gmask) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const uint32_t b = smem_u32(&bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t sb = (smem_u32(sm) + 1023u) & ~1023u;
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) | ((128u >> 4) << 24);
      const long long t0 = clock64();
      for (int i = 0; i < nmma; ++i)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(tmem), "r"(tmem + 384u + (uint32_t)(i & 3) * 8u), "l"(desc(sb + (i & 3) * 32u)), "r"(idesc), "r"(1u));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
      while (!try_wait(b, 0)) {}
      out[0] = clock64() - t0;
      done = 1;
    }
    __syncwarp();
  } else if (warp >= 4) {
    // traffic warps 4..11 (two per TMEM lane quarter)
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t tb = tmem + ((q * 32u) << 16) + 128u + (uint32_t)((warp - 4) >> 2) * 64u;  // cols 128..255
    float acc = 0.f;
    long long ops = 0;
    const float4* ls = reinterpret_cast<const float4*>(sm + 65536);
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = j;
    long long gi = (long long)(warp * 32 + lane) * 4;
    while (!done) {
      for (int it = 0; it < 8; ++it) {
        if (mode == 1 || mode == 6) {
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                       ::"r"(tb + (it & 3) * 16u), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                         "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        if (mode == 2) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                         "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                       : "r"(tb + (it & 3) * 16u));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          acc += __uint_as_float(v[3]);
        }
        if (mode == 3) {
          float4 f = ls[(threadIdx.x * 4 + it * 97) & 4095];
          acc += f.x;
        }
        if (mode == 4 || mode == 5 || mode == 6) {
          float4 f0 = __ldg(gsrc + ((gi + it * 4096) & gmask));
          float4 f1 = __ldg(gsrc + ((gi + it * 4096 + 1) & gmask));
          float4 f2 = __ldg(gsrc + ((gi + it * 4096 + 2) & gmask));
          float4 f3 = __ldg(gsrc + ((gi + it * 4096 + 3) & gmask));
          acc += f0.x + f1.y + f2.z + f3.w;
        }
        ++ops;
      }
      gi += 8 * 4096;
    }
    if (acc == 1234.5f) out[3] = 1;
    if (warp == 4 && lane == 0) out[1] = ops;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  long long* d; cudaMalloc(&d, 32); long long h[4];
  float4* g; cudaMalloc(&g, 64 << 20); cudaMemset(g, 0, 64 << 20);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 << 10);
  const char* names[] = {"none", "STTM", "LDTM", "LDS.128", "LDG.128 L1", "LDG.128 L2", "STTM+LDG L2"};
  const int NM = 4800;
  for (int grid : {1, 148})
    for (int mode = 0; mode < 7; ++mode) {
      long long mask = (mode == 4) ? ((32 << 10) / 16 - 1) : ((8 << 20) / 16 - 1);
      k<<<grid, 384, 160 << 10>>>(d, g, NM, mode, mask);
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("grid=%3d traffic=%-12s mma %.1f cyc/mma (floor 64)   traffic iters/warp %lld\n", grid, names[mode],
             (double)h[0] / NM, h[1]);
    }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
