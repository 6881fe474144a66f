// Microbenchmark (profiling aid, not product): the conv kernel's exact per-K-chunk MMA
// mix on one issuing thread, no operand barriers -- is ~1240 cycles per chunk a
// pipe-internal cost or the synchronization skeleton?
//   per half chunk hf (A half-stage hs = 2g + hf mod 8, B stage g mod 4):
//     2 main MMAs  D_main[(g/2)&1] += A_hi * B_hi       (k8 steps 2hf, 2hf+1)
//     4 corr MMAs  D_corr += A_lo * B_hi, A_hi * B_lo
// mode 0: the mix; 1: + the kernel's commits (emptyA per half, emptyB per chunk, accf
// every 2 chunks); 2: 12 MMAs into one accumulator, same A/B addresses; 3: the mix
// with the correction products into the main accumulator (no accumulator switch);
// 4: mode 0 without the A-operand column changes (always half-stage 0); 5: per k8 step
// main, lo*Bhi, hi*Blo (same per-accumulator order); 6: 5 + commits.
#include <cstdint>
#include <cstdio>
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
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

constexpr int BN = 128;
__global__ void __launch_bounds__(128, 1) k(long long* out, int nchunks, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
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
    const uint32_t stage_bytes = BN * 256u;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t corr = tmem + 2 * BN, a_col0 = 3 * BN;
    const long long t0 = clock64();
    for (int g = 0; g < nchunks; ++g) {
      const uint32_t acc = (uint32_t)(g >> 1) & 1u, sB = (uint32_t)g & 3u;
      for (uint32_t hf = 0; hf < 2; ++hf) {
        const uint32_t hs = mode == 4 ? 0u : ((uint32_t)(2 * g) + hf) & 3u;  // 4 half-stages (BN=128)
        const uint32_t a_hi = tmem + a_col0 + hs * 32u, a_lo = a_hi + 16u;
        const uint32_t b_hi = sb + sB * stage_bytes + hf * 64u, b_lo = b_hi + (uint32_t)BN * 128u;
        const uint32_t d_main = tmem + acc * BN;
        const uint32_t d_corr = (mode == 2 || mode == 3) ? d_main : corr;
        if (mode >= 5) {  // per k8 step: main, then both corrections -- consecutive MMAs share B_hi
          for (int kk = 0; kk < 2; ++kk) {
            mma(d_main, a_hi + kk * 8u, desc(b_hi + kk * 32u), idesc, 1u);
            mma(corr, a_lo + kk * 8u, desc(b_hi + kk * 32u), idesc, 1u);
            mma(corr, a_hi + kk * 8u, desc(b_lo + kk * 32u), idesc, 1u);
          }
        } else {
        for (int kk = 0; kk < 2; ++kk) mma(d_main, a_hi + kk * 8u, desc(b_hi + kk * 32u), idesc, 1u);
        }
        for (int kk = 0; kk < 2 && mode < 5; ++kk) {
          if (mode == 2) {
            mma(d_main, a_hi + kk * 8u, desc(b_hi + kk * 32u), idesc, 1u);
            mma(d_main, a_hi + kk * 8u, desc(b_hi + kk * 32u), idesc, 1u);
          } else {
            mma(d_corr, a_lo + kk * 8u, desc(b_hi + kk * 32u), idesc, 1u);
            mma(d_corr, a_hi + kk * 8u, desc(b_lo + kk * 32u), idesc, 1u);
          }
        }
        if (mode == 1 || mode == 6) {
          commit(smem_u32(&bars[1 + hf]));
          if (hf == 1) {
            commit(smem_u32(&bars[3]));
            if (g & 1) commit(smem_u32(&bars[4]));
          }
        }
      }
    }
    commit(smem_u32(&bars[0]));
    while (!try_wait(smem_u32(&bars[0]), 0)) {
    }
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  long long h[148];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 << 10);
  const int NC = 400;
  const char* names[] = {"mix", "mix+commits", "12 main MMAs", "mix, one accumulator", "mix, fixed A cols",
                         "M,C,C per k8", "M,C,C per k8 + commits"};
  for (int grid : {1, 148})
    for (int mode = 0; mode < 7; ++mode) {
      k<<<grid, 128, 160 << 10>>>(d, NC, mode);
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("grid=%3d %-22s %7.1f cycles per K chunk (12 MMAs, floor 768)\n", grid, names[mode], (double)mx / NC);
    }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
