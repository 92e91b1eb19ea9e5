// CTA-pair (cta_group::2) protocol check: cluster of 2 CTAs; each CTA fills
// its smem A half (128 x 64 bf16 = rank+1) and B half (64 x 64 bf16 = 1);
// the leader issues one M=256 N=128 K=64 MMA (4 x K=16), commits multicast;
// each CTA reads its TMEM lanes and writes D[lane][col] to global.  Expected
// D = (rank+1) * 64 for every element.  Steps can be disabled to localise a
// hang: argv[1] = mode (0 alloc only, 1 + mma, 2 + TMA-to-leader barrier).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__global__ void __cluster_dims__(2, 1, 1) k(int mode, float* out) {
  const int mode0 = mode;
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2[2];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32;
  // A half: 128 rows x 64 k, all = rank+1 ; B half: 64 rows x 64 k all = 1 (bf16 1.0 = 0x3f80, 2.0 = 0x4000)
  const uint32_t av = rank == 0 ? 0x3f803f80u : 0x40004000u;
  for (int i = threadIdx.x; i < 128 * 64 / 2; i += blockDim.x) ((uint32_t*)s)[i] = av;
  if (mode == 7) {   // random bf16 operands (|x| ~ 1), mode 6 timing
    for (int i = threadIdx.x; i < 32768 / 4 * 2; i += blockDim.x) {
      uint32_t h = (uint32_t)i * 2654435761u ^ (rank * 977u);
      h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
      const uint32_t lo = 0x3f00u | (h & 0x80ffu), hi = 0x3f00u | ((h >> 16) & 0x80ffu);
      ((uint32_t*)s)[i] = lo | (hi << 16);
    }
    mode = 6;
  }
  if (mode0 != 7) for (int i = threadIdx.x; i < 64 * 64 / 2; i += blockDim.x) ((uint32_t*)(s + 16384))[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar2[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar2[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = slot;
  if (threadIdx.x == 0 && mode == 0) printf("rank %u tmem base %x\n", rank, tbase);
  if (mode >= 3) {   // rate: 3 = pair M=256 N=128 (leader issues), 4 = each CTA M=128 N=128 (cta_group::1)
    const int R = 4096;
    long long t0 = clock64();
    if (mode == 3 && rank == 0 && warp == 1) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      for (int r = 0; r < R; ++r)
        for (int k = 0; k < 4; ++k)
          asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
                       "l"(desc(su(s)) + 2 * k), "l"(desc(su(s + 16384)) + 2 * k), "r"(idesc), "r"(k));
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n"
                   ::"r"(su(&bar)), "h"((uint16_t)3) : "memory");
    }
    if (mode == 4 && warp == 1) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      for (int r = 0; r < R; ++r)
        for (int k = 0; k < 4; ++k)
          asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
                       "l"(desc(su(s)) + 2 * k), "l"(desc(su(s + 16384)) + 2 * k), "r"(idesc), "r"(k));
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                   ::"r"(su(&bar)) : "memory");
    }
    if (mode >= 5 && warp == 1) {   // 5: commits only; 6: 16 MMAs + 2 commits per iteration (cta_group::1)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      for (int r = 0; r < R / 4; ++r) {
        if (mode == 6)
          for (int k = 0; k < 16; ++k)
            asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
                         "l"(desc(su(s)) + 2 * (k & 3)), "l"(desc(su(s + 16384)) + 2 * (k & 3)), "r"(idesc), "r"(k));
        for (int c = 0; c < 2; ++c)
          asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                       ::"r"(su(&bar2[c])) : "memory");
        __syncwarp();
      }
      long long t1 = clock64();
      if (threadIdx.x == 32) printf("mode %d rank %u: %.1f cycles per iteration (issue side)\n", mode0, rank, (double)(t1 - t0) / (R / 4));
    }
    if (mode < 5)
    asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(su(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0 && mode < 5) printf("mode %d rank %u: %.1f cycles per MMA instruction\n", mode, rank, (double)(t1 - t0) / (4.0 * R));
  } else if (mode >= 1) {
    if (rank == 0 && warp == 1) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      for (int k = 0; k < 4; ++k) {
        asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                     "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
                     "l"(desc(su(s)) + 2 * k), "l"(desc(su(s + 16384)) + 2 * k), "r"(idesc), "r"(k));
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n"
                   ::"r"(su(&bar)), "h"((uint16_t)3) : "memory");
    }
    // all threads wait for the commit (phase 0)
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
      uint32_t r0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(tbase + ((uint32_t)(warp * 32) << 16) + 5));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      out[rank * 128 + warp * 32 + threadIdx.x % 32] = __uint_as_float(r0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 1;
  float* out;
  cudaMalloc(&out, 256 * 4);
  cudaMemset(out, 0, 256 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<2, 128, 64 * 1024>>>(mode, out);
  cudaError_t e = cudaDeviceSynchronize();
  float h[256];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode %d: %s  leader lanes %g %g  peer lanes %g %g (expect 64 / 128)\n", mode, cudaGetErrorString(e), h[0],
         h[127], h[128], h[255]);
  return 0;
}
