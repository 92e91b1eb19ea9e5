// tcgen05.mma issue/execution rate: one CTA per SM, one thread issues NMMA
// back-to-back kind::f16 MMAs (M=128, K=16) with A from smem (SS) or TMEM (TS)
// and B from smem, N in {32, 64, 128, 256}; prints cycles per MMA vs the
// floor 128*N/256.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
template <int N, bool TS>
__global__ void k(int nmma, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < (128 + N) * 64 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0x3c003c00u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t sa = su32(s), sb = su32(s + 128 * 128);
    const uint32_t d = slot + 256;
    unsigned long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint64_t bd = desc(sb + (i & 3) * 32);
      if (TS) {
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(d), "r"(slot + (uint32_t)((i & 7) * 8)),
                     "l"(bd), "r"(idesc));
      } else {
        const uint64_t ad = desc(sa + (i & 3) * 32);
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int N, bool TS>
void run() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  const int smem = 1024 + (128 + N) * 128;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nmma = 8192;
  k<N, TS><<<148, 128, smem>>>(nmma, cyc);
  k<N, TS><<<148, 128, smem>>>(nmma, cyc);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s N=%3d: %.1f cyc/MMA (floor %d)  %s\n", TS ? "TS" : "SS", N, mx / nmma, 128 * N / 256,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  run<32, false>(); run<64, false>(); run<128, false>(); run<256, false>();
  run<32, true>(); run<64, true>(); run<128, true>(); run<256, true>();
  return 0;
}
