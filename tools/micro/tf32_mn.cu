// MN-major B operand with kind::tf32 (SWIZZLE_128B): B(n, k) stored as K rows
// of 32 fp32 (128 B, one MN chunk), row k's 16-B chunk q at q ^ (k & 7).
// A(m, k) = [k == kk] (K-major), so D[m][n] = B(n, kk) -> prints whether the
// MN-major descriptor reads B as intended (for LBO / SBO variants).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__global__ void k(int kk, uint32_t lbo, uint32_t sbo, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  float* A = (float*)s;              // 128 rows x 32 fp32 (K-major, one 128-B row per m)
  float* Bm = (float*)(s + 16384);   // MN-major: 2 chunks (n 0..31, 32..63) x 32 k-rows x 128 B
  for (int i = threadIdx.x; i < (16384 + 8192) / 4; i += blockDim.x) ((float*)s)[i] = 0.f;
  __syncthreads();
  if (threadIdx.x < 128) {
    const int m = threadIdx.x;
    A[m * 32 + (((kk >> 2) ^ (m & 7)) * 4) + (kk & 3)] = 1.f;
  }
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {     // B(n, k) = 100 k + n
    const int n = e % 64, kr = e / 64, ch = n / 32, nn = n % 32;
    Bm[ch * 1024 + kr * 32 + (((nn >> 2) ^ (kr & 7)) * 4) + (nn & 3)] = 100.f * kr + n;
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    for (int st = 0; st < 4; ++st)    // 4 k-steps of 8
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(slot),
                   "l"(desc(su32(A), 16, 1024) + st * 2), "l"(desc(su32(Bm), lbo, sbo) + st * 64), "r"(idesc),
                   "r"(st ? 1 : 0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = threadIdx.x / 32;
  for (int n = 0; n < 64; ++n) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(slot + n + ((uint32_t)(w * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[threadIdx.x * 64 + n] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(slot));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 64 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 30000);
  for (int kk : {0, 5, 13, 31})
    for (auto ls : {std::pair<int, int>{4096, 1024}, {1024, 4096}, {4096, 128}, {128, 4096}}) {
      k<<<1, 128, 30000>>>(kk, ls.first, ls.second, d);
      float h[128 * 64];
      cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) bad += h[m * 64 + n] != 100.f * kk + n;
      printf("kk %2d lbo %4d sbo %4d: D[0][0..3] = %g %g %g %g, D[0][40] = %g, mismatches %d [%s]\n", kk, ls.first,
             ls.second, h[0], h[1], h[2], h[3], h[40], bad, cudaGetErrorString(e));
    }
  return 0;
}
