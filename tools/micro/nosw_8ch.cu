// SWIZZLE_NONE operand layouts for the 8-channel image gathers (16-B rows):
// test 1: K-major A, 8 taps x 8 channels per 64-wide k-block, tap t's 128 x 16 B
//         box at t * 2048 (core matrices: 8 rows x 16 B, SBO = 128 B between
//         8-row groups, LBO = 2048 B between 8-k groups); B K-major SW128.
// test 2: MN-major B, 16 taps x 8 channels = 128 columns, tap t's 64 k-rows x
//         16 B box at t * 1024; A K-major SW128.  Prints mismatches per
//         (LBO, SBO) variant.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// test 1: A(m,k) = 100*(k/8) + (k%8) + 1000*(m%4) ... keep values exact in bf16: small ints
__global__ void k1(int j, uint32_t lbo, uint32_t sbo, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __nv_bfloat16* A = (__nv_bfloat16*)s;            // 16 KB no-swizzle
  __nv_bfloat16* Bm = (__nv_bfloat16*)(s + 16384); // 16 rows x 128 B SW128 (K-major)
  for (int i = threadIdx.x; i < (16384 + 2048) / 2; i += blockDim.x) ((__nv_bfloat16*)s)[i] = __float2bfloat16(0.f);
  __syncthreads();
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    const int m = e / 64, k = e % 64, t = k / 8, c = k % 8;
    A[(t * 2048 + m * 16 + c * 2) / 2] = __float2bfloat16((float)(k + 64 * (m % 3)));
  }
  if (threadIdx.x < 16) {            // B[n][k] = (k == n + 16 j): SW128 row n, element k at chunk (k/8 ^ n&7)
    const int n = threadIdx.x, k = n + 16 * j;
    Bm[n * 64 + (((k >> 3) ^ (n & 7)) << 3) + (k & 7)] = __float2bfloat16(1.f);
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    for (int st = 0; st < 4; ++st)
      mma(slot, desc(su32(A) + st * 2 * 2048, lbo, sbo, 0), desc(su32(Bm), 16, 1024, 2) + st * 2, idesc, st);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = threadIdx.x / 32;
  for (int n = 0; n < 16; ++n) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(slot + n + ((uint32_t)(w * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[threadIdx.x * 16 + n] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}

// test 2: B(n, k) = n + 128 * (k % 2), MN-major no-swizzle, tap t (8 n) box: 64 k-rows x 16 B at t*1024
__global__ void k2(int kk, uint32_t lbo, uint32_t sbo, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __nv_bfloat16* A = (__nv_bfloat16*)s;            // 128 x 64 SW128 K-major
  __nv_bfloat16* Bm = (__nv_bfloat16*)(s + 16384); // 16 KB
  for (int i = threadIdx.x; i < 32768 / 2; i += blockDim.x) ((__nv_bfloat16*)s)[i] = __float2bfloat16(0.f);
  __syncthreads();
  if (threadIdx.x < 128) {
    const int m = threadIdx.x;
    A[m * 64 + (((kk >> 3) ^ (m & 7)) << 3) + (kk & 7)] = __float2bfloat16(1.f);
  }
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    const int n = e % 128, k = e / 128, t = n / 8, c = n % 8;
    Bm[(t * 1024 + k * 16 + c * 2) / 2] = __float2bfloat16((float)(n + 128 * (k % 2)));
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    for (int st = 0; st < 4; ++st)   // K-step of 16 rows: +256 B in the no-swizzle MN-major B (2 core groups of 8 rows)
      mma(slot, desc(su32(A), 16, 1024, 2) + st * 2, desc(su32(Bm) + st * 256, lbo, sbo, 0), idesc, st);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = threadIdx.x / 32;
  for (int n = 0; n < 128; ++n) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(slot + n + ((uint32_t)(w * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[threadIdx.x * 128 + n] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(slot));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 128 * 4);
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  static float h[128 * 128];
  for (auto ls : {std::pair<int, int>{128, 1024}}) {
    int bad = 0;
    for (int kk : {0, 1, 9, 30, 63}) {
      k2<<<1, 128, 40000>>>(kk, ls.first, ls.second, d);
      cudaMemcpy(h, d, 128 * 128 * 4, cudaMemcpyDeviceToHost);
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n) bad += h[m * 128 + n] != (float)(n + 128 * (kk % 2));
    }
    printf("MN-major no-swizzle B: lbo %4d sbo %4d -> mismatches %d (D[0][9] kk=63: %g) [%s]\n", ls.first, ls.second,
           bad, h[9], cudaGetErrorString(cudaGetLastError()));
  }
  for (auto ls : {std::pair<int, int>{2048, 128}}) {
    int bad = 0;
    for (int j = 0; j < 4; ++j) {
      k1<<<1, 128, 40000>>>(j, ls.first, ls.second, d);
      cudaMemcpy(h, d, 128 * 16 * 4, cudaMemcpyDeviceToHost);
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) bad += h[m * 16 + n] != (float)(n + 16 * j + 64 * (m % 3));
    }
    printf("K-major no-swizzle A: lbo %4d sbo %4d -> mismatches %d (D[1][3] j=3: %g) [%s]\n", ls.first, ls.second, bad,
           h[1 * 16 + 3], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
