// Does tcgen05.mma.kind::tf32 truncate or round its fp32 operands?  A[m][0] =
// 1 + 3*2^-12 (0.75 tf32 ulp above 1), B[n][0] = 1, all other k zero, so
// D[m][n] = tf32(A[m][0]): 1 (truncation), 1 + 2^-10 (round to nearest) or
// the exact fp32 value (no reduction).  Decides how the 3xTF32 split of the
// fp32 path forms its hi part.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__global__ void k(float aval, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  float* A = (float*)s;             // 128 rows x 128 B
  float* Bm = (float*)(s + 16384);  // 16 rows x 128 B
  for (int i = threadIdx.x; i < (128 + 16) * 32; i += blockDim.x) ((float*)s)[i] = 0.f;
  __syncthreads();
  if (threadIdx.x < 128) {           // element k = 0 of row m sits in 16-B chunk 0 ^ (m & 7)
    const int m = threadIdx.x;
    A[m * 32 + ((0 ^ (m & 7)) * 4)] = aval;
    if (m < 16) Bm[m * 32 + ((0 ^ (m & 7)) * 4)] = 1.f;
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
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 0;" ::"r"(slot), "l"(desc(su32(A))),
                 "l"(desc(su32(Bm))), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = threadIdx.x / 32;
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(slot + ((uint32_t)(w * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[threadIdx.x] = __uint_as_float(r);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000 + 1024);
  for (float a : {1.0f + 3.0f / 4096.0f, 1.0f + 1.0f / 4096.0f, -(1.0f + 3.0f / 4096.0f), 1.0f + 2.0f / 4096.0f}) {
    k<<<1, 128, 20000 + 1024>>>(a, d);
    float h[128];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("a = %.10f -> D = %.10f (rows 0, 77: %.10f)  trunc %.10f  rn %.10f  [%s]\n", a, h[0], h[77],
           (double)(int)(a * 1024.0f) / 1024.0, (double)rintf(a * 1024.0f) / 1024.0, cudaGetErrorString(e));
  }
  return 0;
}
