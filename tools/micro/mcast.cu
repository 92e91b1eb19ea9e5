// Cluster-of-2 TMA multicast + multicast tcgen05.commit: the pipeline the
// conv modes use when a CTA pair shares the B operand.  Each CTA loads HALF
// of a 128-row x 128-B SWIZZLE_128B tile and multicasts it to both CTAs
// (.multicast::cluster, mask 0b11); each CTA's full barrier expects the whole
// tile.  Then each CTA's MMA-side commit arrives on the "empty" barrier of
// BOTH CTAs (tcgen05.commit ... .multicast::cluster), count 2.  Checks tile
// contents in both CTAs and that both barriers complete (bounded spins).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ int spin(uint64_t* bar, uint32_t parity) {
  for (int it = 0; it < 4000000; ++it) {
    uint32_t p;
    asm volatile("{\n.reg .pred q;\nmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\nselp.u32 %0, 1, 0, q;\n}\n"
                 : "=r"(p) : "r"(su(bar)), "r"(parity) : "memory");
    if (p) return 1;
  }
  return 0;
}

__global__ void __cluster_dims__(2, 1, 1) k(const __grid_constant__ CUtensorMap tm, const __nv_bfloat16* src, int* ok) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full, empty;
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) s[i] = 0xAB;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(su(&empty)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  int good = 1;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full)), "r"(16384) : "memory");
    const uint16_t mask = 3;
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
                 " [%0], [%1, {%3, %4}], [%2], %5;"
                 ::"r"(su(s + rank * 8192)), "l"((uint64_t)&tm), "r"(su(&full)), "r"(0), "r"((int)rank * 64), "h"(mask)
                 : "memory");
    good &= spin(&full, 0);
  }
  __syncthreads();
  // contents: row r chunk q at (q ^ (r & 7))
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    int r = i / 64, c = i % 64, q = c / 8, e = c % 8;
    const __nv_bfloat16* got = (const __nv_bfloat16*)(s + r * 128 + ((q ^ (r & 7)) * 16)) + e;
    if (__bfloat162float(*got) != __bfloat162float(src[r * 64 + c])) good = 0;
  }
  good = __syncthreads_and(good);
  if (threadIdx.x < 32) {
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n"
                 ::"r"(su(&empty)), "h"((uint16_t)3) : "memory");
  }
  if (threadIdx.x == 0) good &= spin(&empty, 0);
  good = __syncthreads_and(good);
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
  if (threadIdx.x == 0) ok[blockIdx.x] = good;
}

int main() {
  std::vector<__nv_bfloat16> h(128 * 64);
  for (int i = 0; i < 128 * 64; ++i) h[i] = __float2bfloat16((float)((i * 7) % 251));
  __nv_bfloat16* d; cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  cuuint64_t dims[2] = {64, 128};
  cuuint64_t str[1] = {128};
  cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  int* ok; cudaMalloc(&ok, 8 * sizeof(int));
  cudaMemset(ok, 0, 8 * sizeof(int));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
  k<<<4, 128, 20480>>>(tm, d, ok);
  cudaError_t e = cudaDeviceSynchronize();
  int hk[8];
  cudaMemcpy(hk, ok, sizeof(hk), cudaMemcpyDeviceToHost);
  printf("%s: ok = %d %d %d %d\n", cudaGetErrorString(e), hk[0], hk[1], hk[2], hk[3]);
  return (e == cudaSuccess && hk[0] && hk[1] && hk[2] && hk[3]) ? 0 : 1;
}
