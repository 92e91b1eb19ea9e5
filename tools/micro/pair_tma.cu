// CTA-pair TMA + barrier protocol check: each CTA of a 2-CTA cluster loads a
// 64 x 64 bf16 tile with cp.async.bulk.tensor.cta_group::2 whose completion is
// signalled on the LEADER's mbarrier (mapa address); the leader arms the
// barrier with both CTAs' bytes and waits; then the peer arrives remotely on a
// second leader barrier (count 1) that the leader waits on.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void waitp(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(bar), "r"(par));
}
__global__ void __cluster_dims__(2, 1, 1) k(const __grid_constant__ CUtensorMap tm, int mode, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar[2];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t bar0_leader, bar1_leader;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(bar0_leader) : "r"(su(&bar[0])));
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(bar1_leader) : "r"(su(&bar[1])));
  if (threadIdx.x == 0) {
    if (rank == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[0])), "r"(2 * 8192) : "memory");
    if (mode == 0)
      asm volatile("cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(s)), "l"((uint64_t)&tm), "r"(bar0_leader), "r"(0), "r"((int)rank * 64), "r"(0) : "memory");
    else   // mode 1: plain TMA with a cluster-address barrier (no cta_group)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su(s)), "l"((uint64_t)&tm), "r"(bar0_leader), "r"(0), "r"((int)rank * 64), "r"(0) : "memory");
  }
  if (rank == 0) waitp(su(&bar[0]), 0);
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  // remote arrive: the peer arrives on the leader's bar[1]
  if (rank == 1 && threadIdx.x == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar1_leader) : "memory");
  if (rank == 0) waitp(su(&bar[1]), 0);
  if (threadIdx.x == 0) out[rank] = __bfloat162float(((__nv_bfloat16*)s)[1]);
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  __nv_bfloat16* g;
  cudaMalloc(&g, 128 * 64 * 2);
  __nv_bfloat16 h[128 * 64];
  for (int i = 0; i < 128 * 64; ++i) h[i] = __float2bfloat16((float)(i / 64 < 64 ? 1 : 2));
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {64, 128, 1};
  cuuint64_t str[2] = {128, 128 * 128};
  cuuint32_t box[3] = {64, 64, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  float* out;
  cudaMalloc(&out, 8);
  cudaMemset(out, 0, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<<<2, 128, 64 * 1024>>>(tm, mode, out);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[2];
  cudaMemcpy(ho, out, 8, cudaMemcpyDeviceToHost);
  printf("mode %d: enc %d, %s, leader got %g peer got %g (expect 1 2)\n", mode, (int)r, cudaGetErrorString(e), ho[0], ho[1]);
  return 0;
}
