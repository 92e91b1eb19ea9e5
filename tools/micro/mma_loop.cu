// Replica of k_lbm_fwd's MMA issue loop without producers/consumers: per
// chunk 2 blocks x 2 k-blocks x 4 k-steps of M=128 N=128 K=16 (SW128
// K-major), D = acc*256 + j*128, commits to two barriers.  Flags select
// variations to find what separates it from the 64 cyc/MMA floor.
//   flags bit4: 8 epilogue warps wait tfull / arrive tempty, MMA waits tempty;
//         bit5: producer warp waits empty / arrives full, MMA waits full
//   argv[1] bit0: rotate B stage (3 x 32 KB)   bit1: alternate acc
//          bit2: W rows 128 apart per block (as kernel)   bit3: wait each commit
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__global__ void k(int flags, int nch, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* wres = s;              // 64 KB
  uint8_t* ast = s + 65536;       // 3 x 32 KB
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[8];
  __shared__ __align__(8) uint64_t tempty[2], fullb[3], done_bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (65536 + 98304) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    ((uint32_t*)s)[i] = (0x3f00u | (h & 0x80ffu)) | ((0x3f00u | ((h >> 16) & 0x80ffu)) << 16);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[i])));
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su(&tempty[i])));
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&fullb[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&done_bar)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&done_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = slot;
  const bool two = flags & 64;   // bit6: two MMA warps (1: even chunks / acc 0, 2: odd chunks / acc 1)
  if (warp == 1 || (two && warp == 2)) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    for (int ch = two ? warp - 1 : 0; ch < nch; ch += two ? 2 : 1) {
      const int acc = ch & 1, stage = ch % 3;
      if (flags & 16) {
        const uint32_t par = ((ch >> 1) & 1) ^ 1;
        asm volatile("{\n.reg .pred p;\nW1: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1;\n}\n" ::"r"(su(&tempty[acc])), "r"(par));
      }
      if (flags & 32) {
        const uint32_t par = (ch / 3) & 1;
        asm volatile("{\n.reg .pred p;\nW3: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W3;\n}\n" ::"r"(su(&fullb[stage])), "r"(par));
      }
      if (flags & 128) {   // two try_waits on barriers whose phase 0 completed long ago
        asm volatile("{\n.reg .pred p;\nW6: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W6;\n}\n" ::"r"(su(&done_bar)), "r"(0));
        asm volatile("{\n.reg .pred p;\nW7: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W7;\n}\n" ::"r"(su(&done_bar)), "r"(0));
      }
      if (two && (flags & 256) && ch > 0)   // token: the other warp finished issuing chunk ch-1
        asm volatile("bar.sync %0, 64;" ::"r"(1 + (ch & 1)) : "memory");
      const uint64_t bd0 = desc(su(ast + ((flags & 1) ? stage : 0) * 32768));
      for (int j = 0; j < 2; ++j) {
        const uint32_t d = tbase + (uint32_t)(((flags & 2) ? acc : 0) * 256 + j * 128);
        const uint64_t ad0 = desc(su(wres + ((flags & 4) ? j * 32768 : 0)));
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = ad0 + (uint64_t)(kb * 1024 + 2 * kk);
            const uint64_t bd = bd0 + (uint64_t)(kb * 1024 + 2 * kk);
            asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                         "l"(ad), "l"(bd), "r"(idesc), "r"(kb | kk));
          }
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                   ::"r"(su(&bars[stage])) : "memory");
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                   ::"r"(su(&bars[4 + acc])) : "memory");
      if (two && (flags & 256) && ch + 1 < nch)   // pass the token to the other warp (it issues ch+1)
        asm volatile("bar.arrive %0, 64;" ::"r"(1 + ((ch + 1) & 1)) : "memory");
      __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  }
  if (warp >= 4 && (flags & 16)) {   // epilogue: wait tfull[acc] (bars[4+acc]), arrive tempty
    int acc = 0;
    uint32_t ph[2] = {0, 0};
    for (int ch = 0; ch < nch; ++ch) {
      asm volatile("{\n.reg .pred p;\nW4: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W4;\n}\n" ::"r"(su(&bars[4 + acc])), "r"(ph[acc]));
      ph[acc] ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&tempty[acc])) : "memory");
      if (++acc == 2) acc = 0;
    }
  }
  if (warp == 0 && (flags & 32)) {   // producer: wait empty[stage] (bars[stage]), arrive full
    int stage = 0;
    uint32_t ph[3] = {1, 1, 1};
    if ((threadIdx.x & 31) == 0)
      for (int ch = 0; ch < nch; ++ch) {
        asm volatile("{\n.reg .pred p;\nW5: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W5;\n}\n" ::"r"(su(&bars[stage])), "r"(ph[stage]));
        ph[stage] ^= 1;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&fullb[stage])) : "memory");
        if (++stage == 3) stage = 0;
      }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main(int argc, char** argv) {
  int nblk = argc > 2 ? atoi(argv[2]) : 1;
  long long* out;
  cudaMalloc(&out, 1024 * 8);
  const int smem = 1024 + 65536 + 98304;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int f : {7, 7 + 48, 7 + 48 + 64, 7 + 48 + 64 + 256, 7 + 64 + 256}) {
    const int nch = 2000;
    k<<<nblk, 384, smem>>>(f, nch, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, out, 8 * nblk, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < nblk; ++i) m += h[i];
    printf("flags %2d blocks %d: %s  %.1f cycles per chunk (16 MMAs; floor 1024)\n", f, nblk, cudaGetErrorString(e), m / nblk / nch);
  }
  return 0;
}
