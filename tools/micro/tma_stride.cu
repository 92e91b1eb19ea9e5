// TMA tiled-mode traversal strides (elementStrides = 2 along W and H) on a
// 5-D map {C, W, H, N, B}: the strided-gather box the implicit-GEMM conv
// producer relies on.  Checks (a) how many bytes one box delivers (expect_tx),
// (b) that out-of-bounds (negative) coordinates zero-fill, (c) the SWIZZLE_128B
// row order ((n * BOH + i) * BOW + j).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tm, int w0, int h0, int n0, int b0, uint32_t bytes,
                  __nv_bfloat16* out, int* ok) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) s[i] = 0xFF;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                 ::"r"(su(s)), "l"((uint64_t)&tm), "r"(su(&bar)), "r"(0), "r"(w0), "r"(h0), "r"(n0), "r"(b0) : "memory");
    int done = 0;
    for (int it = 0; it < 2000000 && !done; ++it) {
      uint32_t p;
      asm volatile("{\n.reg .pred q;\nmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\nselp.u32 %0, 1, 0, q;\n}\n"
                   : "=r"(p) : "r"(su(&bar)) : "memory");
      done = p;
    }
    *ok = done;
  }
  __syncthreads();
  // un-swizzle rows of 128 B: chunk q of row r at (q ^ (r & 7))
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    int r = i / 64, c = i % 64, q = c / 8, e = c % 8;
    const __nv_bfloat16* src = (const __nv_bfloat16*)(s + r * 128 + ((q ^ (r & 7)) * 16)) + e;
    out[i] = *src;
  }
}

int main() {
  const int C = 64, W = 8, H = 8, N = 4, B = 2;
  std::vector<__nv_bfloat16> hx((size_t)B * N * H * W * C);
  for (int b = 0; b < B; ++b) for (int n = 0; n < N; ++n) for (int h = 0; h < H; ++h) for (int w = 0; w < W; ++w)
    for (int c = 0; c < C; ++c) {
      float v = c == 0 ? (float)(h * 16 + w) : c == 1 ? (float)(n + 10 * b) : (float)c;
      hx[((((size_t)b * N + n) * H + h) * W + w) * C + c] = __float2bfloat16(v);
    }
  void* dx; cudaMalloc(&dx, hx.size() * 2);
  cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  cuuint64_t dims[5] = {C, W, H, N, B};
  cuuint64_t str[4] = {C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, (cuuint64_t)N * H * W * C * 2};
  const int BOW = 4, BOH = 4, BNI = 2;
  cuuint32_t box[5] = {64, 2 * BOW, 2 * BOH, BNI, 1};
  cuuint32_t es[5] = {1, 2, 2, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, dx, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  __nv_bfloat16* dout; cudaMalloc(&dout, 128 * 64 * 2);
  int* dok; cudaMalloc(&dok, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  const int rows = BOW * BOH * BNI;
  for (uint32_t bytes : {(uint32_t)(rows * 128), (uint32_t)(64 * 2 * 2 * BOW * 2 * BOH * BNI)}) {
    int w0 = -1, h0 = -1, n0 = 1, b0 = 1;
    cudaMemset(dout, 0, 128 * 64 * 2);
    k<<<1, 256, 20000>>>(tm, w0, h0, n0, b0, bytes, dout, dok);
    cudaError_t e = cudaDeviceSynchronize();
    int ok = 0; cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
    std::vector<__nv_bfloat16> ho(128 * 64);
    cudaMemcpy(ho.data(), dout, ho.size() * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int n = 0; n < BNI; ++n) for (int i = 0; i < BOH; ++i) for (int j = 0; j < BOW; ++j) {
      int row = (n * BOH + i) * BOW + j;
      int h = h0 + 2 * i, w = w0 + 2 * j;
      bool in = h >= 0 && h < H && w >= 0 && w < W;
      float v0 = __bfloat162float(ho[row * 64 + 0]), v1 = __bfloat162float(ho[row * 64 + 1]);
      float e0 = in ? (float)(h * 16 + w) : 0.f, e1 = in ? (float)(n0 + n + 10 * b0) : 0.f;
      if (v0 != e0 || v1 != e1) { if (bad < 5) printf("row %d: got %g %g want %g %g\n", row, v0, v1, e0, e1); ++bad; }
    }
    printf("expect_tx %u: completed %d, err %s, bad rows %d of %d (row %d ch0 = %g)\n", bytes, ok,
           cudaGetErrorString(e), bad, rows, rows, __bfloat162float(ho[rows * 64]));
  }
  return 0;
}
