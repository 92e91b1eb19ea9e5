// Does a TMA tiled STORE honour traversal strides (elementStrides = 2 along W
// and H)?  The sub-pixel conv epilogue would write its phase (ph, pw) rows to
// pixels (2i + ph, 2j + pw) with one such store.  Image [N=2][H=8][W=8][C=64]
// bf16 zeroed; a 16-row x 128-B SWIZZLE_128B smem tile (row r = 1000 + r in
// channel 0, r's chunk q at q ^ (r & 7)) stored with box {64, 8, 8, 1},
// es {1, 2, 2, 1} at (0, x0 = 1, y0 = 0, n = 1); expect row (i, j) at pixel
// (n 1, y 2i, x 2j + 1) and every other pixel still 0.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) {
    int r = i / 64, c = i % 64, q = c / 8, e = c % 8;
    __nv_bfloat16* dst = (__nv_bfloat16*)(s + r * 128 + ((q ^ (r & 7)) * 16)) + e;
    *dst = __float2bfloat16(c == 0 ? (float)(1000 + r) : (float)c);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"((uint64_t)&tm),
                 "r"(su(s)), "r"(0), "r"(1), "r"(0), "r"(1) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int C = 64, W = 8, H = 8, N = 2;
  void* dx; cudaMalloc(&dx, (size_t)N * H * W * C * 2);
  cudaMemset(dx, 0, (size_t)N * H * W * C * 2);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  cuuint64_t dims[4] = {C, W, H, N};
  cuuint64_t str[3] = {C * 2, W * C * 2, H * W * C * 2};
  cuuint32_t box[4] = {64, 8, 8, 1}, es[4] = {1, 2, 2, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dx, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  k<<<1, 128, 8192>>>(tm);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<__nv_bfloat16> h((size_t)N * H * W * C);
  cudaMemcpy(h.data(), dx, h.size() * 2, cudaMemcpyDeviceToHost);
  int bad = 0, written = 0;
  for (int n = 0; n < N; ++n) for (int y = 0; y < H; ++y) for (int x = 0; x < W; ++x) {
    float v0 = __bfloat162float(h[(((size_t)n * H + y) * W + x) * C]);
    float v5 = __bfloat162float(h[(((size_t)n * H + y) * W + x) * C + 5]);
    bool target = n == 1 && y % 2 == 0 && x % 2 == 1;
    if (target) {
      int i = y / 2, j = (x - 1) / 2;
      printf("pixel n%d y%d x%d (i%d j%d): %g %g\n", n, y, x, i, j, v0, v5);
      if (v0 != 1000 + i * 4 + j || v5 != 5) ++bad;
      ++written;
    } else if (v0 != 0 || v5 != 0) {
      if (bad < 5) printf("stray write n%d y%d x%d: %g\n", n, y, x, v0);
      ++bad;
    }
  }
  printf("%s: %d target pixels, %d bad\n", cudaGetErrorString(e), written, bad);
  return bad == 0 && e == cudaSuccess ? 0 : 1;
}
