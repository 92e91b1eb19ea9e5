// FFMA vs FFMA2 (fma.rn.f32x2) issue throughput per SM: 8 independent
// accumulator chains per thread, 1024 threads per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1(float* out, int n, float a) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, 0.5f * i);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, int n, float a) {
  unsigned long long x[8];
  for (int i = 0; i < 8; ++i) {
    float lo = threadIdx.x * 0.001f + i, hi = lo + 1.f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(lo), "f"(hi));
  }
  unsigned long long av, cv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(cv) : "f"(0.5f));
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(av), "l"(cv));
  float s = 0;
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 1024 * 4 * 4);
  const int n = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k1<<<148 * 2, 512>>>(o, n, 0.999f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms1; cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0);
    k2<<<148 * 2, 512>>>(o, n, 0.999f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    const double f1 = 2.0 * 148 * 2 * 512 * 8.0 * n, f2 = 2 * f1;
    printf("FFMA  %.3f ms  %.1f TFLOP/s\nFFMA2 %.3f ms  %.1f TFLOP/s\n", ms1, f1 / ms1 / 1e9, ms2, f2 / ms2 / 1e9);
  }
  return 0;
}
