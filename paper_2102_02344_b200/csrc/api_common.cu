// api_common.cu -- init, error reporting, launch accounting, small utilities.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <set>
#include <tuple>

#include "common.cuh"

namespace hfta {

static thread_local std::string g_err;
static std::atomic<int> g_sms{0};
static std::atomic<int> g_init{0};
static std::atomic<uint64_t> g_launches{0};
static int g_sync = -1;

hfta_status fail(hfta_status code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

hfta_status check_init() {
  if (!g_init.load()) return fail(HFTA_ERR_NOT_INITIALIZED, "hfta_init() has not succeeded");
  return HFTA_OK;
}

int num_sms() { return g_sms.load(); }
void count_launches(uint64_t n) { g_launches += n; }

void set_max_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, size_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert(std::make_tuple(kern, dev, bytes)).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

hfta_status post_launch(cudaStream_t s, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HFTA_ERR_CUDA, "%s: launch failed: %s", what, cudaGetErrorString(e));
  if (g_sync < 0) {
    const char* v = getenv("HFTA_SYNC");
    g_sync = (v && v[0] == '1') ? 1 : 0;
  }
  if (g_sync) {
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(HFTA_ERR_CUDA, "%s: kernel failed: %s", what, cudaGetErrorString(e));
  }
  return HFTA_OK;
}

__global__ void k_cast_f32_bf16(int64_t n, const float* __restrict__ s, __nv_bfloat16* __restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

__global__ void k_step_inc(int64_t* step) { *step += 1; }

template <typename T>
__global__ void k_add(int64_t rows, int64_t cols, const T* __restrict__ x1, int64_t bs1, int64_t ld1,
                      const T* __restrict__ x2, int64_t bs2, int64_t ld2, T* __restrict__ y, int64_t bsy,
                      int64_t ldy) {
  const int b = blockIdx.y;
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    stf(y + b * bsy + r * ldy + c, ldf(x1 + b * bs1 + r * ld1 + c) + ldf(x2 + b * bs2 + r * ld2 + c));
  }
}

// dense bf16 rows: flat runs, 8 elements per 16-B access (packed FADD2 via bf16x2 unpack)
__global__ void k_add_flat(int64_t n8, const __nv_bfloat16* __restrict__ x1, int64_t bs1,
                           const __nv_bfloat16* __restrict__ x2, int64_t bs2, __nv_bfloat16* __restrict__ y,
                           int64_t bsy) {
  const int b = blockIdx.y;
  const uint4* a4 = reinterpret_cast<const uint4*>(x1 + b * bs1);
  const uint4* c4 = reinterpret_cast<const uint4*>(x2 + b * bs2);
  uint4* y4 = reinterpret_cast<uint4*>(y + b * bsy);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 av = a4[i], cv = c4[i];
    const uint32_t as[4] = {av.x, av.y, av.z, av.w}, cs[4] = {cv.x, cv.y, cv.z, cv.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float al, ah, cl, ch;
      unpack_bf2(as[e], al, ah);
      unpack_bf2(cs[e], cl, ch);
      o[e] = pack_bf2(al + cl, ah + ch);
    }
    y4[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace hfta

using namespace hfta;

extern "C" {

hfta_status hfta_init(int device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(HFTA_ERR_ARCH, "hfta_init: no CUDA device (%s)", e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(HFTA_ERR_INVALID_VALUE, "hfta_init: device %d of %d", device, n);
  if ((e = cudaSetDevice(device)) != cudaSuccess) return fail(HFTA_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess)
    return fail(HFTA_ERR_CUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
  if (prop.major != 10 || prop.minor != 0)
    return fail(HFTA_ERR_ARCH, "hfta_init: device %d is %s (CC %d.%d); libhfta requires CC 10.0 (B200, sm_100a)",
                device, prop.name, prop.major, prop.minor);
  g_sms = prop.multiProcessorCount;
  g_init = 1;
  return HFTA_OK;
}

const char* hfta_last_error(void) { return g_err.c_str(); }
const char* hfta_version(void) { return "libhfta 0.1 (sm_100a)"; }
uint64_t hfta_launch_count(void) { return g_launches.load(); }

hfta_status hfta_cast_f32_bf16(int64_t n, const float* src, void* dst, hfta_stream stream) {
  if (hfta_status s = check_init()) return s;
  HFTA_REQUIRE(n >= 0 && (n == 0 || (src && dst)), HFTA_ERR_INVALID_VALUE, "hfta_cast_f32_bf16: bad args");
  if (n == 0) return HFTA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int grid = (int)std::min<int64_t>(cdiv(n, 256), (int64_t)num_sms() * 8);
  k_cast_f32_bf16<<<grid, 256, 0, st>>>(n, src, (__nv_bfloat16*)dst);
  count_launches(1);
  return post_launch(st, "hfta_cast_f32_bf16");
}

hfta_status hfta_add(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_in X1, hfta_in X2, hfta_out Y,
                     hfta_stream stream) {
  if (hfta_status s = check_init()) return s;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(rows >= 1 && cols >= 1 && X1.ptr && X2.ptr && Y.ptr, HFTA_ERR_INVALID_VALUE, "hfta_add: bad args");
  HFTA_REQUIRE(X1.ld >= cols && X2.ld >= cols && Y.ld >= cols && (Y.bstride > 0 || B == 1), HFTA_ERR_SHAPE,
               "hfta_add: strides");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = rows * cols;
  if (dt == HFTA_BF16 && X1.ld == cols && X2.ld == cols && Y.ld == cols && n % 8 == 0 && X1.bstride % 8 == 0 &&
      X2.bstride % 8 == 0 && Y.bstride % 8 == 0 && aligned16(X1.ptr) && aligned16(X2.ptr) && aligned16(Y.ptr)) {
    dim3 g((unsigned)std::min<int64_t>(cdiv(n / 8, 256), 4 * 148), B);
    k_add_flat<<<g, 256, 0, st>>>(n / 8, (const __nv_bfloat16*)X1.ptr, X1.bstride, (const __nv_bfloat16*)X2.ptr,
                                  X2.bstride, (__nv_bfloat16*)Y.ptr, Y.bstride);
    count_launches(1);
    return post_launch(st, "hfta_add");
  }
  dim3 grid((unsigned)std::min<int64_t>(cdiv(rows * cols, 256), 2048), B);
  if (dt == HFTA_F32)
    k_add<float><<<grid, 256, 0, st>>>(rows, cols, (const float*)X1.ptr, X1.bstride, X1.ld, (const float*)X2.ptr,
                                       X2.bstride, X2.ld, (float*)Y.ptr, Y.bstride, Y.ld);
  else
    k_add<__nv_bfloat16><<<grid, 256, 0, st>>>(rows, cols, (const __nv_bfloat16*)X1.ptr, X1.bstride, X1.ld,
                                               (const __nv_bfloat16*)X2.ptr, X2.bstride, X2.ld,
                                               (__nv_bfloat16*)Y.ptr, Y.bstride, Y.ld);
  count_launches(1);
  return post_launch(st, "hfta_add");
}

hfta_status hfta_step_increment(int64_t* step, hfta_stream stream) {
  if (hfta_status s = check_init()) return s;
  HFTA_REQUIRE(step, HFTA_ERR_INVALID_VALUE, "hfta_step_increment: step is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  k_step_inc<<<1, 1, 0, st>>>(step);
  count_launches(1);
  return post_launch(st, "hfta_step_increment");
}

}  // extern "C"
