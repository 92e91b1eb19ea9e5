// pool.cu -- fused MaxPool2d and AdaptiveAvgPool2d((1,1)) for B models
// (App. B rows MaxPool2d / AdaptiveAvgPool2d; the ResNet-18
// family of NEXT-4).  The fused operator pools each of the B x C channels on
// its own, so one launch covers all models: grid-stride over
// [B][N][pixels][C / VEC] with 16-B channel vectors (NHWC per model).
// MaxPool: padded positions take no part (-inf), the first window tap
// (ky * k + kx order) wins exact ties, the tap index is kept (uint8) for the
// backward, which GATHERS per input pixel over the windows that contain it
// (fixed order, no atomics: deterministic).
#include <cfloat>

#include "common.cuh"

namespace hfta {
namespace {

struct PoolGeo {
  int N, H, W, C, Ho, Wo, k, s, p;
};

template <typename T, int VEC>
__global__ void k_maxpool_fwd(int B, PoolGeo g, const T* __restrict__ X, int64_t xbs, T* __restrict__ Y,
                              int64_t ybs, uint8_t* __restrict__ am, int64_t abs_) {
  const int cv = g.C / VEC;
  const int64_t per = (int64_t)g.N * g.Ho * g.Wo * cv;
  const int64_t total = per * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / per);
    int64_t r = i - b * per;
    const int c = (int)(r % cv) * VEC; r /= cv;
    const int ox = (int)(r % g.Wo); r /= g.Wo;
    const int oy = (int)(r % g.Ho);
    const int n = (int)(r / g.Ho);
    float best[VEC];
    int arg[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) { best[v] = -FLT_MAX; arg[v] = 0; }
    bool any[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) any[v] = false;
    const T* Xb = X + (int64_t)b * xbs;
    for (int ky = 0; ky < g.k; ++ky) {
      const int iy = oy * g.s - g.p + ky;
      if (iy < 0 || iy >= g.H) continue;
      for (int kx = 0; kx < g.k; ++kx) {
        const int ix = ox * g.s - g.p + kx;
        if (ix < 0 || ix >= g.W) continue;
        float x[VEC];
        ld_vec<T, VEC>(Xb + (((int64_t)n * g.H + iy) * g.W + ix) * g.C + c, x);
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          if (!any[v] || x[v] > best[v]) { best[v] = x[v]; arg[v] = ky * g.k + kx; any[v] = true; }
      }
    }
    const int64_t o = (((int64_t)n * g.Ho + oy) * g.Wo + ox) * g.C + c;
    st_vec<T, VEC>(Y + (int64_t)b * ybs + o, best);
#pragma unroll
    for (int v = 0; v < VEC; ++v) am[(int64_t)b * abs_ + o + v] = (uint8_t)arg[v];
  }
}

template <typename T, int VEC>
__global__ void k_maxpool_bwd(int B, PoolGeo g, const T* __restrict__ dY, int64_t dybs,
                              const uint8_t* __restrict__ am, int64_t abs_, T* __restrict__ dX, int64_t dxbs) {
  const int cv = g.C / VEC;
  const int64_t per = (int64_t)g.N * g.H * g.W * cv;
  const int64_t total = per * B;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / per);
    int64_t r = i - b * per;
    const int c = (int)(r % cv) * VEC; r /= cv;
    const int ix = (int)(r % g.W); r /= g.W;
    const int iy = (int)(r % g.H);
    const int n = (int)(r / g.H);
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    // windows containing (iy, ix): oy*s - p + ky = iy, 0 <= ky < k
    const int oy0 = max(0, (iy + g.p - g.k + g.s) / g.s), oy1 = min(g.Ho - 1, (iy + g.p) / g.s);
    const int ox0 = max(0, (ix + g.p - g.k + g.s) / g.s), ox1 = min(g.Wo - 1, (ix + g.p) / g.s);
    for (int oy = oy0; oy <= oy1; ++oy) {
      const int ky = iy + g.p - oy * g.s;
      if (ky < 0 || ky >= g.k) continue;
      for (int ox = ox0; ox <= ox1; ++ox) {
        const int kx = ix + g.p - ox * g.s;
        if (kx < 0 || kx >= g.k) continue;
        const int tap = ky * g.k + kx;
        const int64_t o = (((int64_t)n * g.Ho + oy) * g.Wo + ox) * g.C + c;
        const uint8_t* a = am + (int64_t)b * abs_ + o;
        float d[VEC];
        ld_vec<T, VEC>(dY + (int64_t)b * dybs + o, d);
#pragma unroll
        for (int v = 0; v < VEC; ++v)
          if (a[v] == tap) acc[v] += d[v];
      }
    }
    st_vec<T, VEC>(dX + (int64_t)b * dxbs + (((int64_t)n * g.H + iy) * g.W + ix) * g.C + c, acc);
  }
}

template <typename T, int VEC>
__global__ void k_avgpool_fwd(int B, int64_t N, int64_t HW, int64_t C, const T* __restrict__ X, int64_t xbs,
                              T* __restrict__ Y, int64_t ybs) {
  const int64_t cv = C / VEC;
  const int64_t per = N * cv, total = per * B;
  const float inv = 1.0f / (float)HW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / per);
    const int64_t r = i - b * per;
    const int64_t c = (r % cv) * VEC, n = r / cv;
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    const T* Xb = X + (int64_t)b * xbs + n * HW * C + c;
    for (int64_t q = 0; q < HW; ++q) {                 // fixed order
      float x[VEC];
      ld_vec<T, VEC>(Xb + q * C, x);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] += x[v];
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] *= inv;
    st_vec<T, VEC>(Y + (int64_t)b * ybs + n * C + c, acc);
  }
}

template <typename T, int VEC>
__global__ void k_avgpool_bwd(int B, int64_t N, int64_t HW, int64_t C, const T* __restrict__ dY, int64_t dybs,
                              T* __restrict__ dX, int64_t dxbs) {
  const int64_t cv = C / VEC;
  const int64_t per = N * HW * cv, total = per * B;
  const float inv = 1.0f / (float)HW;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / per);
    const int64_t r = i - b * per;
    const int64_t c = (r % cv) * VEC, nq = r / cv, n = nq / HW;
    float d[VEC];
    ld_vec<T, VEC>(dY + (int64_t)b * dybs + n * C + c, d);
#pragma unroll
    for (int v = 0; v < VEC; ++v) d[v] *= inv;
    st_vec<T, VEC>(dX + (int64_t)b * dxbs + nq * C + c, d);
  }
}

unsigned grid_for(int64_t total) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 16)); }

int pool_vec(hfta_dtype dt, int64_t C, std::initializer_list<const void*> ps, std::initializer_list<int64_t> strides) {
  const int vec = dt == HFTA_BF16 ? 8 : 4;
  if (C % vec) return 1;
  for (const void* p : ps) if (!aligned16(p)) return 1;
  for (int64_t s : strides) if (s % vec) return 1;
  return vec;
}

#define POOL_LAUNCH(KERNEL, vec, total, ...)                                                  \
  do {                                                                                       \
    const unsigned gr_ = grid_for((total) / (vec));                                          \
    if (dt == HFTA_F32) {                                                                    \
      using T = float;                                                                       \
      if (vec == 4) KERNEL<T, 4><<<gr_, 256, 0, s>>>(__VA_ARGS__);                           \
      else KERNEL<T, 1><<<gr_, 256, 0, s>>>(__VA_ARGS__);                                    \
    } else {                                                                                 \
      using T = __nv_bfloat16;                                                               \
      if (vec == 8) KERNEL<T, 8><<<gr_, 256, 0, s>>>(__VA_ARGS__);                           \
      else KERNEL<T, 1><<<gr_, 256, 0, s>>>(__VA_ARGS__);                                    \
    }                                                                                        \
  } while (0)

hfta_status pool_geo(int N, int H, int W, int C, int k, int stride, int pad, PoolGeo* g) {
  HFTA_REQUIRE(N >= 1 && H >= 1 && W >= 1 && C >= 1 && k >= 1 && k <= 15 && stride >= 1 && pad >= 0 && 2 * pad <= k,
               HFTA_ERR_SHAPE, "maxpool: N %d H %d W %d C %d k %d s %d p %d", N, H, W, C, k, stride, pad);
  g->N = N; g->H = H; g->W = W; g->C = C; g->k = k; g->s = stride; g->p = pad;
  g->Ho = (H + 2 * pad - k) / stride + 1;
  g->Wo = (W + 2 * pad - k) / stride + 1;
  HFTA_REQUIRE(g->Ho >= 1 && g->Wo >= 1, HFTA_ERR_SHAPE, "maxpool: empty output");
  return HFTA_OK;
}

}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" {

hfta_status hfta_maxpool2d_fwd(int B, int N, int H, int W, int C, int k, int stride, int pad, hfta_dtype dt,
                               hfta_in X, hfta_out Y, uint8_t* argmax, int64_t am_bstride, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  PoolGeo g;
  if (hfta_status st = pool_geo(N, H, W, C, k, stride, pad, &g)) return st;
  HFTA_REQUIRE(X.ptr && Y.ptr && argmax, HFTA_ERR_INVALID_VALUE, "maxpool_fwd: null argument");
  HFTA_REQUIRE(X.ld == C && Y.ld == C, HFTA_ERR_SHAPE, "maxpool_fwd: dense NHWC required (ld == C)");
  HFTA_REQUIRE((Y.bstride > 0 && am_bstride > 0) || B == 1, HFTA_ERR_SHAPE, "maxpool_fwd: output strides");
  cudaStream_t s = (cudaStream_t)stream;
  const int vec = pool_vec(dt, C, {X.ptr, Y.ptr}, {X.bstride, Y.bstride});
  const int64_t total = (int64_t)B * N * g.Ho * g.Wo * C;
  POOL_LAUNCH(k_maxpool_fwd, vec, total, B, g, (const T*)X.ptr, X.bstride, (T*)Y.ptr, Y.bstride, argmax, am_bstride);
  count_launches(1);
  return post_launch(s, "hfta_maxpool2d_fwd");
}

hfta_status hfta_maxpool2d_bwd(int B, int N, int H, int W, int C, int k, int stride, int pad, hfta_dtype dt,
                               hfta_in dY, const uint8_t* argmax, int64_t am_bstride, hfta_out dX,
                               hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  PoolGeo g;
  if (hfta_status st = pool_geo(N, H, W, C, k, stride, pad, &g)) return st;
  HFTA_REQUIRE(dY.ptr && dX.ptr && argmax, HFTA_ERR_INVALID_VALUE, "maxpool_bwd: null argument");
  HFTA_REQUIRE(dY.ld == C && dX.ld == C, HFTA_ERR_SHAPE, "maxpool_bwd: dense NHWC required (ld == C)");
  HFTA_REQUIRE(dX.bstride > 0 || B == 1, HFTA_ERR_SHAPE, "maxpool_bwd: dX.bstride must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  const int vec = pool_vec(dt, C, {dY.ptr, dX.ptr}, {dY.bstride, dX.bstride});
  const int64_t total = (int64_t)B * N * H * W * C;
  POOL_LAUNCH(k_maxpool_bwd, vec, total, B, g, (const T*)dY.ptr, dY.bstride, argmax, am_bstride, (T*)dX.ptr,
              dX.bstride);
  count_launches(1);
  return post_launch(s, "hfta_maxpool2d_bwd");
}

hfta_status hfta_avgpool2d_fwd(int B, int64_t N, int64_t HW, int64_t C, hfta_dtype dt, hfta_in X, hfta_out Y,
                               hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(N >= 1 && HW >= 1 && C >= 1, HFTA_ERR_SHAPE, "avgpool_fwd: N %lld HW %lld C %lld", (long long)N,
               (long long)HW, (long long)C);
  HFTA_REQUIRE(X.ptr && Y.ptr && X.ld == C && Y.ld == C, HFTA_ERR_SHAPE, "avgpool_fwd: dense [N][HW][C] -> [N][C]");
  HFTA_REQUIRE(Y.bstride > 0 || B == 1, HFTA_ERR_SHAPE, "avgpool_fwd: Y.bstride must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  const int vec = pool_vec(dt, C, {X.ptr, Y.ptr}, {X.bstride, Y.bstride});
  POOL_LAUNCH(k_avgpool_fwd, vec, (int64_t)B * N * C, B, N, HW, C, (const T*)X.ptr, X.bstride, (T*)Y.ptr, Y.bstride);
  count_launches(1);
  return post_launch(s, "hfta_avgpool2d_fwd");
}

hfta_status hfta_avgpool2d_bwd(int B, int64_t N, int64_t HW, int64_t C, hfta_dtype dt, hfta_in dY, hfta_out dX,
                               hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(N >= 1 && HW >= 1 && C >= 1, HFTA_ERR_SHAPE, "avgpool_bwd: bad shape");
  HFTA_REQUIRE(dY.ptr && dX.ptr && dY.ld == C && dX.ld == C, HFTA_ERR_SHAPE, "avgpool_bwd: dense layouts");
  HFTA_REQUIRE(dX.bstride > 0 || B == 1, HFTA_ERR_SHAPE, "avgpool_bwd: dX.bstride must be > 0");
  cudaStream_t s = (cudaStream_t)stream;
  const int vec = pool_vec(dt, C, {dY.ptr, dX.ptr}, {dY.bstride, dX.bstride});
  POOL_LAUNCH(k_avgpool_bwd, vec, (int64_t)B * N * HW * C, B, N, HW, C, (const T*)dY.ptr, dY.bstride, (T*)dX.ptr,
              dX.bstride);
  count_launches(1);
  return post_launch(s, "hfta_avgpool2d_bwd");
}

}  // extern "C"
