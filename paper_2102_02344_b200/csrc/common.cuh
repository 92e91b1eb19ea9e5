// common.cuh -- shared device/host helpers of libhfta (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/hfta.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libhfta is written for sm_100a (B200) only"
#endif

namespace hfta {

// ------------------------------------------------------------- host side --
hfta_status fail(hfta_status code, const char* fmt, ...);
hfta_status check_init();
int num_sms();
void count_launches(uint64_t n);
// Call after every launch sequence: checks the launch status, honours HFTA_SYNC.
hfta_status post_launch(cudaStream_t s, const char* what);

inline size_t dsize(hfta_dtype dt) { return dt == HFTA_BF16 ? 2 : 4; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

#define HFTA_REQUIRE(cond, code, ...) \
  do { if (!(cond)) return ::hfta::fail(code, __VA_ARGS__); } while (0)

#define HFTA_CHECK_B(B) HFTA_REQUIRE((B) >= 1, HFTA_ERR_INVALID_VALUE, "B must be >= 1 (got %d)", (int)(B))

// ----------------------------------------------------------- device side --
template <typename T> struct Cvt;
template <> struct Cvt<float> {
  __device__ __forceinline__ static float to_f(float v) { return v; }
  __device__ __forceinline__ static float from_f(float v) { return v; }
};
template <> struct Cvt<__nv_bfloat16> {
  __device__ __forceinline__ static float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

template <typename T> __device__ __forceinline__ float ldf(const T* p) { return Cvt<T>::to_f(*p); }
template <typename T> __device__ __forceinline__ void stf(T* p, float v) { *p = Cvt<T>::from_f(v); }

// Vector of VEC elements of T loaded/stored as one (or a few) wide accesses.
template <typename T, int VEC>
__device__ __forceinline__ void ld_vec(const T* p, float (&v)[VEC]) {
  if constexpr (VEC == 1) {
    v[0] = Cvt<T>::to_f(*p);
  } else if constexpr (sizeof(T) * VEC == 16) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = Cvt<T>::to_f(e[i]);
  } else if constexpr (sizeof(T) * VEC == 8) {
    uint2 u = *reinterpret_cast<const uint2*>(p);
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = Cvt<T>::to_f(e[i]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = Cvt<T>::to_f(p[i]);
  }
}

template <typename T, int VEC>
__device__ __forceinline__ void st_vec(T* p, const float (&v)[VEC]) {
  if constexpr (VEC == 1) {
    *p = Cvt<T>::from_f(v[0]);
  } else if constexpr (sizeof(T) * VEC == 16) {
    uint4 u;
    T* e = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) e[i] = Cvt<T>::from_f(v[i]);
    *reinterpret_cast<uint4*>(p) = u;
  } else if constexpr (sizeof(T) * VEC == 8) {
    uint2 u;
    T* e = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < VEC; ++i) e[i] = Cvt<T>::from_f(v[i]);
    *reinterpret_cast<uint2*>(p) = u;
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) p[i] = Cvt<T>::from_f(v[i]);
  }
}

__device__ __forceinline__ float act_fwd(float z, int act, float alpha) {
  if (act == HFTA_ACT_RELU) return z > 0.f ? z : 0.f;
  if (act == HFTA_ACT_LEAKY_RELU) return z > 0.f ? z : alpha * z;
  return z;
}
// derivative of act at pre-activation z
__device__ __forceinline__ float act_grad(float z, int act, float alpha) {
  if (act == HFTA_ACT_RELU) return z > 0.f ? 1.f : 0.f;
  if (act == HFTA_ACT_LEAKY_RELU) return z > 0.f ? 1.f : alpha;
  return 1.f;
}

}  // namespace hfta
