// common.cuh -- shared device/host helpers of libhfta (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <type_traits>
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
// Raise a kernel's dynamic shared-memory limit once per (kernel, device):
// mutex-protected registry (safe from several host threads and devices).
void set_max_smem(const void* kern, size_t bytes);
template <typename K_> inline void ensure_smem(K_* kern, size_t bytes) {
  set_max_smem(reinterpret_cast<const void*>(kern), bytes);
}

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

// bf16x2 <-> 2 x fp32 in registers (bit operations: no byte-addressed
// temporaries, which the compiler would place in local memory).
__device__ __forceinline__ void unpack_bf2(uint32_t w, float& lo, float& hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xffff0000u);
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Vector of VEC elements of T loaded/stored as one (or a few) wide accesses.
template <typename T, int VEC>
__device__ __forceinline__ void ld_vec(const T* p, float (&v)[VEC]) {
  if constexpr (VEC == 1) {
    v[0] = Cvt<T>::to_f(*p);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value && VEC == 8) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    unpack_bf2(u.x, v[0], v[1]); unpack_bf2(u.y, v[2], v[3]); unpack_bf2(u.z, v[4], v[5]); unpack_bf2(u.w, v[6], v[7]);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value && VEC == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    unpack_bf2(u.x, v[0], v[1]); unpack_bf2(u.y, v[2], v[3]);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value && VEC == 2) {
    unpack_bf2(*reinterpret_cast<const uint32_t*>(p), v[0], v[1]);
  } else if constexpr (std::is_same<T, float>::value && VEC == 4) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  } else if constexpr (std::is_same<T, float>::value && VEC == 2) {
    const float2 u = *reinterpret_cast<const float2*>(p);
    v[0] = u.x; v[1] = u.y;
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = Cvt<T>::to_f(p[i]);
  }
}

template <typename T, int VEC>
__device__ __forceinline__ void st_vec(T* p, const float (&v)[VEC]) {
  if constexpr (VEC == 1) {
    *p = Cvt<T>::from_f(v[0]);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value && VEC == 8) {
    *reinterpret_cast<uint4*>(p) =
        make_uint4(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]), pack_bf2(v[4], v[5]), pack_bf2(v[6], v[7]));
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value && VEC == 4) {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf2(v[0], v[1]), pack_bf2(v[2], v[3]));
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value && VEC == 2) {
    *reinterpret_cast<uint32_t*>(p) = pack_bf2(v[0], v[1]);
  } else if constexpr (std::is_same<T, float>::value && VEC == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else if constexpr (std::is_same<T, float>::value && VEC == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) p[i] = Cvt<T>::from_f(v[i]);
  }
}

// ---- cp.async (LDGSTS) row pipelines: loads in flight without registers --
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// 16 B of shared memory (8 bf16 or 4 fp32) -> VEC floats
template <typename T, int VEC>
__device__ __forceinline__ void ld_vec_smem(uint32_t saddr, float (&v)[VEC]) {
  static_assert(VEC * sizeof(T) == 16, "16-byte vectors only");
  uint4 u;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(saddr));
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    unpack_bf2(u.x, v[0], v[1]); unpack_bf2(u.y, v[2], v[3]); unpack_bf2(u.z, v[4], v[5]); unpack_bf2(u.w, v[6], v[7]);
  } else {
    v[0] = __uint_as_float(u.x); v[1] = __uint_as_float(u.y); v[2] = __uint_as_float(u.z); v[3] = __uint_as_float(u.w);
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
