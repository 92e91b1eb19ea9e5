// gemm_simt.cu -- SIMT (FFMA) model-batched GEMM, fp32 accumulation.
// Used for the shapes the tensor-core path does not take: K < 16 (PointNet's
// xyz input layers, K = 3), N < 16 (STN fc3 N = 9, dgrad into xyz N = 3), and
// unaligned operands.  Those layers have arithmetic intensity ~1-3 flop/B, so
// they are HBM-bound and FFMA is not the limit.  Model index b = blockIdx.z,
// split-K index = blockIdx.y.
#include <type_traits>

#include "gemm.cuh"

namespace hfta {

namespace {
constexpr int BM = 128, BN = 128, BK = 16, NT = 256;

// Tile BM_ x BN_ with 256 threads, each owning a contiguous RM x RN block
// (vector shared-memory reads): 128 x 128 -> 16 x 16 threads of 8 x 8;
// 32 x 64 (per-sample FC layers, M = batch = 32: more CTAs per model) ->
// 8 x 32 threads of 4 x 2.  The next K slab is loaded into registers while
// the current one is multiplied (one-deep software pipeline).
template <typename Tin, typename Tout, bool AK, bool BKM, int BM_, int BN_, int BK>
__global__ void __launch_bounds__(NT) k_gemm_simt(GemmP p) {
  constexpr int TY = BM_ == 128 ? 16 : 8, TX = NT / TY;   // thread grid
  constexpr int RM = BM_ / TY, RN = BN_ / TX;             // outputs per thread
  constexpr int LA = (BM_ * BK) / NT, LB = (BN_ * BK) / NT;
  __shared__ __align__(16) float As[BK][BM_ + 4];
  __shared__ __align__(16) float Bs[BK][BN_ + 4];
  const int b = blockIdx.z;
  const int split = blockIdx.y;
  const int64_t tiles_n = (p.N + BN_ - 1) / BN_;
  const int64_t m0 = (blockIdx.x / tiles_n) * BM_;
  const int64_t n0 = (blockIdx.x % tiles_n) * BN_;
  const int64_t kbeg = (int64_t)split * p.k_chunk;
  const int64_t kend = min(p.K, kbeg + p.k_chunk);
  const Tin* A = reinterpret_cast<const Tin*>(p.A) + (int64_t)b * p.a_bs;
  const Tin* Bm = reinterpret_cast<const Tin*>(p.Bm) + (int64_t)b * p.b_bs;
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;

  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;

  float ra[LA], rb[LB];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = tid + i * NT;
      const int mm = AK ? e / BK : e % BM_, kk = AK ? e % BK : e / BM_;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[i] = (gm < p.M && gk < kend) ? ldf(AK ? A + gm * p.a_ld + gk : A + gk * p.a_ld + gm) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = tid + i * NT;
      const int nn = BKM ? e / BK : e % BN_, kk = BKM ? e % BK : e / BN_;
      const int64_t gn = n0 + nn, gk = k0 + kk;
      rb[i] = (gn < p.N && gk < kend) ? ldf(BKM ? Bm + gn * p.b_ld + gk : Bm + gk * p.b_ld + gn) : 0.f;
    }
  };
  if (kbeg < kend) load(kbeg);
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = tid + i * NT;
      As[AK ? e % BK : e / BM_][AK ? e / BK : e % BM_] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = tid + i * NT;
      Bs[BKM ? e % BK : e / BN_][BKM ? e / BK : e % BN_] = rb[i];
    }
    __syncthreads();
    if (k0 + BK < kend) load(k0 + BK);       // in flight during the FMAs below
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[RM], bb[RN];
#pragma unroll
      for (int i = 0; i < RM; i += 4) {
        const float4 t = *reinterpret_cast<const float4*>(&As[kk][ty * RM + i]);
        a[i] = t.x; a[i + 1] = t.y; a[i + 2] = t.z; a[i + 3] = t.w;
      }
      if constexpr (RN == 1) {
        bb[0] = Bs[kk][tx];
      } else if constexpr (RN % 4 == 0) {
#pragma unroll
        for (int j = 0; j < RN; j += 4) {
          const float4 t = *reinterpret_cast<const float4*>(&Bs[kk][tx * RN + j]);
          bb[j] = t.x; bb[j + 1] = t.y; bb[j + 2] = t.z; bb[j + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < RN; j += 2) {
          const float2 t = *reinterpret_cast<const float2*>(&Bs[kk][tx * RN + j]);
          bb[j] = t.x; bb[j + 1] = t.y;
        }
      }
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }

  if (p.splits > 1) {
    float* part = p.part + ((int64_t)split * p.B + b) * p.M * p.N;
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      const int64_t gm = m0 + ty * RM + i;
      if (gm >= p.M) continue;
#pragma unroll
      for (int j = 0; j < RN; ++j) {
        const int64_t gn = n0 + tx * RN + j;
        if (gn < p.N) part[gm * p.N + gn] = acc[i][j];
      }
    }
    return;
  }
  Tout* C = reinterpret_cast<Tout*>(p.C) + (int64_t)b * p.c_bs;
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int64_t gm = m0 + ty * RM + i;
    if (gm >= p.M) continue;
    const float* brow = p.bias ? p.bias + (int64_t)b * p.bias_bs + (p.bias_div > 0 ? (gm / p.bias_div) * p.bias_ld : 0) : nullptr;
    if constexpr (std::is_same<Tout, float>::value && RN % 4 == 0) {
      // contiguous RN outputs per thread: 16-B stores (full sectors) when possible
      const int64_t gn0 = n0 + tx * RN;
      Tout* c = C + gm * p.c_ld + gn0;
      if (!brow && !p.accumulate && gn0 + RN <= p.N && (reinterpret_cast<uintptr_t>(c) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < RN; j += 4)
          *reinterpret_cast<float4*>(c + j) = make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
        continue;
      }
    }
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int64_t gn = n0 + tx * RN + j;
      if (gn >= p.N) continue;
      float v = acc[i][j];
      if (brow) v += brow[gn];
      Tout* c = C + gm * p.c_ld + gn;
      if (p.accumulate) v += ldf(c);
      stf(c, v);
    }
  }
}

__global__ void k_splitk_reduce(GemmP p) {
  const int b = blockIdx.y;
  const int64_t MN = p.M * p.N;
  float* C = reinterpret_cast<float*>(p.C) + (int64_t)b * p.c_bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = e / p.N, n = e % p.N;
    float v = 0.f;
    for (int s = 0; s < p.splits; ++s) v += p.part[((int64_t)s * p.B + b) * MN + e];   // fixed order
    float* c = C + m * p.c_ld + n;
    *c = p.accumulate ? *c + v : v;
  }
}

template <typename Tin, typename Tout, int BM_, int BN_, int BK_>
void launch_bm(const GemmP& p, dim3 grid, cudaStream_t s) {
  if (p.a_kmajor && p.b_kmajor) k_gemm_simt<Tin, Tout, true, true, BM_, BN_, BK_><<<grid, NT, 0, s>>>(p);
  else if (p.a_kmajor) k_gemm_simt<Tin, Tout, true, false, BM_, BN_, BK_><<<grid, NT, 0, s>>>(p);
  else if (p.b_kmajor) k_gemm_simt<Tin, Tout, false, true, BM_, BN_, BK_><<<grid, NT, 0, s>>>(p);
  else k_gemm_simt<Tin, Tout, false, false, BM_, BN_, BK_><<<grid, NT, 0, s>>>(p);
}
// M <= 32 (per-sample FC layers): 32 x 64 tiles (measured best of 32x32x32,
// 32x64x16 at B = 64: these layers are load-latency bound).
template <typename Tin, typename Tout>
void launch(const GemmP& p, dim3 grid, cudaStream_t s) {
  if (p.M <= 32) launch_bm<Tin, Tout, 32, 64, 16>(p, grid, s);
  else launch_bm<Tin, Tout, 128, 128, BK>(p, grid, s);
}
}  // namespace

hfta_status gemm_simt(const GemmP& p, hfta_dtype dt_in, bool out_f32, cudaStream_t s) {
  const int bm = p.M <= 32 ? 32 : BM, bn = p.M <= 32 ? 64 : BN;
  dim3 grid((unsigned)(cdiv(p.M, bm) * cdiv(p.N, bn)), (unsigned)p.splits, (unsigned)p.B);
  if (dt_in == HFTA_F32) launch<float, float>(p, grid, s);
  else if (out_f32) launch<__nv_bfloat16, float>(p, grid, s);
  else launch<__nv_bfloat16, __nv_bfloat16>(p, grid, s);
  count_launches(1);
  return post_launch(s, "gemm_simt");
}

__global__ void k_colsum_reduce(GemmP p) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)p.B * p.M) return;
  const int64_t b = i / p.M, m = i % p.M;
  float v = 0.f;
  for (int s = 0; s < p.splits; ++s) v += p.colsum_part[((int64_t)s * p.B + b) * p.M + m];   // fixed order
  float* o = p.colsum + b * p.colsum_bs + m;
  *o = p.colsum_acc ? *o + v : v;
}

hfta_status colsum_reduce(const GemmP& p, cudaStream_t s) {
  k_colsum_reduce<<<(unsigned)cdiv((int64_t)p.B * p.M, 256), 256, 0, s>>>(p);
  count_launches(1);
  return post_launch(s, "colsum_reduce");
}

hfta_status splitk_reduce(const GemmP& p, cudaStream_t s) {
  int64_t MN = p.M * p.N;
  dim3 grid((unsigned)std::min<int64_t>(cdiv(MN, 256), 4096), (unsigned)p.B);
  k_splitk_reduce<<<grid, 256, 0, s>>>(p);
  count_launches(1);
  return post_launch(s, "splitk_reduce");
}

}  // namespace hfta
