// gemm_simt.cu -- SIMT (FFMA) model-batched GEMM, fp32 accumulation.
// Used for the shapes the tensor-core path does not take: K < 16 (PointNet's
// xyz input layers, K = 3), N < 16 (STN fc3 N = 9, dgrad into xyz N = 3), and
// unaligned operands.  Those layers have arithmetic intensity ~1-3 flop/B, so
// they are HBM-bound and FFMA is not the limit.  Model index b = blockIdx.z,
// split-K index = blockIdx.y.
#include "gemm.cuh"

namespace hfta {

namespace {
constexpr int BM = 128, BN = 128, BK = 16, NT = 256;

// Tile BM_ x 128 with 256 threads: BM_ = 128 -> 16 x 16 threads of 8 x 8 outputs;
// BM_ = 32 (per-sample FC layers, M = batch = 32) -> 8 x 32 threads of 4 x 4.
template <typename Tin, typename Tout, bool AK, bool BKM, int BM_>
__global__ void __launch_bounds__(NT) k_gemm_simt(GemmP p) {
  constexpr int TY = BM_ == 128 ? 16 : 8, TX = NT / TY;   // thread grid
  constexpr int RM = BM_ / TY, RN = BN / TX;               // outputs per thread
  __shared__ float As[BK][BM_ + 4];
  __shared__ float Bs[BK][BN + 4];
  const int b = blockIdx.z;
  const int split = blockIdx.y;
  const int64_t tiles_n = (p.N + BN - 1) / BN;
  const int64_t m0 = (blockIdx.x / tiles_n) * BM_;
  const int64_t n0 = (blockIdx.x % tiles_n) * BN;
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

  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
    for (int i = 0; i < (BM_ * BK) / NT; ++i) {
      int e = tid + i * NT;
      int mm, kk;
      if (AK) { mm = e / BK; kk = e % BK; } else { mm = e % BM_; kk = e / BM_; }
      int64_t gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < p.M && gk < kend) v = ldf(AK ? A + gm * p.a_ld + gk : A + gk * p.a_ld + gm);
      As[kk][mm] = v;
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / NT; ++i) {
      int e = tid + i * NT;
      int nn, kk;
      if (BKM) { nn = e / BK; kk = e % BK; } else { nn = e % BN; kk = e / BN; }
      int64_t gn = n0 + nn, gk = k0 + kk;
      float v = 0.f;
      if (gn < p.N && gk < kend) v = ldf(BKM ? Bm + gn * p.b_ld + gk : Bm + gk * p.b_ld + gn);
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[RM], bb[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) a[i] = As[kk][ty + TY * i];
#pragma unroll
      for (int j = 0; j < RN; ++j) bb[j] = Bs[kk][tx + TX * j];
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
      int64_t gm = m0 + ty + TY * i;
      if (gm >= p.M) continue;
#pragma unroll
      for (int j = 0; j < RN; ++j) {
        int64_t gn = n0 + tx + TX * j;
        if (gn < p.N) part[gm * p.N + gn] = acc[i][j];
      }
    }
    return;
  }
  Tout* C = reinterpret_cast<Tout*>(p.C) + (int64_t)b * p.c_bs;
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    int64_t gm = m0 + ty + TY * i;
    if (gm >= p.M) continue;
    const float* brow = p.bias ? p.bias + (int64_t)b * p.bias_bs + (p.bias_div > 0 ? (gm / p.bias_div) * p.bias_ld : 0) : nullptr;
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      int64_t gn = n0 + tx + TX * j;
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

template <typename Tin, typename Tout, int BM_>
void launch_bm(const GemmP& p, dim3 grid, cudaStream_t s) {
  if (p.a_kmajor && p.b_kmajor) k_gemm_simt<Tin, Tout, true, true, BM_><<<grid, NT, 0, s>>>(p);
  else if (p.a_kmajor) k_gemm_simt<Tin, Tout, true, false, BM_><<<grid, NT, 0, s>>>(p);
  else if (p.b_kmajor) k_gemm_simt<Tin, Tout, false, true, BM_><<<grid, NT, 0, s>>>(p);
  else k_gemm_simt<Tin, Tout, false, false, BM_><<<grid, NT, 0, s>>>(p);
}
template <typename Tin, typename Tout>
void launch(const GemmP& p, dim3 grid, cudaStream_t s) {
  if (p.M <= 32) launch_bm<Tin, Tout, 32>(p, grid, s);
  else launch_bm<Tin, Tout, 128>(p, grid, s);
}
}  // namespace

hfta_status gemm_simt(const GemmP& p, hfta_dtype dt_in, bool out_f32, cudaStream_t s) {
  const int bm = p.M <= 32 ? 32 : BM;
  dim3 grid((unsigned)(cdiv(p.M, bm) * cdiv(p.N, BN)), (unsigned)p.splits, (unsigned)p.B);
  if (dt_in == HFTA_F32) launch<float, float>(p, grid, s);
  else if (out_f32) launch<__nv_bfloat16, float>(p, grid, s);
  else launch<__nv_bfloat16, __nv_bfloat16>(p, grid, s);
  count_launches(1);
  return post_launch(s, "gemm_simt");
}

hfta_status splitk_reduce(const GemmP& p, cudaStream_t s) {
  int64_t MN = p.M * p.N;
  dim3 grid((unsigned)std::min<int64_t>(cdiv(MN, 256), 4096), (unsigned)p.B);
  k_splitk_reduce<<<grid, 256, 0, s>>>(p);
  count_launches(1);
  return post_launch(s, "splitk_reduce");
}

}  // namespace hfta
