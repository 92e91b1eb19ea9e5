// ftrans.cu -- PointNet feature transform (STNkd head output -> 64 x 64
// per-cloud transform) and its orthogonality regularizer (the
// "Feature Transformation" hyper-parameter of the PointNet tuning space;
// reading R30: the cited implementation's loss += 0.001 * mean_n
// ||T_n T_n^T - I||_F).
//
//   hfta_feature_transform_make: Tt[b][n] = (F3[b][n] viewed K x K + I)^T in
//     the compute dtype -- the K-major weight operand of the per-cloud
//     transform x' = x T, run as a fused Linear over B*N "models".
//   hfta_feature_transform_reg: per (b, n) with T = F3 + I, A = T T^T - I,
//     f = ||A||_F: dF3[i K + j] = dTt[j][i] + w * 2 (A T)[i][j] / (N f), and
//     loss[b] += w * mean_n f (fixed-order sums), mean_loss refreshed.
#include "common.cuh"

namespace hfta {
namespace {

constexpr int KMAXT = 64;

template <typename T>
__global__ void k_ft_make(int64_t N, int K, const float* __restrict__ F3, int64_t fbs, T* __restrict__ Tt, int64_t tbs) {
  const int b = blockIdx.y;
  const int64_t total = N * K * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / (K * K);
    const int r = (int)(e % (K * K)), j = r / K, i = r % K;        // Tt[n][j][i] = T[n][i][j]
    const float v = F3[(int64_t)b * fbs + n * K * K + (int64_t)i * K + j] + (i == j ? 1.f : 0.f);
    stf(Tt + (int64_t)b * tbs + e, v);
  }
}

__global__ void __launch_bounds__(256) k_ft_reg(int64_t N, int K, const float* __restrict__ F3, int64_t fbs,
                                                const float* __restrict__ dTt, int64_t dtbs, float w,
                                                float* __restrict__ dF3, int64_t dfbs, float* __restrict__ fn) {
  __shared__ float Ts[KMAXT][KMAXT + 1], As[KMAXT][KMAXT + 1];
  __shared__ float red[256];
  const int64_t bn = blockIdx.x;                        // (b, n) flattened
  const int64_t b = bn / N, n = bn % N;
  const float* f3 = F3 + b * fbs + n * K * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int i = e / K, j = e % K;
    Ts[i][j] = f3[e] + (i == j ? 1.f : 0.f);
  }
  __syncthreads();
  float s2 = 0.f;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {      // A = T T^T - I
    const int i = e / K, j = e % K;
    float a = 0.f;
    for (int l = 0; l < K; ++l) a = fmaf(Ts[i][l], Ts[j][l], a);
    a -= (i == j ? 1.f : 0.f);
    As[i][j] = a;
    s2 = fmaf(a, a, s2);
  }
  red[threadIdx.x] = s2;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const float f = sqrtf(red[0]);
  const float c = f > 0.f ? 2.f * w / ((float)N * f) : 0.f;
  const float* dt = dTt + b * dtbs + n * K * K;
  float* df = dF3 + b * dfbs + n * K * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {      // dF3 = dTt^T + c (A T)
    const int i = e / K, j = e % K;
    float at = 0.f;
    for (int l = 0; l < K; ++l) at = fmaf(As[i][l], Ts[l][j], at);
    df[e] = dt[(int64_t)j * K + i] + c * at;
  }
  if (threadIdx.x == 0) fn[bn] = f;
}

// loss[b] += w * (1/N) sum_n f[b][n] (fixed order), then mean_loss = (1/B) sum_b loss[b]
__global__ void k_ft_reg_fin(int B, int64_t N, float w, const float* __restrict__ fn, float* __restrict__ loss,
                             float* __restrict__ mean_loss) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int b = warp; b < B; b += nw) {
    double s = 0.0;
    for (int64_t n = lane; n < N; n += 32) s += fn[(int64_t)b * N + n];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) loss[b] = (float)((double)loss[b] + (double)w * s / (double)N);
  }
  __syncthreads();
  if (threadIdx.x == 0 && mean_loss) {
    double tot = 0.0;
    for (int b = 0; b < B; ++b) tot += loss[b];
    *mean_loss = (float)(tot / B);
  }
}

}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" {

hfta_status hfta_feature_transform_make(int B, int64_t N, int64_t K, hfta_dtype dt, const float* F3,
                                        int64_t f_bstride, hfta_out Tt, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(F3 && Tt.ptr && N >= 1 && K >= 1 && K <= KMAXT, HFTA_ERR_INVALID_VALUE,
               "feature_transform_make: F3/Tt required, 1 <= K <= %d (K = %lld)", KMAXT, (long long)K);
  HFTA_REQUIRE(dt == HFTA_F32 || dt == HFTA_BF16, HFTA_ERR_UNSUPPORTED, "feature_transform_make: dtype");
  HFTA_REQUIRE(Tt.bstride >= N * K * K || B == 1, HFTA_ERR_SHAPE, "feature_transform_make: Tt.bstride");
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)std::min<int64_t>(cdiv(N * K * K, 256), 1024), (unsigned)B);
  if (dt == HFTA_F32) k_ft_make<float><<<grid, 256, 0, s>>>(N, (int)K, F3, f_bstride, (float*)Tt.ptr, Tt.bstride);
  else k_ft_make<__nv_bfloat16><<<grid, 256, 0, s>>>(N, (int)K, F3, f_bstride, (__nv_bfloat16*)Tt.ptr, Tt.bstride);
  count_launches(1);
  return post_launch(s, "hfta_feature_transform_make");
}

size_t hfta_feature_transform_reg_workspace(int B, int64_t N) {
  return (B < 1 || N < 1) ? 0 : align_up((size_t)B * N * sizeof(float), 256);
}

hfta_status hfta_feature_transform_reg(int B, int64_t N, int64_t K, const float* F3, int64_t f_bstride,
                                       const float* dTt, int64_t dt_bstride, float weight, float* dF3,
                                       int64_t df_bstride, float* loss, float* mean_loss, void* ws, size_t ws_bytes,
                                       hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(F3 && dTt && dF3 && loss && N >= 1 && K >= 1 && K <= KMAXT, HFTA_ERR_INVALID_VALUE,
               "feature_transform_reg: F3, dTt, dF3, loss required, 1 <= K <= %d", KMAXT);
  HFTA_REQUIRE(ws && ws_bytes >= hfta_feature_transform_reg_workspace(B, N), HFTA_ERR_WORKSPACE,
               "feature_transform_reg: workspace");
  cudaStream_t s = (cudaStream_t)stream;
  float* fn = reinterpret_cast<float*>(ws);
  k_ft_reg<<<(unsigned)((int64_t)B * N), 256, 0, s>>>(N, (int)K, F3, f_bstride, dTt, dt_bstride, weight, dF3,
                                                     df_bstride, fn);
  k_ft_reg_fin<<<1, 1024, 0, s>>>(B, N, weight, fn, loss, mean_loss);
  count_launches(2);
  return post_launch(s, "hfta_feature_transform_reg");
}

}  // extern "C"
