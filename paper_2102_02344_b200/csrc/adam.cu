// adam.cu -- fused Adam over the flat per-model parameter arena (K7).
// "The scalar-vector operations (e.g., multiplying a learning
// rate under tuning with the gradients) ... are now replaced by broadcasted
// vector-vector operations (e.g., multiplying a vector of learning rates with
// the concatenated gradients of all models)".  One launch updates every
// parameter of every model; element j of model b reads hyper-parameters [b].
// Form: PyTorch 1.6 Adam (reading R7).  HBM-bound: 28 B/param (p, g, m, v
// read; p, m, v written), +2 B with the bf16 shadow.
#include "common.cuh"

namespace hfta {
namespace {

template <int VEC, bool SHADOW>
__global__ void __launch_bounds__(256) k_adam(int B, int64_t P, float* __restrict__ param,
                                              const float* __restrict__ grad, float* __restrict__ m1,
                                              float* __restrict__ m2, int64_t bs, const float* __restrict__ lr,
                                              const float* __restrict__ beta1, const float* __restrict__ beta2,
                                              const float* __restrict__ eps, const float* __restrict__ wd,
                                              const int64_t* __restrict__ step, __nv_bfloat16* __restrict__ shadow,
                                              int64_t sbs) {
  const int b = blockIdx.y;
  const double t = (double)*step;
  const float b1 = beta1[b], b2 = beta2[b], e = eps[b], w = wd[b];
  // bias corrections in double from fp32 hyper-parameters, then fp32 (as torch computes them on the host)
  const float bc1 = (float)(1.0 - pow((double)b1, t));
  const float rbc2 = (float)(1.0 / sqrt(1.0 - pow((double)b2, t)));
  const float step_size = lr[b] / bc1;
  float* p = param + (int64_t)b * bs;
  const float* g = grad + (int64_t)b * bs;
  float* m = m1 + (int64_t)b * bs;
  float* v = m2 + (int64_t)b * bs;
  const int64_t nvec = P / VEC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    float pp[VEC], gg[VEC], mm[VEC], vv[VEC];
    ld_vec<float, VEC>(p + i * VEC, pp);
    ld_vec<float, VEC>(g + i * VEC, gg);
    ld_vec<float, VEC>(m + i * VEC, mm);
    ld_vec<float, VEC>(v + i * VEC, vv);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      float gk = fmaf(w, pp[k], gg[k]);
      mm[k] = fmaf(b1, mm[k], (1.f - b1) * gk);
      vv[k] = fmaf(b2, vv[k], (1.f - b2) * gk * gk);
      float denom = sqrtf(vv[k]) * rbc2 + e;
      pp[k] = pp[k] - step_size * (mm[k] / denom);
    }
    st_vec<float, VEC>(p + i * VEC, pp);
    st_vec<float, VEC>(m + i * VEC, mm);
    st_vec<float, VEC>(v + i * VEC, vv);
    if (SHADOW) st_vec<__nv_bfloat16, VEC>(shadow + (int64_t)b * sbs + i * VEC, pp);
  }
}

}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" hfta_status hfta_fused_adam(int B, int64_t P, float* param, const float* grad, float* exp_avg,
                                       float* exp_avg_sq, int64_t bstride, const float* lr, const float* beta1,
                                       const float* beta2, const float* eps, const float* weight_decay,
                                       const int64_t* step, void* param_bf16, int64_t bf16_bstride,
                                       hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(P >= 1 && param && grad && exp_avg && exp_avg_sq && lr && beta1 && beta2 && eps && weight_decay && step,
               HFTA_ERR_INVALID_VALUE, "fused_adam: null argument or P < 1");
  HFTA_REQUIRE(bstride >= P || B == 1, HFTA_ERR_SHAPE, "fused_adam: bstride %lld < P %lld", (long long)bstride,
               (long long)P);
  cudaStream_t s = (cudaStream_t)stream;
  bool v4 = P % 4 == 0 && bstride % 4 == 0 && aligned16(param) && aligned16(grad) && aligned16(exp_avg) &&
            aligned16(exp_avg_sq) && (!param_bf16 || (bf16_bstride % 4 == 0 && (reinterpret_cast<uintptr_t>(param_bf16) & 7) == 0));
  int64_t nvec = v4 ? P / 4 : P;
  int64_t per_model_blocks = std::max<int64_t>(1, std::min<int64_t>(cdiv(nvec, 256), cdiv(4 * (int64_t)num_sms(), B) * 4));
  dim3 grid((unsigned)per_model_blocks, B);
  __nv_bfloat16* sh = reinterpret_cast<__nv_bfloat16*>(param_bf16);
  if (v4) {
    if (sh) k_adam<4, true><<<grid, 256, 0, s>>>(B, P, param, grad, exp_avg, exp_avg_sq, bstride, lr, beta1, beta2, eps, weight_decay, step, sh, bf16_bstride);
    else k_adam<4, false><<<grid, 256, 0, s>>>(B, P, param, grad, exp_avg, exp_avg_sq, bstride, lr, beta1, beta2, eps, weight_decay, step, sh, bf16_bstride);
  } else {
    if (sh) k_adam<1, true><<<grid, 256, 0, s>>>(B, P, param, grad, exp_avg, exp_avg_sq, bstride, lr, beta1, beta2, eps, weight_decay, step, sh, bf16_bstride);
    else k_adam<1, false><<<grid, 256, 0, s>>>(B, P, param, grad, exp_avg, exp_avg_sq, bstride, lr, beta1, beta2, eps, weight_decay, step, sh, bf16_bstride);
  }
  count_launches(1);
  return post_launch(s, "hfta_fused_adam");
}
