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

// Fused SGD (+momentum / dampening / Nesterov), PyTorch-1.6 form: the momentum
// buffer is set to d_p on step 1.  16 B/param read+write without momentum.
template <int VEC, bool SHADOW>
__global__ void __launch_bounds__(256) k_sgd(int64_t P, float* __restrict__ param, const float* __restrict__ grad,
                                             float* __restrict__ buf, int64_t bs, const float* __restrict__ lr,
                                             const float* __restrict__ mom, const float* __restrict__ damp,
                                             const float* __restrict__ wd, int nesterov,
                                             const int64_t* __restrict__ step, __nv_bfloat16* __restrict__ shadow,
                                             int64_t sbs) {
  const int b = blockIdx.y;
  const bool first = *step <= 1;
  const float l = lr[b], mu = mom[b], dm = damp[b], w = wd[b];
  float* p = param + (int64_t)b * bs;
  const float* g = grad + (int64_t)b * bs;
  float* m = buf ? buf + (int64_t)b * bs : nullptr;
  const int64_t nvec = P / VEC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    float pp[VEC], gg[VEC], mm[VEC];
    ld_vec<float, VEC>(p + i * VEC, pp);
    ld_vec<float, VEC>(g + i * VEC, gg);
    if (m && mu != 0.f && !first) ld_vec<float, VEC>(m + i * VEC, mm);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      float d = fmaf(w, pp[k], gg[k]);
      if (m && mu != 0.f) {
        mm[k] = first ? d : fmaf(mu, mm[k], (1.f - dm) * d);
        d = nesterov ? fmaf(mu, mm[k], d) : mm[k];
      }
      pp[k] = fmaf(-l, d, pp[k]);
    }
    st_vec<float, VEC>(p + i * VEC, pp);
    if (m && mu != 0.f) st_vec<float, VEC>(m + i * VEC, mm);
    if (SHADOW) st_vec<__nv_bfloat16, VEC>(shadow + (int64_t)b * sbs + i * VEC, pp);
  }
}

// Fused Adadelta, PyTorch-1.6 form.  28 B/param.
template <int VEC, bool SHADOW>
__global__ void __launch_bounds__(256) k_adadelta(int64_t P, float* __restrict__ param, const float* __restrict__ grad,
                                                  float* __restrict__ sq, float* __restrict__ acc, int64_t bs,
                                                  const float* __restrict__ lr, const float* __restrict__ rho,
                                                  const float* __restrict__ eps, const float* __restrict__ wd,
                                                  __nv_bfloat16* __restrict__ shadow, int64_t sbs) {
  const int b = blockIdx.y;
  const float l = lr[b], r = rho[b], e = eps[b], w = wd[b];
  float* p = param + (int64_t)b * bs;
  const float* g = grad + (int64_t)b * bs;
  float* s2 = sq + (int64_t)b * bs;
  float* a2 = acc + (int64_t)b * bs;
  const int64_t nvec = P / VEC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
    float pp[VEC], gg[VEC], ss[VEC], aa[VEC];
    ld_vec<float, VEC>(p + i * VEC, pp);
    ld_vec<float, VEC>(g + i * VEC, gg);
    ld_vec<float, VEC>(s2 + i * VEC, ss);
    ld_vec<float, VEC>(a2 + i * VEC, aa);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const float gk = fmaf(w, pp[k], gg[k]);
      ss[k] = fmaf(r, ss[k], (1.f - r) * gk * gk);
      const float delta = sqrtf(aa[k] + e) / sqrtf(ss[k] + e) * gk;
      aa[k] = fmaf(r, aa[k], (1.f - r) * delta * delta);
      pp[k] = fmaf(-l, delta, pp[k]);
    }
    st_vec<float, VEC>(p + i * VEC, pp);
    st_vec<float, VEC>(s2 + i * VEC, ss);
    st_vec<float, VEC>(a2 + i * VEC, aa);
    if (SHADOW) st_vec<__nv_bfloat16, VEC>(shadow + (int64_t)b * sbs + i * VEC, pp);
  }
}

__global__ void k_steplr(int B, const float* __restrict__ lr0, const float* __restrict__ gamma,
                         const int32_t* __restrict__ period, int64_t epoch, float* __restrict__ lr) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) lr[b] = (float)((double)lr0[b] * pow((double)gamma[b], (double)(epoch / period[b])));
}

bool opt_v4(int64_t P, int64_t bs, const void* a, const void* b, const void* c, const void* d, const void* sh,
            int64_t sbs) {
  return P % 4 == 0 && bs % 4 == 0 && aligned16(a) && aligned16(b) && (!c || aligned16(c)) && (!d || aligned16(d)) &&
         (!sh || (sbs % 4 == 0 && (reinterpret_cast<uintptr_t>(sh) & 7) == 0));
}

dim3 opt_grid(int B, int64_t P, bool v4) {
  int64_t nvec = v4 ? P / 4 : P;
  int64_t per = std::max<int64_t>(1, std::min<int64_t>(cdiv(nvec, 256), cdiv(4 * (int64_t)num_sms(), B) * 4));
  return dim3((unsigned)per, B);
}

}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" hfta_status hfta_fused_sgd(int B, int64_t P, float* param, const float* grad, float* momentum_buf,
                                      int64_t bstride, const float* lr, const float* momentum, const float* dampening,
                                      const float* weight_decay, int nesterov, const int64_t* step, void* param_bf16,
                                      int64_t bf16_bstride, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(P >= 1 && param && grad && lr && momentum && dampening && weight_decay && step,
               HFTA_ERR_INVALID_VALUE, "fused_sgd: null argument or P < 1");
  HFTA_REQUIRE(bstride >= P || B == 1, HFTA_ERR_SHAPE, "fused_sgd: bstride < P");
  cudaStream_t s = (cudaStream_t)stream;
  auto* sh = reinterpret_cast<__nv_bfloat16*>(param_bf16);
  const bool v4 = opt_v4(P, bstride, param, grad, momentum_buf, nullptr, sh, bf16_bstride);
  dim3 grid = opt_grid(B, P, v4);
#define SGD(V, S) k_sgd<V, S><<<grid, 256, 0, s>>>(P, param, grad, momentum_buf, bstride, lr, momentum, dampening, \
                                                   weight_decay, nesterov, step, sh, bf16_bstride)
  if (v4) { if (sh) SGD(4, true); else SGD(4, false); }
  else { if (sh) SGD(1, true); else SGD(1, false); }
#undef SGD
  count_launches(1);
  return post_launch(s, "hfta_fused_sgd");
}

extern "C" hfta_status hfta_fused_adadelta(int B, int64_t P, float* param, const float* grad, float* square_avg,
                                           float* acc_delta, int64_t bstride, const float* lr, const float* rho,
                                           const float* eps, const float* weight_decay, void* param_bf16,
                                           int64_t bf16_bstride, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(P >= 1 && param && grad && square_avg && acc_delta && lr && rho && eps && weight_decay,
               HFTA_ERR_INVALID_VALUE, "fused_adadelta: null argument or P < 1");
  HFTA_REQUIRE(bstride >= P || B == 1, HFTA_ERR_SHAPE, "fused_adadelta: bstride < P");
  cudaStream_t s = (cudaStream_t)stream;
  auto* sh = reinterpret_cast<__nv_bfloat16*>(param_bf16);
  const bool v4 = opt_v4(P, bstride, param, grad, square_avg, acc_delta, sh, bf16_bstride);
  dim3 grid = opt_grid(B, P, v4);
#define ADD(V, S) k_adadelta<V, S><<<grid, 256, 0, s>>>(P, param, grad, square_avg, acc_delta, bstride, lr, rho, eps, \
                                                        weight_decay, sh, bf16_bstride)
  if (v4) { if (sh) ADD(4, true); else ADD(4, false); }
  else { if (sh) ADD(1, true); else ADD(1, false); }
#undef ADD
  count_launches(1);
  return post_launch(s, "hfta_fused_adadelta");
}

extern "C" hfta_status hfta_steplr(int B, const float* lr0, const float* gamma, const int32_t* period, int64_t epoch,
                                   float* lr, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(lr0 && gamma && period && lr && epoch >= 0, HFTA_ERR_INVALID_VALUE, "steplr: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  k_steplr<<<(unsigned)cdiv(B, 128), 128, 0, s>>>(B, lr0, gamma, period, epoch, lr);
  count_launches(1);
  return post_launch(s, "hfta_steplr");
}

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
