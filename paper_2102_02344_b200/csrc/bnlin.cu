// bnlin.cu -- fused Linear (Conv1d k=1) -> BatchNorm(train) -> act with the BN
// statistics and the BN backward taken from K x K Gram quantities of the
// layer input (K11):
//
//   y = x W^T + b  [R][C],  mean_c = (W_c . s)/R + b_c,
//   E[(y_c - b_c)^2] = W_c G W_c^T / R,   G = x^T x [K][K], s = x^T 1 [K]
//
// so the forward is ONE pass: Gram of x (tensor cores, K <= 128 << R) ->
// per-channel scale/shift -> the GEMM whose epilogue applies
// act(scale*acc + shift) and writes the activation directly (the pre-BN y is
// never written nor re-read for statistics / normalisation).  The backward,
// given dZ = dL/dz (already multiplied by act'), is
//
//   dbeta = 1^T dZ,  Zm = dZ^T x [C][K],  dgamma_c = invstd_c (W_c . Zm_c - mean'_c dbeta_c)
//   dY = a dZ + bx (y - b) + cc       (a = gamma invstd, per channel)
//   dW = diag(a) Zm + diag(bx) W G + cc s^T
//   dx = dZ (diag(a) W) + x (W^T diag(bx) W) + 1 (W^T cc)^T
//
// -- dx is ONE tensor-core GEMM with two K segments ([dZ | x]) whose epilogue
// multiplies by the previous layer's act' (its output is the next dZ).  The
// [R][C] tensor dY is never formed.  (App. B rows Conv1d P:L1265-1266 and
// BatchNorm1d P:L1274-1278; the algebra is exact, only rounding order differs
// from the unfused composition: DESIGN.md reading R26.)
#include "gemm.cuh"

namespace hfta {
namespace {

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// Forward statistics from the Gram: one warp per (model, channel).
__global__ void k_bnl_stats(int B, int64_t R, int64_t C, int K, const float* __restrict__ G,
                            const float* __restrict__ sv, const __nv_bfloat16* __restrict__ W, int64_t w_bs,
                            int64_t w_ld, const float* __restrict__ bias, int64_t bias_bs,
                            const float* __restrict__ gamma, const float* __restrict__ beta, int64_t gbs,
                            float* __restrict__ rmean, float* __restrict__ rvar, float momentum, float eps,
                            float* __restrict__ smean, float* __restrict__ sinv, float* __restrict__ scale,
                            float* __restrict__ shift) {
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (gw >= (int64_t)B * C) return;
  const int64_t b = gw / C, c = gw % C;
  const __nv_bfloat16* Wc = W + b * w_bs + c * w_ld;
  const float* Gb = G + b * (int64_t)K * K;
  // q = W_c G W_c^T, m1 = W_c . s  (lanes over k)
  double q = 0.0, m1 = 0.0;
  for (int k = lane; k < K; k += 32) {      // G symmetric: read column k (lanes consecutive -> coalesced)
    double t = 0.0;
    for (int j = 0; j < K; ++j) t += (double)Gb[(int64_t)j * K + k] * (double)__bfloat162float(Wc[j]);
    const double wk = (double)__bfloat162float(Wc[k]);
    q += wk * t;
    m1 += wk * (double)sv[b * K + k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    q += __shfl_xor_sync(0xffffffffu, q, o);
    m1 += __shfl_xor_sync(0xffffffffu, m1, o);
  }
  if (lane != 0) return;
  const double Rd = (double)R;
  const double mean_nb = m1 / Rd;
  double var = q / Rd - mean_nb * mean_nb;
  if (var < 0.0) var = 0.0;
  const double inv = 1.0 / sqrt(var + (double)eps);
  const double bi = bias ? (double)bias[b * bias_bs + c] : 0.0;
  const double mean = mean_nb + bi;
  const int64_t i = b * C + c;
  smean[i] = (float)mean;
  sinv[i] = (float)inv;
  if (rmean) rmean[i] = (float)((1.0 - momentum) * (double)rmean[i] + momentum * mean);
  if (rvar) rvar[i] = (float)((1.0 - momentum) * (double)rvar[i] + momentum * var * Rd / (Rd - 1.0));
  const double ga = gamma[b * gbs + c], be = beta[b * gbs + c];
  scale[i] = (float)(ga * inv);
  shift[i] = (float)(be - ga * inv * mean_nb);     // applied to the bias-free product x W^T
}

// Backward coefficients per (model, channel): dgamma, dbeta, a, bx, cc; also
// writes the first-segment weight diag(a) W in bf16, as [K][C] (K-major, the
// tensor-core dx GEMM) or [C][K] (the skinny dx kernel), and zeroes the
// BN-absorbed bias gradient.
__global__ void k_bnl_coef(int B, int64_t R, int64_t C, int K, const float* __restrict__ Zm,
                           const float* __restrict__ dbeta_in, const __nv_bfloat16* __restrict__ W, int64_t w_bs,
                           int64_t w_ld, const float* __restrict__ bias, int64_t bias_bs,
                           const float* __restrict__ gamma, int64_t gbs, const float* __restrict__ smean,
                           const float* __restrict__ sinv, float* __restrict__ coef, __nv_bfloat16* __restrict__ Wat,
                           __nv_bfloat16* __restrict__ Wab, float* __restrict__ dgamma, float* __restrict__ dbeta,
                           float* __restrict__ dbias, int64_t dbias_bs, int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * C) return;
  const int64_t b = i / C, c = i % C;
  const __nv_bfloat16* Wc = W + b * w_bs + c * w_ld;
  const float* Zc = Zm + (b * C + c) * K;
  double wz = 0.0;
  for (int k = 0; k < K; ++k) wz += (double)__bfloat162float(Wc[k]) * (double)Zc[k];
  const double inv = sinv[i];
  const double bi = bias ? (double)bias[b * bias_bs + c] : 0.0;
  const double mean_nb = (double)smean[i] - bi;
  const double dbe = dbeta_in[i];
  const double dga = inv * (wz - mean_nb * dbe);
  const double a = (double)gamma[b * gbs + c] * inv;
  const double Rd = (double)R;
  const double bx = -a * inv * dga / Rd;
  const double cc = -a * dbe / Rd - bx * mean_nb;
  coef[i * 3 + 0] = (float)a;
  coef[i * 3 + 1] = (float)bx;
  coef[i * 3 + 2] = (float)cc;
  for (int k = 0; k < K; ++k) {
    const float v = (float)(a * (double)__bfloat162float(Wc[k]));
    if (Wat) Wat[(b * K + k) * C + c] = __float2bfloat16_rn(v);   // [K][C]
    if (Wab) Wab[(b * C + c) * K + k] = __float2bfloat16_rn(v);   // [C][K] (skinny path)
  }
  const int64_t go = b * gbs + c;
  if (accumulate) { dgamma[go] += (float)dga; dbeta[go] += (float)dbe; }
  else { dgamma[go] = (float)dga; dbeta[go] = (float)dbe; }
  if (dbias && !accumulate) dbias[b * dbias_bs + c] = 0.f;
}

// dW[c][k] (+)= a_c Zm[c][k] + bx_c (W G)[c][k] + cc_c s[k]; thread per output.
__global__ void k_bnl_dw(int B, int64_t C, int K, const float* __restrict__ Zm, const float* __restrict__ G,
                         const float* __restrict__ sv, const __nv_bfloat16* __restrict__ W, int64_t w_bs, int64_t w_ld,
                         const float* __restrict__ coef, float* __restrict__ dW, int64_t dw_bs, int64_t dw_ld,
                         int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * C * K) return;
  const int64_t k = i % K, c = (i / K) % C, b = i / (K * C);
  const __nv_bfloat16* Wc = W + b * w_bs + c * w_ld;
  const float* Gb = G + b * (int64_t)K * K;
  float wg = 0.f;
  for (int j = 0; j < K; ++j) wg = fmaf(__bfloat162float(Wc[j]), Gb[(int64_t)j * K + k], wg);
  const float* cf = coef + (b * C + c) * 3;
  const float r = fmaf(cf[0], Zm[(b * C + c) * K + k], fmaf(cf[1], wg, cf[2] * sv[b * K + k]));
  float* d = dW + b * dw_bs + c * dw_ld + k;
  *d = accumulate ? *d + r : r;
}

// M = W^T diag(bx) W [K][K] (bf16 for the tensor-core dx GEMM, or fp32 for
// the skinny path) and v = W^T cc [K]; thread per (model, k, k').
__global__ void k_bnl_mv(int B, int64_t C, int K, const __nv_bfloat16* __restrict__ W, int64_t w_bs, int64_t w_ld,
                         const float* __restrict__ coef, __nv_bfloat16* __restrict__ Mb, float* __restrict__ Mf,
                         float* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * K * (K + 1)) return;
  const int64_t b = i / ((int64_t)K * (K + 1)), r = i % ((int64_t)K * (K + 1));
  const int k = (int)(r / (K + 1)), k2 = (int)(r % (K + 1));   // k2 == K: the v entry
  const __nv_bfloat16* Wb = W + b * w_bs;
  float acc = 0.f;
  for (int64_t c = 0; c < C; ++c) {
    const float* cf = coef + (b * C + c) * 3;
    const float wk = __bfloat162float(Wb[c * w_ld + k]);
    acc = k2 < K ? fmaf(wk * cf[1], __bfloat162float(Wb[c * w_ld + k2]), acc) : fmaf(wk, cf[2], acc);
  }
  if (k2 == K) {
    v[b * K + k] = acc;
  } else {
    if (Mb) Mb[(b * K + k) * K + k2] = __float2bfloat16_rn(acc);
    if (Mf) Mf[(b * K + k) * K + k2] = acc;
  }
}

struct FwdL { size_t G, sv, scale, shift, lin, total; };
FwdL fwd_layout(int B, int64_t M, int64_t N, int64_t K) {
  FwdL l{};
  size_t o = 0;
  l.G = o; o += al256((size_t)B * K * K * 4);
  l.sv = o; o += al256((size_t)B * K * 4);
  l.scale = o; o += al256((size_t)B * N * 4);
  l.shift = o; o += al256((size_t)B * N * 4);
  l.lin = o; o += al256(hfta_fused_linear_bwd_workspace(B, M, K, K, HFTA_BF16));
  l.total = o;
  return l;
}
struct BwdL { size_t Zm, db, coef, Wat, Mm, v, lin, total; };
BwdL bwd_layout(int B, int64_t M, int64_t N, int64_t K) {
  BwdL l{};
  size_t o = 0;
  l.Zm = o; o += al256((size_t)B * N * K * 4);
  l.db = o; o += al256((size_t)B * N * 4);
  l.coef = o; o += al256((size_t)B * N * 12);
  l.Wat = o; o += al256((size_t)B * N * K * 4);      // bf16 [K][N] or fp32 [N][K]
  l.Mm = o; o += al256((size_t)B * K * K * 4);
  l.v = o; o += al256((size_t)B * K * 4);
  l.lin = o; o += al256(hfta_fused_linear_bwd_workspace(B, M, N, K, HFTA_BF16));
  l.total = o;
  return l;
}

hfta_status check_args(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt, hfta_in X, hfta_in W) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(dt == HFTA_BF16, HFTA_ERR_UNSUPPORTED, "linear_bn: bf16 operands only (fused tensor-core path)");
  HFTA_REQUIRE(M >= 2 && N >= 1 && K >= 1, HFTA_ERR_SHAPE, "linear_bn: M,N,K = %lld,%lld,%lld", (long long)M,
               (long long)N, (long long)K);
  HFTA_REQUIRE(K <= 8 || (K % 64 == 0 && K <= 128), HFTA_ERR_UNSUPPORTED,
               "linear_bn: K=%lld must be <= 8 (streaming path) or 64/128 (tensor cores)", (long long)K);
  HFTA_REQUIRE(N <= 512, HFTA_ERR_UNSUPPORTED, "linear_bn: N=%lld > 512", (long long)N);
  HFTA_REQUIRE(X.ptr && W.ptr && X.ld >= K && W.ld >= K, HFTA_ERR_SHAPE, "linear_bn: X/W");
  return HFTA_OK;
}

}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" {

size_t hfta_fused_linear_bn_workspace(int B, int64_t M, int64_t N, int64_t K) {
  if (B < 1 || M < 1 || N < 1 || K < 1) return 0;
  return std::max(fwd_layout(B, M, N, K).total, bwd_layout(B, M, N, K).total);
}

hfta_status hfta_fused_linear_bn_fwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt, hfta_in X, hfta_in W,
                                     const float* bias, int64_t bias_bstride, const float* gamma, const float* beta,
                                     int64_t gb_bstride, float* running_mean, float* running_var, float momentum,
                                     float eps, hfta_act act, float act_alpha, hfta_out A, float* save_mean,
                                     float* save_invstd, float* G, float* s, void* ws, size_t ws_bytes,
                                     hfta_stream stream) {
  if (hfta_status st = check_args(B, M, N, K, dt, X, W)) return st;
  HFTA_REQUIRE(gamma && beta && A.ptr && save_mean && save_invstd && G && s, HFTA_ERR_INVALID_VALUE,
               "linear_bn_fwd: gamma, beta, A, save_mean, save_invstd, G, s are required");
  HFTA_REQUIRE(A.ld >= N && (A.bstride > 0 || B == 1), HFTA_ERR_SHAPE, "linear_bn_fwd: A strides");
  const FwdL l = fwd_layout(B, M, N, K);
  HFTA_REQUIRE(ws && ws_bytes >= hfta_fused_linear_bn_workspace(B, M, N, K), HFTA_ERR_WORKSPACE,
               "linear_bn_fwd: workspace too small");
  cudaStream_t st_ = (cudaStream_t)stream;
  char* w = reinterpret_cast<char*>(ws);
  float* scale = reinterpret_cast<float*>(w + l.scale);
  float* shift = reinterpret_cast<float*>(w + l.shift);
  // 1. G = X^T X, s = X^T 1 (wgrad contraction + column sums over the M rows)
  if (hfta_status e = hfta_fused_linear_bwd(B, M, K, K, HFTA_BF16, X, X, W, hfta_out{nullptr, 0, 1}, G, K * K, K, s,
                                            K, 0, w + l.lin, l.total - l.lin, stream))
    return e;
  // 2. statistics -> scale / shift
  const int64_t warps = (int64_t)B * N;
  k_bnl_stats<<<(unsigned)cdiv(warps * 32, 256), 256, 0, st_>>>(
      B, M, N, (int)K, G, s, (const __nv_bfloat16*)W.ptr, B > 1 ? W.bstride : 0, W.ld, bias, bias_bstride, gamma,
      beta, gb_bstride, running_mean, running_var, momentum, eps, save_mean, save_invstd, scale, shift);
  count_launches(1);
  if (hfta_status e = post_launch(st_, "linear_bn_fwd stats")) return e;
  // 3. A = act(scale * (X W^T) + shift): the GEMM with the fused BN-apply epilogue
  GemmP p{};
  p.B = B; p.M = M; p.N = N; p.K = K;
  p.A = X.ptr; p.a_bs = X.bstride; p.a_ld = X.ld; p.a_kmajor = 1;
  p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 1;
  p.C = A.ptr; p.c_bs = A.bstride; p.c_ld = A.ld;
  p.bias = shift; p.bias_bs = N;
  p.scale = scale; p.scale_bs = N;
  p.act = (int)act; p.act_alpha = act_alpha;
  p.splits = 1; p.k_chunk = cdiv(K, 16) * 16;
  return run_gemm(p, HFTA_BF16, false, st_);
}

hfta_status hfta_fused_linear_bn_bwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt, hfta_in dZ, hfta_in X,
                                     hfta_in W, const float* bias, int64_t bias_bstride, const float* gamma,
                                     int64_t gb_bstride, const float* save_mean, const float* save_invstd,
                                     const float* G, const float* s, hfta_out dX, hfta_act dX_act, float dX_alpha,
                                     float* dW, int64_t dW_bstride, int64_t dW_ld, float* dbias,
                                     int64_t dbias_bstride, float* dgamma, float* dbeta, int accumulate, void* ws,
                                     size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_args(B, M, N, K, dt, X, W)) return st;
  HFTA_REQUIRE(dZ.ptr && gamma && save_mean && save_invstd && G && s && dW && dgamma && dbeta, HFTA_ERR_INVALID_VALUE,
               "linear_bn_bwd: dZ, gamma, save_*, G, s, dW, dgamma, dbeta are required");
  HFTA_REQUIRE(dZ.ld >= N && dW_ld >= K, HFTA_ERR_SHAPE, "linear_bn_bwd: dZ / dW strides");
  HFTA_REQUIRE(!dX.ptr || (dX.ld >= K && (dX.bstride > 0 || B == 1)), HFTA_ERR_SHAPE, "linear_bn_bwd: dX strides");
  const BwdL l = bwd_layout(B, M, N, K);
  HFTA_REQUIRE(ws && ws_bytes >= hfta_fused_linear_bn_workspace(B, M, N, K), HFTA_ERR_WORKSPACE,
               "linear_bn_bwd: workspace too small");
  cudaStream_t st_ = (cudaStream_t)stream;
  char* w = reinterpret_cast<char*>(ws);
  float* Zm = reinterpret_cast<float*>(w + l.Zm);
  float* db = reinterpret_cast<float*>(w + l.db);
  float* coef = reinterpret_cast<float*>(w + l.coef);
  const bool tc = K > 8;
  const __nv_bfloat16* Wp = (const __nv_bfloat16*)W.ptr;
  const int64_t wbs = B > 1 ? W.bstride : 0;
  // 1. Zm = dZ^T X [N][K], dbeta = 1^T dZ
  if (hfta_status e = hfta_fused_linear_bwd(B, M, N, K, HFTA_BF16, dZ, X, W, hfta_out{nullptr, 0, 1}, Zm, N * K, K,
                                            db, N, 0, w + l.lin, l.total - l.lin, stream))
    return e;
  // 2. per-channel coefficients, dgamma/dbeta, first-segment weight
  __nv_bfloat16* Wat = (dX.ptr && tc) ? reinterpret_cast<__nv_bfloat16*>(w + l.Wat) : nullptr;
  __nv_bfloat16* Wab = (dX.ptr && !tc) ? reinterpret_cast<__nv_bfloat16*>(w + l.Wat) : nullptr;
  k_bnl_coef<<<(unsigned)cdiv((int64_t)B * N, 128), 128, 0, st_>>>(
      B, M, N, (int)K, Zm, db, Wp, wbs, W.ld, bias, bias_bstride, gamma, gb_bstride, save_mean, save_invstd, coef,
      Wat, Wab, dgamma, dbeta, dbias, dbias_bstride, accumulate);
  // 3. dW = diag(a) Zm + diag(bx) W G + cc s^T
  k_bnl_dw<<<(unsigned)cdiv((int64_t)B * N * K, 256), 256, 0, st_>>>(B, N, (int)K, Zm, G, s, Wp, wbs, W.ld, coef, dW,
                                                                    dW_bstride, dW_ld, accumulate);
  count_launches(2);
  if (!dX.ptr) return post_launch(st_, "linear_bn_bwd");
  // 4. dX = dZ (diag(a) W) + X M + v, times act'(X) of the previous layer
  __nv_bfloat16* Mb = tc ? reinterpret_cast<__nv_bfloat16*>(w + l.Mm) : nullptr;
  float* Mf = tc ? nullptr : reinterpret_cast<float*>(w + l.Mm);
  float* v = reinterpret_cast<float*>(w + l.v);
  k_bnl_mv<<<(unsigned)cdiv((int64_t)B * K * (K + 1), 128), 128, 0, st_>>>(B, N, (int)K, Wp, wbs, W.ld, coef, Mb, Mf,
                                                                          v);
  count_launches(1);
  if (hfta_status e = post_launch(st_, "linear_bn_bwd coef")) return e;
  GemmP p{};
  p.B = B; p.M = M; p.N = K; p.K = N;                          // dX[M][K] = dZ[M][N] * Wa[N][K] + ...
  p.A = dZ.ptr; p.a_bs = dZ.bstride; p.a_ld = dZ.ld; p.a_kmajor = 1;
  if (tc) { p.Bm = Wat; p.b_bs = K * N; p.b_ld = N; p.b_kmajor = 1; }   // (diag(a) W)^T [K][N], K-major
  else { p.Bm = Wab; p.b_bs = N * K; p.b_ld = K; p.b_kmajor = 0; }      // diag(a) W [N][K] (skinny dgrad)
  p.C = dX.ptr; p.c_bs = dX.bstride; p.c_ld = dX.ld;
  p.bias = v; p.bias_bs = K;
  p.A2 = X.ptr; p.a2_bs = X.bstride; p.a2_ld = X.ld; p.K2 = K;
  if (tc) { p.Bm2 = Mb; p.b2_bs = K * K; p.b2_ld = K; }        // M symmetric: [K][K] K-major
  else { p.Bm2 = Mf; p.b2_bs = K * K; p.b2_ld = K; }
  if (dX_act != HFTA_ACT_NONE) {
    p.mask = X.ptr; p.mask_bs = X.bstride; p.mask_ld = X.ld; p.mask_act = (int)dX_act; p.mask_alpha = dX_alpha;
  }
  p.splits = 1; p.k_chunk = cdiv(N, 16) * 16;
  if (!tc) {
    // K <= 8: the skinny dgrad kernel (M fp32 in the second segment)
    HFTA_REQUIRE(skinny_dgrad_ok(p), HFTA_ERR_UNSUPPORTED, "linear_bn_bwd: dX shape not supported (N=%lld)",
                 (long long)N);
    return gemm_skinny(p, HFTA_BF16, nullptr, 0, st_);
  }
  return run_gemm(p, HFTA_BF16, false, st_);
}

}  // extern "C"
