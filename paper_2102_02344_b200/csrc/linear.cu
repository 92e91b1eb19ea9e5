// linear.cu -- C ABI of the fused Linear / Conv1d(k=1) layer (K1/K2).
// App. B rows "Linear -> baddbmm(b[B,1,Fy], x[B,N,Fx], w[B,Fx,Fy])"
// and "Conv1d ... G = B x g": one launch for
// all B models, model index in the grid / tile scheduler.
#include "gemm.cuh"

namespace hfta {
hfta_status colsum_impl(int B, int64_t rows, int64_t C, int64_t group, hfta_dtype dt, hfta_in X,
                        float* S, int64_t S_bstride, int accumulate, void* ws, size_t ws_bytes,
                        cudaStream_t s);
size_t colsum_ws(int B, int64_t rows, int64_t C, int64_t group);

hfta_status run_gemm(GemmP& p, hfta_dtype dt, bool out_f32, cudaStream_t s, void* ws, size_t wsb) {
  const bool epi = p.scale || p.act != HFTA_ACT_NONE || p.mask || p.K2 > 0;
  // the streaming fwd/dgrad kernels write C in the input dtype: not for bf16 -> fp32 (HFTA_BF16_F32)
  const bool same_out = !out_f32 || dt == HFTA_F32;
  if ((same_out && (skinny_fwd_ok(p) || skinny_dgrad_ok(p))) || skinny_wgrad_ok(p))
    return gemm_skinny(p, dt, ws, wsb, s);
  if (gemm_tc_supported(p, dt, out_f32)) return gemm_tc(p, dt, out_f32, s);
  if (epi) return fail(HFTA_ERR_UNSUPPORTED, "fused epilogue / second K segment needs the tensor-core or skinny path");
  if (dt == HFTA_F32 && gemm_tf32_supported(p)) return gemm_tf32(p, s);     // fp32: 3xTF32 tensor cores
  return gemm_simt(p, dt, out_f32, s);
}

namespace {
// split-K policy of the weight-gradient contraction (reduction over M rows).
struct Split { int splits; int64_t chunk; };
Split wgrad_split(int B, int64_t M, int64_t N, int64_t K, int bn = 128) {
  // Split the reduction over M so the persistent grid's last wave is full:
  // the busiest CTA streams ceil(tiles / SMs) tiles, each (M/s) rows of
  // (N + K) bf16 plus an N x K fp32 partial written and re-read by the
  // reduction; pick the split count s minimising that.
  const int64_t sms = std::max(num_sms(), 1);
  const int64_t tiles = cdiv(N, 128) * cdiv(K, bn) * (int64_t)B;   // bn: the tile width along K
  const int64_t maxs = std::max<int64_t>(1, M / 1024);
  int64_t best_s = 1;
  double best = -1.0;
  for (int64_t s = 1; s <= std::min<int64_t>(maxs, 64); ++s) {
    const int64_t chunk = cdiv(cdiv(M, s), 128) * 128;
    const int64_t sp = cdiv(M, chunk);
    const double per_tile = (double)chunk * (double)(N + K) * 2.0 + (sp > 1 ? (double)N * K * 8.0 : 0.0);
    const double cost = (double)cdiv(tiles * sp, sms) * per_tile;
    if (best < 0.0 || cost < best * 0.999) { best = cost; best_s = sp; }
  }
  const int64_t chunk = cdiv(cdiv(M, best_s), 128) * 128;
  return {(int)cdiv(M, chunk), chunk};
}
}  // namespace

// the same policy for callers outside this file (implicit-GEMM conv wgrad)
void wgrad_split_rows(int B, int64_t rows, int64_t N, int64_t K, int* splits, int64_t* chunk, int bn) {
  Split sp = wgrad_split(B, rows, N, K, bn);
  *splits = sp.splits;
  *chunk = sp.chunk;
}

namespace {

hfta_status check_in(const hfta_in& t, const char* name, int B) {
  HFTA_REQUIRE(t.ptr, HFTA_ERR_INVALID_VALUE, "%s.ptr is NULL", name);
  HFTA_REQUIRE(t.bstride >= 0 && t.ld >= 1, HFTA_ERR_SHAPE, "%s: bstride %lld / ld %lld invalid", name,
               (long long)t.bstride, (long long)t.ld);
  (void)B;
  return HFTA_OK;
}
hfta_status check_out(const hfta_out& t, const char* name, int B) {
  HFTA_REQUIRE(t.ptr, HFTA_ERR_INVALID_VALUE, "%s.ptr is NULL", name);
  HFTA_REQUIRE(t.ld >= 1 && (t.bstride > 0 || B == 1), HFTA_ERR_SHAPE,
               "%s: output needs bstride > 0 (got %lld) and ld >= 1", name, (long long)t.bstride);
  return HFTA_OK;
}
}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" {

hfta_status hfta_fused_linear_fwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt,
                                  hfta_in X, hfta_in W, const float* bias, int64_t bias_bstride,
                                  int64_t bias_ld, int64_t bias_row_div, hfta_out Y,
                                  hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(M >= 1 && N >= 1 && K >= 1, HFTA_ERR_SHAPE, "linear_fwd: M,N,K = %lld,%lld,%lld",
               (long long)M, (long long)N, (long long)K);
  HFTA_REQUIRE(dt == HFTA_F32 || dt == HFTA_BF16 || dt == HFTA_BF16_F32, HFTA_ERR_UNSUPPORTED, "linear_fwd: dtype %d",
               (int)dt);
  const bool mixed = dt == HFTA_BF16_F32;         // bf16 operands, fp32 Y
  if (hfta_status st = check_in(X, "X", B)) return st;
  if (hfta_status st = check_in(W, "W", B)) return st;
  if (hfta_status st = check_out(Y, "Y", B)) return st;
  HFTA_REQUIRE(X.ld >= K, HFTA_ERR_SHAPE, "linear_fwd: X [%lld x %lld] has ld %lld < K", (long long)M,
               (long long)K, (long long)X.ld);
  HFTA_REQUIRE(W.ld >= K, HFTA_ERR_SHAPE, "linear_fwd: W [%lld x %lld] has ld %lld < K", (long long)N,
               (long long)K, (long long)W.ld);
  HFTA_REQUIRE(Y.ld >= N, HFTA_ERR_SHAPE, "linear_fwd: Y [%lld x %lld] has ld %lld < N", (long long)M,
               (long long)N, (long long)Y.ld);
  GemmP p{};
  p.B = B; p.M = M; p.N = N; p.K = K;
  p.A = X.ptr; p.a_bs = X.bstride; p.a_ld = X.ld; p.a_kmajor = 1;
  p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 1;
  p.C = Y.ptr; p.c_bs = Y.bstride; p.c_ld = Y.ld;
  p.bias = bias; p.bias_bs = bias_bstride; p.bias_ld = bias_ld;
  p.bias_div = (bias_ld > 0 && bias_row_div > 0) ? bias_row_div : 0;
  p.splits = 1; p.k_chunk = cdiv(K, 16) * 16;
  return run_gemm(p, mixed ? HFTA_BF16 : dt, mixed, (cudaStream_t)stream);
}

size_t hfta_linear_colstat_size(int B, int64_t M, int64_t N) {
  if (B < 1 || M < 1 || N < 1) return 0;
  return (size_t)B * cdiv(M, 32) * 2 * N * sizeof(float);
}

hfta_status hfta_fused_linear_fwd_stats(int B, int64_t M, int64_t N, int64_t K, hfta_in X, hfta_in W,
                                        const float* bias, int64_t bias_bstride, int64_t bias_ld,
                                        int64_t bias_row_div, hfta_out Y, float* colstat, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(M >= 1 && N >= 1 && K >= 1 && colstat, HFTA_ERR_INVALID_VALUE,
               "linear_fwd_stats: M,N,K = %lld,%lld,%lld, colstat %p", (long long)M, (long long)N, (long long)K,
               (void*)colstat);
  if (hfta_status st = check_in(X, "X", B)) return st;
  if (hfta_status st = check_in(W, "W", B)) return st;
  if (hfta_status st = check_out(Y, "Y", B)) return st;
  HFTA_REQUIRE(X.ld >= K && W.ld >= K && Y.ld >= N, HFTA_ERR_SHAPE, "linear_fwd_stats: ld < extent");
  GemmP p{};
  p.B = B; p.M = M; p.N = N; p.K = K;
  p.A = X.ptr; p.a_bs = X.bstride; p.a_ld = X.ld; p.a_kmajor = 1;
  p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 1;
  p.C = Y.ptr; p.c_bs = Y.bstride; p.c_ld = Y.ld;
  p.bias = bias; p.bias_bs = bias_bstride; p.bias_ld = bias_ld;
  p.bias_div = (bias_ld > 0 && bias_row_div > 0) ? bias_row_div : 0;
  p.splits = 1; p.k_chunk = cdiv(K, 16) * 16;
  p.colstat = colstat; p.colstat_bs = cdiv(M, 32) * 2 * N;
  HFTA_REQUIRE(!skinny_fwd_ok(p) && gemm_tc_supported(p, HFTA_BF16, false), HFTA_ERR_UNSUPPORTED,
               "linear_fwd_stats: the statistics ride on the bf16 tensor-core epilogue (K %lld, N %lld not eligible)",
               (long long)K, (long long)N);
  return gemm_tc(p, HFTA_BF16, false, (cudaStream_t)stream);
}

size_t hfta_fused_linear_bwd_workspace(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt) {
  if (B < 1 || M < 1 || N < 1 || K < 1) return 0;
  Split sp = wgrad_split(B, M, N, K);
  size_t part = sp.splits > 1 ? (size_t)sp.splits * B * N * K * sizeof(float) : 0;
  part = std::max(part, skinny_wgrad_ws(B, M, N, K));
  size_t cs = colsum_ws(B, M, N, M);
  size_t csp = sp.splits > 1 ? (size_t)sp.splits * B * N * sizeof(float) : 0;   // fused column-sum partials
  return align_up(part, 256) + align_up(std::max(cs, csp), 256);
  (void)dt;
}

hfta_status hfta_fused_linear_bwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt,
                                  hfta_in dY, hfta_in X, hfta_in W, hfta_out dX, float* dW,
                                  int64_t dW_bstride, int64_t dW_ld, float* dbias, int64_t dbias_bstride,
                                  int accumulate, void* ws, size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(M >= 1 && N >= 1 && K >= 1, HFTA_ERR_SHAPE, "linear_bwd: M,N,K = %lld,%lld,%lld",
               (long long)M, (long long)N, (long long)K);
  HFTA_REQUIRE(dt == HFTA_F32 || dt == HFTA_BF16 || dt == HFTA_BF16_F32, HFTA_ERR_UNSUPPORTED, "linear_bwd: dtype %d",
               (int)dt);
  const bool mixed = dt == HFTA_BF16_F32;         // bf16 operands, fp32 dX
  if (mixed) dt = HFTA_BF16;
  if (hfta_status st = check_in(dY, "dY", B)) return st;
  HFTA_REQUIRE(dY.ld >= N, HFTA_ERR_SHAPE, "linear_bwd: dY ld %lld < N %lld", (long long)dY.ld, (long long)N);
  cudaStream_t s = (cudaStream_t)stream;
  size_t need = hfta_fused_linear_bwd_workspace(B, M, N, K, dt);
  HFTA_REQUIRE(ws_bytes >= need && (need == 0 || ws), HFTA_ERR_WORKSPACE,
               "linear_bwd: workspace %zu < required %zu bytes", ws_bytes, need);
  if (dX.ptr) {
    if (hfta_status st = check_in(W, "W", B)) return st;
    if (hfta_status st = check_out(dX, "dX", B)) return st;
    HFTA_REQUIRE(dX.ld >= K && W.ld >= K, HFTA_ERR_SHAPE, "linear_bwd: dX/W ld < K");
    GemmP p{};
    p.B = B; p.M = M; p.N = K; p.K = N;                         // dX[M,K] = dY[M,N] W[N,K]
    p.A = dY.ptr; p.a_bs = dY.bstride; p.a_ld = dY.ld; p.a_kmajor = 1;
    p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 0;
    p.C = dX.ptr; p.c_bs = dX.bstride; p.c_ld = dX.ld;
    p.splits = 1; p.k_chunk = cdiv(N, 16) * 16;
    if (hfta_status st = run_gemm(p, dt, mixed, s)) return st;
  }
  if (dW) {
    if (hfta_status st = check_in(X, "X", B)) return st;
    HFTA_REQUIRE(X.ld >= K, HFTA_ERR_SHAPE, "linear_bwd: X ld %lld < K %lld", (long long)X.ld, (long long)K);
    HFTA_REQUIRE(dW_ld >= K, HFTA_ERR_SHAPE, "linear_bwd: dW_ld %lld < K %lld", (long long)dW_ld, (long long)K);
    HFTA_REQUIRE(dW_bstride >= N * dW_ld || B == 1, HFTA_ERR_SHAPE, "linear_bwd: dW_bstride %lld < N*dW_ld",
                 (long long)dW_bstride);
    GemmP p{};
    p.B = B; p.M = N; p.N = K; p.K = M;                         // dW[N,K] = dY^T[N,M] X[M,K]
    p.A = dY.ptr; p.a_bs = dY.bstride; p.a_ld = dY.ld; p.a_kmajor = 0;
    p.Bm = X.ptr; p.b_bs = X.bstride; p.b_ld = X.ld; p.b_kmajor = 0;
    p.C = dW; p.c_bs = dW_bstride; p.c_ld = dW_ld;
    p.accumulate = accumulate;
    p.splits = 1; p.k_chunk = M;
    if (skinny_wgrad_ok(p)) {
      if (dbias && skinny_wgrad_ok_base(p)) {   // dbias fused into the streaming wgrad (column k = K)
        p.colsum = dbias; p.colsum_bs = dbias_bstride; p.colsum_acc = accumulate;
        dbias = nullptr;
      }
      if (hfta_status st = gemm_skinny(p, dt, ws, ws_bytes, s)) return st;
    } else {
      Split sp = wgrad_split(B, M, N, K);
      p.splits = sp.splits; p.k_chunk = sp.chunk;
      p.part = sp.splits > 1 ? reinterpret_cast<float*>(ws) : nullptr;
      if (dbias && gemm_tc_supported(p, dt, true)) {
        // dbias = column sums of dY, fused into the tensor-core wgrad (ones operand)
        const size_t off = align_up(std::max(sp.splits > 1 ? (size_t)sp.splits * B * N * K * sizeof(float) : 0,
                                             skinny_wgrad_ws(B, M, N, K)), 256);
        p.colsum = dbias; p.colsum_bs = dbias_bstride; p.colsum_acc = accumulate;
        p.colsum_part = sp.splits > 1 ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + off) : nullptr;
        dbias = nullptr;
      }
      if (hfta_status st = run_gemm(p, dt, true, s)) return st;
      if (sp.splits > 1) {
        if (hfta_status st = splitk_reduce(p, s)) return st;
        if (p.colsum)
          if (hfta_status st = colsum_reduce(p, s)) return st;
      }
    }
  }
  if (dbias) {
    Split sp = wgrad_split(B, M, N, K);
    size_t off = align_up(std::max(sp.splits > 1 ? (size_t)sp.splits * B * N * K * sizeof(float) : 0,
                                   skinny_wgrad_ws(B, M, N, K)), 256);
    char* cws = ws ? reinterpret_cast<char*>(ws) + off : nullptr;
    if (hfta_status st = colsum_impl(B, M, N, M, dt, dY, dbias, dbias_bstride, accumulate, cws,
                                     ws_bytes > off ? ws_bytes - off : 0, s))
      return st;
  }
  return HFTA_OK;
}

}  // extern "C"
