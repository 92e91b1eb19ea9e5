// gemm_skinny.cu -- HBM-bound "skinny" model-batched contractions: the
// PointNet layers that touch the 3-wide xyz input (Conv1d 3->64, K = 3; its
// dgrad into xyz, N = 3; its wgrad dW[64][3]).  Arithmetic intensity is
// ~1-3 flop/B, far below every tensor-core ridge, so these are written as
// streaming kernels: one pass over the wide operand with 128-bit accesses,
// the narrow operand (weights, <= 8 per row) held in registers/smem.
#include "gemm.cuh"

namespace hfta {
namespace {

constexpr int NT = 256;
constexpr int KMAX = 8;

// fwd, small K: C[m][n] = sum_k A[m][k] * Bw[n][k] + bias.  Thread = (row, VEC columns).
template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_skinny_fwd(GemmP p, int tpr, int rpb, int64_t rows_per_block) {
  __shared__ float w[KMAX * 512];
  const int b = blockIdx.y;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* Bw = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  T* C = reinterpret_cast<T*>(p.C) + (int64_t)b * p.c_bs;
  const int K = (int)p.K, N = (int)p.N;
  for (int i = threadIdx.x; i < N * K; i += NT) w[(i % K) * N + i / K] = ldf(Bw + (int64_t)(i / K) * p.b_ld + i % K);
  __syncthreads();
  const int lane = threadIdx.x % tpr, rl = threadIdx.x / tpr;
  const int n0 = lane * VEC;
  if (n0 >= N) return;
  float bias[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) bias[v] = p.bias ? p.bias[(int64_t)b * p.bias_bs + n0 + v] : 0.f;
  const int64_t r0 = blockIdx.x * rows_per_block, r1 = min(p.M, r0 + rows_per_block);
  for (int64_t m = r0 + rl; m < r1; m += rpb) {
    float a[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) a[k] = k < K ? ldf(A + m * p.a_ld + k) : 0.f;
    float o[VEC];
    const float* br = p.bias && p.bias_div > 0 ? p.bias + (int64_t)b * p.bias_bs + (m / p.bias_div) * p.bias_ld : nullptr;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      float acc = br ? br[n0 + v] : bias[v];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) acc = fmaf(a[k], w[k * N + n0 + v], acc);
      o[v] = acc;
    }
    st_vec<T, VEC>(C + m * p.c_ld + n0, o);
  }
}

// dgrad, small N-out: C[m][j] = sum_n A[m][n] * Bw(n, j) with Bw MN-major (W[n][j]), j < N <= 8,
// reduction length K (= layer width, e.g. 64).  Thread per row; A row read with 128-bit loads.
template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_skinny_dgrad(GemmP p) {
  __shared__ float w[KMAX * 1024];
  const int b = blockIdx.y;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* Bw = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  T* C = reinterpret_cast<T*>(p.C) + (int64_t)b * p.c_bs;
  const int Kr = (int)p.K, Nj = (int)p.N;
  for (int i = threadIdx.x; i < Kr * Nj; i += NT) {
    int n = i / Nj, j = i % Nj;                       // element (j, n) of B = W[n][j]
    w[n * KMAX + j] = ldf(Bw + (int64_t)n * p.b_ld + j);
  }
  __syncthreads();
  for (int64_t m = blockIdx.x * (int64_t)NT + threadIdx.x; m < p.M; m += (int64_t)gridDim.x * NT) {
    float acc[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) acc[j] = 0.f;
    const T* a = A + m * p.a_ld;
    for (int n = 0; n < Kr; n += VEC) {
      float av[VEC];
      ld_vec<T, VEC>(a + n, av);
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int j = 0; j < KMAX; ++j) acc[j] = fmaf(av[v], w[(n + v) * KMAX + j], acc[j]);
    }
    for (int j = 0; j < Nj; ++j) stf(C + m * p.c_ld + j, acc[j]);
  }
}

// wgrad, small K-out: part[chunk][b][n][k] = sum_{rows in chunk} A(n, r) * Bx(k, r), both MN-major:
// A = dY[r][n] (n < N), Bx = X[r][k] (k < K_out <= 8).  Thread = (row lane, VEC n-columns).
template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_skinny_wgrad(GemmP p, int tpr, int rpb, int64_t rows_per_chunk,
                                                     float* __restrict__ part) {
  __shared__ float red[NT * VEC * 3];
  const int b = blockIdx.y, chunk = blockIdx.x;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* X = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  const int N = (int)p.M, Ko = (int)p.N;               // dW is [N][Ko]
  const int lane = threadIdx.x % tpr, rl = threadIdx.x / tpr;
  const int n0 = lane * VEC;
  float acc[VEC][3];
#pragma unroll
  for (int v = 0; v < VEC; ++v)
#pragma unroll
    for (int k = 0; k < 3; ++k) acc[v][k] = 0.f;
  if (n0 < N) {
    const int64_t r0 = (int64_t)chunk * rows_per_chunk, r1 = min(p.K, r0 + rows_per_chunk);
    for (int64_t r = r0 + rl; r < r1; r += rpb) {
      float dy[VEC];
      ld_vec<T, VEC>(A + r * p.a_ld + n0, dy);
      float x[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) x[k] = k < Ko ? ldf(X + r * p.b_ld + k) : 0.f;
#pragma unroll
      for (int v = 0; v < VEC; ++v)
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[v][k] = fmaf(dy[v], x[k], acc[v][k]);
    }
  }
  const int cb = tpr * VEC;
#pragma unroll
  for (int v = 0; v < VEC; ++v)
#pragma unroll
    for (int k = 0; k < 3; ++k) red[(rl * cb + lane * VEC + v) * 3 + k] = acc[v][k];
  __syncthreads();
  for (int e = threadIdx.x; e < cb * 3; e += NT) {
    const int col = e / 3, k = e % 3;
    if (col >= N || k >= Ko) continue;
    float s = 0.f;
    for (int r = 0; r < rpb; ++r) s += red[(r * cb + col) * 3 + k];
    part[(((int64_t)chunk * p.B + b) * N + col) * Ko + k] = s;
  }
}

__global__ void k_skinny_wgrad_fin(GemmP p, int chunks, const float* __restrict__ part) {
  const int N = (int)p.M, Ko = (int)p.N;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)p.B * N * Ko) return;
  int64_t b = i / (N * Ko), rem = i % (N * Ko), n = rem / Ko, k = rem % Ko;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += part[(((int64_t)c * p.B + b) * N + n) * Ko + k];
  float* o = reinterpret_cast<float*>(p.C) + b * p.c_bs + n * p.c_ld + k;
  *o = p.accumulate ? *o + (float)s : (float)s;
}

int pow2ceil(int64_t x) { int q = 1; while (q < x) q <<= 1; return q; }

// ---- tiny output width / tiny reduction (e.g. DCGAN D c5: Conv 512->1 on 4x4) ----
// fwd, N <= 8 outputs per row, long K: one warp per row, lanes split K.
template <typename T>
__global__ void k_gemv_fwd(GemmP p) {
  const int b = blockIdx.y;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* Bw = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  T* C = reinterpret_cast<T*>(p.C) + (int64_t)b * p.c_bs;
  for (int64_t m = warp; m < p.M; m += nwarps) {
    float acc[KMAX];
#pragma unroll
    for (int n = 0; n < KMAX; ++n) acc[n] = 0.f;
    for (int64_t k = lane; k < p.K; k += 32) {
      const float a = ldf(A + m * p.a_ld + k);
#pragma unroll
      for (int n = 0; n < KMAX; ++n)
        if (n < p.N) acc[n] = fmaf(a, ldf(Bw + n * p.b_ld + k), acc[n]);
    }
#pragma unroll
    for (int n = 0; n < KMAX; ++n) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], o);
    }
    if (lane == 0)
      for (int n = 0; n < p.N; ++n) {
        float v = acc[n];
        if (p.bias) v += p.bias[(int64_t)b * p.bias_bs + (p.bias_div > 0 ? (m / p.bias_div) * p.bias_ld : 0) + n];
        stf(C + m * p.c_ld + n, v);
      }
  }
}

// any majorness, reduction K <= 8: C[m][n] = sum_k A(m,k) B(n,k); thread per output element.
template <typename T, bool AK, bool BKM>
__global__ void k_smallk(GemmP p) {
  const int b = blockIdx.y;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* Bw = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  T* C = reinterpret_cast<T*>(p.C) + (int64_t)b * p.c_bs;
  const int64_t tot = p.M * p.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / p.N, n = i % p.N;
    float acc = 0.f;
    for (int64_t k = 0; k < p.K; ++k)
      acc = fmaf(ldf(AK ? A + m * p.a_ld + k : A + k * p.a_ld + m), ldf(BKM ? Bw + n * p.b_ld + k : Bw + k * p.b_ld + n),
                 acc);
    if (p.bias) acc += p.bias[(int64_t)b * p.bias_bs + (p.bias_div > 0 ? (m / p.bias_div) * p.bias_ld : 0) + n];
    stf(C + m * p.c_ld + n, acc);
  }
}

// wgrad with M <= 8 output rows (both operands MN-major), fp32 out, fixed-order chunks:
// part[chunk][b][m][n] = sum_{r in chunk} A[r][m] * X[r][n]; thread = column n.
template <typename T>
__global__ void k_smallm_wgrad(GemmP p, int64_t rows_per_chunk, float* __restrict__ part) {
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= p.N) return;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* X = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  float acc[KMAX];
#pragma unroll
  for (int m = 0; m < KMAX; ++m) acc[m] = 0.f;
  const int64_t r0 = chunk * rows_per_chunk, r1 = min(p.K, r0 + rows_per_chunk);
  for (int64_t r = r0; r < r1; ++r) {
    const float x = ldf(X + r * p.b_ld + n);
#pragma unroll
    for (int m = 0; m < KMAX; ++m)
      if (m < p.M) acc[m] = fmaf(ldf(A + r * p.a_ld + m), x, acc[m]);
  }
  for (int m = 0; m < p.M; ++m) part[(((int64_t)chunk * p.B + b) * p.M + m) * p.N + n] = acc[m];
}

__global__ void k_smallm_fin(GemmP p, int chunks, const float* __restrict__ part) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)p.B * p.M * p.N) return;
  const int64_t b = i / (p.M * p.N), rem = i % (p.M * p.N), m = rem / p.N, n = rem % p.N;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += part[(((int64_t)c * p.B + b) * p.M + m) * p.N + n];
  float* o = reinterpret_cast<float*>(p.C) + b * p.c_bs + m * p.c_ld + n;
  *o = p.accumulate ? *o + (float)s : (float)s;
}

}  // namespace

// ---- dispatch predicates (called from linear.cu / conv.cu) ----
static bool gemv_fwd_ok(const GemmP& p) { return p.a_kmajor && p.b_kmajor && p.N <= KMAX && p.splits == 1; }
static bool smallk_ok(const GemmP& p) { return p.a_kmajor && p.K <= KMAX && p.splits == 1 && !p.accumulate; }
static bool smallm_wgrad_ok(const GemmP& p) { return !p.a_kmajor && !p.b_kmajor && p.M <= KMAX; }
bool skinny_fwd_ok_base(const GemmP& p) { return p.a_kmajor && p.b_kmajor && p.K <= KMAX && p.N <= 512 && p.splits == 1; }
bool skinny_dgrad_ok(const GemmP& p) {
  return p.a_kmajor && !p.b_kmajor && p.N <= KMAX && p.K <= 1024 && p.splits == 1 && p.K % 8 == 0 && p.a_ld % 8 == 0;
}
bool skinny_wgrad_ok_base(const GemmP& p) { return !p.a_kmajor && !p.b_kmajor && p.N <= 3 && p.M <= 128; }
bool skinny_fwd_ok(const GemmP& p) { return skinny_fwd_ok_base(p) || gemv_fwd_ok(p) || smallk_ok(p); }
bool skinny_wgrad_ok(const GemmP& p) { return skinny_wgrad_ok_base(p) || smallm_wgrad_ok(p); }

static int64_t smallm_chunks(int B, int64_t rows, int64_t N) {
  const int64_t colblocks = cdiv(N, 256);
  return std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * 148, (int64_t)B * colblocks), cdiv(rows, 64)));
}

size_t skinny_wgrad_ws(int B, int64_t rows, int64_t N, int64_t Ko) {
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * 148, B), cdiv(rows, 2048)));
  size_t a = (size_t)chunks * B * N * Ko * sizeof(float);
  size_t c = N <= KMAX ? (size_t)smallm_chunks(B, rows, Ko) * B * N * Ko * sizeof(float) : 0;   // dW is [N][Ko]
  return std::max(a, c);
}

hfta_status gemm_skinny(const GemmP& p, hfta_dtype dt, void* ws, size_t ws_bytes, cudaStream_t s) {
  const bool bf = dt == HFTA_BF16;
  if (!skinny_fwd_ok_base(p) && !skinny_dgrad_ok(p) && !skinny_wgrad_ok_base(p)) {
    if (smallm_wgrad_ok(p)) {
      const int64_t chunks = smallm_chunks(p.B, p.K, p.N);
      const int64_t rpc = cdiv(p.K, chunks);
      const size_t need = (size_t)chunks * p.B * p.M * p.N * sizeof(float);
      HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "small-M wgrad: workspace %zu < %zu", ws_bytes, need);
      float* part = reinterpret_cast<float*>(ws);
      dim3 grid((unsigned)cdiv(p.N, 256), (unsigned)chunks, p.B);
      if (bf) k_smallm_wgrad<__nv_bfloat16><<<grid, 256, 0, s>>>(p, rpc, part);
      else k_smallm_wgrad<float><<<grid, 256, 0, s>>>(p, rpc, part);
      k_smallm_fin<<<(unsigned)cdiv((int64_t)p.B * p.M * p.N, 256), 256, 0, s>>>(p, (int)chunks, part);
      count_launches(2);
      return post_launch(s, "gemm_smallm_wgrad");
    }
    if (gemv_fwd_ok(p)) {
      dim3 grid((unsigned)std::min<int64_t>(cdiv(p.M, 8), 1024), p.B);
      if (bf) k_gemv_fwd<__nv_bfloat16><<<grid, 256, 0, s>>>(p);
      else k_gemv_fwd<float><<<grid, 256, 0, s>>>(p);
      count_launches(1);
      return post_launch(s, "gemm_gemv_fwd");
    }
    if (smallk_ok(p)) {
      dim3 grid((unsigned)std::min<int64_t>(cdiv(p.M * p.N, 256), 8192), p.B);
#define SK(AK, BK) (bf ? (void)k_smallk<__nv_bfloat16, AK, BK><<<grid, 256, 0, s>>>(p) : (void)k_smallk<float, AK, BK><<<grid, 256, 0, s>>>(p))
      if (p.a_kmajor && p.b_kmajor) SK(true, true);
      else if (p.a_kmajor) SK(true, false);
      else if (p.b_kmajor) SK(false, true);
      else SK(false, false);
#undef SK
      count_launches(1);
      return post_launch(s, "gemm_smallk");
    }
  }
  if (skinny_fwd_ok_base(p)) {
    int vec = bf ? 8 : 4;
    if (p.N % vec || p.c_ld % vec || !aligned16(p.C) || p.c_bs % vec) vec = 1;
    int tpr = std::min(32, pow2ceil(cdiv(p.N, vec)));
    int rpb = NT / tpr;
    int64_t blocks_per = std::max<int64_t>(1, std::min<int64_t>(cdiv(p.M, rpb * 4), cdiv(8 * 148, p.B)));
    int64_t rows_per_block = cdiv(p.M, blocks_per);
    dim3 grid((unsigned)cdiv(p.M, rows_per_block), p.B);
    if (bf) {
      if (vec == 8) k_skinny_fwd<__nv_bfloat16, 8><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
      else k_skinny_fwd<__nv_bfloat16, 1><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
    } else {
      if (vec == 4) k_skinny_fwd<float, 4><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
      else k_skinny_fwd<float, 1><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
    }
    count_launches(1);
    return post_launch(s, "gemm_skinny_fwd");
  }
  if (skinny_dgrad_ok(p)) {
    dim3 grid((unsigned)std::min<int64_t>(cdiv(p.M, NT), cdiv(8 * 148, p.B)), p.B);
    const bool v = aligned16(p.A) && (p.a_bs % 8 == 0);
    if (bf) {
      if (v) k_skinny_dgrad<__nv_bfloat16, 8><<<grid, NT, 0, s>>>(p);
      else k_skinny_dgrad<__nv_bfloat16, 1><<<grid, NT, 0, s>>>(p);
    } else {
      if (v) k_skinny_dgrad<float, 4><<<grid, NT, 0, s>>>(p);
      else k_skinny_dgrad<float, 1><<<grid, NT, 0, s>>>(p);
    }
    count_launches(1);
    return post_launch(s, "gemm_skinny_dgrad");
  }
  if (skinny_wgrad_ok_base(p)) {
    const int64_t rows = p.K, N = p.M, Ko = p.N;
    int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * 148, p.B), cdiv(rows, 2048)));
    size_t need = (size_t)chunks * p.B * N * Ko * sizeof(float);
    HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "skinny wgrad: workspace %zu < %zu", ws_bytes, need);
    int vec = bf ? 8 : 4;
    if (N % vec || p.a_ld % vec || !aligned16(p.A) || p.a_bs % vec) vec = 1;
    int tpr = std::min(32, pow2ceil(cdiv(N, vec)));
    int rpb = NT / tpr;
    int64_t rows_per_chunk = cdiv(rows, chunks);
    chunks = cdiv(rows, rows_per_chunk);
    float* part = reinterpret_cast<float*>(ws);
    dim3 grid((unsigned)chunks, p.B);
    if (bf) {
      if (vec == 8) k_skinny_wgrad<__nv_bfloat16, 8><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_chunk, part);
      else k_skinny_wgrad<__nv_bfloat16, 1><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_chunk, part);
    } else {
      if (vec == 4) k_skinny_wgrad<float, 4><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_chunk, part);
      else k_skinny_wgrad<float, 1><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_chunk, part);
    }
    k_skinny_wgrad_fin<<<(unsigned)cdiv((int64_t)p.B * N * Ko, 256), 256, 0, s>>>(p, (int)chunks, part);
    count_launches(2);
    return post_launch(s, "gemm_skinny_wgrad");
  }
  return fail(HFTA_ERR_UNSUPPORTED, "gemm_skinny: shape not skinny");
}

}  // namespace hfta
