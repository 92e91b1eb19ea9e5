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
constexpr int XTILE = 1024;   // rows of the narrow operand staged in smem per step

// fwd, small K: C[m][n] = sum_k A[m][k] * Bw[n][k] + bias.  Thread = (row, VEC
// columns) with its KT x VEC weights and VEC biases in registers (KT = K, a
// compile-time constant: 3 for the xyz layers; 0 = generic K <= KMAX from smem).
template <typename T, int VEC, int KT>
__global__ void __launch_bounds__(NT) k_skinny_fwd(GemmP p, int tpr, int rpb, int64_t rows_per_block) {
  __shared__ float w[KMAX * 512];
  const int b = blockIdx.y;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* Bw = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  T* C = reinterpret_cast<T*>(p.C) + (int64_t)b * p.c_bs;
  const int K = KT > 0 ? KT : (int)p.K, N = (int)p.N;
  for (int i = threadIdx.x; i < N * K; i += NT) w[(i % K) * N + i / K] = ldf(Bw + (int64_t)(i / K) * p.b_ld + i % K);
  __syncthreads();
  const int lane = threadIdx.x % tpr, rl = threadIdx.x / tpr;
  const int n0 = lane * VEC;
  float bias[VEC], sc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    bias[v] = (p.bias && n0 + v < N) ? p.bias[(int64_t)b * p.bias_bs + n0 + v] : 0.f;
    sc[v] = (p.scale && n0 + v < N) ? p.scale[(int64_t)b * p.scale_bs + n0 + v] : 1.f;   // fused BN apply
  }
  constexpr int KR = KT > 0 ? KT : 1;
  float wr[KR][VEC];
  if constexpr (KT > 0) {
#pragma unroll
    for (int k = 0; k < KT; ++k)
#pragma unroll
      for (int v = 0; v < VEC; ++v) wr[k][v] = n0 + v < N ? w[k * N + n0 + v] : 0.f;
  }
  const int64_t r0 = blockIdx.x * rows_per_block, r1 = min(p.M, r0 + rows_per_block);
  if constexpr (KT > 0) {
    // the block's narrow input rows are staged through smem XTILE rows at a
    // time (one cooperative copy), so the row loop only streams its stores
    __shared__ float xs[XTILE * KT];
    for (int64_t t0 = r0; t0 < r1; t0 += XTILE) {
      const int nr = (int)min((int64_t)XTILE, r1 - t0);
      __syncthreads();
      for (int i = threadIdx.x; i < nr * KT; i += NT) {
        const int rr = i / KT, k = i - rr * KT;
        xs[i] = ldf(A + (t0 + rr) * p.a_ld + k);
      }
      __syncthreads();
      if (n0 >= N) continue;
#pragma unroll 4
      for (int rr = rl; rr < nr; rr += rpb) {
        const int64_t m = t0 + rr;
        float o[VEC];
        const float* br = p.bias && p.bias_div > 0 ? p.bias + (int64_t)b * p.bias_bs + (m / p.bias_div) * p.bias_ld : nullptr;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < KT; ++k) acc = fmaf(xs[rr * KT + k], wr[k][v], acc);
          o[v] = act_fwd(fmaf(acc, sc[v], br ? br[n0 + v] : bias[v]), p.act, p.act_alpha);
        }
        st_vec<T, VEC>(C + m * p.c_ld + n0, o);
      }
    }
    return;
  }
  if (n0 >= N) return;
#pragma unroll 2
  for (int64_t m = r0 + rl; m < r1; m += rpb) {
    float a[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) a[k] = k < K ? ldf(A + m * p.a_ld + k) : 0.f;
    float o[VEC];
    const float* br = p.bias && p.bias_div > 0 ? p.bias + (int64_t)b * p.bias_bs + (m / p.bias_div) * p.bias_ld : nullptr;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < K) acc = fmaf(a[k], w[k * N + n0 + v], acc);
      o[v] = act_fwd(fmaf(acc, sc[v], br ? br[n0 + v] : bias[v]), p.act, p.act_alpha);
    }
    st_vec<T, VEC>(C + m * p.c_ld + n0, o);
  }
}

// dgrad, small N-out: C[m][j] = sum_n A[m][n] * Bw(n, j) with Bw MN-major
// (W[n][j]), j < NJ <= 4, reduction length K (layer width, e.g. 64, a
// multiple of VEC).  A row is read by TPR = K/VEC threads with one 16-B load
// each (coalesced), partial sums combined with shuffles.
template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_skinny_dgrad(GemmP p, int tpr) {
  __shared__ float4 w[1024];                           // w[n] = (W[n][0..3])
  __shared__ float4 m2s[32];                           // M2[k][0..3] (K2 <= 32)
  const int b = blockIdx.y;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* Bw = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  T* C = reinterpret_cast<T*>(p.C) + (int64_t)b * p.c_bs;
  const int Kr = (int)p.K, Nj = (int)p.N, K2 = (int)p.K2;
  for (int n = threadIdx.x; n < Kr; n += NT) {
    float e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = j < Nj ? ldf(Bw + (int64_t)n * p.b_ld + j) : 0.f;
    w[n] = make_float4(e[0], e[1], e[2], e[3]);
  }
  if (K2 > 0) {
    const float* M2 = reinterpret_cast<const float*>(p.Bm2) + (int64_t)b * p.b2_bs;
    for (int k = threadIdx.x; k < K2; k += NT) {
      float e[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) e[j] = j < Nj ? M2[k * Nj + j] : 0.f;
      m2s[k] = make_float4(e[0], e[1], e[2], e[3]);
    }
  }
  float bj[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) bj[j] = (p.bias && j < Nj) ? p.bias[(int64_t)b * p.bias_bs + j] : 0.f;
  __syncthreads();
  const int lane = threadIdx.x % tpr, rl = threadIdx.x / tpr, rpb = NT / tpr;
  const int n0 = lane * VEC;
  // this lane's W slice (VEC rows x 4 outputs) and M2 row in registers: no
  // shared-memory traffic in the row loop
  float4 wr[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) wr[v] = w[n0 + v];
  const float4 mr = (K2 > 0 && lane < K2) ? m2s[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  const T* A2 = K2 > 0 ? reinterpret_cast<const T*>(p.A2) + (int64_t)b * p.a2_bs : nullptr;
  const T* Mk = p.mask ? reinterpret_cast<const T*>(p.mask) + (int64_t)b * p.mask_bs : nullptr;
  const float neg = p.mask_act == HFTA_ACT_LEAKY_RELU ? p.mask_alpha : 0.f;
  constexpr int U = 2;                                 // rows per group in flight
  const int64_t stride = (int64_t)gridDim.x * rpb;
  for (int64_t m0 = blockIdx.x * (int64_t)rpb + rl; m0 < p.M; m0 += stride * U) {
    float av[U][VEC];
    float xa[U], mk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {                      // all loads of U rows issued up front
      const int64_t m = m0 + u * stride;
      const bool ok = m < p.M;
      if (ok) ld_vec<T, VEC>(A + m * p.a_ld + n0, av[u]);
      else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) av[u][v] = 0.f;
      }
      xa[u] = (ok && lane < K2) ? ldf(A2 + m * p.a2_ld + lane) : 0.f;     // lane k holds x[m][k]
      mk[u] = (ok && Mk && lane < Nj) ? ldf(Mk + m * p.mask_ld + lane) : 1.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t m = m0 + u * stride;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        acc[0] = fmaf(av[u][v], wr[v].x, acc[0]); acc[1] = fmaf(av[u][v], wr[v].y, acc[1]);
        acc[2] = fmaf(av[u][v], wr[v].z, acc[2]); acc[3] = fmaf(av[u][v], wr[v].w, acc[3]);
      }
      // the Gram-form BN backward's X M2 term, one k per lane (mr = 0 on the other lanes)
      acc[0] = fmaf(xa[u], mr.x, acc[0]); acc[1] = fmaf(xa[u], mr.y, acc[1]);
      acc[2] = fmaf(xa[u], mr.z, acc[2]); acc[3] = fmaf(xa[u], mr.w, acc[3]);
      for (int o = tpr / 2; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
      if (m < p.M && lane < Nj) {                      // lane j stores column j
        float vj = acc[0];
#pragma unroll
        for (int j = 1; j < 4; ++j)
          if (lane == j) vj = acc[j];
        vj += bj[0];
#pragma unroll
        for (int j = 1; j < 4; ++j)
          if (lane == j) vj += bj[j] - bj[0];
        if (Mk) vj *= mk[u] > 0.f ? 1.f : neg;
        stf(C + m * p.c_ld + lane, vj);
      }
    }
  }
}

// dgrad fallback (K not a power-of-two multiple of the vector width): thread per row.
template <typename T>
__global__ void __launch_bounds__(NT) k_skinny_dgrad_row(GemmP p) {
  const int b = blockIdx.y;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* Bw = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  T* C = reinterpret_cast<T*>(p.C) + (int64_t)b * p.c_bs;
  for (int64_t m = blockIdx.x * (int64_t)NT + threadIdx.x; m < p.M; m += (int64_t)gridDim.x * NT) {
    for (int j = 0; j < (int)p.N; ++j) {
      float acc = 0.f;
      for (int64_t n = 0; n < p.K; ++n) acc = fmaf(ldf(A + m * p.a_ld + n), ldf(Bw + n * p.b_ld + j), acc);
      stf(C + m * p.c_ld + j, acc);
    }
  }
}

// dgrad, thread per row (bf16, K = 8 KB8): C[m][j] = sum_n A[m][n] W[n][j] (+ A2[m] M2
// + bias, x mask) with W (and M2) broadcast from smem; each thread streams its
// whole A row with KB8 independent 16-B loads, so no cross-lane reduction is
// needed and every row's bytes are in flight at once.
template <int KB8>
__global__ void __launch_bounds__(NT) k_skinny_dgrad_rows(GemmP p) {
  __shared__ float4 w[KB8 * 8];                        // w[n] = (W[n][0..3])
  __shared__ float4 m2s[8];
  const int b = blockIdx.y;
  const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(p.A) + (int64_t)b * p.a_bs;
  const __nv_bfloat16* Bw = reinterpret_cast<const __nv_bfloat16*>(p.Bm) + (int64_t)b * p.b_bs;
  __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)b * p.c_bs;
  const int Nj = (int)p.N, K2 = (int)p.K2;
  for (int n = threadIdx.x; n < KB8 * 8; n += NT) {
    float e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = j < Nj ? ldf(Bw + (int64_t)n * p.b_ld + j) : 0.f;
    w[n] = make_float4(e[0], e[1], e[2], e[3]);
  }
  if (K2 > 0 && threadIdx.x < K2) {
    const float* M2 = reinterpret_cast<const float*>(p.Bm2) + (int64_t)b * p.b2_bs;
    float e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = j < Nj ? M2[threadIdx.x * Nj + j] : 0.f;
    m2s[threadIdx.x] = make_float4(e[0], e[1], e[2], e[3]);
  }
  float bj[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) bj[j] = (p.bias && j < Nj) ? p.bias[(int64_t)b * p.bias_bs + j] : 0.f;
  __syncthreads();
  const __nv_bfloat16* A2 = K2 > 0 ? reinterpret_cast<const __nv_bfloat16*>(p.A2) + (int64_t)b * p.a2_bs : nullptr;
  const __nv_bfloat16* Mk = p.mask ? reinterpret_cast<const __nv_bfloat16*>(p.mask) + (int64_t)b * p.mask_bs : nullptr;
  const float neg = p.mask_act == HFTA_ACT_LEAKY_RELU ? p.mask_alpha : 0.f;
  for (int64_t m = blockIdx.x * (int64_t)NT + threadIdx.x; m < p.M; m += (int64_t)gridDim.x * NT) {
    uint4 raw[KB8];
    const uint4* ar = reinterpret_cast<const uint4*>(A + m * p.a_ld);
#pragma unroll
    for (int q = 0; q < KB8; ++q) raw[q] = __ldg(ar + q);
    float xa[8], mk[4];
#pragma unroll
    for (int k = 0; k < 8; ++k) xa[k] = k < K2 ? __bfloat162float(A2[m * p.a2_ld + k]) : 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) mk[j] = (Mk && j < Nj) ? __bfloat162float(Mk[m * p.mask_ld + j]) : 1.f;
    float acc[4] = {bj[0], bj[1], bj[2], bj[3]};
#pragma unroll
    for (int q = 0; q < KB8; ++q) {
      const uint32_t u4[4] = {raw[q].x, raw[q].y, raw[q].z, raw[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float lo, hi;
        unpack_bf2(u4[e], lo, hi);
        const float4 w0 = w[q * 8 + 2 * e], w1 = w[q * 8 + 2 * e + 1];
        acc[0] = fmaf(lo, w0.x, acc[0]); acc[1] = fmaf(lo, w0.y, acc[1]);
        acc[2] = fmaf(lo, w0.z, acc[2]); acc[3] = fmaf(lo, w0.w, acc[3]);
        acc[0] = fmaf(hi, w1.x, acc[0]); acc[1] = fmaf(hi, w1.y, acc[1]);
        acc[2] = fmaf(hi, w1.z, acc[2]); acc[3] = fmaf(hi, w1.w, acc[3]);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < K2) {
        const float4 mv = m2s[k];
        acc[0] = fmaf(xa[k], mv.x, acc[0]); acc[1] = fmaf(xa[k], mv.y, acc[1]);
        acc[2] = fmaf(xa[k], mv.z, acc[2]); acc[3] = fmaf(xa[k], mv.w, acc[3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j < Nj) {
        const float vj = Mk ? acc[j] * (mk[j] > 0.f ? 1.f : neg) : acc[j];
        C[m * p.c_ld + j] = __float2bfloat16_rn(vj);
      }
    }
  }
}

// wgrad, small K-out: part[chunk][b][n][k] = sum_{rows in chunk} A(n, r) * Bx(k, r), both MN-major:
// A = dY[r][n] (n < N), Bx = X[r][k] (k < K_out <= 3).  Thread = (row lane, VEC n-columns).
// With p.colsum, a 4th column k = 3 accumulates sum_r A(n, r) (x = 1): the fused dbias.
template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_skinny_wgrad(GemmP p, int tpr, int rpb, int64_t rows_per_chunk,
                                                     float* __restrict__ part) {
  __shared__ float red[NT * VEC * 4];
  const int b = blockIdx.y, chunk = blockIdx.x;
  const T* A = reinterpret_cast<const T*>(p.A) + (int64_t)b * p.a_bs;
  const T* X = reinterpret_cast<const T*>(p.Bm) + (int64_t)b * p.b_bs;
  const int N = (int)p.M, Ko = (int)p.N;               // dW is [N][Ko]
  const int KE = p.colsum ? Ko + 1 : Ko;              // columns written to part
  const int lane = threadIdx.x % tpr, rl = threadIdx.x / tpr;
  const int n0 = lane * VEC;
  float acc[VEC][4];
#pragma unroll
  for (int v = 0; v < VEC; ++v)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[v][k] = 0.f;
  {
    // the narrow operand X (<= 3 columns) is staged through smem XTILE rows at
    // a time (one cooperative copy): the row loop only streams dY
    __shared__ float xs[XTILE * 3];
    const int64_t r0 = (int64_t)chunk * rows_per_chunk, r1 = min(p.K, r0 + rows_per_chunk);
    for (int64_t t0 = r0; t0 < r1; t0 += XTILE) {
      const int nr = (int)min((int64_t)XTILE, r1 - t0);
      __syncthreads();
      for (int i = threadIdx.x; i < nr * 3; i += NT) {
        const int rr = i / 3, k = i - rr * 3;
        xs[i] = k < Ko ? ldf(X + (t0 + rr) * p.b_ld + k) : 0.f;
      }
      __syncthreads();
      if (n0 >= N) continue;
#pragma unroll 4
      for (int rr = rl; rr < nr; rr += rpb) {
        float dy[VEC];
        ld_vec<T, VEC>(A + (t0 + rr) * p.a_ld + n0, dy);
        const float x0 = xs[rr * 3], x1 = xs[rr * 3 + 1], x2 = xs[rr * 3 + 2];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          acc[v][0] = fmaf(dy[v], x0, acc[v][0]);
          acc[v][1] = fmaf(dy[v], x1, acc[v][1]);
          acc[v][2] = fmaf(dy[v], x2, acc[v][2]);
          acc[v][3] += dy[v];
        }
      }
    }
  }
  const int cb = tpr * VEC;
#pragma unroll
  for (int v = 0; v < VEC; ++v)
#pragma unroll
    for (int k = 0; k < 4; ++k) red[(rl * cb + lane * VEC + v) * 4 + k] = acc[v][k];
  __syncthreads();
  for (int e = threadIdx.x; e < cb * 4; e += NT) {
    const int col = e / 4, k = e % 4;
    const int kk = k == 3 ? Ko : k;                   // slot 3 = column sum
    if (col >= N || (k < 3 && k >= Ko) || (k == 3 && !p.colsum)) continue;
    float sum = 0.f;
    for (int r = 0; r < rpb; ++r) sum += red[(r * cb + col) * 4 + k];
    part[(((int64_t)chunk * p.B + b) * N + col) * KE + kk] = sum;
  }
}

__global__ void k_skinny_wgrad_fin(GemmP p, int chunks, const float* __restrict__ part) {
  const int N = (int)p.M, Ko = (int)p.N;
  const int KE = p.colsum ? Ko + 1 : Ko;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)p.B * N * KE) return;
  int64_t b = i / (N * KE), rem = i % (N * KE), n = rem / KE, k = rem % KE;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += part[(((int64_t)c * p.B + b) * N + n) * KE + k];
  float* o = k < Ko ? reinterpret_cast<float*>(p.C) + b * p.c_bs + n * p.c_ld + k : p.colsum + b * p.colsum_bs + n;
  const int acc = k < Ko ? p.accumulate : p.colsum_acc;
  *o = acc ? *o + (float)s : (float)s;
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
    if (lane == 0) {
#pragma unroll
      for (int n = 0; n < KMAX; ++n) {
        if (n >= p.N) break;
        float v = acc[n];
        if (p.bias) v += p.bias[(int64_t)b * p.bias_bs + (p.bias_div > 0 ? (m / p.bias_div) * p.bias_ld : 0) + n];
        stf(C + m * p.c_ld + n, v);
      }
    }
  }
}

// gemv fwd with 16-B vectors (bf16, K % 8 == 0, aligned rows): lane l reads
// A[m][8 l + 256 i ..] and B[n][..] as uint4 -- a warp moves 512 B per step.
template <int NMAX>
__global__ void k_gemv_fwd_v8(GemmP p) {
  const int b = blockIdx.y;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(p.A) + (int64_t)b * p.a_bs;
  const __nv_bfloat16* Bw = reinterpret_cast<const __nv_bfloat16*>(p.Bm) + (int64_t)b * p.b_bs;
  __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)b * p.c_bs;
  for (int64_t m = warp; m < p.M; m += nwarps) {
    float acc[NMAX];
#pragma unroll
    for (int n = 0; n < NMAX; ++n) acc[n] = 0.f;
    const uint4* ar = reinterpret_cast<const uint4*>(A + m * p.a_ld);
    for (int64_t q = lane; q < p.K / 8; q += 32) {
      float a[8];
      ld_vec<__nv_bfloat16, 8>(reinterpret_cast<const __nv_bfloat16*>(ar + q), a);
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n >= p.N) break;
        float w[8];
        ld_vec<__nv_bfloat16, 8>(Bw + n * p.b_ld + q * 8, w);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[n] = fmaf(a[e], w[e], acc[n]);
      }
    }
#pragma unroll
    for (int n = 0; n < NMAX; ++n) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int n = 0; n < NMAX; ++n) {
        if (n >= p.N) break;
        float v = acc[n];
        if (p.bias) v += p.bias[(int64_t)b * p.bias_bs + (p.bias_div > 0 ? (m / p.bias_div) * p.bias_ld : 0) + n];
        stf(C + m * p.c_ld + n, v);
      }
    }
  }
}

// outer-product-like small K with B MN-major ([K][N], n contiguous), bf16,
// N % 8 == 0: thread = (row m, 8 consecutive n), 16-B loads / stores.
__global__ void k_smallk_v8(GemmP p) {
  const int b = blockIdx.y;
  const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(p.A) + (int64_t)b * p.a_bs;
  const __nv_bfloat16* Bw = reinterpret_cast<const __nv_bfloat16*>(p.Bm) + (int64_t)b * p.b_bs;
  __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)b * p.c_bs;
  const int64_t nv = p.N / 8, tot = p.M * nv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / nv, n0 = (i - m * nv) * 8;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int64_t k = 0; k < p.K; ++k) {
      const float a = ldf(A + m * p.a_ld + k);
      float w[8];
      ld_vec<__nv_bfloat16, 8>(Bw + k * p.b_ld + n0, w);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fmaf(a, w[e], acc[e]);
    }
    if (p.bias) {
      const float* br = p.bias + (int64_t)b * p.bias_bs + (p.bias_div > 0 ? (m / p.bias_div) * p.bias_ld : 0) + n0;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += br[e];
    }
    st_vec<__nv_bfloat16, 8>(C + m * p.c_ld + n0, acc);
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
#pragma unroll
  for (int m = 0; m < KMAX; ++m)
    if (m < p.M) part[(((int64_t)chunk * p.B + b) * p.M + m) * p.N + n] = acc[m];
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
static bool plain(const GemmP& p) { return !p.scale && p.act == HFTA_ACT_NONE && !p.mask && p.K2 == 0; }
static bool gemv_fwd_ok(const GemmP& p) { return p.a_kmajor && p.b_kmajor && p.N <= KMAX && p.splits == 1 && plain(p); }
static bool smallk_ok(const GemmP& p) { return p.a_kmajor && p.K <= KMAX && p.splits == 1 && !p.accumulate && plain(p); }
static bool smallm_wgrad_ok(const GemmP& p) { return !p.a_kmajor && !p.b_kmajor && p.M <= KMAX; }
bool skinny_fwd_ok_base(const GemmP& p) { return p.a_kmajor && p.b_kmajor && p.K <= KMAX && p.N <= 512 && p.splits == 1; }
bool skinny_dgrad_ok(const GemmP& p) {
  return p.a_kmajor && !p.b_kmajor && p.N <= 4 && p.K <= 1024 && p.splits == 1 && p.K % 8 == 0 && p.a_ld % 8 == 0 &&
         p.K / 8 <= 32;
}
bool skinny_wgrad_ok_base(const GemmP& p) { return !p.a_kmajor && !p.b_kmajor && p.N <= 3 && p.M <= 128; }
bool skinny_fwd_ok(const GemmP& p) { return skinny_fwd_ok_base(p) || gemv_fwd_ok(p) || smallk_ok(p); }
bool skinny_wgrad_ok(const GemmP& p) { return skinny_wgrad_ok_base(p) || smallm_wgrad_ok(p); }

static int64_t smallm_chunks(int B, int64_t rows, int64_t N) {
  const int64_t colblocks = cdiv(N, 256);
  return std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * 148, (int64_t)B * colblocks), cdiv(rows, 64)));
}

size_t skinny_wgrad_ws(int B, int64_t rows, int64_t N, int64_t Ko) {
  int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(16 * 148, B), cdiv(rows, 1024)));
  size_t a = (size_t)chunks * B * N * (Ko + 1) * sizeof(float);   // + fused column sums
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
      const bool v8 = bf && p.K % 8 == 0 && p.a_ld % 8 == 0 && p.b_ld % 8 == 0 && p.a_bs % 8 == 0 &&
                      p.b_bs % 8 == 0 && aligned16(p.A) && aligned16(p.Bm);
      if (v8) k_gemv_fwd_v8<KMAX><<<grid, 256, 0, s>>>(p);
      else if (bf) k_gemv_fwd<__nv_bfloat16><<<grid, 256, 0, s>>>(p);
      else k_gemv_fwd<float><<<grid, 256, 0, s>>>(p);
      count_launches(1);
      return post_launch(s, "gemm_gemv_fwd");
    }
    if (smallk_ok(p)) {
      dim3 grid((unsigned)std::min<int64_t>(cdiv(p.M * p.N, 256), 8192), p.B);
      if (bf && !p.b_kmajor && p.N % 8 == 0 && p.b_ld % 8 == 0 && p.b_bs % 8 == 0 && p.c_ld % 8 == 0 &&
          p.c_bs % 8 == 0 && aligned16(p.Bm) && aligned16(p.C)) {
        dim3 g8((unsigned)std::min<int64_t>(cdiv(p.M * p.N / 8, 256), 8192), p.B);
        k_smallk_v8<<<g8, 256, 0, s>>>(p);
        count_launches(1);
        return post_launch(s, "gemm_smallk");
      }
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
    int64_t blocks_per = std::max<int64_t>(1, std::min<int64_t>(cdiv(p.M, rpb * 4), cdiv(16 * 148, p.B)));
    int64_t rows_per_block = cdiv(p.M, blocks_per);
    dim3 grid((unsigned)cdiv(p.M, rows_per_block), p.B);
    const bool k3 = p.K == 3;
    if (bf) {
      if (vec == 8 && k3) k_skinny_fwd<__nv_bfloat16, 8, 3><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
      else if (vec == 8) k_skinny_fwd<__nv_bfloat16, 8, 0><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
      else k_skinny_fwd<__nv_bfloat16, 1, 0><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
    } else {
      if (vec == 4 && k3) k_skinny_fwd<float, 4, 3><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
      else if (vec == 4) k_skinny_fwd<float, 4, 0><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
      else k_skinny_fwd<float, 1, 0><<<grid, NT, 0, s>>>(p, tpr, rpb, rows_per_block);
    }
    count_launches(1);
    return post_launch(s, "gemm_skinny_fwd");
  }
  if (skinny_dgrad_ok(p)) {
    if (bf && aligned16(p.A) && p.a_bs % 8 == 0 && p.a_ld % 8 == 0 && p.K2 <= 8 && (p.K == 64 || p.K == 128)) {
      dim3 grid((unsigned)std::min<int64_t>(cdiv(p.M, NT), cdiv(32 * 148, p.B)), p.B);
      if (p.K == 64) k_skinny_dgrad_rows<8><<<grid, NT, 0, s>>>(p);
      else k_skinny_dgrad_rows<16><<<grid, NT, 0, s>>>(p);
      count_launches(1);
      return post_launch(s, "gemm_skinny_dgrad_rows");
    }
    const bool v = aligned16(p.A) && (p.a_bs % 8 == 0);
    const int vec = v ? (bf ? 8 : 4) : 1;
    int tpr = 1;
    while (tpr * vec < p.K && tpr < 32) tpr <<= 1;     // K / vec lanes per row (power of 2 up to 32)
    if (tpr * vec != p.K) { tpr = 1; }
    if (tpr > 1 && (tpr < p.N || tpr < p.K2 || p.K2 > 32)) tpr = 1;   // lane j stores column j, lane k holds x[k]
    const int rpb = NT / tpr;
    dim3 grid((unsigned)std::min<int64_t>(cdiv(p.M, rpb), cdiv(16 * 148, p.B)), p.B);
    HFTA_REQUIRE(tpr > 1 || plain(p), HFTA_ERR_UNSUPPORTED, "skinny dgrad: fused terms need K %% 8 == 0");
    if (tpr == 1) {   // generic: one thread per row, the whole row
      if (bf) k_skinny_dgrad_row<__nv_bfloat16><<<grid, NT, 0, s>>>(p);
      else k_skinny_dgrad_row<float><<<grid, NT, 0, s>>>(p);
    } else if (bf) {
      k_skinny_dgrad<__nv_bfloat16, 8><<<grid, NT, 0, s>>>(p, tpr);
    } else {
      k_skinny_dgrad<float, 4><<<grid, NT, 0, s>>>(p, tpr);
    }
    count_launches(1);
    return post_launch(s, "gemm_skinny_dgrad");
  }
  if (skinny_wgrad_ok_base(p)) {
    const int64_t rows = p.K, N = p.M, Ko = p.N;
    int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(16 * 148, p.B), cdiv(rows, 1024)));
    size_t need = (size_t)chunks * p.B * N * (p.colsum ? Ko + 1 : Ko) * sizeof(float);
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
    k_skinny_wgrad_fin<<<(unsigned)cdiv((int64_t)p.B * N * (Ko + 1), 256), 256, 0, s>>>(p, (int)chunks, part);
    count_launches(2);
    return post_launch(s, "gemm_skinny_wgrad");
  }
  return fail(HFTA_ERR_UNSUPPORTED, "gemm_skinny: shape not skinny");
}

}  // namespace hfta
