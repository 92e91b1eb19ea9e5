// loss.cu -- fused per-model losses (K8d).  App. C: the fused
// loss L = (1/B) sum_b l_b (Eq. 1, sum over b = 0..B-1, reading R8) needs
// scaling by B so that each model receives its serial gradient (Eq. 3).  The
// kernels write d l_b / d logits directly -- analytically the same as
// back-propagating B*L (reading R9) -- plus loss[B] and L.
#include "common.cuh"

namespace hfta {
namespace {

constexpr int NT = 256;
constexpr int ROWS_PER_BLOCK = 64;

// grid (chunks, B): one warp per row; lanes stride over the K classes.
template <typename T>
__global__ void __launch_bounds__(NT) k_nll(int64_t rows, int64_t K, const T* __restrict__ Z, int64_t zbs,
                                            int64_t zld, const int32_t* __restrict__ y, int64_t ybs,
                                            T* __restrict__ dZ, int64_t dbs, int64_t dld, float* __restrict__ part) {
  __shared__ float wsum[NT / 32];
  const int b = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float inv_rows = 1.0f / (float)rows;
  float lsum = 0.f;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS_PER_BLOCK;
  const int64_t r1 = min(rows, r0 + ROWS_PER_BLOCK);
  for (int64_t r = r0 + warp; r < r1; r += NT / 32) {
    const T* z = Z + (int64_t)b * zbs + r * zld;
    float m = -INFINITY;
    for (int64_t k = lane; k < K; k += 32) m = fmaxf(m, ldf(z + k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float se = 0.f;
    for (int64_t k = lane; k < K; k += 32) se += expf(ldf(z + k) - m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const float lse = m + logf(se);
    const int32_t t = y[(int64_t)b * ybs + r];
    if (lane == 0) lsum += lse - ldf(z + t);
    T* d = dZ + (int64_t)b * dbs + r * dld;
    for (int64_t k = lane; k < K; k += 32) {
      float pk = expf(ldf(z + k) - lse);
      stf(d + k, (pk - (k == t ? 1.f : 0.f)) * inv_rows);
    }
  }
  if (lane == 0) wsum[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < NT / 32; ++w) s += wsum[w];
    part[(int64_t)b * gridDim.x + blockIdx.x] = s;
  }
}

// bf16, K <= 8 KV classes, 16-B rows: one thread per row holding the whole
// row (KV 16-B loads in flight; no shuffles), grid (cdiv(rows, NT), B); the
// block's loss partial lands in part[b][blockIdx.x] (chunks of NT rows).
template <int KV>
__global__ void __launch_bounds__(NT) k_nll_rows(int64_t rows, int K, const __nv_bfloat16* __restrict__ Z,
                                                 int64_t zbs, int64_t zld, const int32_t* __restrict__ y,
                                                 int64_t ybs, __nv_bfloat16* __restrict__ dZ, int64_t dbs,
                                                 int64_t dld, float* __restrict__ part, int64_t part_stride) {
  __shared__ float wsum[NT / 32];
  const int b = blockIdx.y;
  const int64_t r = (int64_t)blockIdx.x * NT + threadIdx.x;
  float lterm = 0.f;
  if (r < rows) {
    const uint4* zr = reinterpret_cast<const uint4*>(Z + (int64_t)b * zbs + r * zld);
    uint4 raw[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) raw[q] = __ldg(zr + q);
    const int32_t t = y[(int64_t)b * ybs + r];
    float v[KV * 8];
#pragma unroll
    for (int q = 0; q < KV; ++q) {
      const uint32_t u[4] = {raw[q].x, raw[q].y, raw[q].z, raw[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        v[8 * q + 2 * e] = __uint_as_float(u[e] << 16);
        v[8 * q + 2 * e + 1] = __uint_as_float(u[e] & 0xffff0000u);
      }
    }
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < KV * 8; ++k)
      if (k < K) m = fmaxf(m, v[k]);
    float se = 0.f;
#pragma unroll
    for (int k = 0; k < KV * 8; ++k)
      if (k < K) se += expf(v[k] - m);
    const float lse = m + logf(se);
    float zt = 0.f;
#pragma unroll
    for (int k = 0; k < KV * 8; ++k)
      if (k == t) zt = v[k];
    lterm = lse - zt;
    const float inv_rows = 1.0f / (float)rows;
    uint4* dr = reinterpret_cast<uint4*>(dZ + (int64_t)b * dbs + r * dld);
#pragma unroll
    for (int q = 0; q < KV; ++q) {
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float g[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = 8 * q + 2 * e + h;
          g[h] = k < K ? (expf(v[k] - lse) - (k == t ? 1.f : 0.f)) * inv_rows : 0.f;
        }
        o[e] = pack_bf2(g[0], g[1]);
      }
      dr[q] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lterm += __shfl_xor_sync(0xffffffffu, lterm, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = lterm;
  __syncthreads();
  if (threadIdx.x == 0) {
    float sum = 0.f;
    for (int w = 0; w < NT / 32; ++w) sum += wsum[w];
    part[(int64_t)b * part_stride + blockIdx.x] = sum;
  }
}

template <typename T>
__global__ void __launch_bounds__(NT) k_mse(int64_t rows, int64_t C, const T* __restrict__ A, int64_t abs_,
                                            int64_t ald, const float* __restrict__ Tg, int64_t tbs, int64_t tld,
                                            T* __restrict__ dA, int64_t dbs, int64_t dld, float* __restrict__ part) {
  __shared__ float red[NT];
  const int b = blockIdx.y;
  const float scale = 2.0f / ((float)rows * (float)C);
  float s = 0.f;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS_PER_BLOCK;
  const int64_t r1 = min(rows, r0 + ROWS_PER_BLOCK);
  const int64_t n = (r1 - r0) * C;
  for (int64_t e = threadIdx.x; e < n; e += NT) {
    int64_t r = r0 + e / C, c = e % C;
    float d = ldf(A + (int64_t)b * abs_ + r * ald + c) - Tg[(int64_t)b * tbs + r * tld + c];
    s = fmaf(d, d, s);
    stf(dA + (int64_t)b * dbs + r * dld + c, d * scale);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)b * gridDim.x + blockIdx.x] = red[0];
}

template <typename T>
__global__ void __launch_bounds__(NT) k_bce(int64_t rows, const T* __restrict__ Z, int64_t zbs, int64_t zld,
                                            float y, T* __restrict__ dZ, int64_t dbs, int64_t dld,
                                            float* __restrict__ part) {
  __shared__ float red[NT];
  const int b = blockIdx.y;
  float s = 0.f;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS_PER_BLOCK;
  const int64_t r1 = min(rows, r0 + ROWS_PER_BLOCK);
  for (int64_t r = r0 + threadIdx.x; r < r1; r += NT) {
    const float z = ldf(Z + (int64_t)b * zbs + r * zld);
    // log p = -softplus(-z), log(1-p) = -softplus(z), both clamped at -100 (BCELoss)
    const float sp_pos = fmaxf(z, 0.f) + log1pf(expf(-fabsf(z)));     // softplus(z)
    const float lp = fmaxf(-(sp_pos - z), -100.f);
    const float l1p = fmaxf(-sp_pos, -100.f);
    s -= y * lp + (1.f - y) * l1p;
    // BCELoss backward x sigmoid' (reading R29): (p - y) q / max(q, 1e-12),
    // q = p (1 - p) = sigmoid(z) sigmoid(-z), all from e = exp(-|z|) so that a
    // saturated logit keeps its exact (tiny) q instead of rounding p to 1
    const float e = expf(-fabsf(z));
    const float ri = 1.f / (1.f + e);
    const float sg_pos = z >= 0.f ? ri : e * ri;                       // sigmoid(z)
    const float sg_neg = z >= 0.f ? e * ri : ri;                       // sigmoid(-z)
    const float q = e * ri * ri;
    const float pmy = (y == 1.f) ? -sg_neg : sg_pos - y;
    const float g = q >= 1e-12f ? pmy : pmy * (q * 1e12f);
    stf(dZ + (int64_t)b * dbs + r * dld, g / (float)rows);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = NT / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(int64_t)b * gridDim.x + blockIdx.x] = red[0];
}

// loss[b] = scale * sum_chunks part (fixed order, fp64); mean over b.  One
// warp per model: lane l sums chunks l, l + 32, ... in order, then a fixed
// xor tree (deterministic); thread 0 sums the B losses in order.
__global__ void __launch_bounds__(1024) k_loss_fin(int B, int chunks, const float* __restrict__ part, double scale,
                                                   float* __restrict__ loss, float* __restrict__ mean_loss) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int b = warp; b < B; b += nw) {
    double s = 0.0;
    for (int k = lane; k < chunks; k += 32) s += part[(int64_t)b * chunks + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) loss[b] = (float)(s * scale);
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

size_t hfta_loss_workspace(int B, int64_t rows) {
  if (B < 1 || rows < 1) return 0;
  return align_up((size_t)B * cdiv(rows, ROWS_PER_BLOCK) * sizeof(float), 256);
}

hfta_status hfta_loss_nll(int B, int64_t rows, int64_t K, hfta_dtype dt, hfta_in logits, const int32_t* labels,
                          int64_t labels_bstride, float* loss, float* mean_loss, hfta_out dlogits, void* ws,
                          size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(rows >= 1 && K >= 1 && logits.ptr && labels && loss && dlogits.ptr, HFTA_ERR_INVALID_VALUE,
               "loss_nll: bad args");
  HFTA_REQUIRE(logits.ld >= K && dlogits.ld >= K && (dlogits.bstride > 0 || B == 1), HFTA_ERR_SHAPE,
               "loss_nll: strides");
  size_t need = hfta_loss_workspace(B, rows);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "loss_nll: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  int chunks = (int)cdiv(rows, ROWS_PER_BLOCK);
  float* part = reinterpret_cast<float*>(ws);
  const bool rows_path = dt == HFTA_BF16 && K <= 64 && logits.ld % 8 == 0 && dlogits.ld % 8 == 0 &&
                         logits.bstride % 8 == 0 && dlogits.bstride % 8 == 0 && aligned16(logits.ptr) &&
                         aligned16(dlogits.ptr) && cdiv(K, 8) * 8 <= std::min(logits.ld, dlogits.ld);
  if (rows_path) {                              // thread per row (seg: 50 classes per point)
    const int nb = (int)cdiv(rows, NT);
    const int kv = (int)cdiv(K, 8);
    dim3 g2((unsigned)nb, (unsigned)B);
#define HFTA_NLL_ROWS(KVC)                                                                                          \
  k_nll_rows<KVC><<<g2, NT, 0, s>>>(rows, (int)K, (const __nv_bfloat16*)logits.ptr, logits.bstride, logits.ld, labels, \
                                    labels_bstride, (__nv_bfloat16*)dlogits.ptr, dlogits.bstride, dlogits.ld, part, nb)
    switch (kv) {
      case 1: HFTA_NLL_ROWS(1); break;
      case 2: HFTA_NLL_ROWS(2); break;
      case 3: HFTA_NLL_ROWS(3); break;
      case 4: HFTA_NLL_ROWS(4); break;
      case 5: HFTA_NLL_ROWS(5); break;
      case 6: HFTA_NLL_ROWS(6); break;
      case 7: HFTA_NLL_ROWS(7); break;
      default: HFTA_NLL_ROWS(8); break;
    }
#undef HFTA_NLL_ROWS
    k_loss_fin<<<1, 1024, 0, s>>>(B, nb, part, 1.0 / (double)rows, loss, mean_loss);
    count_launches(2);
    return post_launch(s, "hfta_loss_nll");
  }
  dim3 grid(chunks, B);
  if (dt == HFTA_F32)
    k_nll<float><<<grid, NT, 0, s>>>(rows, K, (const float*)logits.ptr, logits.bstride, logits.ld, labels,
                                    labels_bstride, (float*)dlogits.ptr, dlogits.bstride, dlogits.ld, part);
  else
    k_nll<__nv_bfloat16><<<grid, NT, 0, s>>>(rows, K, (const __nv_bfloat16*)logits.ptr, logits.bstride, logits.ld,
                                            labels, labels_bstride, (__nv_bfloat16*)dlogits.ptr, dlogits.bstride,
                                            dlogits.ld, part);
  k_loss_fin<<<1, 1024, 0, s>>>(B, chunks, part, 1.0 / (double)rows, loss, mean_loss);
  count_launches(2);
  return post_launch(s, "hfta_loss_nll");
}

hfta_status hfta_loss_bce_logits(int B, int64_t rows, hfta_dtype dt, hfta_in Z, float target, float* loss,
                                 float* mean_loss, hfta_out dZ, void* ws, size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(rows >= 1 && Z.ptr && loss && dZ.ptr, HFTA_ERR_INVALID_VALUE, "loss_bce: bad args");
  HFTA_REQUIRE(dZ.bstride > 0 || B == 1, HFTA_ERR_SHAPE, "loss_bce: dZ stride");
  size_t need = hfta_loss_workspace(B, rows);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "loss_bce: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  int chunks = (int)cdiv(rows, ROWS_PER_BLOCK);
  float* part = reinterpret_cast<float*>(ws);
  dim3 grid(chunks, B);
  if (dt == HFTA_F32)
    k_bce<float><<<grid, NT, 0, s>>>(rows, (const float*)Z.ptr, Z.bstride, Z.ld, target, (float*)dZ.ptr, dZ.bstride,
                                    dZ.ld, part);
  else
    k_bce<__nv_bfloat16><<<grid, NT, 0, s>>>(rows, (const __nv_bfloat16*)Z.ptr, Z.bstride, Z.ld, target,
                                            (__nv_bfloat16*)dZ.ptr, dZ.bstride, dZ.ld, part);
  k_loss_fin<<<1, 1024, 0, s>>>(B, chunks, part, 1.0 / (double)rows, loss, mean_loss);
  count_launches(2);
  return post_launch(s, "hfta_loss_bce_logits");
}

hfta_status hfta_loss_mse(int B, int64_t rows, int64_t C, hfta_dtype dt, hfta_in A, const float* T, int64_t T_bstride,
                          int64_t T_ld, float* loss, float* mean_loss, hfta_out dA, void* ws, size_t ws_bytes,
                          hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(rows >= 1 && C >= 1 && A.ptr && T && loss && dA.ptr, HFTA_ERR_INVALID_VALUE, "loss_mse: bad args");
  HFTA_REQUIRE(A.ld >= C && T_ld >= C && dA.ld >= C && (dA.bstride > 0 || B == 1), HFTA_ERR_SHAPE,
               "loss_mse: strides");
  size_t need = hfta_loss_workspace(B, rows);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "loss_mse: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  int chunks = (int)cdiv(rows, ROWS_PER_BLOCK);
  float* part = reinterpret_cast<float*>(ws);
  dim3 grid(chunks, B);
  if (dt == HFTA_F32)
    k_mse<float><<<grid, NT, 0, s>>>(rows, C, (const float*)A.ptr, A.bstride, A.ld, T, T_bstride, T_ld,
                                    (float*)dA.ptr, dA.bstride, dA.ld, part);
  else
    k_mse<__nv_bfloat16><<<grid, NT, 0, s>>>(rows, C, (const __nv_bfloat16*)A.ptr, A.bstride, A.ld, T, T_bstride,
                                            T_ld, (__nv_bfloat16*)dA.ptr, dA.bstride, dA.ld, part);
  k_loss_fin<<<1, 1024, 0, s>>>(B, chunks, part, 1.0 / ((double)rows * (double)C), loss, mean_loss);
  count_launches(2);
  return post_launch(s, "hfta_loss_mse");
}

}  // extern "C"
