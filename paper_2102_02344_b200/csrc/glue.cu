// glue.cu -- PointNet glue kernels (K8b/K8c) and segmented column sums.
//  * input transform x' = x * T (STN, the cited PointNet model; reading R1)
//  * dropout with a Philox4x32-10 counter-based mask (App. B row Dropout,
//    P:L1295-1296; reading R14)
//  * segmented column sums (dbias, and the per-sample sums of the seg
//    split-weight rewrite)
#include "common.cuh"

namespace hfta {
namespace {

// ---------------------------------------------------- transform points --
template <typename T>
__global__ void k_transform_fwd(int64_t N, int64_t L, const float* __restrict__ X, int64_t xbs, int64_t xld,
                                const float* __restrict__ F, int64_t fbs, int64_t fld, int add_id, T* __restrict__ Y,
                                int64_t ybs, int64_t yld) {
  const int b = blockIdx.y;
  const int64_t R = N * L;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = r / L;
    const float* t = F + (int64_t)b * fbs + n * fld;
    const float* x = X + (int64_t)b * xbs + r * xld;
    float x0 = x[0], x1 = x[1], x2 = x[2];
    T* y = Y + (int64_t)b * ybs + r * yld;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      float t0 = ldf(t + 0 * 3 + j) + (add_id && j == 0 ? 1.f : 0.f);
      float t1 = ldf(t + 1 * 3 + j) + (add_id && j == 1 ? 1.f : 0.f);
      float t2 = ldf(t + 2 * 3 + j) + (add_id && j == 2 ? 1.f : 0.f);
      stf(y + j, fmaf(x0, t0, fmaf(x1, t1, x2 * t2)));
    }
  }
}

// dF[b][n][i*3+j] = sum_l x[n*L+l][i] * dY[b][n*L+l][j]; one block per (n, b).
template <typename T>
__global__ void k_transform_bwd(int64_t N, int64_t L, const float* __restrict__ X, int64_t xbs, int64_t xld,
                                const T* __restrict__ dY, int64_t dbs, int64_t dld, float* __restrict__ dF,
                                int64_t fbs, int64_t fld) {
  __shared__ float red[9][256];
  const int b = blockIdx.y;
  const int64_t n = blockIdx.x;
  float acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.f;
  for (int64_t l = threadIdx.x; l < L; l += blockDim.x) {
    const int64_t r = n * L + l;
    const float* x = X + (int64_t)b * xbs + r * xld;
    const T* d = dY + (int64_t)b * dbs + r * dld;
    float dj[3] = {ldf(d), ldf(d + 1), ldf(d + 2)};
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) acc[i * 3 + j] = fmaf(x[i], dj[j], acc[i * 3 + j]);
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) red[q][threadIdx.x] = acc[q];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
#pragma unroll
      for (int q = 0; q < 9; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < 9) dF[(int64_t)b * fbs + n * fld + threadIdx.x] = red[threadIdx.x][0];
}

// ------------------------------------------------------------- Philox --
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

template <typename T>
__global__ void k_dropout(int64_t rows, int64_t cols, const T* __restrict__ X, int64_t xbs, int64_t xld,
                          T* __restrict__ Y, int64_t ybs, int64_t yld, uint32_t k0, uint32_t k1, uint32_t step_arg,
                          const int64_t* __restrict__ step_ptr, uint32_t layer, uint32_t thr, float scale,
                          uint32_t model_offset, const int32_t* __restrict__ model_ids) {
  const int b = blockIdx.y;
  const uint32_t gid = model_ids ? (uint32_t)model_ids[b] : model_offset + (uint32_t)b;   // global model index
  const uint32_t step = step_ptr ? (uint32_t)(*step_ptr + (int64_t)step_arg) : step_arg;   // device counter: graphs
  const int64_t n = rows * cols;
  const int64_t groups = (n + 3) / 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < groups; q += (int64_t)gridDim.x * blockDim.x) {
    U4 w = philox4x32_10(U4{(uint32_t)q, gid, step, layer}, k0, k1);
    uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int64_t i = q * 4 + e;
      if (i >= n) break;
      int64_t r = i / cols, c = i % cols;
      float v = ldf(X + (int64_t)b * xbs + r * xld + c);
      stf(Y + (int64_t)b * ybs + r * yld + c, ws[e] >= thr ? v * scale : 0.f);
    }
  }
}

// ------------------------------------------------------------- colsum --
// grid (cdiv(C, tpr*VEC), ngroups*cpg, B), 256 threads = tpr column lanes x
// (256/tpr) row lanes; each thread sums VEC adjacent columns (one 16-B load
// per row for bf16 VEC=8), then a shared-memory reduction over the row lanes.
template <typename T, int VEC>
__global__ void __launch_bounds__(256) k_colsum_part(int64_t C, int64_t group, int cpg, int64_t rpc, int tpr,
                                                     const T* __restrict__ X, int64_t xbs, int64_t xld,
                                                     float* __restrict__ part) {
  __shared__ float red[256 * VEC];
  const int b = blockIdx.z;
  const int64_t chunk = blockIdx.y;
  const int64_t g = chunk / cpg, j = chunk % cpg;
  const int lane = threadIdx.x % tpr, rl = threadIdx.x / tpr, rpb = 256 / tpr;
  const int64_t cbase = (int64_t)blockIdx.x * tpr * VEC;
  const int64_t c0 = cbase + (int64_t)lane * VEC;
  const int64_t r0 = g * group + j * rpc;
  const int64_t r1 = min((g + 1) * group, r0 + rpc);
  float a0[VEC], a1[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) a0[v] = a1[v] = 0.f;
  if (c0 < C) {
    const T* Xb = X + (int64_t)b * xbs + c0;
    int64_t r = r0 + rl;
    for (; r + rpb < r1; r += 2 * rpb) {
      float x0[VEC], x1[VEC];
      ld_vec<T, VEC>(Xb + r * xld, x0);
      ld_vec<T, VEC>(Xb + (r + rpb) * xld, x1);
#pragma unroll
      for (int v = 0; v < VEC; ++v) { a0[v] += x0[v]; a1[v] += x1[v]; }
    }
    if (r < r1) {
      float x0[VEC];
      ld_vec<T, VEC>(Xb + r * xld, x0);
#pragma unroll
      for (int v = 0; v < VEC; ++v) a0[v] += x0[v];
    }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) red[(rl * tpr + lane) * VEC + v] = a0[v] + a1[v];
  __syncthreads();
  const int t = threadIdx.x;
  if (t < tpr * VEC && cbase + t < C) {
    float sum = 0.f;
    for (int y = 0; y < rpb; ++y) sum += red[(y * tpr + t / VEC) * VEC + t % VEC];
    part[((int64_t)b * gridDim.y + chunk) * C + cbase + t] = sum;
  }
}

__global__ void k_colsum_fin(int B, int64_t C, int64_t ngroups, int cpg, const float* __restrict__ part,
                             float* __restrict__ S, int64_t sbs, int accumulate) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * ngroups * C) return;
  int64_t b = i / (ngroups * C), rem = i % (ngroups * C), g = rem / C, c = rem % C;
  double s = 0.0;
  for (int j = 0; j < cpg; ++j) s += part[((b * ngroups + g) * cpg + j) * C + c];
  float* o = S + b * sbs + g * C + c;
  *o = accumulate ? *o + (float)s : (float)s;
}

struct ColsumGeo { int64_t ngroups; int cpg; int64_t rpc; };
ColsumGeo colsum_geo(int B, int64_t rows, int64_t C, int64_t group) {
  ColsumGeo g;
  g.ngroups = cdiv(rows, group);
  int64_t blocks_per = cdiv(C, 128) * (int64_t)B * g.ngroups;
  int64_t target = 8 * (int64_t)std::max(num_sms(), 148);
  int64_t cpg = std::max<int64_t>(1, std::min<int64_t>(cdiv(target, blocks_per), cdiv(group, 256)));
  g.rpc = cdiv(group, cpg);
  g.cpg = (int)cdiv(group, g.rpc);
  return g;
}

template <typename T>
__global__ void k_act(int64_t rows, int64_t cols, int act, float alpha, const T* __restrict__ X, int64_t xbs,
                      int64_t xld, const T* __restrict__ D, int64_t dbs, int64_t dld, T* __restrict__ Y, int64_t ybs,
                      int64_t yld, int bwd) {
  const int b = blockIdx.y;
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const float x = ldf(X + b * xbs + r * xld + c);
    float out;
    if (!bwd) {
      if (act == HFTA_ACT_TANH) out = tanhf(x);
      else if (act == HFTA_ACT_SIGMOID) out = 1.f / (1.f + expf(-x));
      else out = act_fwd(x, act, alpha);
    } else {
      const float d = ldf(D + b * dbs + r * dld + c);
      if (act == HFTA_ACT_TANH) out = d * (1.f - x * x);            // x is the output y
      else if (act == HFTA_ACT_SIGMOID) out = d * x * (1.f - x);
      else out = d * act_grad(x, act, alpha);
    }
    stf(Y + b * ybs + r * yld + c, out);
  }
}

// dense rows (ld == cols): the tensor of each model is one flat run of n
// elements, 8 bf16 per thread per 16-B access, no index arithmetic per element
__device__ __forceinline__ float act_apply(float x, float d, int act, float alpha, int bwd) {
  if (!bwd) {
    if (act == HFTA_ACT_TANH) return tanhf(x);
    if (act == HFTA_ACT_SIGMOID) return 1.f / (1.f + expf(-x));
    return act_fwd(x, act, alpha);
  }
  if (act == HFTA_ACT_TANH) return d * (1.f - x * x);            // x is the output y
  if (act == HFTA_ACT_SIGMOID) return d * x * (1.f - x);
  return d * act_grad(x, act, alpha);
}
__global__ void k_act_flat(int64_t n8, int act, float alpha, const __nv_bfloat16* __restrict__ X, int64_t xbs,
                           const __nv_bfloat16* __restrict__ D, int64_t dbs, __nv_bfloat16* __restrict__ Y,
                           int64_t ybs, int bwd) {
  const int b = blockIdx.y;
  const uint4* x4 = reinterpret_cast<const uint4*>(X + b * xbs);
  const uint4* d4 = bwd ? reinterpret_cast<const uint4*>(D + b * dbs) : nullptr;
  uint4* y4 = reinterpret_cast<uint4*>(Y + b * ybs);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 xv = x4[i];
    const uint4 dv = bwd ? d4[i] : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t xs[4] = {xv.x, xv.y, xv.z, xv.w}, ds[4] = {dv.x, dv.y, dv.z, dv.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float xl, xh, dl, dh;
      unpack_bf2(xs[e], xl, xh);
      unpack_bf2(ds[e], dl, dh);
      o[e] = pack_bf2(act_apply(xl, dl, act, alpha, bwd), act_apply(xh, dh, act, alpha, bwd));
    }
    y4[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

}  // namespace

size_t colsum_ws(int B, int64_t rows, int64_t C, int64_t group) {
  if (B < 1 || rows < 1 || C < 1 || group < 1) return 0;
  ColsumGeo g = colsum_geo(B, rows, C, group);
  return align_up((size_t)B * g.ngroups * g.cpg * C * sizeof(float), 256);
}

hfta_status colsum_impl(int B, int64_t rows, int64_t C, int64_t group, hfta_dtype dt, hfta_in X, float* S,
                        int64_t S_bstride, int accumulate, void* ws, size_t ws_bytes, cudaStream_t s) {
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(rows >= 1 && C >= 1 && group >= 1 && X.ptr && S, HFTA_ERR_INVALID_VALUE, "colsum: bad args");
  size_t need = colsum_ws(B, rows, C, group);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "colsum: workspace %zu < %zu", ws_bytes, need);
  ColsumGeo g = colsum_geo(B, rows, C, group);
  float* part = reinterpret_cast<float*>(ws);
  const int esz = dt == HFTA_F32 ? 4 : 2;
  const int vec = (esz == 2 && C % 8 == 0 && X.ld % 8 == 0 && X.bstride % 8 == 0 && aligned16(X.ptr)) ? 8
                  : (esz == 4 && C % 4 == 0 && X.ld % 4 == 0 && X.bstride % 4 == 0 && aligned16(X.ptr)) ? 4 : 1;
  int tpr = 1;
  while (tpr < 32 && tpr * vec < C) tpr <<= 1;
  dim3 grid((unsigned)cdiv(C, (int64_t)tpr * vec), (unsigned)(g.ngroups * g.cpg), B);
  if (dt == HFTA_F32) {
    if (vec == 4)
      k_colsum_part<float, 4><<<grid, 256, 0, s>>>(C, group, g.cpg, g.rpc, tpr, (const float*)X.ptr, X.bstride, X.ld,
                                                   part);
    else
      k_colsum_part<float, 1><<<grid, 256, 0, s>>>(C, group, g.cpg, g.rpc, tpr, (const float*)X.ptr, X.bstride, X.ld,
                                                   part);
  } else {
    if (vec == 8)
      k_colsum_part<__nv_bfloat16, 8><<<grid, 256, 0, s>>>(C, group, g.cpg, g.rpc, tpr, (const __nv_bfloat16*)X.ptr,
                                                           X.bstride, X.ld, part);
    else
      k_colsum_part<__nv_bfloat16, 1><<<grid, 256, 0, s>>>(C, group, g.cpg, g.rpc, tpr, (const __nv_bfloat16*)X.ptr,
                                                           X.bstride, X.ld, part);
  }
  int64_t tot = (int64_t)B * g.ngroups * C;
  k_colsum_fin<<<(unsigned)cdiv(tot, 256), 256, 0, s>>>(B, C, g.ngroups, g.cpg, part, S, S_bstride, accumulate);
  count_launches(2);
  return post_launch(s, "colsum");
}

}  // namespace hfta

using namespace hfta;

extern "C" {

hfta_status hfta_transform_points_fwd(int B, int64_t N, int64_t L, hfta_dtype dt, hfta_in X, hfta_in F,
                                      int add_identity, hfta_out Xout, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(N >= 1 && L >= 1 && X.ptr && F.ptr && Xout.ptr, HFTA_ERR_INVALID_VALUE, "transform_fwd: bad args");
  HFTA_REQUIRE(X.ld >= 3 && F.ld >= 9 && Xout.ld >= 3 && (Xout.bstride > 0 || B == 1), HFTA_ERR_SHAPE,
               "transform_fwd: strides");
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)std::min<int64_t>(cdiv(N * L, 256), 1024), B);
  if (dt == HFTA_F32)
    k_transform_fwd<float><<<grid, 256, 0, s>>>(N, L, (const float*)X.ptr, X.bstride, X.ld, (const float*)F.ptr,
                                               F.bstride, F.ld, add_identity, (float*)Xout.ptr, Xout.bstride, Xout.ld);
  else
    k_transform_fwd<__nv_bfloat16><<<grid, 256, 0, s>>>(N, L, (const float*)X.ptr, X.bstride, X.ld,
                                                       (const float*)F.ptr, F.bstride, F.ld, add_identity,
                                                       (__nv_bfloat16*)Xout.ptr, Xout.bstride, Xout.ld);
  count_launches(1);
  return post_launch(s, "hfta_transform_points_fwd");
}

hfta_status hfta_transform_points_bwd(int B, int64_t N, int64_t L, hfta_dtype dt, hfta_in X, hfta_in dXout,
                                      hfta_out dF, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(N >= 1 && L >= 1 && X.ptr && dXout.ptr && dF.ptr, HFTA_ERR_INVALID_VALUE, "transform_bwd: bad args");
  HFTA_REQUIRE(dF.ld >= 9 && (dF.bstride > 0 || B == 1), HFTA_ERR_SHAPE, "transform_bwd: dF strides");
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)N, B);
  if (dt == HFTA_F32)
    k_transform_bwd<float><<<grid, 256, 0, s>>>(N, L, (const float*)X.ptr, X.bstride, X.ld, (const float*)dXout.ptr,
                                               dXout.bstride, dXout.ld, (float*)dF.ptr, dF.bstride, dF.ld);
  else
    k_transform_bwd<__nv_bfloat16><<<grid, 256, 0, s>>>(N, L, (const float*)X.ptr, X.bstride, X.ld,
                                                       (const __nv_bfloat16*)dXout.ptr, dXout.bstride, dXout.ld,
                                                       (float*)dF.ptr, dF.bstride, dF.ld);
  count_launches(1);
  return post_launch(s, "hfta_transform_points_bwd");
}

static hfta_status dropout_common(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_in X, hfta_out Y,
                                  uint64_t seed, int64_t step, const int64_t* step_ptr, int32_t layer, float p,
                                  int32_t model_offset, const int32_t* model_ids, hfta_stream stream,
                                  const char* what) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(rows >= 1 && cols >= 1 && X.ptr && Y.ptr, HFTA_ERR_INVALID_VALUE, "%s: bad args", what);
  HFTA_REQUIRE(p >= 0.f && p < 1.f, HFTA_ERR_INVALID_VALUE, "%s: p=%g not in [0,1)", what, (double)p);
  HFTA_REQUIRE(X.ld >= cols && Y.ld >= cols && (Y.bstride > 0 || B == 1), HFTA_ERR_SHAPE, "%s: strides", what);
  cudaStream_t s = (cudaStream_t)stream;
  double t = floor((double)p * 4294967296.0);
  uint32_t thr = (uint32_t)(t > 4294967295.0 ? 4294967295.0 : t);
  float scale = 1.0f / (1.0f - p);
  int64_t groups = cdiv(rows * cols, 4);
  dim3 grid((unsigned)std::min<int64_t>(cdiv(groups, 256), 2048), B);
  uint32_t k0 = (uint32_t)(seed & 0xffffffffu), k1 = (uint32_t)(seed >> 32);
  if (dt == HFTA_F32)
    k_dropout<float><<<grid, 256, 0, s>>>(rows, cols, (const float*)X.ptr, X.bstride, X.ld, (float*)Y.ptr, Y.bstride,
                                         Y.ld, k0, k1, (uint32_t)step, step_ptr, (uint32_t)layer, thr, scale,
                                         (uint32_t)model_offset, model_ids);
  else
    k_dropout<__nv_bfloat16><<<grid, 256, 0, s>>>(rows, cols, (const __nv_bfloat16*)X.ptr, X.bstride, X.ld,
                                                 (__nv_bfloat16*)Y.ptr, Y.bstride, Y.ld, k0, k1, (uint32_t)step,
                                                 step_ptr, (uint32_t)layer, thr, scale, (uint32_t)model_offset,
                                                 model_ids);
  count_launches(1);
  return post_launch(s, what);
}

hfta_status hfta_dropout_fwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_in X, hfta_out Y, uint64_t seed,
                             int64_t step, const int64_t* step_ptr, int32_t layer, float p, int32_t model_offset,
                             const int32_t* model_ids, hfta_stream stream) {
  return dropout_common(B, rows, cols, dt, X, Y, seed, step, step_ptr, layer, p, model_offset, model_ids, stream,
                        "hfta_dropout_fwd");
}

hfta_status hfta_dropout_bwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_in dY, hfta_out dX,
                             uint64_t seed, int64_t step, const int64_t* step_ptr, int32_t layer, float p,
                             int32_t model_offset, const int32_t* model_ids, hfta_stream stream) {
  return dropout_common(B, rows, cols, dt, dY, dX, seed, step, step_ptr, layer, p, model_offset, model_ids, stream,
                        "hfta_dropout_bwd");
}

static hfta_status act_common(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_act act, float alpha,
                              hfta_in X, hfta_in D, hfta_out Y, int bwd, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(rows >= 1 && cols >= 1 && X.ptr && Y.ptr && (!bwd || D.ptr), HFTA_ERR_INVALID_VALUE, "act: bad args");
  HFTA_REQUIRE((int)act >= 1 && (int)act <= 4, HFTA_ERR_UNSUPPORTED, "act: activation %d", (int)act);
  HFTA_REQUIRE(X.ld >= cols && Y.ld >= cols && (Y.bstride > 0 || B == 1), HFTA_ERR_SHAPE, "act: strides");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = rows * cols;
  if (dt == HFTA_BF16 && X.ld == cols && Y.ld == cols && (!bwd || D.ld == cols) && n % 8 == 0 &&
      X.bstride % 8 == 0 && Y.bstride % 8 == 0 && (!bwd || D.bstride % 8 == 0) && aligned16(X.ptr) &&
      aligned16(Y.ptr) && (!bwd || aligned16(D.ptr))) {
    dim3 g((unsigned)std::min<int64_t>(cdiv(n / 8, 256), 4 * 148), B);
    k_act_flat<<<g, 256, 0, s>>>(n / 8, (int)act, alpha, (const __nv_bfloat16*)X.ptr, X.bstride,
                                 (const __nv_bfloat16*)D.ptr, D.bstride, (__nv_bfloat16*)Y.ptr, Y.bstride, bwd);
    count_launches(1);
    return post_launch(s, bwd ? "hfta_act_bwd" : "hfta_act_fwd");
  }
  dim3 grid((unsigned)std::min<int64_t>(cdiv(rows * cols, 256), 4096), B);
  if (dt == HFTA_F32)
    k_act<float><<<grid, 256, 0, s>>>(rows, cols, (int)act, alpha, (const float*)X.ptr, X.bstride, X.ld,
                                     (const float*)D.ptr, D.bstride, D.ld, (float*)Y.ptr, Y.bstride, Y.ld, bwd);
  else
    k_act<__nv_bfloat16><<<grid, 256, 0, s>>>(rows, cols, (int)act, alpha, (const __nv_bfloat16*)X.ptr, X.bstride,
                                             X.ld, (const __nv_bfloat16*)D.ptr, D.bstride, D.ld,
                                             (__nv_bfloat16*)Y.ptr, Y.bstride, Y.ld, bwd);
  count_launches(1);
  return post_launch(s, bwd ? "hfta_act_bwd" : "hfta_act_fwd");
}

hfta_status hfta_act_fwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_act act, float alpha, hfta_in X,
                         hfta_out Y, hfta_stream stream) {
  return act_common(B, rows, cols, dt, act, alpha, X, hfta_in{nullptr, 0, 1}, Y, 0, stream);
}

hfta_status hfta_act_bwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_act act, float alpha, hfta_in XY,
                         hfta_in dY, hfta_out dX, hfta_stream stream) {
  return act_common(B, rows, cols, dt, act, alpha, XY, dY, dX, 1, stream);
}

size_t hfta_colsum_workspace(int B, int64_t rows, int64_t C, int64_t group) { return colsum_ws(B, rows, C, group); }

hfta_status hfta_colsum(int B, int64_t rows, int64_t C, int64_t group, hfta_dtype dt, hfta_in X, float* S,
                        int64_t S_bstride, int accumulate, void* ws, size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  return colsum_impl(B, rows, C, group, dt, X, S, S_bstride, accumulate, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
