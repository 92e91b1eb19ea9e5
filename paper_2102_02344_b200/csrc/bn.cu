// bn.cu -- fused BatchNorm forward/backward with per-model statistics (K6)
// and the PointNet BN-apply + max-over-points fusion (K8a).
// App. B rows BatchNorm1d/BatchNorm2d: the fused BN runs over
// B*C channels, i.e. statistics per (model b, channel c) (reading R13).
// HBM-bound: 128-bit loads along C (4 fp32 / 8 bf16 per access), one CTA row
// of threads per row slice, fixed-order partial merges in fp64.
#include <cstdlib>
#include <initializer_list>
#include <tuple>

#include "common.cuh"

namespace hfta {
namespace {

constexpr int NT = 256;

// Pre-activation z = a*x + c of a BN column, a = gamma*invstd,
// c = beta - mean*a: ONE fp32 rounding order shared by every forward and
// backward kernel, so the act'(z) decision recomputed in backward is
// bit-identical to the one the forward took (reading R15c).
__device__ __forceinline__ void bn_affine(float ga, float be, float m, float is, float& a, float& c) {
  a = ga * is;
  c = fmaf(-m, a, be);
}
constexpr int UNRM = 1;     // max-over-points: rows in flight per thread (loop-carried max)
constexpr int UNR = 1;      // rows per thread per iteration (UNR=4 measured slower: 76-150 regs cut occupancy)

struct Geo {
  int vec, tpr, cb, rpb, colgroups, chunks;
  int64_t rows_per_chunk;
};

int pow2ceil(int64_t x) { int p = 1; while (p < x) p <<= 1; return p; }

int bn_blocks_per_sm() {   // row-chunk parallelism target (env HFTA_BN_BPS for tuning)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HFTA_BN_BPS");
    v = e ? atoi(e) : 4;
    if (v < 1) v = 4;
  }
  return v;
}

bool vec_ok(const void* p, int64_t ld, int64_t bs, int64_t C, int vec) {
  return p == nullptr || (aligned16(p) && ld % vec == 0 && bs % vec == 0 && C % vec == 0);
}

// RUN: the most rows one thread sums sequentially in fp32 (the reductions'
// per-thread runs; error ~RUN u of a run, then fixed-order fp64 combination
// across threads and chunks -- reading R15c: a 2000-row fp32 run had moved
// the BN output z by 5e-5 of a channel's spread)
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
int bn_run() { static int v = env_int("HFTA_BN_RUN", 128); return v; }
// fewest rows one thread streams per chunk (small-R layers: blocks long enough
// to amortise their setup and the partial merge)
int bn_min_rows() { static int v = std::max(1, env_int("HFTA_BN_MINROWS", 8)); return v; }

// run > 0: chunks short enough that one thread sums <= run rows (reductions);
// run == 0: apply passes (no reduction, chunks sized for parallelism only)
Geo make_geo(int B, int64_t R, int64_t C, int vec, int bps = 0, int run = 0) {
  Geo g;
  g.vec = vec;
  g.tpr = (int)std::min<int64_t>(32, pow2ceil(cdiv(C, vec)));
  g.cb = g.tpr * vec;
  g.rpb = NT / g.tpr;
  g.colgroups = (int)cdiv(C, g.cb);
  int64_t target = (int64_t)(bps > 0 ? bps : bn_blocks_per_sm()) * std::max(num_sms(), 148);
  int64_t chunks = std::max<int64_t>(1, target / ((int64_t)g.colgroups * B));
  chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, cdiv(R, (int64_t)g.rpb * bn_min_rows())));
  if (run > 0) chunks = std::max<int64_t>(chunks, cdiv(R, (int64_t)g.rpb * run));   // runs of <= run rows per thread
  g.rows_per_chunk = cdiv(cdiv(R, chunks), g.rpb) * g.rpb;
  g.chunks = (int)cdiv(R, g.rows_per_chunk);
  return g;
}

// Welford-free stable stats: per-thread fp32 sums of (x - shift) and (x - shift)^2
// with shift = x[row 0] of the column; merged across row lanes in fixed order.
template <typename T, int VEC, int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_stats(int64_t R, int64_t C, const T* __restrict__ X,
                                                 int64_t xbs, int64_t ld, Geo g,
                                                 double* __restrict__ p1, double* __restrict__ p2) {
  // each thread sums <= RUN rows in fp32 (4 rows' loads in flight), blocks
  // combine their threads and chunks in fp64, fixed order (reading R15c)
  __shared__ double s1[NT * VEC], s2[NT * VEC];
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  const T* Xb = X + (int64_t)b * xbs;
  float a1[VEC], a2[VEC], sh[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { a1[v] = 0.f; a2[v] = 0.f; sh[v] = 0.f; }
  if (c0 < C) {
    ld_vec<T, VEC>(Xb + c0, sh);
    const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
    const int64_t r1 = min(R, r0 + g.rows_per_chunk);
    for (int64_t r = r0 + rl; r < r1; r += U * g.rpb) {
      float x[U][VEC];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r + u * g.rpb < r1) ld_vec<T, VEC>(Xb + (r + u * g.rpb) * ld + c0, x[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r + u * g.rpb < r1) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const float d = x[u][v] - sh[v];
            a1[v] += d;
            a2[v] = fmaf(d, d, a2[v]);
          }
        }
    }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    s1[rl * g.cb + lane * VEC + v] = a1[v];
    s2[rl * g.cb + lane * VEC + v] = a2[v];
  }
  __syncthreads();
  for (int col = threadIdx.x; col < g.cb; col += NT) {
    int64_t c = (int64_t)blockIdx.x * g.cb + col;
    if (c >= C) continue;
    double t1 = 0.0, t2 = 0.0;
    for (int r = 0; r < g.rpb; ++r) { t1 += s1[r * g.cb + col]; t2 += s2[r * g.cb + col]; }
    int64_t o = ((int64_t)b * g.chunks + chunk) * C + c;
    p1[o] = t1;
    p2[o] = t2;
  }
}

// Chunk partials -> per-(model, channel) sums: block = (32 channels, model b),
// 8 warps take chunks w, w + 8, ... (lane = channel: coalesced), then warp 0
// adds the 8 warp sums in order (fixed order: deterministic).
__device__ __forceinline__ bool chunk_sums(int64_t C, int chunks, const double* __restrict__ p1,
                                           const double* __restrict__ p2, double& s1, double& s2) {
  __shared__ double r1[8][32], r2[8][32];
  const int b = blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double a1 = 0.0, a2 = 0.0;
  if (c < C)
    for (int k = w; k < chunks; k += 8) {
      a1 += p1[((int64_t)b * chunks + k) * C + c];
      a2 += p2[((int64_t)b * chunks + k) * C + c];
    }
  r1[w][lane] = a1;
  r2[w][lane] = a2;
  __syncthreads();
  if (w != 0 || c >= C) return false;
  s1 = 0.0; s2 = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) { s1 += r1[q][lane]; s2 += r2[q][lane]; }
  return true;
}

template <typename T>
__global__ void k_bn_finalize(int B, int64_t R, int64_t C, const T* __restrict__ X, int64_t xbs, int chunks,
                              const double* __restrict__ p1, const double* __restrict__ p2, float eps,
                              float momentum, float* __restrict__ rmean, float* __restrict__ rvar,
                              float* __restrict__ smean, float* __restrict__ sinv) {
  double s1, s2;
  if (!chunk_sums(C, chunks, p1, p2, s1, s2)) return;
  const int64_t b = blockIdx.y, c = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t i = b * C + c;
  double shift = (double)ldf(X + b * xbs + c);
  double md = s1 / (double)R;
  double var = s2 / (double)R - md * md;
  if (var < 0.0) var = 0.0;
  double mean = shift + md;
  smean[i] = (float)mean;
  sinv[i] = (float)(1.0 / sqrt(var + (double)eps));
  if (rmean) rmean[i] = (float)((1.0 - momentum) * (double)rmean[i] + momentum * mean);
  if (rvar) rvar[i] = (float)((1.0 - momentum) * (double)rvar[i] + momentum * var * (double)R / (double)(R - 1));
}

// Statistics from the producing GEMM's epilogue partials (hfta_fused_linear_fwd_stats):
// colstat[b][blk][0|1][c] = sum / sum of squares of 32 stored rows; fixed-order fp64 merge
// (8 warps take blocks w, w + 8, ..., then warp 0 adds the 8 warp sums in order).
__global__ void k_bn_finalize_colstat(int B, int64_t R, int64_t C, int64_t nblk, const float* __restrict__ cs,
                                      float eps, float momentum, float* __restrict__ rmean,
                                      float* __restrict__ rvar, float* __restrict__ smean,
                                      float* __restrict__ sinv) {
  __shared__ double r1[8][32], r2[8][32];
  const int b = blockIdx.y, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double a1 = 0.0, a2 = 0.0;
  if (c < C)
    for (int64_t k = w; k < nblk; k += 8) {
      const float* q = cs + (((int64_t)b * nblk + k) * 2) * C + c;
      a1 += (double)q[0];
      a2 += (double)q[C];
    }
  r1[w][lane] = a1;
  r2[w][lane] = a2;
  __syncthreads();
  if (w != 0 || c >= C) return;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) { s1 += r1[q][lane]; s2 += r2[q][lane]; }
  const int64_t i = (int64_t)b * C + c;
  const double mean = s1 / (double)R;
  double var = s2 / (double)R - mean * mean;
  if (var < 0.0) var = 0.0;
  smean[i] = (float)mean;
  sinv[i] = (float)(1.0 / sqrt(var + (double)eps));
  if (rmean) rmean[i] = (float)((1.0 - momentum) * (double)rmean[i] + momentum * mean);
  if (rvar) rvar[i] = (float)((1.0 - momentum) * (double)rvar[i] + momentum * var * (double)R / (double)(R - 1));
}

template <typename T, int VEC, int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_apply(int64_t R, int64_t C, const T* __restrict__ X, int64_t xbs,
                                                 int64_t xld, T* __restrict__ Y, int64_t ybs, int64_t yld,
                                                 const float* __restrict__ gamma, const float* __restrict__ beta,
                                                 int64_t gbs, const float* __restrict__ smean,
                                                 const float* __restrict__ sinv, int act, float alpha, Geo g) {
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  if (c0 >= C) return;
  float sc[VEC], sf[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    float m = smean[(int64_t)b * C + c0 + v], is = sinv[(int64_t)b * C + c0 + v];
    float ga = gamma[(int64_t)b * gbs + c0 + v], be = beta[(int64_t)b * gbs + c0 + v];
    bn_affine(ga, be, m, is, sc[v], sf[v]);
  }
  const T* Xb = X + (int64_t)b * xbs + c0;
  T* Yb = Y + (int64_t)b * ybs + c0;
  const int r0 = (int)((int64_t)chunk * g.rows_per_chunk);
  const int r1 = (int)min(R, (int64_t)r0 + g.rows_per_chunk);
  for (int r = r0 + rl; r < r1; r += U * g.rpb) {
    float x[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r + u * g.rpb < r1) ld_vec<T, VEC>(Xb + (int64_t)(r + u * g.rpb) * xld, x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r + u * g.rpb < r1) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) x[u][v] = act_fwd(fmaf(x[u][v], sc[v], sf[v]), act, alpha);
        st_vec<T, VEC>(Yb + (int64_t)(r + u * g.rpb) * yld, x[u]);
      }
  }
}

// ------------------------------------------------------------- backward --
// Per column the pre-activation is z = a*x + c (a = gamma*invstd, c = beta - mean*a);
// act'(z) is a select on the sign of z.  The reduce pass accumulates sum dz and
// sum dz*(x - mean) (shifted by the exact mean: no cancellation); the apply pass
// evaluates dx = A*act'(z)*dy + Bx*x + Cc with three per-column constants.
// Few live per-column values keep these kernels at <= 80 registers (3 CTAs/SM).
template <typename T, int VEC, int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_bwd_reduce(int64_t R, int64_t C, const T* __restrict__ dY, int64_t dbs,
                                                         int64_t dld, const T* __restrict__ X, int64_t xbs, int64_t xld,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ beta, int64_t gbs,
                                                         const float* __restrict__ smean,
                                                         const float* __restrict__ sinv, int act, float alpha, Geo g,
                                                         double* __restrict__ p1, double* __restrict__ p2) {
  __shared__ double s1[NT * VEC], s2[NT * VEC];
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  float a1[VEC], a2[VEC];          // <= RUN rows per thread in fp32, fp64 across threads / chunks
#pragma unroll
  for (int v = 0; v < VEC; ++v) { a1[v] = 0.f; a2[v] = 0.f; }
  if (c0 < C) {
    float ka[VEC], kc[VEC], m[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      m[v] = smean[(int64_t)b * C + c0 + v];
      bn_affine(gamma[(int64_t)b * gbs + c0 + v], beta[(int64_t)b * gbs + c0 + v], m[v],
                sinv[(int64_t)b * C + c0 + v], ka[v], kc[v]);
    }
    const T* Xb = X + (int64_t)b * xbs;
    const T* Db = dY + (int64_t)b * dbs;
    const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
    const int64_t r1 = min(R, r0 + g.rows_per_chunk);
    for (int64_t r = r0 + rl; r < r1; r += U * g.rpb) {
      float x[U][VEC], d[U][VEC];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r + u * g.rpb < r1) {
          ld_vec<T, VEC>(Xb + (r + u * g.rpb) * xld + c0, x[u]);
          ld_vec<T, VEC>(Db + (r + u * g.rpb) * dld + c0, d[u]);
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (r + u * g.rpb < r1) {
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const float dz = d[u][v] * act_grad(fmaf(ka[v], x[u][v], kc[v]), act, alpha);
            a1[v] += dz;
            a2[v] = fmaf(dz, x[u][v] - m[v], a2[v]);
          }
        }
    }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    s1[rl * g.cb + lane * VEC + v] = a1[v];
    s2[rl * g.cb + lane * VEC + v] = a2[v];
  }
  __syncthreads();
  for (int col = threadIdx.x; col < g.cb; col += NT) {
    int64_t c = (int64_t)blockIdx.x * g.cb + col;
    if (c >= C) continue;
    double t1 = 0.0, t2 = 0.0;
    for (int r = 0; r < g.rpb; ++r) { t1 += s1[r * g.cb + col]; t2 += s2[r * g.cb + col]; }
    int64_t o = ((int64_t)b * g.chunks + chunk) * C + c;
    p1[o] = t1;
    p2[o] = t2;
  }
}

// dbeta = sum dz, dgamma = invstd * sum dz (x - mean) (fp32, written to the
// gradient arena) and the apply-pass constants in ws (5 x [B][C]):
// A = gamma*invstd, Bx = -A*invstd*dgamma/R, Cc = A*(mean*invstd*dgamma/R - dbeta/R),
// ka = gamma*invstd, kc = beta - mean*ka.
__global__ void k_bn_bwd_finalize(int B, int64_t R, int64_t C, int chunks, const double* __restrict__ p1,
                                  const double* __restrict__ p2, const float* __restrict__ gamma,
                                  const float* __restrict__ beta, int64_t gbs, const float* __restrict__ smean,
                                  const float* __restrict__ sinv, float* __restrict__ dgamma,
                                  float* __restrict__ dbeta, int accumulate, float* __restrict__ coef) {
  double s1, s2;
  if (!chunk_sums(C, chunks, p1, p2, s1, s2)) return;
  const int64_t b = blockIdx.y, c = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t i = b * C + c;
  const double is = sinv[i], m = smean[i], ga = gamma[b * gbs + c], be = beta[b * gbs + c];
  const double db = s1, dg = s2 * is;
  if (dbeta) dbeta[b * gbs + c] = accumulate ? dbeta[b * gbs + c] + (float)db : (float)db;
  if (dgamma) dgamma[b * gbs + c] = accumulate ? dgamma[b * gbs + c] + (float)dg : (float)dg;
  const double A = ga * is, k2 = db / (double)R, k3 = dg / (double)R;
  const int64_t BC = (int64_t)B * C;
  coef[i] = (float)A;
  coef[BC + i] = (float)(-A * k3 * is);
  coef[2 * BC + i] = (float)(A * (k3 * m * is - k2));
  float fa, fc;                                   // the forward's z = a x + c, same rounding
  bn_affine(gamma[b * gbs + c], beta[b * gbs + c], smean[i], sinv[i], fa, fc);
  coef[3 * BC + i] = fa;
  coef[4 * BC + i] = fc;
}

template <typename T, int VEC, int U, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_bwd_apply(int B, int64_t R, int64_t C, const T* __restrict__ dY,
                                                        int64_t dbs, int64_t dld, const T* __restrict__ X, int64_t xbs,
                                                        int64_t xld, T* __restrict__ dX, int64_t obs, int64_t old,
                                                        int act, float alpha, Geo g, const float* __restrict__ coef) {
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  if (c0 >= C) return;
  const int64_t BC = (int64_t)B * C;
  float kA[VEC], kB[VEC], kC[VEC], ka[VEC], kc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    int64_t i = (int64_t)b * C + c0 + v;
    kA[v] = coef[i]; kB[v] = coef[BC + i]; kC[v] = coef[2 * BC + i];
    ka[v] = coef[3 * BC + i]; kc[v] = coef[4 * BC + i];
  }
  const T* Xb = X + (int64_t)b * xbs;
  const T* Db = dY + (int64_t)b * dbs;
  T* Ob = dX + (int64_t)b * obs;
  const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
  const int64_t r1 = min(R, r0 + g.rows_per_chunk);
  for (int64_t r = r0 + rl; r < r1; r += U * g.rpb) {
    float x[U][VEC], d[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r + u * g.rpb < r1) {
        ld_vec<T, VEC>(Xb + (r + u * g.rpb) * xld + c0, x[u]);
        ld_vec<T, VEC>(Db + (r + u * g.rpb) * dld + c0, d[u]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (r + u * g.rpb < r1) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const float gd = d[u][v] * act_grad(fmaf(ka[v], x[u][v], kc[v]), act, alpha);
          x[u][v] = fmaf(kA[v], gd, fmaf(kB[v], x[u][v], kC[v]));
        }
        st_vec<T, VEC>(Ob + (r + u * g.rpb) * old + c0, x[u]);
      }
  }
}

// ------------------------------------------- cp.async row pipelines ------
// 16-B vectors (8 bf16 / 4 fp32 per thread): each thread streams its rows
// rbeg, rbeg + step, ... through a private S-stage ring in shared memory
// (LDGSTS, no registers held by loads in flight): S rows x NS streams x 16 B
// per thread, S x NS x 4 KB per CTA.  Measured on the seg head shapes: the
// register-staged loops above reach 2.8-3.9 TB/s on the reductions (one or
// two rows in flight per thread).
template <int NS, int S>
struct Ring {
  static constexpr uint32_t SLOT = NS * NT * 16;     // bytes per stage
  static constexpr size_t BYTES = (size_t)S * SLOT;
};

template <typename T, int NS, int S, typename F>
__device__ __forceinline__ void row_pipe(const T* g0, int64_t ld0, const T* g1, int64_t ld1, int64_t rbeg,
                                         int64_t rend, int step, uint32_t ring, F&& f) {
  constexpr uint32_t SLOT = Ring<NS, S>::SLOT;
  const int n = rbeg < rend ? (int)((rend - rbeg + step - 1) / step) : 0;
  const uint32_t tslot = ring + threadIdx.x * 16;
  auto issue = [&](int k) {
    const int64_t r = rbeg + (int64_t)k * step;
    const uint32_t a = tslot + (uint32_t)(k % S) * SLOT;
    cp_async16(a, g0 + r * ld0);
    if constexpr (NS == 2) cp_async16(a + NT * 16, g1 + r * ld1);
  };
#pragma unroll
  for (int k = 0; k < S - 1; ++k) {
    if (k < n) issue(k);
    cp_async_commit();
  }
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
    if (i + S - 1 < n) issue(i + S - 1);
    cp_async_commit();
    cp_async_wait<S - 1>();                          // row i's group has landed
    const uint32_t a = tslot + (uint32_t)(i % S) * SLOT;
    f(rbeg + (int64_t)i * step, a, a + NT * 16);
  }
  cp_async_wait<0>();
}

// fixed-order fp64 merge of the per-thread fp32 runs of a CTA (reuses the ring)
template <int VEC>
__device__ __forceinline__ void block_merge(double* s1, double* s2, const float (&a1)[VEC], const float (&a2)[VEC],
                                            int rl, int lane, const Geo& g, int64_t C, int b, int chunk,
                                            double* __restrict__ p1, double* __restrict__ p2) {
  __syncthreads();                                   // every thread is done with its ring slots
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    s1[rl * g.cb + lane * VEC + v] = a1[v];
    s2[rl * g.cb + lane * VEC + v] = a2[v];
  }
  __syncthreads();
  for (int col = threadIdx.x; col < g.cb; col += NT) {
    int64_t c = (int64_t)blockIdx.x * g.cb + col;
    if (c >= C) continue;
    double t1 = 0.0, t2 = 0.0;
    for (int r = 0; r < g.rpb; ++r) { t1 += s1[r * g.cb + col]; t2 += s2[r * g.cb + col]; }
    int64_t o = ((int64_t)b * g.chunks + chunk) * C + c;
    p1[o] = t1;
    p2[o] = t2;
  }
}

template <typename T, int VEC> constexpr size_t merge_bytes() { return 2 * (size_t)NT * VEC * sizeof(double); }
template <typename T, int VEC, int NS, int S> constexpr size_t pipe_smem() {
  return Ring<NS, S>::BYTES > merge_bytes<T, VEC>() ? Ring<NS, S>::BYTES : merge_bytes<T, VEC>();
}

template <typename T, int VEC, int S, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_stats_p(int64_t R, int64_t C, const T* __restrict__ X, int64_t xbs,
                                                        int64_t ld, Geo g, double* __restrict__ p1,
                                                        double* __restrict__ p2) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  const T* Xb = X + (int64_t)b * xbs + c0;
  float a1[VEC], a2[VEC], sh[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { a1[v] = 0.f; a2[v] = 0.f; sh[v] = 0.f; }
  if (c0 < C) {
    ld_vec<T, VEC>(Xb, sh);
    const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
    row_pipe<T, 1, S>(Xb, ld, Xb, ld, r0 + rl, min(R, r0 + g.rows_per_chunk), g.rpb, (uint32_t)__cvta_generic_to_shared(smem_raw),
                      [&](int64_t, uint32_t sx, uint32_t) {
                        float x[VEC];
                        ld_vec_smem<T, VEC>(sx, x);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) {
                          const float d = x[v] - sh[v];
                          a1[v] += d;
                          a2[v] = fmaf(d, d, a2[v]);
                        }
                      });
  }
  double* s1 = reinterpret_cast<double*>(smem_raw);
  block_merge<VEC>(s1, s1 + NT * VEC, a1, a2, rl, lane, g, C, b, chunk, p1, p2);
}

template <typename T, int VEC, int S, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_apply_p(int64_t R, int64_t C, const T* __restrict__ X, int64_t xbs,
                                                        int64_t xld, T* __restrict__ Y, int64_t ybs, int64_t yld,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, int64_t gbs,
                                                        const float* __restrict__ smean,
                                                        const float* __restrict__ sinv, int act, float alpha, Geo g) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  if (c0 >= C) return;
  float sc[VEC], sf[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    float m = smean[(int64_t)b * C + c0 + v], is = sinv[(int64_t)b * C + c0 + v];
    float ga = gamma[(int64_t)b * gbs + c0 + v], be = beta[(int64_t)b * gbs + c0 + v];
    bn_affine(ga, be, m, is, sc[v], sf[v]);
  }
  const T* Xb = X + (int64_t)b * xbs + c0;
  T* Yb = Y + (int64_t)b * ybs + c0;
  const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
  row_pipe<T, 1, S>(Xb, xld, Xb, xld, r0 + rl, min(R, r0 + g.rows_per_chunk), g.rpb, (uint32_t)__cvta_generic_to_shared(smem_raw),
                    [&](int64_t r, uint32_t sx, uint32_t) {
                      float x[VEC];
                      ld_vec_smem<T, VEC>(sx, x);
#pragma unroll
                      for (int v = 0; v < VEC; ++v) x[v] = act_fwd(fmaf(x[v], sc[v], sf[v]), act, alpha);
                      st_vec<T, VEC>(Yb + r * yld, x);
                    });
}

template <typename T, int VEC, int S, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_bwd_reduce_p(int64_t R, int64_t C, const T* __restrict__ dY,
                                                             int64_t dbs, int64_t dld, const T* __restrict__ X,
                                                             int64_t xbs, int64_t xld,
                                                             const float* __restrict__ gamma,
                                                             const float* __restrict__ beta, int64_t gbs,
                                                             const float* __restrict__ smean,
                                                             const float* __restrict__ sinv, int act, float alpha,
                                                             Geo g, double* __restrict__ p1, double* __restrict__ p2) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  float a1[VEC], a2[VEC];            // fp32 runs of <= run rows per thread, fp64 across threads / chunks
#pragma unroll
  for (int v = 0; v < VEC; ++v) { a1[v] = 0.f; a2[v] = 0.f; }
  if (c0 < C) {
    float ka[VEC], kc[VEC], m[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      m[v] = smean[(int64_t)b * C + c0 + v];
      bn_affine(gamma[(int64_t)b * gbs + c0 + v], beta[(int64_t)b * gbs + c0 + v], m[v],
                sinv[(int64_t)b * C + c0 + v], ka[v], kc[v]);
    }
    const T* Xb = X + (int64_t)b * xbs + c0;
    const T* Db = dY + (int64_t)b * dbs + c0;
    const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
    row_pipe<T, 2, S>(Xb, xld, Db, dld, r0 + rl, min(R, r0 + g.rows_per_chunk), g.rpb, (uint32_t)__cvta_generic_to_shared(smem_raw),
                      [&](int64_t, uint32_t sx, uint32_t sd) {
                        float x[VEC], d[VEC];
                        ld_vec_smem<T, VEC>(sx, x);
                        ld_vec_smem<T, VEC>(sd, d);
#pragma unroll
                        for (int v = 0; v < VEC; ++v) {
                          const float dz = d[v] * act_grad(fmaf(ka[v], x[v], kc[v]), act, alpha);
                          a1[v] += dz;
                          a2[v] = fmaf(dz, x[v] - m[v], a2[v]);
                        }
                      });
  }
  double* s1 = reinterpret_cast<double*>(smem_raw);
  block_merge<VEC>(s1, s1 + NT * VEC, a1, a2, rl, lane, g, C, b, chunk, p1, p2);
}

template <typename T, int VEC, int S, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_bn_bwd_apply_p(int B, int64_t R, int64_t C, const T* __restrict__ dY,
                                                            int64_t dbs, int64_t dld, const T* __restrict__ X,
                                                            int64_t xbs, int64_t xld, T* __restrict__ dX, int64_t obs,
                                                            int64_t old, int act, float alpha, Geo g,
                                                            const float* __restrict__ coef) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  if (c0 >= C) return;
  const int64_t BC = (int64_t)B * C;
  float kA[VEC], kB[VEC], kC[VEC], ka[VEC], kc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    int64_t i = (int64_t)b * C + c0 + v;
    kA[v] = coef[i]; kB[v] = coef[BC + i]; kC[v] = coef[2 * BC + i];
    ka[v] = coef[3 * BC + i]; kc[v] = coef[4 * BC + i];
  }
  const T* Xb = X + (int64_t)b * xbs + c0;
  const T* Db = dY + (int64_t)b * dbs + c0;
  T* Ob = dX + (int64_t)b * obs + c0;
  const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
  row_pipe<T, 2, S>(Xb, xld, Db, dld, r0 + rl, min(R, r0 + g.rows_per_chunk), g.rpb, (uint32_t)__cvta_generic_to_shared(smem_raw),
                    [&](int64_t r, uint32_t sx, uint32_t sd) {
                      float x[VEC], d[VEC];
                      ld_vec_smem<T, VEC>(sx, x);
                      ld_vec_smem<T, VEC>(sd, d);
#pragma unroll
                      for (int v = 0; v < VEC; ++v) {
                        const float gd = d[v] * act_grad(fmaf(ka[v], x[v], kc[v]), act, alpha);
                        x[v] = fmaf(kA[v], gd, fmaf(kB[v], x[v], kC[v]));
                      }
                      st_vec<T, VEC>(Ob + r * old, x);
                    });
}

// --------------------------------------------------- BN + act + max (K8a) --
// grid (colgroups, N, B); block reduces max/argmax over the L rows of sample n.
template <typename T, int VEC>
__global__ void __launch_bounds__(NT, 4) k_bn_max_fwd(int64_t L, int64_t C, const T* __restrict__ X, int64_t xbs,
                                                   int64_t xld, const float* __restrict__ gamma,
                                                   const float* __restrict__ beta, int64_t gbs,
                                                   const float* __restrict__ smean, const float* __restrict__ sinv,
                                                   int act, float alpha, float* __restrict__ out, int64_t obs,
                                                   int64_t old, int32_t* __restrict__ amax, int64_t N, Geo g) {
  __shared__ float sv[NT * VEC];
  __shared__ int si[NT * VEC];
  const int b = blockIdx.z;
  const int64_t n = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  float best[VEC];
  int bi[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { best[v] = -INFINITY; bi[v] = 0x7fffffff; }
  if (c0 < C) {
    float sc[VEC], sf[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      float m = smean[(int64_t)b * C + c0 + v], is = sinv[(int64_t)b * C + c0 + v];
      float ga = gamma[(int64_t)b * gbs + c0 + v], be = beta[(int64_t)b * gbs + c0 + v];
      bn_affine(ga, be, m, is, sc[v], sf[v]);
    }
    const T* Xb = X + (int64_t)b * xbs + n * L * xld;
    // two rows in flight per thread (bulk), then the tail row: loads issued before use
    int64_t l = rl;
    for (; l + g.rpb < L; l += 2 * g.rpb) {
      float x0[VEC], x1[VEC];
      ld_vec<T, VEC>(Xb + l * xld + c0, x0);
      ld_vec<T, VEC>(Xb + (l + g.rpb) * xld + c0, x1);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const float z0 = act_fwd(fmaf(x0[v], sc[v], sf[v]), act, alpha);
        const float z1 = act_fwd(fmaf(x1[v], sc[v], sf[v]), act, alpha);
        if (z0 > best[v]) { best[v] = z0; bi[v] = (int)l; }          // increasing l per lane
        if (z1 > best[v]) { best[v] = z1; bi[v] = (int)(l + g.rpb); }
      }
    }
    if (l < L) {
      float x0[VEC];
      ld_vec<T, VEC>(Xb + l * xld + c0, x0);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const float z0 = act_fwd(fmaf(x0[v], sc[v], sf[v]), act, alpha);
        if (z0 > best[v]) { best[v] = z0; bi[v] = (int)l; }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    sv[rl * g.cb + lane * VEC + v] = best[v];
    si[rl * g.cb + lane * VEC + v] = bi[v];
  }
  __syncthreads();
  for (int col = threadIdx.x; col < g.cb; col += NT) {
    int64_t c = (int64_t)blockIdx.x * g.cb + col;
    if (c >= C) continue;
    float bv = -INFINITY;
    int bidx = 0x7fffffff;
    for (int r = 0; r < g.rpb; ++r) {
      float v = sv[r * g.cb + col];
      int ix = si[r * g.cb + col];
      if (v > bv || (v == bv && ix < bidx)) { bv = v; bidx = ix; }   // first index on ties (R15)
    }
    out[(int64_t)b * obs + n * old + c] = bv;
    amax[((int64_t)b * N + n) * C + c] = bidx;
  }
}

// step 1 of the max backward: per (b, c) loop over samples n: dz at the argmax
// row, dbeta = sum dz, dgamma = sum dz*xhat; writes coef (k1,k2,k3) and dz [B][N][C].
template <typename T>
__global__ void k_bn_max_bwd_small(int B, int64_t N, int64_t L, int64_t C, const float* __restrict__ dG, int64_t gbs_,
                                   int64_t gld, const T* __restrict__ X, int64_t xbs, int64_t xld,
                                   const int32_t* __restrict__ amax, const float* __restrict__ gamma,
                                   const float* __restrict__ beta, int64_t gbs, const float* __restrict__ smean,
                                   const float* __restrict__ sinv, int act, float alpha, float* __restrict__ dgamma,
                                   float* __restrict__ dbeta, float* __restrict__ coef, float* __restrict__ dz_out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * C) return;
  int64_t b = i / C, c = i % C;
  float m = smean[i], is = sinv[i], ga = gamma[b * gbs + c], be = beta[b * gbs + c];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t n = 0; n < N; ++n) {
    int64_t l = amax[(b * N + n) * C + c];
    float x = ldf(X + b * xbs + (n * L + l) * xld + c);
    float xh = (x - m) * is;
    float fa, fc;
    bn_affine(ga, be, m, is, fa, fc);
    float dz = dG[b * gbs_ + n * gld + c] * act_grad(fmaf(x, fa, fc), act, alpha);
    dz_out[(b * N + n) * C + c] = dz;
    s1 += dz;
    s2 += (double)dz * xh;
  }
  float db = (float)s1, dg = (float)s2;
  dbeta[b * gbs + c] = db;
  dgamma[b * gbs + c] = dg;
  const double R = (double)(N * L);
  coef[i] = ga * is;
  coef[(int64_t)B * C + i] = (float)(s1 / R);
  coef[2 * (int64_t)B * C + i] = (float)(s2 / R);
}

// step 2: dense dX = k1 * (0 - k2 - xhat*k3) for every row (the scattered
// gradient is zero off the argmax rows), grid (colgroups, chunks, B).
template <typename T, int VEC>
__global__ void __launch_bounds__(NT) k_bn_max_bwd_apply(int B, int64_t N, int64_t L, int64_t C,
                                                         const T* __restrict__ X, int64_t xbs, int64_t xld,
                                                         T* __restrict__ dX, int64_t obs, int64_t old,
                                                         const float* __restrict__ smean,
                                                         const float* __restrict__ sinv,
                                                         const float* __restrict__ coef, Geo g) {
  const int b = blockIdx.z, chunk = blockIdx.y;
  const int lane = threadIdx.x % g.tpr, rl = threadIdx.x / g.tpr;
  const int64_t c0 = (int64_t)blockIdx.x * g.cb + (int64_t)lane * VEC;
  if (c0 >= C) return;
  const int64_t BC = (int64_t)B * C;
  float sc[VEC], sf[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    int64_t i = (int64_t)b * C + c0 + v;
    // k1*(-k2 - (x - m)*is*k3) = x*(-k1*is*k3) + k1*(m*is*k3 - k2)
    const float k1 = coef[i], k2 = coef[BC + i], k3 = coef[2 * BC + i], m = smean[i], is = sinv[i];
    sc[v] = -k1 * is * k3;
    sf[v] = k1 * (m * is * k3 - k2);
  }
  const int64_t R = N * L;
  const T* Xb = X + (int64_t)b * xbs;
  T* Ob = dX + (int64_t)b * obs;
  const int64_t r0 = (int64_t)chunk * g.rows_per_chunk;
  const int64_t r1 = min(R, r0 + g.rows_per_chunk);
  for (int64_t r = r0 + rl; r < r1; r += UNR * g.rpb) {
    float x[UNR][VEC];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (r + u * g.rpb < r1) ld_vec<T, VEC>(Xb + (r + u * g.rpb) * xld + c0, x[u]);
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      if (r + u * g.rpb < r1) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) x[u][v] = fmaf(x[u][v], sc[v], sf[v]);
        st_vec<T, VEC>(Ob + (r + u * g.rpb) * old + c0, x[u]);
      }
  }
}

// step 3: the argmax rows, recomputed in full: dX = k1 * (dz - k2 - xhat*k3).
template <typename T>
__global__ void k_bn_max_bwd_scatter(int B, int64_t N, int64_t L, int64_t C, const T* __restrict__ X, int64_t xbs,
                                     int64_t xld, const int32_t* __restrict__ amax, const float* __restrict__ dz,
                                     T* __restrict__ dX, int64_t obs, int64_t old, const float* __restrict__ smean,
                                     const float* __restrict__ sinv, const float* __restrict__ coef) {
  const int64_t tot = (int64_t)B * N * C;
  const int64_t BC = (int64_t)B * C;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < tot; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = j / (N * C), c = j % C, n = (j / C) % N;
    const int64_t r = n * L + amax[j];
    const int64_t i = b * C + c;
    const float xh = (ldf(X + b * xbs + r * xld + c) - smean[i]) * sinv[i];
    stf(dX + b * obs + r * old + c, coef[i] * (dz[j] - coef[BC + i] - xh * coef[2 * BC + i]));
  }
}

int pick_vec(hfta_dtype dt, int64_t C, std::initializer_list<std::tuple<const void*, int64_t, int64_t>> ts) {
  int vec = dt == HFTA_BF16 ? 8 : 4;
  for (auto& t : ts)
    if (!vec_ok(std::get<0>(t), std::get<1>(t), std::get<2>(t), C, vec)) return 1;
  return vec;
}

// backward passes read 2 tensors: more row chunks in flight (measured)
int bn_bwd_bps() { static int v = env_int("HFTA_BN_BWD_BPS", 32); return v; }
int bn_s1() { static int v = env_int("HFTA_BN_S1", 16); return v; }   // ring stages, one-stream kernels
int bn_s2() { static int v = env_int("HFTA_BN_S2", 8); return v; }    // ring stages, two-stream kernels

template <typename K_, typename... A>
void launch_pipe(K_* kern, size_t smem, dim3 grid, cudaStream_t s, A... args) {
  ensure_smem(kern, smem);
  kern<<<grid, NT, smem, s>>>(args...);
}
// one-stream kernels (stats, apply) at S1 in {8, 16}; two-stream (bwd reduce / apply) at S2 in {4, 8}
#define LAUNCH_P1(T, KERNEL, GRID, ...)                                                        \
  do {                                                                                        \
    constexpr int V_ = 16 / (int)sizeof(T);                                                   \
    if (bn_s1() <= 8) launch_pipe(KERNEL<T, V_, 8, 4>, pipe_smem<T, V_, 1, 8>(), GRID, s, __VA_ARGS__);   \
    else launch_pipe(KERNEL<T, V_, 16, 3>, pipe_smem<T, V_, 1, 16>(), GRID, s, __VA_ARGS__);             \
  } while (0)
#define LAUNCH_P2(T, KERNEL, GRID, ...)                                                        \
  do {                                                                                        \
    constexpr int V_ = 16 / (int)sizeof(T);                                                   \
    if (bn_s2() <= 4) launch_pipe(KERNEL<T, V_, 4, 3>, pipe_smem<T, V_, 2, 4>(), GRID, s, __VA_ARGS__);   \
    else launch_pipe(KERNEL<T, V_, 8, 3>, pipe_smem<T, V_, 2, 8>(), GRID, s, __VA_ARGS__);               \
  } while (0)

size_t bn_parts_bytes(int B, int64_t R, int64_t C) {
  int ch = 1;
  for (int vec : {1, 4, 8})
    for (int bps : {0, bn_bwd_bps()}) ch = std::max(ch, make_geo(B, R, C, vec, bps, bn_run()).chunks);
  return align_up(2 * (size_t)B * ch * C * sizeof(double), 256);
}

// fallback of the epilogue statistics: thread = (model b, 32-row block, column)
template <typename T>
__global__ void k_colstat_rows(int B, int64_t M, int64_t N, const T* __restrict__ Y, int64_t ybs, int64_t yld,
                               float* __restrict__ cs) {
  const int64_t nblk = (M + 31) / 32;
  const int64_t total = (int64_t)B * nblk * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i % N, k = (i / N) % nblk, b = i / (N * nblk);
    const T* y = Y + b * ybs + 32 * k * yld + n;
    const int rows = (int)min((int64_t)32, M - 32 * k);
    float s1 = 0.f, s2 = 0.f;
    for (int r = 0; r < rows; ++r) {
      const float x = ldf(y + r * yld);
      s1 += x;
      s2 = fmaf(x, x, s2);
    }
    float* o = cs + ((b * nblk + k) * 2) * N + n;
    o[0] = s1;
    o[N] = s2;
  }
}

}  // namespace

hfta_status colstat_rows(int B, int64_t M, int64_t N, hfta_dtype dt, hfta_in Y, float* colstat, cudaStream_t s) {
  const int64_t total = (int64_t)B * ((M + 31) / 32) * N;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 16);
  if (dt == HFTA_F32) k_colstat_rows<float><<<grid, 256, 0, s>>>(B, M, N, (const float*)Y.ptr, Y.bstride, Y.ld, colstat);
  else k_colstat_rows<__nv_bfloat16><<<grid, 256, 0, s>>>(B, M, N, (const __nv_bfloat16*)Y.ptr, Y.bstride, Y.ld,
                                                         colstat);
  count_launches(1);
  return HFTA_OK;
}
}  // namespace hfta

using namespace hfta;

#define LAUNCH_VEC(T, vec, KERNEL, GRID, ...)                                                   \
  do {                                                                                        \
    if (vec == 1) KERNEL<T, 1><<<GRID, NT, 0, s>>>(__VA_ARGS__);                               \
    else if (vec == 4) KERNEL<T, 4><<<GRID, NT, 0, s>>>(__VA_ARGS__);                          \
    else KERNEL<T, 8><<<GRID, NT, 0, s>>>(__VA_ARGS__);                                        \
  } while (0)

// the register-staged kernels serve unaligned / odd-width tensors (VEC = 1)
#define LAUNCH_V1(T, KERNEL, GRID, ...) KERNEL<T, 1, 1, 3><<<GRID, NT, 0, s>>>(__VA_ARGS__)

#define DT_DISPATCH(dt, ...)                                                                   \
  do {                                                                                        \
    if (dt == HFTA_F32) { using T = float; __VA_ARGS__; }                                     \
    else { using T = __nv_bfloat16; __VA_ARGS__; }                                            \
  } while (0)

extern "C" {

size_t hfta_fused_bn_workspace(int B, int64_t R, int64_t C) {
  if (B < 1 || R < 1 || C < 1) return 0;
  return bn_parts_bytes(B, R, C) + align_up(5 * (size_t)B * C * sizeof(float), 256);
}

hfta_status hfta_fused_bn_fwd(int B, int64_t R, int64_t C, hfta_dtype dt, hfta_in X, const float* gamma,
                              const float* beta, int64_t gb_bstride, float* running_mean, float* running_var,
                              float momentum, float eps, hfta_act act, float act_alpha, hfta_out Y,
                              float* save_mean, float* save_invstd, void* ws, size_t ws_bytes,
                              hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(R >= 2 && C >= 1, HFTA_ERR_SHAPE, "bn_fwd: R=%lld (needs >= 2), C=%lld", (long long)R, (long long)C);
  HFTA_REQUIRE(X.ptr && gamma && beta && save_mean && save_invstd, HFTA_ERR_INVALID_VALUE,
               "bn_fwd: X, gamma, beta, save_mean, save_invstd are required");
  HFTA_REQUIRE(X.ld >= C && (!Y.ptr || Y.ld >= C), HFTA_ERR_SHAPE, "bn_fwd: ld < C");
  HFTA_REQUIRE(!Y.ptr || Y.bstride > 0 || B == 1, HFTA_ERR_SHAPE, "bn_fwd: Y.bstride must be > 0");
  size_t need = hfta_fused_bn_workspace(B, R, C);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "bn_fwd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  int vec = pick_vec(dt, C, {{X.ptr, X.ld, X.bstride}, {Y.ptr, Y.ld, Y.bstride}});
  Geo g = make_geo(B, R, C, vec, 0, bn_run());
  Geo ga = make_geo(B, R, C, vec);
  double* p1 = reinterpret_cast<double*>(ws);
  double* p2 = p1 + (size_t)B * g.chunks * C;
  dim3 grid(g.colgroups, g.chunks, B), grida(ga.colgroups, ga.chunks, B);
    DT_DISPATCH(dt, {
    if (vec > 1) LAUNCH_P1(T, k_bn_stats_p, grid, R, C, (const T*)X.ptr, X.bstride, X.ld, g, p1, p2);
    else LAUNCH_V1(T, k_bn_stats, grid, R, C, (const T*)X.ptr, X.bstride, X.ld, g, p1, p2);
    k_bn_finalize<T><<<dim3((unsigned)cdiv(C, 32), (unsigned)B), 256, 0, s>>>(
        B, R, C, (const T*)X.ptr, X.bstride, g.chunks, p1, p2, eps, momentum, running_mean, running_var,
        save_mean, save_invstd);
    if (Y.ptr)
    {
      if (vec > 1)
        LAUNCH_P1(T, k_bn_apply_p, grida, R, C, (const T*)X.ptr, X.bstride, X.ld, (T*)Y.ptr, Y.bstride, Y.ld,
                  gamma, beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha, ga);
      else
        LAUNCH_V1(T, k_bn_apply, grida, R, C, (const T*)X.ptr, X.bstride, X.ld, (T*)Y.ptr, Y.bstride, Y.ld,
                  gamma, beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha, ga);
    }
  });
  count_launches(Y.ptr ? 3 : 2);
  return post_launch(s, "hfta_fused_bn_fwd");
}

hfta_status hfta_fused_bn_fwd_colstat(int B, int64_t R, int64_t C, hfta_dtype dt, hfta_in X, const float* gamma,
                                      const float* beta, int64_t gb_bstride, float* running_mean, float* running_var,
                                      float momentum, float eps, hfta_act act, float act_alpha, hfta_out Y,
                                      float* save_mean, float* save_invstd, const float* colstat,
                                      hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(R >= 2 && C >= 1, HFTA_ERR_SHAPE, "bn_fwd_colstat: R=%lld (needs >= 2), C=%lld", (long long)R,
               (long long)C);
  HFTA_REQUIRE(X.ptr && Y.ptr && gamma && beta && save_mean && save_invstd && colstat, HFTA_ERR_INVALID_VALUE,
               "bn_fwd_colstat: X, Y, gamma, beta, save_mean, save_invstd, colstat are required");
  HFTA_REQUIRE(X.ld >= C && Y.ld >= C && (Y.bstride > 0 || B == 1), HFTA_ERR_SHAPE, "bn_fwd_colstat: strides");
  cudaStream_t s = (cudaStream_t)stream;
  k_bn_finalize_colstat<<<dim3((unsigned)cdiv(C, 32), (unsigned)B), 256, 0, s>>>(
      B, R, C, cdiv(R, 32), colstat, eps, momentum, running_mean, running_var, save_mean, save_invstd);
  const int vec = pick_vec(dt, C, {{X.ptr, X.ld, X.bstride}, {Y.ptr, Y.ld, Y.bstride}});
  Geo ga = make_geo(B, R, C, vec);
  dim3 grida(ga.colgroups, ga.chunks, B);
  DT_DISPATCH(dt, {
    if (vec > 1)
      LAUNCH_P1(T, k_bn_apply_p, grida, R, C, (const T*)X.ptr, X.bstride, X.ld, (T*)Y.ptr, Y.bstride, Y.ld, gamma,
                beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha, ga);
    else
      LAUNCH_V1(T, k_bn_apply, grida, R, C, (const T*)X.ptr, X.bstride, X.ld, (T*)Y.ptr, Y.bstride, Y.ld, gamma, beta,
                gb_bstride, save_mean, save_invstd, (int)act, act_alpha, ga);
  });
  count_launches(2);
  return post_launch(s, "hfta_fused_bn_fwd_colstat");
}

hfta_status hfta_fused_bn_bwd(int B, int64_t R, int64_t C, hfta_dtype dt, hfta_in dY, hfta_in X,
                              const float* gamma, const float* beta, int64_t gb_bstride, const float* save_mean,
                              const float* save_invstd, hfta_act act, float act_alpha, hfta_out dX,
                              float* dgamma, float* dbeta, int accumulate, void* ws, size_t ws_bytes,
                              hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(R >= 2 && C >= 1, HFTA_ERR_SHAPE, "bn_bwd: R=%lld, C=%lld", (long long)R, (long long)C);
  HFTA_REQUIRE(dY.ptr && X.ptr && gamma && beta && save_mean && save_invstd && dX.ptr, HFTA_ERR_INVALID_VALUE,
               "bn_bwd: dY, X, gamma, beta, save_mean, save_invstd, dX are required");
  HFTA_REQUIRE(dX.bstride > 0 || B == 1, HFTA_ERR_SHAPE, "bn_bwd: dX.bstride must be > 0");
  size_t need = hfta_fused_bn_workspace(B, R, C);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "bn_bwd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  int vec = pick_vec(dt, C, {{X.ptr, X.ld, X.bstride}, {dY.ptr, dY.ld, dY.bstride}, {dX.ptr, dX.ld, dX.bstride}});
  Geo g = make_geo(B, R, C, vec, bn_bwd_bps(), bn_run());
  Geo ga = make_geo(B, R, C, vec, bn_bwd_bps());
  double* p1 = reinterpret_cast<double*>(ws);
  double* p2 = p1 + (size_t)B * g.chunks * C;
  size_t parts_bytes = bn_parts_bytes(B, R, C);
  float* coef = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + parts_bytes);
  dim3 grid(g.colgroups, g.chunks, B), grida(ga.colgroups, ga.chunks, B);
    DT_DISPATCH(dt, {
    if (vec > 1) LAUNCH_P2(T, k_bn_bwd_reduce_p, grid, R, C, (const T*)dY.ptr, dY.bstride, dY.ld, (const T*)X.ptr,
               X.bstride, X.ld, gamma, beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha, g, p1, p2);
    else LAUNCH_V1(T, k_bn_bwd_reduce, grid, R, C, (const T*)dY.ptr, dY.bstride, dY.ld, (const T*)X.ptr,
               X.bstride, X.ld, gamma, beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha, g, p1, p2);
    k_bn_bwd_finalize<<<dim3((unsigned)cdiv(C, 32), (unsigned)B), 256, 0, s>>>(
        B, R, C, g.chunks, p1, p2, gamma, beta, gb_bstride, save_mean, save_invstd, dgamma, dbeta, accumulate, coef);
    if (vec > 1) LAUNCH_P2(T, k_bn_bwd_apply_p, grida, B, R, C, (const T*)dY.ptr, dY.bstride, dY.ld, (const T*)X.ptr,
              X.bstride, X.ld, (T*)dX.ptr, dX.bstride, dX.ld, (int)act, act_alpha, ga, coef);
    else LAUNCH_V1(T, k_bn_bwd_apply, grida, B, R, C, (const T*)dY.ptr, dY.bstride, dY.ld, (const T*)X.ptr,
              X.bstride, X.ld, (T*)dX.ptr, dX.bstride, dX.ld, (int)act, act_alpha, ga, coef);
  });
  count_launches(3);
  return post_launch(s, "hfta_fused_bn_bwd");
}

hfta_status hfta_bn_max_fwd(int B, int64_t N, int64_t L, int64_t C, hfta_dtype dt, hfta_in X, const float* gamma,
                            const float* beta, int64_t gb_bstride, const float* save_mean,
                            const float* save_invstd, hfta_act act, float act_alpha, hfta_out out,
                            int32_t* argmax, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(N >= 1 && L >= 1 && C >= 1, HFTA_ERR_SHAPE, "bn_max_fwd: N,L,C = %lld,%lld,%lld", (long long)N,
               (long long)L, (long long)C);
  HFTA_REQUIRE(X.ptr && gamma && beta && save_mean && save_invstd && out.ptr && argmax, HFTA_ERR_INVALID_VALUE,
               "bn_max_fwd: null argument");
  HFTA_REQUIRE(out.ld >= C && (out.bstride > 0 || B == 1), HFTA_ERR_SHAPE, "bn_max_fwd: out stride");
  cudaStream_t s = (cudaStream_t)stream;
  int vec = pick_vec(dt, C, {{X.ptr, X.ld, X.bstride}});
  Geo g = make_geo(B, N * L, C, vec);
  dim3 grid(g.colgroups, (unsigned)N, B);
  DT_DISPATCH(dt, {
    LAUNCH_VEC(T, vec, k_bn_max_fwd, grid, L, C, (const T*)X.ptr, X.bstride, X.ld, gamma, beta, gb_bstride,
               save_mean, save_invstd, (int)act, act_alpha, (float*)out.ptr, out.bstride, out.ld, argmax, N, g);
  });
  count_launches(1);
  return post_launch(s, "hfta_bn_max_fwd");
}

size_t hfta_bn_max_bwd_workspace(int B, int64_t N, int64_t C) {
  if (B < 1 || N < 1 || C < 1) return 0;
  return align_up(3 * (size_t)B * C * sizeof(float), 256) + align_up((size_t)B * N * C * sizeof(float), 256);
}

hfta_status hfta_bn_max_bwd(int B, int64_t N, int64_t L, int64_t C, hfta_dtype dt, hfta_in dG, hfta_in X,
                            const int32_t* argmax, const float* gamma, const float* beta, int64_t gb_bstride,
                            const float* save_mean, const float* save_invstd, hfta_act act, float act_alpha,
                            hfta_out dX, float* dgamma, float* dbeta, void* ws, size_t ws_bytes,
                            hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(N >= 1 && L >= 1 && C >= 1 && N * L >= 2, HFTA_ERR_SHAPE, "bn_max_bwd: bad N,L,C");
  HFTA_REQUIRE(dG.ptr && X.ptr && argmax && gamma && beta && save_mean && save_invstd && dX.ptr && dgamma && dbeta,
               HFTA_ERR_INVALID_VALUE, "bn_max_bwd: null argument");
  size_t need = hfta_bn_max_bwd_workspace(B, N, C);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "bn_max_bwd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  float* coef = reinterpret_cast<float*>(ws);
  float* dz = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + align_up(3 * (size_t)B * C * sizeof(float), 256));
  int vec = pick_vec(dt, C, {{X.ptr, X.ld, X.bstride}, {dX.ptr, dX.ld, dX.bstride}});
  Geo g = make_geo(B, N * L, C, vec);
  dim3 grid(g.colgroups, g.chunks, B);
  DT_DISPATCH(dt, {
    k_bn_max_bwd_small<T><<<(unsigned)cdiv((int64_t)B * C, 128), 128, 0, s>>>(
        B, N, L, C, (const float*)dG.ptr, dG.bstride, dG.ld, (const T*)X.ptr, X.bstride, X.ld, argmax, gamma, beta,
        gb_bstride, save_mean, save_invstd, (int)act, act_alpha, dgamma, dbeta, coef, dz);
    LAUNCH_VEC(T, vec, k_bn_max_bwd_apply, grid, B, N, L, C, (const T*)X.ptr, X.bstride, X.ld,
               (T*)dX.ptr, dX.bstride, dX.ld, save_mean, save_invstd, coef, g);
    k_bn_max_bwd_scatter<T><<<(unsigned)std::min<int64_t>(cdiv((int64_t)B * N * C, 256), 4096), 256, 0, s>>>(
        B, N, L, C, (const T*)X.ptr, X.bstride, X.ld, argmax, dz, (T*)dX.ptr, dX.bstride, dX.ld, save_mean,
        save_invstd, coef);
  });
  count_launches(3);
  return post_launch(s, "hfta_bn_max_bwd");
}

}  // extern "C"
