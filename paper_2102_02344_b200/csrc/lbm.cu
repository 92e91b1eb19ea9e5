// lbm.cu -- the fused PointNet point-feature block on tensor cores (K10):
//
//   Y = X W^T (+ bias)         Conv1d(k=1) K -> C over the R = N*L points   (App. B)
//   Z = act(BN_train(Y))       BatchNorm1d over all R points                (App. B)
//   G[n][c] = max_l Z[n*L+l][c]   max over the L points of cloud n          (App. B)
//
// for all B models in one persistent launch per pass, WITHOUT materialising
// the [B][R][C] pre-BN activation Y in HBM:
//
//  forward   k_lbm_fwd: Y^T chunks (channels on the TMEM lanes, points on the
//            columns) are produced by tcgen05 into TMEM and reduced by the
//            epilogue warps straight out of TMEM -- per (model, cloud,
//            channel): sum Y, sum Y^2, and the extreme value + first index
//            (max over l of act(gamma*xhat+beta) sits at max_l Y when
//            gamma >= 0 and at min_l Y when gamma < 0; the sign is folded into
//            a flipped copy of W so the epilogue always takes a max).
//            k_lbm_fwd_fin combines the per-cloud moments (Chan et al.,
//            fp64), writes mean/invstd/running statistics and the pooled
//            output.  HBM traffic: X once (+ W, + B*N*C partials) instead of
//            writing Y and reading it twice.
//  backward  dY = gamma*invstd*(dZ - dbeta/R - xhat*dgamma/R) with dZ nonzero
//            only at the argmax rows (dZ = act'(z) * dG there), i.e.
//            dY[r][c] = bx_c * Y[r][c] + cc_c  (+ a_c*dz at r = argmax),
//            an affine function of the recomputable Y.  k_lbm_dgrad
//            (dX = dY W) and k_lbm_wgrad (dW = dY^T X) each recompute their
//            Y^T tile in TMEM (tensor cores are idle otherwise: the layer is
//            HBM-bound by 8x), transform it into a bf16 dY tile in shared
//            memory (UMMA layout, argmax rows patched) and feed it straight
//            back into tcgen05 -- dY never reaches HBM either.
//
// Roles per CTA (320 threads, 1 CTA/SM, persistent): warp 0 TMA producer,
// warp 1 single-thread MMA issuer, warps 2..9 epilogue / transform (two per
// TMEM lane quarter).
#include "tc_common.cuh"

namespace hfta {
namespace {

constexpr int LT = 320;
constexpr int NEPIW = 8;
constexpr int CBLK = 128;                      // channels per UMMA M block
constexpr uint32_t WKB = CBLK * 64 * 2;        // one 64-wide k block of a 128-channel W block: 16 KB
// forward
constexpr int FR = 128;                        // points per chunk (UMMA N): smem operand reads 8 KB / 64 MMA cycles
constexpr int FG = 2;                          // channel blocks per unit: TMEM 2 x FG x FR = 512 columns
constexpr int FSTAGES = 3;
constexpr int NBW = FG / 2;                    // channel blocks per epilogue warp
constexpr int LPB = FR / 32;                   // 32-column TMEM loads per block and chunk
static_assert(NBW * LPB == 4, "epilogue load schedule assumes 4 loads per warp and chunk");
constexpr uint32_t FA_KB = FR * 64 * 2;        // 8 KB per k block of an X chunk
// backward
constexpr int BR = 128;                        // points per tile / chunk
constexpr uint32_t BA_KB = BR * 64 * 2;        // 16 KB per k block of an X tile
constexpr uint32_t DY_BYTES = 2 * CBLK * 64 * 2;   // dY^T tile [128 c][128 r] as two [128][64] sub-tiles
constexpr int DG_WST = 3;                      // dgrad: W block stages
constexpr int WG_AST = 3;                      // wgrad: X chunk stages

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}
__device__ __forceinline__ void st_shared_u16(uint32_t addr, unsigned short v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void tmem_alloc512(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_free512(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}
__device__ __forceinline__ void ld64(uint32_t ta, uint32_t (&u)[64]) {
  tmem_ld32_nowait(ta, *reinterpret_cast<uint32_t(*)[32]>(&u[0]));
  tmem_ld32_nowait(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&u[32]));
  tmem_wait_ld();
}

// ================================================================ forward ==

struct FwdArgs {
  int B, Ncl, nblk, ngroups, teams, nkb, a_shared, mode;
  int64_t L, C;
  float* s1; float* s2; float* mx; int32_t* idx;   // per-cloud partials [B][Ncl][C]
};

// Packed fp32x2 arithmetic (FADD2 / FFMA2) and 3-input max (FMNMX3) keep the
// epilogue's issue count at ~2 instructions per accumulator element, below
// the MMA rate for K = 128 (one 64-point chunk: 1024 MMA cycles per SM).
__device__ __forceinline__ unsigned long long pk2(uint32_t lo, uint32_t hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ void add2(unsigned long long& acc, unsigned long long v) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(v));
}
__device__ __forceinline__ void sq2(unsigned long long& acc, unsigned long long v) {
  asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(v));
}
__device__ __forceinline__ float hsum2(unsigned long long v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo + hi;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float uf(uint32_t x) { return __uint_as_float(x); }

// Per-channel running state of the forward epilogue: packed sums, running
// max m and the 16-point group it came from; the group's values sit in this
// lane's smem slot so the exact first index is resolved once per cloud.
struct FwdAcc {
  unsigned long long s1[2], s2[2];
  float m;
  int gid;
};

// One 16-point group (values u[o..o+15]) of one channel.  FULL = all valid.
template <bool FULL>
__device__ __forceinline__ void fwd_group(const uint32_t* u, int valid, int gid, FwdAcc& A, uint32_t slot) {
  uint32_t v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = (FULL || j < valid) ? u[j] : 0u;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const unsigned long long w = pk2(v[2 * q], v[2 * q + 1]);
    add2(A.s1[q & 1], w);
    sq2(A.s2[q & 1], w);
  }
  if (!FULL) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = j < valid ? v[j] : __float_as_uint(-INFINITY);
  }
  const float a0 = max3(uf(v[0]), uf(v[1]), uf(v[2])), a1 = max3(uf(v[3]), uf(v[4]), uf(v[5]));
  const float a2 = max3(uf(v[6]), uf(v[7]), uf(v[8])), a3 = max3(uf(v[9]), uf(v[10]), uf(v[11]));
  const float a4 = max3(uf(v[12]), uf(v[13]), uf(v[14]));
  const float gm = fmaxf(max3(a0, a1, a2), max3(a3, a4, uf(v[15])));
  const bool p = gm > A.m;
  if (__any_sync(0xffffffffu, p)) {
    if (p) {
      A.m = gm;
      A.gid = gid;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        st_shared_v4(slot + q * 512, make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    }
  }
}

__global__ void __launch_bounds__(LT, 1)
k_lbm_fwd(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, FwdArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* wres = smem;                                        // FG blocks x 2 k blocks x 16 KB
  uint8_t* ast = wres + FG * 2 * WKB;                          // FSTAGES x 2 k blocks x 8 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(ast + FSTAGES * 2 * FA_KB);
  uint64_t* empty = full + FSTAGES;
  uint64_t* tfull = empty + FSTAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* wfull = tempty + 2;
  uint64_t* wempty = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
  uint8_t* slot_base = reinterpret_cast<uint8_t*>(full) + 256;        // NEPIW x NBW ch x 4 x 32 lanes x 16 B

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < FSTAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], NEPIW); }
    mbar_init(wfull, 1);
    mbar_init(wempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Team schedule: CTA (team, g) handles channel group g for a contiguous run
  // of (model, cloud) pairs; the ngroups CTAs of a team read the same X chunks
  // at the same time (L2 hits) and each keeps its W group resident across the
  // clouds of a model.
  const int g = blockIdx.x % p.ngroups, team = blockIdx.x / p.ngroups;
  const int64_t npairs = (int64_t)p.B * p.Ncl;
  const int64_t u0 = npairs * team / p.teams, u1 = npairs * (team + 1) / p.teams;
  const int nch = (int)((p.L + FR - 1) / FR);
  const int blk0 = g * FG;
  const int nb = min(FG, p.nblk - blk0);

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
      int stage = 0, curb = -1;
      uint32_t ph = 0, wep = 0;
      for (int64_t u = u0; u < u1; ++u) {
        const int b = (int)(u / p.Ncl), n = (int)(u % p.Ncl);
        if (b != curb) {
          if (curb >= 0) mbar_wait(wempty, (wep - 1) & 1);
          mbar_expect_tx(wfull, (uint32_t)(nb * p.nkb) * WKB);
          for (int j = 0; j < nb; ++j)
            for (int kb = 0; kb < p.nkb; ++kb)
              tma_load_3d(wres + (j * 2 + kb) * WKB, &tmW, wfull, kb * 64, (blk0 + j) * CBLK, b);
          curb = b;
          ++wep;
        }
        const int ba = p.a_shared ? 0 : b;
        for (int ch = 0; ch < nch; ++ch) {
          mbar_wait(&empty[stage], ph ^ 1);
          mbar_expect_tx(&full[stage], (uint32_t)p.nkb * FA_KB);
          for (int kb = 0; kb < p.nkb; ++kb)
            tma_load_3d(ast + (stage * 2 + kb) * FA_KB, &tmA, &full[stage], kb * 64, (int)(n * p.L + ch * FR), ba);
          if (++stage == FSTAGES) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t IDESC = idesc_bf16(CBLK, FR, false, false);
    int stage = 0, acc = 0, curb = -1;
    uint32_t ph = 0, aph = 0, wep = 0;
    for (int64_t u = u0; u < u1; ++u) {
      const int b = (int)(u / p.Ncl);
      if (b != curb) {
        if (curb >= 0) tc_commit_w(wempty);
        __syncwarp();
        mbar_wait(wfull, wep & 1);
        curb = b;
        ++wep;
      }
      for (int ch = 0; ch < nch; ++ch) {
        mbar_wait(&tempty[acc], aph ^ 1);
        mbar_wait(&full[stage], ph);
        tc_fence_after();
        {
          const uint64_t bd0 = smem_desc(smem_u32(ast + stage * 2 * FA_KB), 16, 1024);
          for (int j = 0; j < nb; ++j) {
            const uint32_t d = tmem_base + (uint32_t)(acc * FG * FR + j * FR);
            const uint64_t ad0 = smem_desc(smem_u32(wres + j * 2 * WKB), 16, 1024);
            for (int kb = 0; kb < p.nkb; ++kb) {
#pragma unroll
              for (int k = 0; k < 4; ++k)   // +32 B per k step, +WKB / FA_KB per k block (descriptor units of 16 B)
                tc_mma_ss(d, ad0 + (uint64_t)(kb * (WKB >> 4) + 2 * k), bd0 + (uint64_t)(kb * (FA_KB >> 4) + 2 * k), IDESC,
                          (kb | k) != 0 ? 1u : 0u);
            }
          }
          tc_commit_w(&empty[stage]);
          tc_commit_w(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == FSTAGES) { stage = 0; ph ^= 1; }
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else {
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    // per-lane slots [warp][jj][q][lane] x 16 B (conflict-free v4 stores)
    const uint32_t slots = smem_u32(slot_base) + (uint32_t)(((warp - 2) * (NBW * 4 * 32) + lane) * 16);
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t u = u0; u < u1; ++u) {
      const int b = (int)(u / p.Ncl), n = (int)(u % p.Ncl);
      FwdAcc A[NBW];
#pragma unroll
      for (int jj = 0; jj < NBW; ++jj) {
        A[jj].s1[0] = A[jj].s1[1] = A[jj].s2[0] = A[jj].s2[1] = 0ull;
        A[jj].m = -INFINITY;
        A[jj].gid = 0;
      }
      // this warp owns blocks half + 2 jj (when present): nld 32-column loads per chunk
      int nld = 0;
#pragma unroll
      for (int jj = 0; jj < NBW; ++jj) nld += half + 2 * jj < nb ? LPB : 0;
      for (int ch = 0; ch < nch; ++ch) {
        const int valid = (int)min((int64_t)FR, p.L - (int64_t)ch * FR);
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t ta = tmem_base + (uint32_t)(acc * FG * FR + half * FR) + ((uint32_t)(quarter * 32) << 16);
        auto release = [&]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        };
        // load i+1 is in flight while load i is reduced; i -> (block jj = i/2, columns hh = i%2)
        auto proc = [&](const uint32_t (&r)[32], int i) {
          const int jj = i / LPB, hh = i % LPB;
          const int g0 = ch * (FR / 16) + hh * 2;
          const uint32_t sl = slots + (uint32_t)(jj * 4 * 32 * 16);
          if (p.mode == 1) {
            if (r[0] == 0x7f800001u && r[31] == 0x7f800001u) A[jj].m = 1.f;   // diagnostics: keep the load live
          } else if (valid == FR) {
            fwd_group<true>(r, 16, g0, A[jj], sl);
            fwd_group<true>(r + 16, 16, g0 + 1, A[jj], sl);
          } else {
            fwd_group<false>(r, valid - hh * 32, g0, A[jj], sl);
            fwd_group<false>(r + 16, valid - hh * 32 - 16, g0 + 1, A[jj], sl);
          }
        };
        uint32_t r0[32], r1[32];
        if (nld == 0) {
          release();
        } else {
          tmem_ld32_nowait(ta, r0);
          tmem_wait_ld();
          auto col = [](int i) { return (uint32_t)(2 * (i / LPB) * FR + (i % LPB) * 32); };
          tmem_ld32_nowait(ta + col(1), r1);
          proc(r0, 0);
          tmem_wait_ld();
          if (nld == 4) tmem_ld32_nowait(ta + col(2), r0);
          else release();
          proc(r1, 1);
          if (nld == 4) {
            tmem_wait_ld();
            tmem_ld32_nowait(ta + col(3), r1);
            proc(r0, 2);
            tmem_wait_ld();
            release();
            proc(r1, 3);
          }
        }
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
#pragma unroll
      for (int jj = 0; jj < NBW; ++jj) {
        const int j = half + 2 * jj;
        if (j >= nb) continue;
        int first = 15;                               // first point of the winning group equal to the max
#pragma unroll
        for (int q = 3; q >= 0; --q) {
          const float4 t4 = ld_shared_f4(slots + (uint32_t)((jj * 4 + q) * 512));
          if (t4.w == A[jj].m) first = 4 * q + 3;
          if (t4.z == A[jj].m) first = 4 * q + 2;
          if (t4.y == A[jj].m) first = 4 * q + 1;
          if (t4.x == A[jj].m) first = 4 * q;
        }
        const int64_t c = (int64_t)(blk0 + j) * CBLK + quarter * 32 + lane;
        const int64_t o = ((int64_t)b * p.Ncl + n) * p.C + c;
        p.s1[o] = hsum2(A[jj].s1[0]) + hsum2(A[jj].s1[1]);
        p.s2[o] = hsum2(A[jj].s2[0]) + hsum2(A[jj].s2[1]);
        p.mx[o] = A[jj].m;
        p.idx[o] = A[jj].gid * 16 + first;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free512(tmem_base);
  }
}

// W' = s_c * W (s_c = -1 where gamma_c < 0): the forward kernel then always
// reduces a max.  Sign flips are exact, so Y' = s * Y bit for bit.
__global__ void k_lbm_flip(int B, int64_t C, int64_t K, const __nv_bfloat16* __restrict__ W, int64_t wbs, int64_t wld,
                           const float* __restrict__ gamma, int64_t gbs, __nv_bfloat16* __restrict__ Wf) {
  const int64_t n = (int64_t)B * C * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i % K, c = (i / K) % C, b = i / (K * C);
    const __nv_bfloat16 w = W[b * wbs + c * wld + k];
    Wf[i] = gamma[b * gbs + c] < 0.f ? __hneg(w) : w;
  }
}

// Per (model, channel): Chan's parallel combination of the per-cloud moments
// in fp64 (fixed cloud order), then statistics, running averages and the
// pooled outputs.
__global__ void k_lbm_fwd_fin(int B, int Ncl, int64_t L, int64_t C, const float* __restrict__ s1,
                              const float* __restrict__ s2, const float* __restrict__ mx,
                              const int32_t* __restrict__ idx, const float* __restrict__ bias, int64_t bias_bs,
                              const float* __restrict__ gamma, const float* __restrict__ beta, int64_t gbs,
                              float* __restrict__ rmean, float* __restrict__ rvar, float momentum, float eps, int act,
                              float alpha, float* __restrict__ G, int64_t g_bs, int64_t g_ld,
                              int32_t* __restrict__ amax, int64_t am_bs, int64_t am_ld, float* __restrict__ ext,
                              int64_t ext_bs, int64_t ext_ld, float* __restrict__ smean, float* __restrict__ sinv) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * C) return;
  const int64_t b = i / C, c = i % C;
  const float ga = gamma[b * gbs + c], be = beta[b * gbs + c];
  const double sg = ga < 0.f ? -1.0 : 1.0;
  const float bi = bias ? bias[b * bias_bs + c] : 0.f;
  double mean = 0.0, M2 = 0.0, cnt = 0.0;
  const double Ld = (double)L;
  for (int n = 0; n < Ncl; ++n) {
    const int64_t o = (b * Ncl + n) * C + c;
    const double t1 = s1[o], t2 = s2[o];
    const double mn = t1 / Ld;
    double m2 = t2 - t1 * mn;
    if (m2 < 0.0) m2 = 0.0;
    const double tot = cnt + Ld, d = mn - mean;
    mean += d * Ld / tot;
    M2 += m2 + d * d * cnt * Ld / tot;
    cnt = tot;
  }
  const double R = cnt;
  const double var = M2 / R;
  const double mean_y = sg * mean;                 // statistics of Y (bias excluded)
  const double inv = 1.0 / sqrt(var + (double)eps);
  const double mean_b = mean_y + (double)bi;       // the layer output includes its bias
  smean[i] = (float)mean_b;
  sinv[i] = (float)inv;
  if (rmean) rmean[i] = (float)((1.0 - momentum) * (double)rmean[i] + momentum * mean_b);
  if (rvar) rvar[i] = (float)((1.0 - momentum) * (double)rvar[i] + momentum * var * R / (R - 1.0));
  const float scale = (float)((double)ga * inv);
  const float mean_f = (float)mean_y;
  for (int n = 0; n < Ncl; ++n) {
    const int64_t o = (b * Ncl + n) * C + c;
    const float ey = (float)(sg * (double)mx[o]);   // Y at the argmax row (bias excluded)
    const float z = scale * (ey - mean_f) + be;
    G[b * g_bs + n * g_ld + c] = act_fwd(z, act, alpha);
    amax[b * am_bs + n * am_ld + c] = idx[o];
    ext[b * ext_bs + n * ext_ld + c] = ey + bi;
  }
}

// =============================================================== backward ==

// Per (model, channel): dz at the pooled rows, dgamma/dbeta, and the affine
// form dY = bx*Y + cc (+ a*dz at the argmax row; pv = the full value there).
__global__ void k_lbm_bwd_coef(int B, int Ncl, int64_t L, int64_t C, const float* __restrict__ dG, int64_t dg_bs,
                               int64_t dg_ld, const float* __restrict__ ext, int64_t ext_bs, int64_t ext_ld,
                               const float* __restrict__ bias, int64_t bias_bs, const float* __restrict__ gamma,
                               const float* __restrict__ beta, int64_t gbs, const float* __restrict__ smean,
                               const float* __restrict__ sinv, int act, float alpha, float2* __restrict__ coef,
                               float* __restrict__ pv, float* __restrict__ dgamma, float* __restrict__ dbeta,
                               float* __restrict__ dbias, int64_t dbias_bs, int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * C) return;
  const int64_t b = i / C, c = i % C;
  const float ga = gamma[b * gbs + c], be = beta[b * gbs + c];
  const float mb = smean[i], inv = sinv[i];
  const float bi = bias ? bias[b * bias_bs + c] : 0.f;
  double dbe = 0.0, dga = 0.0;
  for (int n = 0; n < Ncl; ++n) {
    const float xh = (ext[b * ext_bs + n * ext_ld + c] - mb) * inv;
    const float dz = dG[b * dg_bs + n * dg_ld + c] * act_grad(ga * xh + be, act, alpha);
    dbe += dz;
    dga += (double)dz * xh;
  }
  const double R = (double)Ncl * (double)L;
  const double a = (double)ga * inv;
  const double bx = -a * inv * dga / R;
  const double cc = -a * dbe / R - bx * ((double)mb - (double)bi);
  coef[i] = make_float2((float)bx, (float)cc);
  for (int n = 0; n < Ncl; ++n) {
    const float e = ext[b * ext_bs + n * ext_ld + c];
    const float xh = (e - mb) * inv;
    const float dz = dG[b * dg_bs + n * dg_ld + c] * act_grad(ga * xh + be, act, alpha);
    pv[(b * Ncl + n) * C + c] = (float)(a * dz + bx * ((double)e - (double)bi) + cc);
  }
  const int64_t go = b * gbs + c;
  if (accumulate) { dgamma[go] += (float)dga; dbeta[go] += (float)dbe; }
  else { dgamma[go] = (float)dga; dbeta[go] = (float)dbe; }
  if (dbias && !accumulate) dbias[b * dbias_bs + c] = 0.f;   // BN-absorbed bias: exact zero
}

struct BwdArgs {
  int B, Ncl, nblk, nkb, a_shared, splits;
  int64_t L, C, R, K, tiles, rps;
  const float2* coef; const float* pv;          // [B][C], [B][Ncl][C]
  const int32_t* am; int64_t am_bs, am_ld;      // argmax (point index within its cloud)
  __nv_bfloat16* dX; int64_t dx_bs, dx_ld;      // dgrad output
  float* dW; int64_t dw_bs, dw_ld; int accumulate;
  float* part;                                  // wgrad split partials [S][B][C][K]
};

// Per-thread operands of one transform (channel c, points r0h..r0h+63):
// the affine coefficients and the argmax rows of the (at most two) clouds
// overlapping the points.  Loaded BEFORE the wait for the recomputed tile so
// their global-load latency overlaps it.
struct BwdPre {
  float bx, cc, v0, v1;
  int a0, a1;            // argmax point index within cloud n0 / n0 + 1 (-1: none)
  int n0, slow;          // slow: more than two clouds overlap (L < 64)
};

__device__ __forceinline__ BwdPre bwd_prefetch(const BwdArgs& p, int b, int64_t c, int64_t r0h) {
  BwdPre q;
  const float2 cf = p.coef[(int64_t)b * p.C + c];
  q.bx = cf.x;
  q.cc = cf.y;
  q.a0 = q.a1 = -1;
  q.v0 = q.v1 = 0.f;
  q.slow = 0;
  q.n0 = 0;
  if (r0h < p.R) {
    const int L = (int)p.L;
    const int n_lo = (int)r0h / L;
    const int n_hi = min(p.Ncl - 1, ((int)r0h + 63) / L);
    q.n0 = n_lo;
    if (n_hi - n_lo > 1) {
      q.slow = 1;
    } else {
      const int32_t* am = p.am + (int64_t)b * p.am_bs + c;
      const float* pv = p.pv + (int64_t)b * p.Ncl * p.C + c;
      q.a0 = am[(int64_t)n_lo * p.am_ld];
      q.v0 = pv[(int64_t)n_lo * p.C];
      if (n_hi > n_lo) {
        q.a1 = am[(int64_t)n_hi * p.am_ld];
        q.v1 = pv[(int64_t)n_hi * p.C];
      }
    }
  }
  return q;
}

__device__ __forceinline__ void patch_u16(uint32_t rowaddr, uint32_t sw, int64_t j, float v) {
  if (j >= 0 && j < 64) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    st_shared_u16(rowaddr + ((((uint32_t)j >> 3) ^ sw) << 4) + ((uint32_t)j & 7) * 2,
                  *reinterpret_cast<const unsigned short*>(&h));
  }
}

// Transform one thread's 64 recomputed Y^T values (channel c, points
// r0h..r0h+63) into bf16 dY in the dY^T sub-tile row (SW128 layout: 16-B chunk
// q of row cl at q ^ (cl & 7)), then patch the argmax rows.
__device__ __forceinline__ void bwd_transform(const uint32_t (&u)[64], const BwdPre& q, const BwdArgs& p, int b,
                                              int64_t c, int64_t r0h, uint32_t rowaddr, uint32_t sw) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint4 w4;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      h[e] = __floats2bfloat162_rn(fmaf(q.bx, __uint_as_float(u[8 * k + 2 * e]), q.cc),
                                   fmaf(q.bx, __uint_as_float(u[8 * k + 2 * e + 1]), q.cc));
    st_shared_v4(rowaddr + (((uint32_t)k ^ sw) << 4), w4);
  }
  if (r0h >= p.R) return;
  if (!q.slow) {
    if (q.a0 >= 0) patch_u16(rowaddr, sw, (int64_t)q.n0 * p.L + q.a0 - r0h, q.v0);
    if (q.a1 >= 0) patch_u16(rowaddr, sw, (int64_t)(q.n0 + 1) * p.L + q.a1 - r0h, q.v1);
    return;
  }
  const int n_hi = (int)min((int64_t)p.Ncl - 1, (r0h + 63) / p.L);
  for (int n = q.n0; n <= n_hi; ++n) {
    const int64_t row = (int64_t)n * p.L + p.am[(int64_t)b * p.am_bs + (int64_t)n * p.am_ld + c];
    patch_u16(rowaddr, sw, row - r0h, p.pv[((int64_t)b * p.Ncl + n) * p.C + c]);
  }
}

// ---------------------------------------------------------------- dgrad --
// Unit = (model, 128-point tile).  Per channel block cb: recompute Y^T[cb]
// (M = 128 channels, N = 128 points, K), transform to dY^T[cb] in smem, then
// dX_tile += dY[cb] W[cb] (M = 128 points from the MN-major dY^T tile,
// N = K from the MN-major W block, K = 128 channels).  The recompute of cb+1
// overlaps the transform of cb.
__global__ void __launch_bounds__(LT, 1)
k_lbm_dgrad(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, BwdArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* at = smem;                                  // 2 x 2 k blocks x 16 KB
  uint8_t* wst = at + 2 * 2 * BA_KB;                   // DG_WST x 2 k blocks x 16 KB
  uint8_t* dyt = wst + DG_WST * 2 * WKB;               // 2 x 32 KB
  uint64_t* a_full = reinterpret_cast<uint64_t*>(dyt + 2 * DY_BYTES);
  uint64_t* a_empty = a_full + 2;
  uint64_t* w_full = a_empty + 2;
  uint64_t* w_empty = w_full + DG_WST;
  uint64_t* y_full = w_empty + DG_WST;
  uint64_t* y_empty = y_full + 2;
  uint64_t* dy_full = y_empty + 2;
  uint64_t* dy_empty = dy_full + 2;
  uint64_t* d_full = dy_empty + 2;
  uint64_t* d_empty = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a_full[s], 1); mbar_init(&a_empty[s], 1);
      mbar_init(&y_full[s], 1); mbar_init(&y_empty[s], NEPIW);
      mbar_init(&dy_full[s], NEPIW); mbar_init(&dy_empty[s], 1);
      mbar_init(&d_full[s], 1); mbar_init(&d_empty[s], NEPIW);
    }
    for (int s = 0; s < DG_WST; ++s) { mbar_init(&w_full[s], 1); mbar_init(&w_empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;           // cols [0,256): Y^T x2, [256,512): dX x2
  const int64_t total = (int64_t)p.B * p.tiles;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
      int ab = 0, ws = 0;
      uint32_t aph = 0, wph = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        const int b = (int)(t / p.tiles);
        const int r0 = (int)((t % p.tiles) * BR);
        mbar_wait(&a_empty[ab], aph ^ 1);
        mbar_expect_tx(&a_full[ab], (uint32_t)p.nkb * BA_KB);
        for (int kb = 0; kb < p.nkb; ++kb)
          tma_load_3d(at + (ab * 2 + kb) * BA_KB, &tmA, &a_full[ab], kb * 64, r0, p.a_shared ? 0 : b);
        if (++ab == 2) { ab = 0; aph ^= 1; }
        for (int cb = 0; cb < p.nblk; ++cb) {
          mbar_wait(&w_empty[ws], wph ^ 1);
          mbar_expect_tx(&w_full[ws], (uint32_t)p.nkb * WKB);
          for (int kb = 0; kb < p.nkb; ++kb)
            tma_load_3d(wst + (ws * 2 + kb) * WKB, &tmW, &w_full[ws], kb * 64, cb * CBLK, b);
          if (++ws == DG_WST) { ws = 0; wph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc_y = idesc_bf16(CBLK, BR, false, false);
    const uint32_t idesc_d = idesc_bf16(BR, (int)p.K, true, true);
    int ab = 0, ws = 0, yb = 0, dyb = 0, db = 0;
    uint32_t aph = 0, wph = 0, yph = 0, dyph = 0, dph = 0;
    int pws = 0;                                      // W stage of the block awaiting its dgrad
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      mbar_wait(&a_full[ab], aph);
      mbar_wait(&d_empty[db], dph ^ 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(at + ab * 2 * BA_KB);
      const uint32_t dacc = tmem_base + 256 + (uint32_t)(db * 128);
      for (int cb = 0; cb <= p.nblk; ++cb) {
        if (cb < p.nblk) {                              // recompute Y^T[cb]
          mbar_wait(&w_full[ws], wph);
          mbar_wait(&y_empty[yb], yph ^ 1);
          tc_fence_after();
          {
            const uint64_t ad0 = smem_desc(smem_u32(wst + ws * 2 * WKB), 16, 1024), bd0 = smem_desc(sa, 16, 1024);
            const uint32_t d = tmem_base + (uint32_t)(yb * 128);
            for (int kb = 0; kb < p.nkb; ++kb) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc_mma_ss(d, ad0 + (uint64_t)(kb * (WKB >> 4) + 2 * k), bd0 + (uint64_t)(kb * (BA_KB >> 4) + 2 * k), idesc_y,
                          (kb | k) != 0 ? 1u : 0u);
            }
            tc_commit_w(&y_full[yb]);
            if (cb == p.nblk - 1) tc_commit_w(&a_empty[ab]);
          }
          __syncwarp();
          if (++yb == 2) { yb = 0; yph ^= 1; }
        }
        if (cb > 0) {                                   // dX += dY[cb-1] W[cb-1]
          mbar_wait(&dy_full[dyb], dyph);
          tc_fence_after();
          {
            const uint64_t ad0 = smem_desc(smem_u32(dyt + dyb * DY_BYTES), CBLK * 128, 1024);
            const uint64_t bd0 = smem_desc(smem_u32(wst + pws * 2 * WKB), WKB, 1024);
#pragma unroll
            for (int k = 0; k < CBLK / 16; ++k)   // MN-major: +16 rows x 128 B per k step
              tc_mma_ss(dacc, ad0 + (uint64_t)(k * 128), bd0 + (uint64_t)(k * 128), idesc_d, (cb > 1 || k > 0) ? 1u : 0u);
            tc_commit_w(&dy_empty[dyb]);
            tc_commit_w(&w_empty[pws]);
            if (cb == p.nblk) tc_commit_w(&d_full[db]);
          }
          __syncwarp();
          if (++dyb == 2) { dyb = 0; dyph ^= 1; }
        }
        if (cb < p.nblk) {
          pws = ws;
          if (++ws == DG_WST) { ws = 0; wph ^= 1; }
        }
      }
      if (++ab == 2) { ab = 0; aph ^= 1; }
      if (++db == 2) { db = 0; dph ^= 1; }
    }
  } else {
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int cl = quarter * 32 + lane;               // channel within the block (TMEM lane)
    const uint32_t sw = (uint32_t)(cl & 7);
    int yb = 0, dyb = 0, db = 0;
    uint32_t yph = 0, dyph = 0, dph = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const int b = (int)(t / p.tiles);
      const int64_t r0 = (t % p.tiles) * BR;
      for (int cb = 0; cb < p.nblk; ++cb) {
        uint32_t u[64];
        const BwdPre pre = bwd_prefetch(p, b, (int64_t)cb * CBLK + cl, r0 + half * 64);
        mbar_wait(&y_full[yb], yph);
        tc_fence_after();
        ld64(tmem_base + (uint32_t)(yb * 128 + half * 64) + ((uint32_t)(quarter * 32) << 16), u);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&y_empty[yb]);
        if (++yb == 2) { yb = 0; yph ^= 1; }
        mbar_wait(&dy_empty[dyb], dyph ^ 1);
        const uint32_t rowaddr = smem_u32(dyt + dyb * DY_BYTES + half * (CBLK * 128)) + cl * 128;
        bwd_transform(u, pre, p, b, (int64_t)cb * CBLK + cl, r0 + half * 64, rowaddr, sw);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&dy_full[dyb]);
        if (++dyb == 2) { dyb = 0; dyph ^= 1; }
      }
      // dX tile: TMEM lane = point, columns = k
      mbar_wait(&d_full[db], dph);
      tc_fence_after();
      const int64_t r = r0 + quarter * 32 + lane;
      if (half * 64 < p.K) {
        uint32_t u[64];
        ld64(tmem_base + 256 + (uint32_t)(db * 128 + half * 64) + ((uint32_t)(quarter * 32) << 16), u);
        if (r < p.R) {
          __nv_bfloat16* dst = p.dX + (int64_t)b * p.dx_bs + r * p.dx_ld + half * 64;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint4 w4;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              h[e] = __floats2bfloat162_rn(__uint_as_float(u[8 * q + 2 * e]), __uint_as_float(u[8 * q + 2 * e + 1]));
            *reinterpret_cast<uint4*>(dst + 8 * q) = w4;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_empty[db]);
      if (++db == 2) { db = 0; dph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free512(tmem_base);
  }
}

// ---------------------------------------------------------------- wgrad --
// Unit = (model, point split, channel block cb), cb fastest so the nblk CTAs
// of one (model, split) stream the same X chunks together (L2 hits).  Per
// 128-point chunk: recompute Y^T[cb] chunk, transform to dY^T, then
// dW[cb] += dY^T X_chunk (M = 128 channels, K-major dY^T; N = K, MN-major X).
__global__ void __launch_bounds__(LT, 1)
k_lbm_wgrad(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, BwdArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* wr = smem;                                  // W[cb]: 2 k blocks x 16 KB
  uint8_t* ast = wr + 2 * WKB;                         // WG_AST x 2 k blocks x 16 KB
  uint8_t* dyt = ast + WG_AST * 2 * BA_KB;             // 2 x 32 KB
  uint64_t* a_full = reinterpret_cast<uint64_t*>(dyt + 2 * DY_BYTES);
  uint64_t* a_empty = a_full + WG_AST;
  uint64_t* w_full = a_empty + WG_AST;
  uint64_t* w_empty = w_full + 1;
  uint64_t* y_full = w_empty + 1;
  uint64_t* y_empty = y_full + 2;
  uint64_t* dy_full = y_empty + 2;
  uint64_t* dy_empty = dy_full + 2;
  uint64_t* d_full = dy_empty + 2;
  uint64_t* d_empty = d_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&y_full[s], 1); mbar_init(&y_empty[s], NEPIW);
      mbar_init(&dy_full[s], NEPIW); mbar_init(&dy_empty[s], 1);
      mbar_init(&d_full[s], 1); mbar_init(&d_empty[s], NEPIW);
    }
    for (int s = 0; s < WG_AST; ++s) { mbar_init(&a_full[s], 1); mbar_init(&a_empty[s], 1); }
    mbar_init(w_full, 1);
    mbar_init(w_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;           // cols [0,256): Y^T x2, [256,512): dW x2
  const int64_t total = (int64_t)p.B * p.splits * p.nblk;

  auto unit = [&](int64_t t, int& b, int& cb, int64_t& rbeg, int& nch) {
    cb = (int)(t % p.nblk);
    const int64_t r = t / p.nblk;
    const int s = (int)(r % p.splits);
    b = (int)(r / p.splits);
    rbeg = (int64_t)s * p.rps;
    const int64_t rend = min(p.R, rbeg + p.rps);
    nch = rend > rbeg ? (int)((rend - rbeg + BR - 1) / BR) : 0;
  };

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
      int st = 0;
      uint32_t ph = 0, wep = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        int b, cb, nch;
        int64_t rbeg;
        unit(t, b, cb, rbeg, nch);
        if (wep > 0) mbar_wait(w_empty, (wep - 1) & 1);
        mbar_expect_tx(w_full, (uint32_t)p.nkb * WKB);
        for (int kb = 0; kb < p.nkb; ++kb) tma_load_3d(wr + kb * WKB, &tmW, w_full, kb * 64, cb * CBLK, b);
        ++wep;
        for (int j = 0; j < nch; ++j) {
          mbar_wait(&a_empty[st], ph ^ 1);
          mbar_expect_tx(&a_full[st], (uint32_t)p.nkb * BA_KB);
          for (int kb = 0; kb < p.nkb; ++kb)
            tma_load_3d(ast + (st * 2 + kb) * BA_KB, &tmA, &a_full[st], kb * 64, (int)(rbeg + (int64_t)j * BR),
                        p.a_shared ? 0 : b);
          if (++st == WG_AST) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc_y = idesc_bf16(CBLK, BR, false, false);
    const uint32_t idesc_w = idesc_bf16(CBLK, (int)p.K, false, true);
    int st = 0, yb = 0, dyb = 0, db = 0;
    uint32_t ph = 0, yph = 0, dyph = 0, dph = 0, wep = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      int b, cb, nch;
      int64_t rbeg;
      unit(t, b, cb, rbeg, nch);
      mbar_wait(w_full, wep & 1);
      ++wep;
      mbar_wait(&d_empty[db], dph ^ 1);
      tc_fence_after();
      const uint32_t sw = smem_u32(wr);
      const uint32_t dacc = tmem_base + 256 + (uint32_t)(db * 128);
      int pst = 0;
      for (int j = 0; j <= nch; ++j) {
        if (j < nch) {
          mbar_wait(&a_full[st], ph);
          mbar_wait(&y_empty[yb], yph ^ 1);
          tc_fence_after();
          {
            const uint64_t ad0 = smem_desc(sw, 16, 1024), bd0 = smem_desc(smem_u32(ast + st * 2 * BA_KB), 16, 1024);
            const uint32_t d = tmem_base + (uint32_t)(yb * 128);
            for (int kb = 0; kb < p.nkb; ++kb) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                tc_mma_ss(d, ad0 + (uint64_t)(kb * (WKB >> 4) + 2 * k), bd0 + (uint64_t)(kb * (BA_KB >> 4) + 2 * k), idesc_y,
                          (kb | k) != 0 ? 1u : 0u);
            }
            tc_commit_w(&y_full[yb]);
          }
          __syncwarp();
          if (++yb == 2) { yb = 0; yph ^= 1; }
        }
        if (j > 0) {                                    // dW += dY^T[j-1] X[j-1]
          mbar_wait(&dy_full[dyb], dyph);
          tc_fence_after();
          {
            const uint64_t ad0 = smem_desc(smem_u32(dyt + dyb * DY_BYTES), 16, 1024);
            const uint64_t bd0 = smem_desc(smem_u32(ast + pst * 2 * BA_KB), BA_KB, 1024);
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int k = 0; k < 4; ++k)   // A: K-major +32 B per k step; B: MN-major +16 rows x 128 B
                tc_mma_ss(dacc, ad0 + (uint64_t)(h * (CBLK * 128 >> 4) + 2 * k), bd0 + (uint64_t)((h * 64 + k * 16) * 8),
                          idesc_w, (j > 1 || h > 0 || k > 0) ? 1u : 0u);
            tc_commit_w(&dy_empty[dyb]);
            tc_commit_w(&a_empty[pst]);
            if (j == nch) {
              tc_commit_w(&d_full[db]);
              tc_commit_w(w_empty);
            }
          }
          __syncwarp();
          if (++dyb == 2) { dyb = 0; dyph ^= 1; }
        }
        if (j < nch) {
          pst = st;
          if (++st == WG_AST) { st = 0; ph ^= 1; }
        }
      }
      if (nch == 0) {
        if (lane == 0) mbar_arrive(&d_full[db]);
        tc_commit_w(w_empty);
      }
      __syncwarp();
      if (++db == 2) { db = 0; dph ^= 1; }
    }
  } else {
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int cl = quarter * 32 + lane;
    const uint32_t sw = (uint32_t)(cl & 7);
    int yb = 0, dyb = 0, db = 0;
    uint32_t yph = 0, dyph = 0, dph = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      int b, cb, nch;
      int64_t rbeg;
      unit(t, b, cb, rbeg, nch);
      const int64_t c = (int64_t)cb * CBLK + cl;
      for (int j = 0; j < nch; ++j) {
        uint32_t u[64];
        const BwdPre pre = bwd_prefetch(p, b, c, rbeg + (int64_t)j * BR + half * 64);
        mbar_wait(&y_full[yb], yph);
        tc_fence_after();
        ld64(tmem_base + (uint32_t)(yb * 128 + half * 64) + ((uint32_t)(quarter * 32) << 16), u);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&y_empty[yb]);
        if (++yb == 2) { yb = 0; yph ^= 1; }
        mbar_wait(&dy_empty[dyb], dyph ^ 1);
        const uint32_t rowaddr = smem_u32(dyt + dyb * DY_BYTES + half * (CBLK * 128)) + cl * 128;
        bwd_transform(u, pre, p, b, c, rbeg + (int64_t)j * BR + half * 64, rowaddr, sw);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&dy_full[dyb]);
        if (++dyb == 2) { dyb = 0; dyph ^= 1; }
      }
      // dW[cb] block: TMEM lane = channel, columns = k
      mbar_wait(&d_full[db], dph);
      tc_fence_after();
      if (half * 64 < p.K) {
        uint32_t u[64];
        if (nch > 0) ld64(tmem_base + 256 + (uint32_t)(db * 128 + half * 64) + ((uint32_t)(quarter * 32) << 16), u);
        else {
#pragma unroll
          for (int q = 0; q < 64; ++q) u[q] = 0u;
        }
        const int s = (int)((t / p.nblk) % p.splits);
        float* dst;
        bool acc_into = false;
        if (p.splits > 1) {
          dst = p.part + (((int64_t)s * p.B + b) * p.C + c) * p.K + half * 64;
        } else {
          dst = p.dW + (int64_t)b * p.dw_bs + c * p.dw_ld + half * 64;
          acc_into = p.accumulate != 0;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float4 v = make_float4(__uint_as_float(u[4 * q]), __uint_as_float(u[4 * q + 1]), __uint_as_float(u[4 * q + 2]),
                                 __uint_as_float(u[4 * q + 3]));
          if (acc_into) {
            dst[4 * q] += v.x; dst[4 * q + 1] += v.y; dst[4 * q + 2] += v.z; dst[4 * q + 3] += v.w;
          } else if (p.splits > 1) {
            *reinterpret_cast<float4*>(dst + 4 * q) = v;
          } else {
            dst[4 * q] = v.x; dst[4 * q + 1] = v.y; dst[4 * q + 2] = v.z; dst[4 * q + 3] = v.w;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_empty[db]);
      if (++db == 2) { db = 0; dph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free512(tmem_base);
  }
}

// dW = sum_s part[s] in split order (deterministic).
__global__ void k_lbm_wreduce(int B, int S, int64_t C, int64_t K, const float* __restrict__ part, float* __restrict__ dW,
                              int64_t dw_bs, int64_t dw_ld, int accumulate) {
  const int64_t n = (int64_t)B * C * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < S; ++s) a += part[(int64_t)s * n + i];
    const int64_t k = i % K, c = (i / K) % C, b = i / (K * C);
    float* d = dW + b * dw_bs + c * dw_ld + k;
    *d = accumulate ? *d + a : a;
  }
}

// ------------------------------------------------------------ host side --
constexpr size_t FWD_SMEM = 1024 + FG * 2 * WKB + FSTAGES * 2 * FA_KB + 256 + NEPIW * NBW * 4 * 32 * 16;
constexpr size_t DG_SMEM = 1024 + 2 * 2 * BA_KB + DG_WST * 2 * WKB + 2 * DY_BYTES + 256;
constexpr size_t WG_SMEM = 1024 + 2 * WKB + WG_AST * 2 * BA_KB + 2 * DY_BYTES + 256;
static_assert(FWD_SMEM <= 232448 && DG_SMEM <= 232448 && WG_SMEM <= 232448, "shared memory budget");

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

int wgrad_splits(int B, int64_t C, int64_t R) {
  const int64_t nblk = C / CBLK;
  int64_t s = cdiv(4 * 148, (int64_t)B * nblk);
  s = std::max<int64_t>(1, std::min<int64_t>(s, 16));
  s = std::min<int64_t>(s, std::max<int64_t>(1, cdiv(R, BR)));
  return (int)s;
}

size_t fwd_ws(int B, int64_t N, int64_t C, int64_t K) {
  return al256((size_t)B * C * K * 2) + 4 * al256((size_t)B * N * C * 4);
}
size_t bwd_ws(int B, int64_t N, int64_t L, int64_t C, int64_t K) {
  const int S = wgrad_splits(B, C, N * L);
  return al256((size_t)B * C * 8) + al256((size_t)B * N * C * 4) + (S > 1 ? al256((size_t)S * B * C * K * 4) : 0);
}

template <typename K_>
void set_smem(K_ kern, size_t bytes, bool& done) {
  if (!done) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    done = true;
  }
}

hfta_status check_common(int B, int64_t N, int64_t L, int64_t C, int64_t K, hfta_dtype dt, hfta_in X, hfta_in W) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  HFTA_REQUIRE(dt == HFTA_BF16, HFTA_ERR_UNSUPPORTED, "linear_bn_max: bf16 operands only (tensor-core path)");
  HFTA_REQUIRE(N >= 1 && L >= 1 && N * L >= 2, HFTA_ERR_SHAPE, "linear_bn_max: N=%lld L=%lld", (long long)N,
               (long long)L);
  HFTA_REQUIRE(C >= CBLK && C % CBLK == 0, HFTA_ERR_UNSUPPORTED, "linear_bn_max: C=%lld must be a multiple of 128",
               (long long)C);
  HFTA_REQUIRE(K == 64 || K == 128, HFTA_ERR_UNSUPPORTED, "linear_bn_max: K=%lld must be 64 or 128", (long long)K);
  HFTA_REQUIRE(N * L <= INT32_MAX && C * B <= INT32_MAX, HFTA_ERR_SHAPE, "linear_bn_max: sizes exceed int32");
  HFTA_REQUIRE(X.ptr && W.ptr, HFTA_ERR_INVALID_VALUE, "linear_bn_max: X and W are required");
  HFTA_REQUIRE(aligned16(X.ptr) && aligned16(W.ptr) && (X.ld * 2) % 16 == 0 && (X.bstride * 2) % 16 == 0 &&
                   (W.ld * 2) % 16 == 0 && (W.bstride * 2) % 16 == 0 && X.ld >= K && W.ld >= K,
               HFTA_ERR_UNSUPPORTED, "linear_bn_max: X/W must be 16-B aligned with 16-B row strides");
  return HFTA_OK;
}

}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" {

size_t hfta_fused_linear_bn_max_workspace(int B, int64_t N, int64_t L, int64_t C, int64_t K) {
  if (B < 1 || N < 1 || L < 1 || C < 1 || K < 1) return 0;
  return std::max(fwd_ws(B, N, C, K), bwd_ws(B, N, L, C, K));
}

hfta_status hfta_fused_linear_bn_max_fwd(int B, int64_t N, int64_t L, int64_t C, int64_t K, hfta_dtype dt, hfta_in X,
                                         hfta_in W, const float* bias, int64_t bias_bstride, const float* gamma,
                                         const float* beta, int64_t gb_bstride, float* running_mean,
                                         float* running_var, float momentum, float eps, hfta_act act,
                                         float act_alpha, hfta_out G, int32_t* argmax, hfta_out ext,
                                         float* save_mean, float* save_invstd, void* ws, size_t ws_bytes,
                                         hfta_stream stream) {
  if (hfta_status st = check_common(B, N, L, C, K, dt, X, W)) return st;
  HFTA_REQUIRE(gamma && beta && G.ptr && argmax && ext.ptr && save_mean && save_invstd, HFTA_ERR_INVALID_VALUE,
               "linear_bn_max_fwd: gamma, beta, G, argmax, ext, save_mean, save_invstd are required");
  const size_t need = hfta_fused_linear_bn_max_workspace(B, N, L, C, K);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "linear_bn_max_fwd: workspace %zu < %zu", ws_bytes, need);
  if (hfta_status st = get_encode()) return st;
  cudaStream_t s = (cudaStream_t)stream;
  char* w = reinterpret_cast<char*>(ws);
  __nv_bfloat16* wf = reinterpret_cast<__nv_bfloat16*>(w);
  w += al256((size_t)B * C * K * 2);
  const size_t pb = al256((size_t)B * N * C * 4);
  float* s1 = reinterpret_cast<float*>(w);
  float* s2 = reinterpret_cast<float*>(w + pb);
  float* mx = reinterpret_cast<float*>(w + 2 * pb);
  int32_t* idx = reinterpret_cast<int32_t*>(w + 3 * pb);

  const int64_t nw = (int64_t)B * C * K;
  k_lbm_flip<<<(unsigned)std::min<int64_t>(cdiv(nw, 256), 148 * 16), 256, 0, s>>>(
      B, C, K, (const __nv_bfloat16*)W.ptr, W.bstride, W.ld, gamma, gb_bstride, wf);

  CUtensorMap ta, tw;
  const int nba = (X.bstride == 0 && B > 1) ? 1 : B;
  if (hfta_status st = make_map(&ta, X.ptr, K, N * L, X.ld, X.bstride, nba, 64, FR)) return st;
  if (hfta_status st = make_map(&tw, wf, K, C, K, C * K, B, 64, CBLK)) return st;
  FwdArgs a{};
  a.B = B; a.Ncl = (int)N; a.nblk = (int)(C / CBLK); a.ngroups = (int)cdiv(a.nblk, FG); a.nkb = (int)(K / 64);
  a.a_shared = nba == 1 && B > 1;
  a.L = L; a.C = C;
  a.s1 = s1; a.s2 = s2; a.mx = mx; a.idx = idx;
  {
    const char* e = getenv("HFTA_LBM_MODE");   // diagnostics: 1 = epilogue only drains TMEM
    a.mode = e ? atoi(e) : 0;
  }
  const int64_t npairs = (int64_t)B * N;
  a.teams = (int)std::max<int64_t>(1, std::min<int64_t>(npairs, num_sms() / a.ngroups));
  static bool attr = false;
  set_smem(k_lbm_fwd, FWD_SMEM, attr);
  k_lbm_fwd<<<a.teams * a.ngroups, LT, FWD_SMEM, s>>>(ta, tw, a);
  k_lbm_fwd_fin<<<(unsigned)cdiv((int64_t)B * C, 128), 128, 0, s>>>(
      B, (int)N, L, C, s1, s2, mx, idx, bias, bias_bstride, gamma, beta, gb_bstride, running_mean, running_var,
      momentum, eps, (int)act, act_alpha, (float*)G.ptr, G.bstride, G.ld, argmax, N * C, C, (float*)ext.ptr,
      ext.bstride, ext.ld, save_mean, save_invstd);
  count_launches(3);
  return post_launch(s, "hfta_fused_linear_bn_max_fwd");
}

hfta_status hfta_fused_linear_bn_max_bwd(int B, int64_t N, int64_t L, int64_t C, int64_t K, hfta_dtype dt,
                                         hfta_in dG, hfta_in X, hfta_in W, const int32_t* argmax, hfta_in ext,
                                         const float* bias, int64_t bias_bstride, const float* gamma,
                                         const float* beta, int64_t gb_bstride, const float* save_mean,
                                         const float* save_invstd, hfta_act act, float act_alpha, hfta_out dX,
                                         float* dW, int64_t dW_bstride, int64_t dW_ld, float* dbias,
                                         int64_t dbias_bstride, float* dgamma, float* dbeta, int accumulate,
                                         void* ws, size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_common(B, N, L, C, K, dt, X, W)) return st;
  HFTA_REQUIRE(dG.ptr && argmax && ext.ptr && gamma && beta && save_mean && save_invstd && dW && dgamma && dbeta,
               HFTA_ERR_INVALID_VALUE,
               "linear_bn_max_bwd: dG, argmax, ext, gamma, beta, save_*, dW, dgamma, dbeta are required");
  HFTA_REQUIRE(!dX.ptr || (aligned16(dX.ptr) && (dX.ld * 2) % 16 == 0 && (dX.bstride * 2) % 16 == 0 && dX.ld >= K),
               HFTA_ERR_UNSUPPORTED, "linear_bn_max_bwd: dX must be 16-B aligned with 16-B row strides");
  HFTA_REQUIRE(dW_ld >= K, HFTA_ERR_SHAPE, "linear_bn_max_bwd: dW_ld < K");
  const size_t need = hfta_fused_linear_bn_max_workspace(B, N, L, C, K);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "linear_bn_max_bwd: workspace %zu < %zu", ws_bytes, need);
  if (hfta_status st = get_encode()) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t R = N * L;
  const int S = wgrad_splits(B, C, R);
  char* w = reinterpret_cast<char*>(ws);
  float2* coef = reinterpret_cast<float2*>(w);
  w += al256((size_t)B * C * 8);
  float* pv = reinterpret_cast<float*>(w);
  w += al256((size_t)B * N * C * 4);
  float* part = reinterpret_cast<float*>(w);

  k_lbm_bwd_coef<<<(unsigned)cdiv((int64_t)B * C, 128), 128, 0, s>>>(
      B, (int)N, L, C, (const float*)dG.ptr, dG.bstride, dG.ld, (const float*)ext.ptr, ext.bstride, ext.ld, bias,
      bias_bstride, gamma, beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha, coef, pv, dgamma, dbeta,
      dbias, dbias_bstride, accumulate);

  CUtensorMap ta, tw;
  const int nba = (X.bstride == 0 && B > 1) ? 1 : B;
  if (hfta_status st = make_map(&ta, X.ptr, K, R, X.ld, X.bstride, nba, 64, BR)) return st;
  if (hfta_status st = make_map(&tw, W.ptr, K, C, W.ld, W.bstride, B, 64, CBLK)) return st;
  BwdArgs a{};
  a.B = B; a.Ncl = (int)N; a.nblk = (int)(C / CBLK); a.nkb = (int)(K / 64); a.a_shared = nba == 1 && B > 1;
  a.L = L; a.C = C; a.R = R; a.K = K; a.tiles = cdiv(R, BR);
  a.coef = coef; a.pv = pv; a.am = argmax; a.am_bs = N * C; a.am_ld = C;
  a.dX = (__nv_bfloat16*)dX.ptr; a.dx_bs = dX.bstride; a.dx_ld = dX.ld;
  a.dW = dW; a.dw_bs = dW_bstride; a.dw_ld = dW_ld; a.accumulate = accumulate;
  a.splits = S; a.rps = cdiv(cdiv(R, S), BR) * BR; a.part = part;
  int launches = 1;
  if (dX.ptr) {
    static bool attr = false;
    set_smem(k_lbm_dgrad, DG_SMEM, attr);
    const int grid = (int)std::min<int64_t>((int64_t)B * a.tiles, num_sms());
    k_lbm_dgrad<<<grid, LT, DG_SMEM, s>>>(ta, tw, a);
    ++launches;
  }
  {
    static bool attr = false;
    set_smem(k_lbm_wgrad, WG_SMEM, attr);
    const int grid = (int)std::min<int64_t>((int64_t)B * S * a.nblk, num_sms());
    k_lbm_wgrad<<<grid, LT, WG_SMEM, s>>>(ta, tw, a);
    ++launches;
  }
  if (S > 1) {
    k_lbm_wreduce<<<(unsigned)std::min<int64_t>(cdiv((int64_t)B * C * K, 256), 148 * 16), 256, 0, s>>>(
        B, S, C, K, part, dW, dW_bstride, dW_ld, accumulate);
    ++launches;
  }
  count_launches(launches);
  return post_launch(s, "hfta_fused_linear_bn_max_bwd");
}

}  // extern "C"
