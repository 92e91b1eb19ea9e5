// lbm.cu -- the fused PointNet point-feature block on tensor cores (K10):
//
//   Y = X W^T (+ bias)         Conv1d(k=1) K -> C over the R = N*L points   (App. B)
//   Z = act(BN_train(Y))       BatchNorm1d over all R points                (App. B)
//   G[n][c] = max_l Z[n*L+l][c]   max over the L points of cloud n          (App. B)
//
// for all B models in one persistent launch per pass, WITHOUT materialising
// the [B][R][C] pre-BN activation Y in HBM:
//
//  forward   Gram G = X^T X and s = X^T 1 of the layer input (the tcgen05
//            wgrad kernel with fused column sums, X read once), k_lbm_flip
//            (W' = sign(gamma) W, exact), k_lbm_fwd: Y'^T chunks (channels on
//            the TMEM lanes, 128 points on the columns) produced by tcgen05
//            into TMEM and reduced by the epilogue warps straight out of TMEM
//            -- only the per-(model, cloud, channel) maximum of Y' and its
//            first index (max over l of act(gamma*xhat+beta) sits at max_l Y
//            when gamma >= 0 and at min_l Y when gamma < 0).  The batch
//            statistics come from the Gram (reading R27): k_lbm_center forms
//            Gc = G - s s^T / R in fp64, k_lbm_stats evaluates
//            var_c = W_c Gc W_c^T / R and mean_c = W_c s / R + b_c, and
//            k_lbm_fwd_fin writes mean/invstd/running statistics, the pooled
//            output, the argmax and ext = Y at the argmax.
//  backward  dZ is nonzero only at the argmax rows, so the BN backward is
//            dY = bx Y + cc + S (per-channel affine in Y plus one entry per
//            cloud and channel).  Substituting Y = X W^T gives, exactly,
//            dX = X M + 1 v^T + S W  and  dW = diag(bx) W G + cc s^T + S^T X
//            with M = W^T diag(bx) W, v = W^T cc (k_lbm_mv, k_lbm_mv_sum):
//            one R x K x K tcgen05 GEMM (gated by relu' of the layer input in
//            its epilogue), a deterministic sorted scatter of the sparse rows
//            (k_lbm_sparse_dx) and a per-channel dW kernel with G in shared
//            memory (k_lbm_dw).  Neither Y nor dY is ever formed.
//
// k_lbm_fwd roles per CTA (352 threads, 1 CTA/SM, persistent): warp 0 TMA
// producer, warps 1 and 10 two token-passing tcgen05 issuers, warps 2..9
// epilogue (two per TMEM lane quarter).
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "gemm.cuh"
#include "tc_common.cuh"

namespace hfta {
namespace {

constexpr int FWD_LT = 352;         // forward: producer, MMA issuers (warps 1, 10), 8 epilogue warps
constexpr int MMA2_WARP = 10;
constexpr int NEPIW = 8;
constexpr int CBLK = 128;                      // channels per UMMA M block
constexpr uint32_t WKB = CBLK * 64 * 2;        // one 64-wide k block of a 128-channel W block: 16 KB
// forward
constexpr int FR = 128;                        // points per chunk (UMMA N): smem operand reads 8 KB / 64 MMA cycles
constexpr int FG = 2;                          // channel blocks per unit: TMEM 2 x FG x FR = 512 columns
constexpr int FSTAGES = 4;
constexpr int NBW = FG / 2;                    // channel blocks per epilogue warp
constexpr int LPB = FR / 32;                   // 32-column TMEM loads per block and chunk
static_assert(NBW == 1 && LPB == 4, "epilogue: one 128-channel block and four 32-column loads per warp and chunk");
constexpr uint32_t FA_KB = FR * 64 * 2;        // 8 KB per k block of an X chunk

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}
__device__ __forceinline__ void tmem_alloc512(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_free512(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}


#ifdef HFTA_LBM_PROF
// developer build only: per-CTA cycle counters of the forward's waits
}  // namespace
__device__ unsigned long long g_lbm_prof[512][8];
namespace {
#define PROF_WAIT(slot, call)                  \
  do {                                         \
    const long long t0_ = clock64();           \
    call;                                      \
    prof[slot] += clock64() - t0_;             \
  } while (0)
#else
#define PROF_WAIT(slot, call) call
#endif

// ================================================================ forward ==

struct FwdArgs {
  int B, Ncl, nblk, ngroups, teams, nkb, a_shared;
  int64_t L, C;
  float* mx; int32_t* idx;   // per-cloud max of Y' and its first row [B][Ncl][C]
};

// The epilogue reduces only the max: BN statistics come from the Gram of X
// (k_lbm_stats), so per accumulator element the epilogue issues ~0.4
// instructions (FMNMX3 tree) instead of ~2 (sums and squares as well).
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float uf(uint32_t x) { return __uint_as_float(x); }

// Per-channel running state of the forward epilogue: running max m and the
// 16-point group it came from; the group's values sit in this lane's smem
// slot so the exact first index is resolved once per cloud.
struct FwdAcc {
  float m;
  int gid;
};

// One 16-point group (values u[0..15]) of one channel; FULL = all valid.
// Predicated update (no vote / branch): improvements are rare after the
// first groups of a cloud.
template <bool FULL>
__device__ __forceinline__ void fwd_group(const uint32_t* u, int valid, int gid, FwdAcc& A, uint32_t slot) {
  uint32_t v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = (FULL || j < valid) ? u[j] : __float_as_uint(-INFINITY);
  const float a0 = max3(uf(v[0]), uf(v[1]), uf(v[2])), a1 = max3(uf(v[3]), uf(v[4]), uf(v[5]));
  const float a2 = max3(uf(v[6]), uf(v[7]), uf(v[8])), a3 = max3(uf(v[9]), uf(v[10]), uf(v[11]));
  const float a4 = max3(uf(v[12]), uf(v[13]), uf(v[14]));
  const float gm = fmaxf(max3(a0, a1, a2), max3(a3, a4, uf(v[15])));
  const bool p = gm > A.m;
  A.m = p ? gm : A.m;
  A.gid = p ? gid : A.gid;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (p) st_shared_v4(slot + q * 512, make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
}

__global__ void __launch_bounds__(FWD_LT, 1)
k_lbm_fwd(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, FwdArgs p) {
  constexpr int NST = FSTAGES;                                 // X chunk stages
  constexpr uint32_t SKB = FA_KB;                              // bytes per k block of a chunk
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* wres = smem;                                        // FG blocks x 2 k blocks x 16 KB
  uint8_t* ast = wres + FG * 2 * WKB;                          // NST x 2 k blocks x SKB
  uint64_t* full = reinterpret_cast<uint64_t*>(ast + NST * 2 * SKB);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint64_t* wfull = tempty + 2;
  uint64_t* wempty = wfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + 1);
  uint8_t* slot_base = reinterpret_cast<uint8_t*>(full) + 256;        // NEPIW x NBW ch x 4 x 32 lanes x 16 B

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
#ifdef HFTA_LBM_PROF
  long long prof[4] = {0, 0, 0, 0};
  const long long tstart = clock64();
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], NEPIW); }
    mbar_init(wfull, 1);
    mbar_init(wempty, 2);                                      // one commit per issuing warp
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
  const int blk0 = g * FG;                                     // this CTA's channel blocks blk0 + j, j < nb
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
          PROF_WAIT(0, mbar_wait(&empty[stage], ph ^ 1));
          mbar_expect_tx(&full[stage], (uint32_t)p.nkb * SKB);
          for (int kb = 0; kb < p.nkb; ++kb)
            tma_load_3d(ast + (stage * 2 + kb) * SKB, &tmA, &full[stage], kb * 64, (int)(n * p.L + ch * FR), ba);
          if (++stage == NST) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1 || warp == MMA2_WARP) {
    // Two issuing warps alternate chunks (warp 1: even, MMA2_WARP: odd) and
    // pass a token (named barriers 1/2) after each chunk's MMAs are issued:
    // the tcgen05 queue is shallow, so a single issuer's per-chunk barrier
    // waits (~100+ cycles) would idle the tensor pipe; here one warp waits
    // while the other issues.  Accumulator buffer = chunk parity.
    constexpr uint32_t IDESC = idesc_bf16(CBLK, FR, false, false);
    const int mw = warp == 1 ? 0 : 1;
    const int64_t gtot = (u1 - u0) * nch;
    int curb = -1;
    uint32_t wep = 0;
    int64_t gc = 0;
    for (int64_t u = u0; u < u1; ++u) {
      const int b = (int)(u / p.Ncl);
      if (b != curb) {
        if (curb >= 0) tc_commit_w(wempty);   // both issuers' MMAs on the old W (wempty counts 2 commits)
        __syncwarp();
        mbar_wait(wfull, wep & 1);
        curb = b;
        ++wep;
      }
      for (int ch = 0; ch < nch; ++ch, ++gc) {
        if ((int)(gc & 1) != mw) continue;
        const int acc = (int)(gc & 1);
        const int stage = (int)(gc % NST);
        PROF_WAIT(0, mbar_wait(&tempty[acc], (uint32_t)((gc >> 1) & 1) ^ 1u));
        PROF_WAIT(1, mbar_wait(&full[stage], (uint32_t)((gc / NST) & 1)));
        tc_fence_after();
        if (gc > 0) asm volatile("bar.sync %0, 64;" ::"r"(1 + (int)(gc & 1)) : "memory");   // token from chunk gc-1
        const uint64_t bd0 = smem_desc(smem_u32(ast + stage * 2 * SKB), 16, 1024);
        for (int j = 0; j < nb; ++j) {
          const uint32_t d = tmem_base + (uint32_t)(acc * FG * FR + j * FR);
          const uint64_t ad0 = smem_desc(smem_u32(wres + j * 2 * WKB), 16, 1024);
          for (int kb = 0; kb < p.nkb; ++kb) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {   // +32 B per k step, +WKB / SKB per k block (descriptor units of 16 B)
              const uint64_t ad = ad0 + (uint64_t)(kb * (WKB >> 4) + 2 * k);
              const uint64_t bd = bd0 + (uint64_t)(kb * (SKB >> 4) + 2 * k);
              tc_mma_ss(d, ad, bd, IDESC, (kb | k) != 0 ? 1u : 0u);
            }
          }
        }
        tc_commit_w(&empty[stage]);
        tc_commit_w(&tfull[acc]);
        if (gc + 1 < gtot) asm volatile("bar.arrive %0, 64;" ::"r"(1 + (int)((gc + 1) & 1)) : "memory");   // token
        __syncwarp();
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
        A[jj].m = -INFINITY;
        A[jj].gid = 0;
      }
      // this warp owns blocks half + 2 jj (when present): nld 32-column loads per chunk
      int nld = 0;
#pragma unroll
      for (int jj = 0; jj < NBW; ++jj) nld += half + 2 * jj < nb ? LPB : 0;
      for (int ch = 0; ch < nch; ++ch) {
        const int valid = (int)min((int64_t)FR, p.L - (int64_t)ch * FR);
        PROF_WAIT(0, mbar_wait(&tfull[acc], aph));
        tc_fence_after();
        // TMEM reads are the epilogue's bound (128 KB per chunk over 8 warps):
        // the first two 32-column loads land, the last two are issued and
        // the first half is reduced while they are in flight; the
        // accumulator is released once all four have landed
        const uint32_t ta = tmem_base + (uint32_t)(acc * FG * FR + half * FR) + ((uint32_t)(quarter * 32) << 16);
        uint32_t r0[32], r1[32], r2[32], r3[32];
        const bool work = nld != 0;
        if (work) {
          tmem_ld32_nowait(ta, r0);
          tmem_ld32_nowait(ta + 32, r1);
          tmem_wait_ld();
          tmem_ld32_nowait(ta + 64, r2);
          tmem_ld32_nowait(ta + 96, r3);
        }
        const int g0 = ch * (FR / 16);
        if (work) {
          if (valid == FR) {
            fwd_group<true>(r0, 16, g0, A[0], slots);
            fwd_group<true>(r0 + 16, 16, g0 + 1, A[0], slots);
            fwd_group<true>(r1, 16, g0 + 2, A[0], slots);
            fwd_group<true>(r1 + 16, 16, g0 + 3, A[0], slots);
          } else {
            fwd_group<false>(r0, valid, g0, A[0], slots);
            fwd_group<false>(r0 + 16, valid - 16, g0 + 1, A[0], slots);
            fwd_group<false>(r1, valid - 32, g0 + 2, A[0], slots);
            fwd_group<false>(r1 + 16, valid - 48, g0 + 3, A[0], slots);
          }
          tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (work) {
          if (valid == FR) {
            fwd_group<true>(r2, 16, g0 + 4, A[0], slots);
            fwd_group<true>(r2 + 16, 16, g0 + 5, A[0], slots);
            fwd_group<true>(r3, 16, g0 + 6, A[0], slots);
            fwd_group<true>(r3 + 16, 16, g0 + 7, A[0], slots);
          } else {
            fwd_group<false>(r2, valid - 64, g0 + 4, A[0], slots);
            fwd_group<false>(r2 + 16, valid - 80, g0 + 5, A[0], slots);
            fwd_group<false>(r3, valid - 96, g0 + 6, A[0], slots);
            fwd_group<false>(r3 + 16, valid - 112, g0 + 7, A[0], slots);
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
        p.mx[o] = A[jj].m;
        p.idx[o] = A[jj].gid * 16 + first;
      }
    }
  }
#ifdef HFTA_LBM_PROF
  if (lane == 0 && warp <= 2) {
    const int base = warp == 0 ? 0 : warp == 1 ? 2 : 4;
    g_lbm_prof[blockIdx.x][base] = prof[0];
    if (warp == 1) g_lbm_prof[blockIdx.x][base + 1] = prof[1];
    if (warp == 2) g_lbm_prof[blockIdx.x][base + 1] = prof[2];
    if (warp == 2) g_lbm_prof[blockIdx.x][7] = clock64() - tstart;
  }
#endif
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
  // 8 bf16 (16 B) per thread; rows are 16-B aligned (check_common); sign flip = XOR of the sign bits
  const int kv = (int)(K / 8);
  const int64_t n = (int64_t)B * C * kv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / kv;
    const int k8 = (int)(i - row * kv);
    const int64_t b = row / C, c = row - b * C;
    uint4 w = *reinterpret_cast<const uint4*>(W + b * wbs + c * wld + k8 * 8);
    if (gamma[b * gbs + c] < 0.f) { w.x ^= 0x80008000u; w.y ^= 0x80008000u; w.z ^= 0x80008000u; w.w ^= 0x80008000u; }
    *reinterpret_cast<uint4*>(Wf + row * K + k8 * 8) = w;
  }
}

// BN batch statistics of Y = X W^T from the Gram of the layer input (exact
// algebra, reading R27): with mu = s/R and the centred Gram
//   Gc = G - R mu mu^T   (fp64 -> fp32: centring first avoids the
//                         E[y^2] - E[y]^2 cancellation),
//   mean_c = W_c . mu (+ bias_c),   var_c = W_c Gc W_c^T / R   (biased).
// One CTA per (model, 64 channels), Gc [K][K] and W^T [K][64] in smem;
// thread (channel group cg of 4, k group kg of 16) accumulates
// t[c][k] = sum_j Gc[j][k] W_c[j] for 4 channels x K/16 k (register blocked:
// 2-3 LDS.128 per 32 FMA), then the dot with W_c in fp64 reduced over the 16
// k groups of a half-warp.  Writes save_mean / save_invstd and the running
// statistics.  K in {64, 128}.
constexpr int ST_CH = 64;                // channels per CTA

// Gc = G - R mu mu^T in fp64 -> fp32 and mu = s / R (fp64), once per model
// (the statistics CTAs of a model then just copy Gc into shared memory).
__global__ void __launch_bounds__(256) k_lbm_center(int K, int64_t R, const float* __restrict__ G,
                                                    const float* __restrict__ xs, float* __restrict__ Gc,
                                                    double* __restrict__ mu) {
  const int b = blockIdx.y;
  const double Rd = (double)R;
  const float* xb = xs + (int64_t)b * K;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < K) mu[(int64_t)b * K + i] = (double)xb[i] / Rd;
  if (i >= (int64_t)K * K) return;
  const int j = (int)(i / K), k = (int)(i % K);
  const double mj = (double)xb[j] / Rd, mk = (double)xb[k] / Rd;
  Gc[(int64_t)b * K * K + i] = (float)((double)G[(int64_t)b * K * K + i] - Rd * mj * mk);
}

template <int K>
__global__ void __launch_bounds__(256) k_lbm_stats(int B, int64_t R, int64_t C, const float* __restrict__ Gcg,
                                                   const double* __restrict__ mug, const __nv_bfloat16* __restrict__ W,
                                                   int64_t wbs, int64_t wld, const float* __restrict__ bias,
                                                   int64_t bias_bs, float* __restrict__ rmean,
                                                   float* __restrict__ rvar, float momentum, float eps,
                                                   float* __restrict__ smean, float* __restrict__ sinv) {
  extern __shared__ __align__(16) float st_smem[];
  float* Gc = st_smem;                             // [K][K]
  float* Wt = st_smem + K * K;                     // [K][ST_CH]
  __shared__ double mu[128];
  const int b = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * ST_CH;
  const double Rd = (double)R;
  for (int k = threadIdx.x; k < K; k += blockDim.x) mu[k] = mug[(int64_t)b * K + k];
  {   // Gc (fp32, centred once per model by k_lbm_center): 16-B loads, 4 in flight per thread
    const float4* G4 = reinterpret_cast<const float4*>(Gcg + (int64_t)b * K * K);
    float4* S4 = reinterpret_cast<float4*>(Gc);
    constexpr int n4 = K * K / 4;
    for (int i0 = threadIdx.x; i0 < n4; i0 += 4 * 256) {
      float4 g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * 256 < n4) g[u] = __ldg(G4 + i0 + u * 256);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * 256 < n4) S4[i0 + u * 256] = g[u];
    }
  }
  const __nv_bfloat16* Wb = W + (int64_t)b * wbs;
  constexpr int kv = K / 8;                        // 16-B vectors per W row (rows 16-B aligned)
  for (int i0 = threadIdx.x; i0 < ST_CH * kv; i0 += 2 * blockDim.x) {
    uint4 wv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * blockDim.x;
      const int cl = i % ST_CH, k8 = i / ST_CH;    // lanes over channels: conflict-free transposed stores
      const int64_t c = c0 + cl;
      wv[u] = (i < ST_CH * kv && c < C) ? __ldg(reinterpret_cast<const uint4*>(Wb + c * wld) + k8)
                                        : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i >= ST_CH * kv) continue;
      const int cl = i % ST_CH, k8 = i / ST_CH;
      const uint32_t e[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Wt[(k8 * 8 + 2 * q) * ST_CH + cl] = __uint_as_float(e[q] << 16);
        Wt[(k8 * 8 + 2 * q + 1) * ST_CH + cl] = __uint_as_float(e[q] & 0xffff0000u);
      }
    }
  }
  __syncthreads();
  const int kg = threadIdx.x & 15, cg = threadIdx.x >> 4;     // 16 channel groups x 16 k groups
  constexpr int nh = K / 64;                                  // k = kg*4 + 64*h + i, h < nh, i < 4
  float t[4][8];
#pragma unroll
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int i = 0; i < 8; ++i) t[c][i] = 0.f;
  for (int j = 0; j < K; ++j) {
    const float4 w4 = *reinterpret_cast<const float4*>(Wt + j * ST_CH + cg * 4);
    const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h < nh) {
        const float4 g4 = *reinterpret_cast<const float4*>(Gc + j * K + kg * 4 + 64 * h);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          t[c][4 * h + 0] = fmaf(g4.x, wv[c], t[c][4 * h + 0]);
          t[c][4 * h + 1] = fmaf(g4.y, wv[c], t[c][4 * h + 1]);
          t[c][4 * h + 2] = fmaf(g4.z, wv[c], t[c][4 * h + 2]);
          t[c][4 * h + 3] = fmaf(g4.w, wv[c], t[c][4 * h + 3]);
        }
      }
    }
  }
  double q[4], m1[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    q[c] = 0.0;
    m1[c] = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h < nh) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = kg * 4 + 64 * h + i;
          const double wk = (double)Wt[k * ST_CH + cg * 4 + c];
          q[c] += wk * (double)t[c][4 * h + i];
          m1[c] += wk * mu[k];
        }
      }
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      q[c] += __shfl_xor_sync(0xffffffffu, q[c], o);
      m1[c] += __shfl_xor_sync(0xffffffffu, m1[c], o);
    }
  }
  if (kg >= 4) return;
  const int c_ = kg;                               // lanes kg = 0..3 write channel cg*4 + kg
  double qq = q[0], mm = m1[0];
#pragma unroll
  for (int c = 1; c < 4; ++c)
    if (c_ == c) { qq = q[c]; mm = m1[c]; }
  const int64_t c = c0 + cg * 4 + c_;
  if (c >= C) return;
  double var = qq / Rd;
  if (var < 0.0) var = 0.0;
  const double bi = bias ? (double)bias[(int64_t)b * bias_bs + c] : 0.0;
  const double mean = mm + bi;                     // the layer output includes its bias
  const int64_t i = (int64_t)b * C + c;
  smean[i] = (float)mean;
  sinv[i] = (float)(1.0 / sqrt(var + (double)eps));
  if (rmean) rmean[i] = (float)((1.0 - momentum) * (double)rmean[i] + momentum * mean);
  if (rvar) rvar[i] = (float)((1.0 - momentum) * (double)rvar[i] + momentum * var * Rd / (Rd - 1.0));
}
size_t stats_smem(int K) { return ((size_t)K * K + (size_t)K * ST_CH) * 4; }

// Per (model, channel, cloud): the pooled output from the per-cloud max of
// Y' = s_c Y (sign-flipped), the statistics and the affine BN.
__global__ void k_lbm_fwd_fin(int B, int Ncl, int64_t C, const float* __restrict__ mx, const int32_t* __restrict__ idx,
                              const float* __restrict__ bias, int64_t bias_bs, const float* __restrict__ gamma,
                              const float* __restrict__ beta, int64_t gbs, const float* __restrict__ smean,
                              const float* __restrict__ sinv, int act, float alpha, float* __restrict__ G,
                              int64_t g_bs, int64_t g_ld, int32_t* __restrict__ amax, int64_t am_bs, int64_t am_ld,
                              float* __restrict__ ext, int64_t ext_bs, int64_t ext_ld) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * Ncl * C) return;
  const int64_t c = i % C, n = (i / C) % Ncl, b = i / (C * Ncl);
  const float ga = gamma[b * gbs + c], be = beta[b * gbs + c];
  const float bi = bias ? bias[b * bias_bs + c] : 0.f;
  const float inv = sinv[b * C + c];
  const float mean_y = smean[b * C + c] - bi;      // statistics of Y (bias excluded)
  const float ey = ga < 0.f ? -mx[i] : mx[i];      // Y at the argmax row (bias excluded)
  const float z = ga * inv * (ey - mean_y) + be;
  G[b * g_bs + n * g_ld + c] = act_fwd(z, act, alpha);
  amax[b * am_bs + n * am_ld + c] = idx[i];
  ext[b * ext_bs + n * ext_ld + c] = ey + bi;
}

// =============================================================== backward ==
//
// With dZ nonzero only at the argmax rows, the BN backward is
//   dY[r][c] = bx_c Y[r][c] + cc_c + S[r][c],   S = a_c dz at r = argmax(n, c),
// an affine map of Y = X W^T plus a sparse matrix, so both contractions
// collapse onto K x K quantities of the layer input (K = 128 << C = 1024):
//   dX = dY W   = X M + 1 v^T + S W,       M = W^T diag(bx) W,  v = W^T cc
//   dW = dY^T X = diag(bx) W G + cc s^T + S^T X,   G = X^T X,  s = X^T 1
// (exact algebra; only the rounding order differs from forming dY).  The
// dense parts are one Gram contraction over the R points (tensor cores,
// hfta_fused_linear_bwd's wgrad path) and one R x K x K GEMM (dX = X M^T + v,
// M symmetric); the sparse parts touch one row per (cloud, channel).  No
// [R][C] tensor is formed, no Y is recomputed: the backward reads X once for
// G/s, once for dX, and writes dX -- HBM-bound.

// Per (model, channel): dz at the pooled rows, dgamma/dbeta, the affine
// coefficients (bx, cc) of dY and the sparse values sp = a*dz.
__global__ void k_lbm_bwd_coef(int B, int Ncl, int64_t L, int64_t C, const float* __restrict__ dG, int64_t dg_bs,
                               int64_t dg_ld, const float* __restrict__ ext, int64_t ext_bs, int64_t ext_ld,
                               const float* __restrict__ bias, int64_t bias_bs, const float* __restrict__ gamma,
                               const float* __restrict__ beta, int64_t gbs, const float* __restrict__ smean,
                               const float* __restrict__ sinv, int act, float alpha, float2* __restrict__ coef,
                               float* __restrict__ sp, float* __restrict__ dgamma, float* __restrict__ dbeta,
                               float* __restrict__ dbias, int64_t dbias_bs, int accumulate) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * C) return;
  const int64_t b = i / C, c = i % C;
  const float ga = gamma[b * gbs + c], be = beta[b * gbs + c];
  const float mb = smean[i], inv = sinv[i];
  const float bi = bias ? bias[b * bias_bs + c] : 0.f;
  const double a = (double)ga * inv;
  double dbe = 0.0, dga = 0.0;
  for (int n = 0; n < Ncl; ++n) {
    const float xh = (ext[b * ext_bs + n * ext_ld + c] - mb) * inv;
    const float dz = dG[b * dg_bs + n * dg_ld + c] * act_grad(ga * xh + be, act, alpha);
    dbe += dz;
    dga += (double)dz * xh;
    sp[(b * Ncl + n) * C + c] = (float)(a * dz);
  }
  const double R = (double)Ncl * (double)L;
  const double bx = -a * inv * dga / R;
  const double cc = -a * dbe / R - bx * ((double)mb - (double)bi);   // affine in Y without its bias
  coef[i] = make_float2((float)bx, (float)cc);
  const int64_t go = b * gbs + c;
  if (accumulate) { dgamma[go] += (float)dga; dbeta[go] += (float)dbe; }
  else { dgamma[go] = (float)dga; dbeta[go] = (float)dbe; }
  if (dbias && !accumulate) dbias[b * dbias_bs + c] = 0.f;   // BN-absorbed bias: exact zero
}

// M[b] = W^T diag(bx) W (bf16, the dX GEMM's weight; symmetric), v[b] = W^T cc.
// Grid (K/64, B): a CTA owns 64 rows of M; thread = 4 rows x 8 columns
// register tile; W streamed through smem 32 channels at a time (fp32).
constexpr int MV_ROWS = 64;
template <int K>
__global__ void __launch_bounds__(256) k_lbm_mv(int64_t C, const __nv_bfloat16* __restrict__ W, int64_t w_bs,
                                                int64_t w_ld, const float2* __restrict__ coef,
                                                float* __restrict__ Mpart, float* __restrict__ vpart) {
  // M[r][c] = sum_ch bx_ch W[ch][r] W[ch][c] over this CTA's channel range:
  // 16 x 16 threads, each an (NH*4) x (NH*4) register tile at rows
  // {4 tr + 64 h + i}, columns {4 tc + 64 h + j} (conflict-free LDS.128:
  // 64 FFMA per 4 shared loads at K = 128)
  constexpr int NH = K / 64;
  __shared__ __align__(16) float swa[32][K];   // bx_c * W[c][k]
  __shared__ __align__(16) float swb[32][K];   // W[c][k]
  __shared__ float scc[32];
  const int b = blockIdx.y;
  const int64_t cs = C * blockIdx.z / gridDim.z, ce = C * (blockIdx.z + 1) / gridDim.z;
  const int t = threadIdx.x, tr = t / 16, tc = t % 16;
  float acc[NH * 4][NH * 4];
#pragma unroll
  for (int i = 0; i < NH * 4; ++i)
#pragma unroll
    for (int j = 0; j < NH * 4; ++j) acc[i][j] = 0.f;
  float vacc[NH * 4];
#pragma unroll
  for (int j = 0; j < NH * 4; ++j) vacc[j] = 0.f;
  const __nv_bfloat16* Wb = W + (int64_t)b * w_bs;
  for (int64_t c0 = cs; c0 < ce; c0 += 32) {
    __syncthreads();
    for (int e = t; e < 32 * (K / 8); e += 256) {          // 8 bf16 per load, two STS.128 per array
      const int q = e / (K / 8), k8 = (e % (K / 8)) * 8;
      float x[8];
      ld_vec<__nv_bfloat16, 8>(Wb + (c0 + q) * w_ld + k8, x);
      const float bx = coef[(int64_t)b * C + c0 + q].x;
      *reinterpret_cast<float4*>(&swb[q][k8]) = make_float4(x[0], x[1], x[2], x[3]);
      *reinterpret_cast<float4*>(&swb[q][k8 + 4]) = make_float4(x[4], x[5], x[6], x[7]);
      *reinterpret_cast<float4*>(&swa[q][k8]) = make_float4(x[0] * bx, x[1] * bx, x[2] * bx, x[3] * bx);
      *reinterpret_cast<float4*>(&swa[q][k8 + 4]) = make_float4(x[4] * bx, x[5] * bx, x[6] * bx, x[7] * bx);
    }
    if (t < 32) scc[t] = coef[(int64_t)b * C + c0 + t].y;
    __syncthreads();
#pragma unroll 2
    for (int q = 0; q < 32; ++q) {
      float av[NH * 4], bv[NH * 4];
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const float4 a4 = *reinterpret_cast<const float4*>(&swa[q][tr * 4 + 64 * h]);
        const float4 b4 = *reinterpret_cast<const float4*>(&swb[q][tc * 4 + 64 * h]);
        av[4 * h] = a4.x; av[4 * h + 1] = a4.y; av[4 * h + 2] = a4.z; av[4 * h + 3] = a4.w;
        bv[4 * h] = b4.x; bv[4 * h + 1] = b4.y; bv[4 * h + 2] = b4.z; bv[4 * h + 3] = b4.w;
      }
#pragma unroll
      for (int i = 0; i < NH * 4; ++i)
#pragma unroll
        for (int j = 0; j < NH * 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      if (tr == 0) {                                        // v = W^T cc on the first row group
        const float cq = scc[q];
#pragma unroll
        for (int j = 0; j < NH * 4; ++j) vacc[j] = fmaf(bv[j], cq, vacc[j]);
      }
    }
  }
  float* Mp = Mpart + ((int64_t)blockIdx.z * gridDim.y + b) * K * K;
#pragma unroll
  for (int hi = 0; hi < NH; ++hi)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int hj = 0; hj < NH; ++hj) {
        const int r = tr * 4 + 64 * hi + i, c = tc * 4 + 64 * hj;
        *reinterpret_cast<float4*>(Mp + (int64_t)r * K + c) =
            make_float4(acc[4 * hi + i][4 * hj], acc[4 * hi + i][4 * hj + 1], acc[4 * hi + i][4 * hj + 2],
                        acc[4 * hi + i][4 * hj + 3]);
      }
  if (tr == 0) {
    float* vp = vpart + ((int64_t)blockIdx.z * gridDim.y + b) * K;
#pragma unroll
    for (int hj = 0; hj < NH; ++hj)
#pragma unroll
      for (int j = 0; j < 4; ++j) vp[tc * 4 + 64 * hj + j] = vacc[4 * hj + j];
  }
}
constexpr int MV_SPLIT = 4;   // channel splits of k_lbm_mv (C >= 128: >= 32 channels each, 512 CTAs at B = 64)

// M (bf16) and v from the MV_SPLIT partials, fixed order.
__global__ void k_lbm_mv_sum(int B, int K, const float* __restrict__ Mpart, const float* __restrict__ vpart,
                             __nv_bfloat16* __restrict__ Mout, float* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nm = (int64_t)B * K * K;
  if (i < nm) {
    float a = 0.f;
#pragma unroll
    for (int z = 0; z < MV_SPLIT; ++z) a += Mpart[z * nm + i];
    Mout[i] = __float2bfloat16_rn(a);
  }
  if (i < (int64_t)B * K) {
    float a = 0.f;
#pragma unroll
    for (int z = 0; z < MV_SPLIT; ++z) a += vpart[z * (int64_t)B * K + i];
    v[i] = a;
  }
}

// Sparse part of dX: dX[n*L + l] += sum over channels c with argmax(n, c) = l
// of sp(n, c) W[c].  One CTA per (model, cloud): a stable radix sort of the
// channels by argmax row (so each row's channels stay in channel order), a
// scan of the segment heads, then (segment, 8-column slice) work items spread
// over all threads; each row is written by exactly one item per slice
// (deterministic, no atomics).
constexpr int SDX_T = 256, SDX_ITEMS = 4;   // C <= 1024
__global__ void __launch_bounds__(SDX_T) k_lbm_sparse_dx(int Ncl, int64_t L, int64_t C, int K, int end_bit,
                                                         const int32_t* __restrict__ am, const float* __restrict__ sp,
                                                         const __nv_bfloat16* __restrict__ W, int64_t w_bs,
                                                         int64_t w_ld, __nv_bfloat16* __restrict__ dX, int64_t dx_bs,
                                                         int64_t dx_ld, const __nv_bfloat16* __restrict__ mask,
                                                         int64_t m_bs, int64_t m_ld, int m_act, float m_alpha) {
  using Sort = cub::BlockRadixSort<uint32_t, SDX_T, SDX_ITEMS, int>;
  using Scan = cub::BlockScan<int, SDX_T>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ uint32_t srow[SDX_T * SDX_ITEMS];
  __shared__ int schan[SDX_T * SDX_ITEMS];
  __shared__ int shead[SDX_T * SDX_ITEMS + 1];
  __shared__ float spv[SDX_T * SDX_ITEMS];      // sp of the sorted channels
  __shared__ int snseg;
  const int b = blockIdx.y, n = blockIdx.x;
  const int t = threadIdx.x;
  const uint32_t sentinel = (1u << end_bit) - 1u;
  uint32_t key[SDX_ITEMS];
  int val[SDX_ITEMS];
  const int32_t* amn = am + ((int64_t)b * Ncl + n) * C;
#pragma unroll
  for (int i = 0; i < SDX_ITEMS; ++i) {
    const int c = t * SDX_ITEMS + i;
    key[i] = c < C ? (uint32_t)amn[c] : sentinel;
    val[i] = c;
  }
  Sort(tmp.sort).Sort(key, val, 0, end_bit);
  const float* spc = sp + ((int64_t)b * Ncl + n) * C;
#pragma unroll
  for (int i = 0; i < SDX_ITEMS; ++i) {
    srow[t * SDX_ITEMS + i] = key[i];
    schan[t * SDX_ITEMS + i] = val[i];
    spv[t * SDX_ITEMS + i] = val[i] < C ? spc[val[i]] : 0.f;
  }
  __syncthreads();
  // segment heads -> compacted list of segment starts
  int flag[SDX_ITEMS], pos[SDX_ITEMS];
#pragma unroll
  for (int i = 0; i < SDX_ITEMS; ++i) {
    const int j = t * SDX_ITEMS + i;
    flag[i] = (j < C && (j == 0 || srow[j - 1] != srow[j])) ? 1 : 0;
  }
  int total;
  Scan(tmp.scan).ExclusiveSum(flag, pos, total);
#pragma unroll
  for (int i = 0; i < SDX_ITEMS; ++i)
    if (flag[i]) shead[pos[i]] = t * SDX_ITEMS + i;
  if (t == 0) { shead[total] = (int)C; snseg = total; }
  __syncthreads();
  const int nseg = snseg;
  const __nv_bfloat16* Wb = W + (int64_t)b * w_bs;
  __nv_bfloat16* dXn = dX + (int64_t)b * dx_bs + (int64_t)n * L * dx_ld;
  // item = (segment = one distinct argmax row, 16-element k slice): the dX
  // slice load is issued with the first W loads, the segment's W rows are
  // gathered two at a time, then one gated add and store
  const int nsl = K / 16;
  for (int it = t; it < nseg * nsl; it += SDX_T) {
    const int sg = it / nsl, k16 = (it % nsl) * 16;
    const int j0 = shead[sg], j1 = shead[sg + 1];
    const int64_t r = srow[j0];
    __nv_bfloat16* d = dXn + r * dx_ld + k16;
    const uint4 y0 = *reinterpret_cast<const uint4*>(d), y1 = *reinterpret_cast<const uint4*>(d + 8);
    uint4 m0 = make_uint4(0u, 0u, 0u, 0u), m1 = m0;
    if (mask) {
      const __nv_bfloat16* mr = mask + (int64_t)b * m_bs + ((int64_t)n * L + r) * m_ld + k16;
      m0 = *reinterpret_cast<const uint4*>(mr);
      m1 = *reinterpret_cast<const uint4*>(mr + 8);
    }
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
    for (int j = j0; j < j1; j += 2) {
      const bool two = j + 1 < j1;
      const __nv_bfloat16* w0 = Wb + (int64_t)schan[j] * w_ld + k16;
      const __nv_bfloat16* w1 = Wb + (int64_t)schan[two ? j + 1 : j] * w_ld + k16;
      const uint4 a0 = *reinterpret_cast<const uint4*>(w0), a1 = *reinterpret_cast<const uint4*>(w0 + 8);
      const uint4 c0 = *reinterpret_cast<const uint4*>(w1), c1 = *reinterpret_cast<const uint4*>(w1 + 8);
      const float s0 = spv[j], s1 = two ? spv[j + 1] : 0.f;
      const uint32_t ua[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const uint32_t uc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float lo, hi;
        unpack_bf2(ua[q], lo, hi);
        acc[2 * q] = fmaf(s0, lo, acc[2 * q]);
        acc[2 * q + 1] = fmaf(s0, hi, acc[2 * q + 1]);
        unpack_bf2(uc[q], lo, hi);
        acc[2 * q] = fmaf(s1, lo, acc[2 * q]);
        acc[2 * q + 1] = fmaf(s1, hi, acc[2 * q + 1]);
      }
    }
    const uint32_t uy[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
    const uint32_t um[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    const float neg = m_act == HFTA_ACT_LEAKY_RELU ? m_alpha : 0.f;
    uint32_t out[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float lo, hi;
      unpack_bf2(uy[q], lo, hi);
      float g0 = acc[2 * q], g1 = acc[2 * q + 1];
      if (mask) {   // the dense part was gated by act'(X) in the GEMM epilogue: gate the sparse part too
        float ml, mh;
        unpack_bf2(um[q], ml, mh);
        g0 *= ml > 0.f ? 1.f : neg;
        g1 *= mh > 0.f ? 1.f : neg;
      }
      out[q] = pack_bf2(lo + g0, hi + g1);
    }
    *reinterpret_cast<uint4*>(d) = make_uint4(out[0], out[1], out[2], out[3]);
    *reinterpret_cast<uint4*>(d + 8) = make_uint4(out[4], out[5], out[6], out[7]);
  }
}

// dW[c] (+)= bx_c (W G)[c] + cc_c s + sum_n sp(n, c) X[n*L + argmax(n, c)].
// CTA = (model, 32 channels), 256 threads = 8 warps x 4 channels; lane l owns
// k = 4l .. 4l+3 (K = 128; K = 64: lanes 0-15).  (W G): the CTA's 32 W rows
// in smem (fp32), one G row segment (L1) per k2 reused by the warp's 4
// channels.  Sparse part: per-cloud (sp, argmax) one per lane, broadcast by
// shuffles, 16 row gathers issued back to back.
__global__ void __launch_bounds__(256, 2) k_lbm_dw(int Ncl, int64_t L, int64_t C, int K, const float* __restrict__ G,
                                                const float* __restrict__ svec, const __nv_bfloat16* __restrict__ W,
                                                int64_t w_bs, int64_t w_ld, const float2* __restrict__ coef,
                                                const int32_t* __restrict__ am, const float* __restrict__ sp,
                                                const __nv_bfloat16* __restrict__ X, int64_t x_bs, int64_t x_ld,
                                                float* __restrict__ dW, int64_t dw_bs, int64_t dw_ld,
                                                int accumulate) {
  __shared__ float sw[32][128];
  extern __shared__ float4 sG4[];                 // G [K][K] fp32 (the model's Gram, shared by all its CTAs)
  const int b = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const __nv_bfloat16* Wb = W + (int64_t)b * w_bs;
  for (int e = threadIdx.x; e < 32 * K; e += 256) {
    const int ci = e / K, k = e % K;
    sw[ci][k] = c0 + ci < C ? __bfloat162float(Wb[(c0 + ci) * w_ld + k]) : 0.f;
  }
  {
    const float4* g4 = reinterpret_cast<const float4*>(G + (int64_t)b * K * K);
    for (int e = threadIdx.x; e < K * K / 4; e += 256) sG4[e] = g4[e];
  }
  __syncthreads();
  const bool on = lane * 4 < K;
  const __nv_bfloat16* Xb = X + (int64_t)b * x_bs;
  const float* sG = reinterpret_cast<const float*>(sG4);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;
  if (on) {
#pragma unroll 2
    for (int k2 = 0; k2 < K; ++k2) {
      const float4 g4 = *reinterpret_cast<const float4*>(sG + k2 * K + lane * 4);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float w = sw[warp * 4 + i][k2];
        acc[i][0] = fmaf(w, g4.x, acc[i][0]); acc[i][1] = fmaf(w, g4.y, acc[i][1]);
        acc[i][2] = fmaf(w, g4.z, acc[i][2]); acc[i][3] = fmaf(w, g4.w, acc[i][3]);
      }
    }
  }
  float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (on) s4 = __ldg(reinterpret_cast<const float4*>(svec + (int64_t)b * K + lane * 4));
  const float ss[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t c = c0 + warp * 4 + i;
    if (c >= C) break;
    float sacc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int nb = 0; nb < Ncl; nb += 32) {          // sparse gathers: 32 clouds per round
      const int nl = nb + lane;
      float vl = 0.f;
      int64_t rl = 0;
      if (nl < Ncl) {
        const int64_t o = ((int64_t)b * Ncl + nl) * C + c;
        vl = sp[o];
        rl = (int64_t)nl * L + am[o];
      }
      const int cnt = min(32, Ncl - nb);
      for (int q0 = 0; q0 < cnt; q0 += 16) {
        float xv[16][4];
        float vv[16];
#pragma unroll
        for (int dq = 0; dq < 16; ++dq) {            // 16 independent row gathers in flight
          const int q = min(q0 + dq, cnt - 1);
          vv[dq] = q0 + dq < cnt ? __shfl_sync(0xffffffffu, vl, q) : 0.f;
          const int64_t row = __shfl_sync(0xffffffffu, rl, q);
          if (on) ld_vec<__nv_bfloat16, 4>(Xb + row * x_ld + lane * 4, xv[dq]);
          else xv[dq][0] = xv[dq][1] = xv[dq][2] = xv[dq][3] = 0.f;
        }
#pragma unroll
        for (int dq = 0; dq < 16; ++dq)
#pragma unroll
          for (int e = 0; e < 4; ++e) sacc[e] = fmaf(vv[dq], xv[dq][e], sacc[e]);
      }
    }
    if (on) {
      const float2 cf = coef[(int64_t)b * C + c];
      float* d = dW + (int64_t)b * dw_bs + c * dw_ld + lane * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float r = fmaf(cf.x, acc[i][e], fmaf(cf.y, ss[e], sacc[e]));
        d[e] = accumulate ? d[e] + r : r;
      }
    }
  }
}

// ------------------------------------------------------------ host side --
constexpr size_t FWD_SMEM = 1024 + FG * 2 * WKB + FSTAGES * 2 * FA_KB + 256 + NEPIW * NBW * 4 * 32 * 16;
static_assert(FWD_SMEM <= 232448, "shared memory budget");

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// forward workspace: flipped W, per-cloud max / argmax, then the Gram call's own
struct FwdWs {
  size_t wf, mx, idx, gc, mu, lin, total;
};
FwdWs fwd_layout(int B, int64_t N, int64_t L, int64_t C, int64_t K) {
  FwdWs w{};
  size_t o = 0;
  w.wf = o; o += al256((size_t)B * C * K * 2);
  w.mx = o; o += al256((size_t)B * N * C * 4);
  w.idx = o; o += al256((size_t)B * N * C * 4);
  w.gc = o; o += al256((size_t)B * K * K * 4);
  w.mu = o; o += al256((size_t)B * K * 8);
  w.lin = o; o += al256(hfta_fused_linear_bwd_workspace(B, N * L, K, K, HFTA_BF16));
  w.total = o;
  return w;
}
// backward workspace: coef, sp, M, v
struct BwdWs {
  size_t coef, sp, M, v, mp, vp, total;
};
BwdWs bwd_layout(int B, int64_t N, int64_t L, int64_t C, int64_t K) {
  BwdWs w{};
  size_t o = 0;
  w.coef = o; o += al256((size_t)B * C * 8);
  w.sp = o; o += al256((size_t)B * N * C * 4);
  w.M = o; o += al256((size_t)B * K * K * 2);
  w.v = o; o += al256((size_t)B * K * 4);
  w.mp = o; o += al256((size_t)MV_SPLIT * B * K * K * 4);
  w.vp = o; o += al256((size_t)MV_SPLIT * B * K * 4);
  w.total = o;
  return w;
}
size_t bwd_ws(int B, int64_t N, int64_t L, int64_t C, int64_t K) { return bwd_layout(B, N, L, C, K).total; }

template <typename K_>
void set_smem(K_ kern, size_t bytes) { ensure_smem(kern, bytes); }

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
  return std::max(fwd_layout(B, N, L, C, K).total, bwd_ws(B, N, L, C, K));
}

hfta_status hfta_fused_linear_bn_max_fwd(int B, int64_t N, int64_t L, int64_t C, int64_t K, hfta_dtype dt, hfta_in X,
                                         hfta_in W, const float* bias, int64_t bias_bstride, const float* gamma,
                                         const float* beta, int64_t gb_bstride, float* running_mean,
                                         float* running_var, float momentum, float eps, hfta_act act,
                                         float act_alpha, hfta_out G, int32_t* argmax, hfta_out ext,
                                         float* save_mean, float* save_invstd, float* gram, float* xsum, void* ws,
                                         size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_common(B, N, L, C, K, dt, X, W)) return st;
  HFTA_REQUIRE(gamma && beta && G.ptr && argmax && ext.ptr && save_mean && save_invstd && gram && xsum,
               HFTA_ERR_INVALID_VALUE,
               "linear_bn_max_fwd: gamma, beta, G, argmax, ext, save_mean, save_invstd, gram, xsum are required");
  const size_t need = hfta_fused_linear_bn_max_workspace(B, N, L, C, K);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "linear_bn_max_fwd: workspace %zu < %zu", ws_bytes, need);
  if (hfta_status st = get_encode()) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const FwdWs lay = fwd_layout(B, N, L, C, K);
  char* w = reinterpret_cast<char*>(ws);
  __nv_bfloat16* wf = reinterpret_cast<__nv_bfloat16*>(w + lay.wf);
  float* mx = reinterpret_cast<float*>(w + lay.mx);
  int32_t* idx = reinterpret_cast<int32_t*>(w + lay.idx);
  const int64_t R = N * L;

  // 1. gram = X^T X, xsum = X^T 1 (tensor-core wgrad contraction + fused column sums); also the backward's input
  if (hfta_status st = hfta_fused_linear_bwd(B, R, K, K, HFTA_BF16, X, X, W, hfta_out{nullptr, 0, 1}, gram, K * K, K,
                                             xsum, K, 0, w + lay.lin, lay.total - lay.lin, stream))
    return st;
  // 2. W' = s_c W (sign of gamma folded in: the epilogue always takes a max)
  const int64_t nw = (int64_t)B * C * K / 8;
  k_lbm_flip<<<(unsigned)std::min<int64_t>(cdiv(nw, 256), 148 * 16), 256, 0, s>>>(
      B, C, K, (const __nv_bfloat16*)W.ptr, W.bstride, W.ld, gamma, gb_bstride, wf);
  // 3. per-cloud max / first argmax of Y' = X W'^T (tensor cores, Y' never leaves TMEM)
  CUtensorMap ta, tw;
  const int nba = (X.bstride == 0 && B > 1) ? 1 : B;
  if (hfta_status st = make_map(&ta, X.ptr, K, N * L, X.ld, X.bstride, nba, 64, FR)) return st;
  if (hfta_status st = make_map(&tw, wf, K, C, K, C * K, B, 64, CBLK)) return st;
  FwdArgs a{};
  a.B = B; a.Ncl = (int)N; a.nblk = (int)(C / CBLK); a.nkb = (int)(K / 64);
  a.ngroups = (int)cdiv(a.nblk, FG);
  a.a_shared = nba == 1 && B > 1;
  a.L = L; a.C = C;
  a.mx = mx; a.idx = idx;
  const int64_t npairs = (int64_t)B * N;
  a.teams = (int)std::max<int64_t>(1, std::min<int64_t>(npairs, num_sms() / a.ngroups));
  set_smem(k_lbm_fwd, FWD_SMEM);
  k_lbm_fwd<<<a.teams * a.ngroups, FWD_LT, FWD_SMEM, s>>>(ta, tw, a);
  // 4. batch statistics from the Gram, 5. pooled outputs
  set_smem(k_lbm_stats<128>, stats_smem(128));
  set_smem(k_lbm_stats<64>, stats_smem(64));
  {
    float* gc = reinterpret_cast<float*>(w + lay.gc);
    double* mu = reinterpret_cast<double*>(w + lay.mu);
    k_lbm_center<<<dim3((unsigned)cdiv(K * K, 256), (unsigned)B), 256, 0, s>>>((int)K, R, gram, xsum, gc, mu);
    const dim3 grid((unsigned)cdiv(C, ST_CH), (unsigned)B);
    const __nv_bfloat16* Wp = (const __nv_bfloat16*)W.ptr;
    const int64_t wbs = B > 1 ? W.bstride : 0;
    if (K == 128)
      k_lbm_stats<128><<<grid, 256, stats_smem(128), s>>>(B, R, C, gc, mu, Wp, wbs, W.ld, bias, bias_bstride,
                                                          running_mean, running_var, momentum, eps, save_mean,
                                                          save_invstd);
    else
      k_lbm_stats<64><<<grid, 256, stats_smem(64), s>>>(B, R, C, gc, mu, Wp, wbs, W.ld, bias, bias_bstride,
                                                        running_mean, running_var, momentum, eps, save_mean,
                                                        save_invstd);
  }
  k_lbm_fwd_fin<<<(unsigned)cdiv((int64_t)B * N * C, 256), 256, 0, s>>>(
      B, (int)N, C, mx, idx, bias, bias_bstride, gamma, beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha,
      (float*)G.ptr, G.bstride, G.ld, argmax, N * C, C, (float*)ext.ptr, ext.bstride, ext.ld);
  count_launches(5);
  return post_launch(s, "hfta_fused_linear_bn_max_fwd");
}

hfta_status hfta_fused_linear_bn_max_bwd(int B, int64_t N, int64_t L, int64_t C, int64_t K, hfta_dtype dt,
                                         hfta_in dG, hfta_in X, hfta_in W, const int32_t* argmax, hfta_in ext,
                                         const float* bias, int64_t bias_bstride, const float* gamma,
                                         const float* beta, int64_t gb_bstride, const float* save_mean,
                                         const float* save_invstd, const float* gram, const float* xsum,
                                         hfta_act act, float act_alpha, hfta_out dX,
                                         hfta_act dX_act, float dX_alpha, float* dW, int64_t dW_bstride,
                                         int64_t dW_ld, float* dbias, int64_t dbias_bstride, float* dgamma,
                                         float* dbeta, int accumulate, void* ws, size_t ws_bytes,
                                         hfta_stream stream) {
  if (hfta_status st = check_common(B, N, L, C, K, dt, X, W)) return st;
  HFTA_REQUIRE(dG.ptr && argmax && ext.ptr && gamma && beta && save_mean && save_invstd && gram && xsum && dW &&
                   dgamma && dbeta,
               HFTA_ERR_INVALID_VALUE,
               "linear_bn_max_bwd: dG, argmax, ext, gamma, beta, save_*, gram, xsum, dW, dgamma, dbeta are required");
  HFTA_REQUIRE(!dX.ptr || (aligned16(dX.ptr) && (dX.ld * 2) % 16 == 0 && (dX.bstride * 2) % 16 == 0 && dX.ld >= K),
               HFTA_ERR_UNSUPPORTED, "linear_bn_max_bwd: dX must be 16-B aligned with 16-B row strides");
  HFTA_REQUIRE(C <= SDX_T * SDX_ITEMS, HFTA_ERR_UNSUPPORTED, "linear_bn_max_bwd: C=%lld > %d", (long long)C,
               SDX_T * SDX_ITEMS);
  HFTA_REQUIRE(dW_ld >= K, HFTA_ERR_SHAPE, "linear_bn_max_bwd: dW_ld < K");
  const size_t need = hfta_fused_linear_bn_max_workspace(B, N, L, C, K);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "linear_bn_max_bwd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t R = N * L;
  const BwdWs lay = bwd_layout(B, N, L, C, K);
  char* w = reinterpret_cast<char*>(ws);
  float2* coef = reinterpret_cast<float2*>(w + lay.coef);
  float* sp = reinterpret_cast<float*>(w + lay.sp);
  __nv_bfloat16* M = reinterpret_cast<__nv_bfloat16*>(w + lay.M);
  float* v = reinterpret_cast<float*>(w + lay.v);
  const __nv_bfloat16* Wp = (const __nv_bfloat16*)W.ptr;
  const int64_t wbs = B > 1 ? W.bstride : 0;

  k_lbm_bwd_coef<<<(unsigned)cdiv((int64_t)B * C, 128), 128, 0, s>>>(
      B, (int)N, L, C, (const float*)dG.ptr, dG.bstride, dG.ld, (const float*)ext.ptr, ext.bstride, ext.ld, bias,
      bias_bstride, gamma, beta, gb_bstride, save_mean, save_invstd, (int)act, act_alpha, coef, sp, dgamma, dbeta,
      dbias, dbias_bstride, accumulate);
  int launches = 2;   // coef, dw
  if (dX.ptr) {
    float* mp = reinterpret_cast<float*>(w + lay.mp);
    float* vp = reinterpret_cast<float*>(w + lay.vp);
    if (K == 128)
      k_lbm_mv<128><<<dim3(1u, (unsigned)B, MV_SPLIT), 256, 0, s>>>(C, Wp, wbs, W.ld, coef, mp, vp);
    else
      k_lbm_mv<64><<<dim3(1u, (unsigned)B, MV_SPLIT), 256, 0, s>>>(C, Wp, wbs, W.ld, coef, mp, vp);
    k_lbm_mv_sum<<<(unsigned)cdiv((int64_t)B * K * K, 256), 256, 0, s>>>(B, (int)K, mp, vp, M, v);
    // dX = X M^T + v (M symmetric), times act'(X) when X is an activation output
    GemmP p{};
    p.B = B; p.M = R; p.N = K; p.K = K;
    p.A = X.ptr; p.a_bs = X.bstride; p.a_ld = X.ld; p.a_kmajor = 1;
    p.Bm = M; p.b_bs = K * K; p.b_ld = K; p.b_kmajor = 1;
    p.C = dX.ptr; p.c_bs = dX.bstride; p.c_ld = dX.ld;
    p.bias = v; p.bias_bs = K;
    if (dX_act != HFTA_ACT_NONE) {
      p.mask = X.ptr; p.mask_bs = X.bstride; p.mask_ld = X.ld; p.mask_act = (int)dX_act; p.mask_alpha = dX_alpha;
    }
    p.splits = 1; p.k_chunk = K;
    if (hfta_status st = run_gemm(p, HFTA_BF16, false, s)) return st;
    int end_bit = 1;
    while ((int64_t(1) << end_bit) <= L) ++end_bit;       // argmax < L < 2^end_bit - 1 (sentinel)
    k_lbm_sparse_dx<<<dim3((unsigned)N, (unsigned)B), SDX_T, 0, s>>>(
        (int)N, L, C, (int)K, end_bit, argmax, sp, Wp, wbs, W.ld, (__nv_bfloat16*)dX.ptr, dX.bstride, dX.ld,
        dX_act != HFTA_ACT_NONE ? (const __nv_bfloat16*)X.ptr : nullptr, X.bstride, X.ld, (int)dX_act, dX_alpha);
    launches += 3;
  }
  set_smem(k_lbm_dw, (size_t)128 * 128 * 4);   // K <= 128
  k_lbm_dw<<<dim3((unsigned)cdiv(C, 32), (unsigned)B), 256, (size_t)K * K * 4, s>>>(
      (int)N, L, C, (int)K, gram, xsum, Wp, wbs, W.ld, coef, argmax, sp, (const __nv_bfloat16*)X.ptr, X.bstride, X.ld, dW,
      dW_bstride, dW_ld, accumulate);
  count_launches(launches);
  return post_launch(s, "hfta_fused_linear_bn_max_bwd");
}

}  // extern "C"

#ifdef HFTA_LBM_PROF
extern "C" __attribute__((visibility("default"))) int hfta_lbm_prof_dump(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, hfta::g_lbm_prof, sizeof(unsigned long long) * 8 * (size_t)n);
}
#endif
