// gemm_tc.cu -- tcgen05 / TMEM / TMA model-batched GEMM (K1 fwd/dgrad, K2 wgrad).
//
// The fused Linear / Conv1d(k=1) of App. B
// for all B models in ONE persistent launch: the model index b is folded into
// the tile scheduler (tile = (b, split, m-tile, n-tile)), so many small
// per-model GEMMs fill the 148 SMs (the paper's "horizontal fusion",
// P:L856-857, done in the scheduler instead of by a grouped library call).
//
// Per CTA (1 per SM, 576 threads = 18 warps):
//   warp 0       TMA producer: 3-D tensor maps [B][rows][cols] (bstride = dim 2),
//                SWIZZLE_128B boxes of 64 elements (128 B) along the contiguous dim.
//   warp 1       MMA issuer: one elected thread issues tcgen05.mma.kind::f16
//                (bf16 x bf16 -> fp32 in TMEM), M=128, N=BN, K=16 per instruction.
//   warps 2..17  epilogue, two groups of 8 warps taking alternate tiles:
//                tcgen05.ld 32x32b -> registers -> bias / BN apply / ReLU' gate ->
//                bf16 SWIZZLE_128B smem staging + TMA store (or fp32 stores);
//                double-buffered TMEM accumulators let the epilogue of tile i
//                overlap the MMAs of i+1.
// Operands: A(m,k), B(n,k) each K-major ([m][k], k contiguous) or MN-major
// ([k][m], m contiguous); MN-major is what the dgrad (B = W) and wgrad
// (A = dY, B = X) contractions need, read without a transpose pass.
#include "gemm.cuh"
#include "tc_common.cuh"

namespace hfta {
namespace {

constexpr int BM = 128;     // UMMA M (one CTA, cta_group::1)
constexpr int BK = 64;      // k per stage: 64 bf16 = 128 B = one swizzle row
// warp 0 TMA, warp 1 MMA, warps 2..17 epilogue: two groups of 8 (2 per TMEM lane
// quarter) that take alternate tiles, so each group has two tiles' time for its
// (latency-bound) epilogue while the tensor core and TMA stream
constexpr int NTHREADS = 576;
constexpr int NEPI = 8;           // epilogue warps per group (= arrivals per tile)
constexpr int NEPI_ALL = 16;
// SWIZZLE_NONE core-matrix strides of the 8-channel image operands (bytes; tools/micro/nosw_8ch.cu)
constexpr uint32_t NOSW_K_LBO = 2048, NOSW_K_SBO = 128;     // K-major: k-adjacent (taps), m-adjacent (8-row groups)
constexpr uint32_t NOSW_MN_LBO = 128, NOSW_MN_SBO = 1024;   // MN-major: k-adjacent (8-row groups), mn-adjacent (taps)

struct TcArgs {
  int B, splits, order;            // order 0: n fastest, 1: m fastest
  int64_t M, N, K, k_chunk;
  int a_shared, b_shared;
  void* C; int64_t c_bs, c_ld;
  const float* bias; int64_t bias_bs, bias_ld, bias_div;
  int accumulate;
  float* part;
  int tiles_m, tiles_n;
  // EPI extensions
  const float* scale; int64_t scale_bs;
  int act; float act_alpha;
  const __nv_bfloat16* mask; int64_t mask_bs, mask_ld; int mask_act; float mask_alpha;
  int64_t K2;                        // second K segment (maps tmA2 / tmB2)
  int mask_kb;                       // >= 0: the gating tensor is the A tile of k-blocks mask_kb..:
                                     // read from the resident smem stage (released by the epilogue)
  float* colsum; int64_t colsum_bs; int colsum_acc; float* colsum_part;   // fused column sums of A
  float* colstat; int64_t colstat_bs;  // BN statistics of the stored bf16 C per 32-row block (see gemm.cuh)
  int ab_same;                       // Gram X^T X (A == B, one 128-wide tile): B is read from the A stage
  // implicit-GEMM convolution geometry (CONV > 0; kernel 4x4, stride 2, pad 1)
  int gw, gh, ghw;                   // the image grid the GEMM rows (CONV 1, 2) / reduction rows (3, 4) enumerate
  int cblk;                          // CONV 1, 2: 64-channel blocks per tap of the image operand
  int cg;                            // CONV 3: channels per tap of B (C_in); CONV 4: rows per tap of A (C_out)
  int y_c, y_h, y_w; int64_t y_bs;   // CONV 2: output image [B][n][y_h][y_w][y_c] the phases interleave into
  // CONV 1, 3, 4 gather geometry: kernel ks x ks, stride cs, pad cp (DCGAN: 4, 2, 1); taps = ks * ks
  int ks, cs, cp, taps;
  uint8_t tkx[64], tky[64];          // tap -> (kx, ky) (row-major; entries past `taps` = tap 0): no division
  int wflip;                         // CONV 1 with B MN-major: B is the 4-D weight view {Cn, taps, Ca} read at
                                     // tap taps-1-t (the stride-1 Conv2d dgrad: flipped, transposed W)
};

// Image coordinate of kernel tap `tap` (row-major ky * ks + kx) for output grid position g
// (gather modes): x = cs * g - cp + kx.  Taps past the kernel (a partial last k-block of an
// 8-channel image) read tap 0: their weight rows are zero (TMA zero-fill past K).
__device__ __forceinline__ void tap_xy(const TcArgs& p, int tap, int gx, int gy, int& x, int& y) {
  if (p.ks == 4 && p.cs == 2 && p.cp == 1) {      // k4 s2 p1 (DCGAN): shifts, no table reads
    x = 2 * gx - 1 + (tap & 3);
    y = 2 * gy - 1 + (tap >> 2);
    return;
  }
  x = p.cs * gx - p.cp + p.tkx[tap & 63];
  y = p.cs * gy - p.cp + p.tky[tap & 63];
}

// Row index r of a dense NHWC grid (gw x gh per image) -> (image, row, col), 32-bit.
__device__ __forceinline__ void grid_pos(uint32_t r, const TcArgs& p, int& n, int& y, int& x) {
  n = (int)(r / (uint32_t)p.ghw);
  const uint32_t rem = r - (uint32_t)n * (uint32_t)p.ghw;
  y = (int)(rem / (uint32_t)p.gw);
  x = (int)(rem - (uint32_t)y * (uint32_t)p.gw);
}

// Sub-pixel taps of a k4 s2 p1 ConvTranspose2d (and of the matching Conv2d
// dgrad, its adjoint): output row 2i + par takes input rows i + off from
// kernel rows kh, for t = 0, 1:  par 0 -> (kh 1, off 0), (kh 3, off -1);
// par 1 -> (kh 0, off +1), (kh 2, off 0).
__device__ __forceinline__ void phase_tap(int par, int t, int& k, int& off) {
  k = par ? (t ? 2 : 0) : (t ? 3 : 1);
  off = par ? (t ? 0 : 1) : (t ? -1 : 0);
}

// (a, b) += (c, d) as one packed FADD2
__device__ __forceinline__ void add_f32x2(float& a, float& b, float c, float d) {
  unsigned long long x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a), "f"(b));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(c), "f"(d));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
}

// Tile t -> (m-tile, n-tile, split, model) in 32-bit arithmetic (tile counts
// fit easily; the int64 divisions cost ~150 instructions per tile per warp)
__device__ __forceinline__ void tile_coords(uint32_t t, const TcArgs& p, int& mt, int& nt, int& split, int& b) {
  uint32_t r = t;
  const uint32_t tn = (uint32_t)p.tiles_n, tm = (uint32_t)p.tiles_m, sp = (uint32_t)p.splits;
  if (p.order == 0) {
    if (tn == 1) nt = 0; else { nt = (int)(r % tn); r /= tn; }
    mt = (int)(r % tm); r /= tm;
  } else {
    mt = (int)(r % tm); r /= tm;
    if (tn == 1) nt = 0; else { nt = (int)(r % tn); r /= tn; }
  }
  if (sp == 1) { split = 0; b = (int)r; } else { split = (int)(r % sp); b = (int)(r / sp); }
}

// BN statistics of one staged 32-row block, lane = column: rows r at base + 128 r,
// 16-B chunk qc ^ (r & 7) (SWIZZLE_128B staging); full blocks unrolled with 4
// independent accumulator pairs (the loop-carried add chain was the epilogue's
// critical path), ragged blocks (and the sub-pixel epilogue: register budget) row by row
template <bool UNROLL>
__device__ __forceinline__ void colstat_sum(uint32_t base, uint32_t qc, int nrow, float& s1, float& s2) {
  if (UNROLL && nrow == 32) {
    float a1[4] = {0.f, 0.f, 0.f, 0.f}, a2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      unsigned short u;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(u) : "r"(base + r * 128 + ((qc ^ (uint32_t)(r & 7)) << 4)));
      const float x = __uint_as_float((uint32_t)u << 16);
      a1[r & 3] += x;
      a2[r & 3] = fmaf(x, x, a2[r & 3]);
    }
    s1 = (a1[0] + a1[1]) + (a1[2] + a1[3]);
    s2 = (a2[0] + a2[1]) + (a2[2] + a2[3]);
    return;
  }
  s1 = 0.f; s2 = 0.f;
  for (int r = 0; r < nrow; ++r) {
    unsigned short u;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(u) : "r"(base + r * 128 + ((qc ^ (uint32_t)(r & 7)) << 4)));
    const float x = __uint_as_float((uint32_t)u << 16);
    s1 += x;
    s2 = fmaf(x, x, s2);
  }
}

// BRES ("B resident", forward layers with K <= 128): the B operand (the
// weight slice of one model / n-tile, <= 2 k-blocks) stays in shared memory
// while the CTA sweeps consecutive m-tiles of the same (model, n-tile) --
// the static schedule gives each CTA ~M/128/148*B such tiles in a row -- so
// only the activation tile streams through the ring (cuts L2->SM traffic 3x).
// EPI (bf16 output): 1 = fused BatchNorm apply, v = act(v * scale + shift);
// 2 = gated dgrad, v = (v + bias) * act'(A) with the gating values read from
// this tile's A (or A2) stage still resident in smem, optionally with a second
// K segment (A2, B2) accumulated into the same tile (non-BRES).  Separate
// instantiations keep each epilogue branch-free and small.
// CONV (implicit-GEMM convolution, no im2col / col2im buffer in HBM; the
// image operand is gathered by TMA with traversal strides, 5-D maps
// {C, W, H, N, B}, SWIZZLE_128B boxes of whole grid rows):
//   1  Conv2d fwd:          A(m = (n,oy,ox), k = (kh,kw,ci)) = X[n][2oy-1+kh][2ox-1+kw][ci]   (stride-2 gather)
//                           B = W [Co][(kh,kw,ci)] K-major
//   2  ConvT2d fwd / Conv2d dgrad, one of 4 sub-pixel phases per `split`:
//                           A(m = (n,i,j), k = (t,c)) = X[n][i+off_t][j+off_t][c]       (shifted box)
//                           B = the tap's weight slice (K-major ConvT, MN-major Conv dgrad);
//                           the epilogue interleaves row (n,i,j) into output pixel (n, 2i+ph, 2j+pw)
//   3  Conv2d wgrad:        A = dY (MN-major), B(k = (n,oy,ox), n = (tap,ci)) gathered (stride 2)
//   4  ConvT2d wgrad:       A(k = (n,i,j), m = (tap,co)) = dY[n][2i-1+kh][2j-1+kw][co] gathered, B = X (MN-major)
//   5  mode 2 for 8 output channels, the 4 phases merged into N = 32 columns (ph, pw, co):
//                           A(m = (n,i,j), k = (dy,dx,c)) = X[n][i+dy][j+dx][c], dy, dx in {-1,0,1} (9 shifted
//                           boxes), B = the phase-merged weights (zeros where a phase skips a tap); each
//                           row's 32 columns are 4 output pixels x 8 channels (four 16-B stores)
// NARROW (CONV 1, 3, 4): the image operand has 8 channels (16-B rows: D's
// input image, G's output image) -- one SWIZZLE_NONE box per kernel tap,
// core-matrix layout: K-major A (mode 1) = 8 taps x 8 channels per k-block,
// tap t's 128 x 16 B box at t * 2048; MN-major (mode 3's B, mode 4's A) = 16
// taps x 8 channels, tap t's 64-row x 16 B box at t * 1024.
template <bool A_MN, bool B_MN, int BN, int STAGES, bool OUT_F32, bool BRES, int EPI, int CONV = 0, bool NARROW = false>
__global__ void __launch_bounds__(NTHREADS, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
          const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmA2,
          const __grid_constant__ CUtensorMap tmB2, TcArgs p) {
  // CSUM (wgrad, fp32 out): B is augmented with a constant 64-column MN-major
  // atom of ones after its BN columns, and MMAs of column-sum tiles use
  // N = BN + 16: accumulator columns BN..BN+15 then hold sum_k A(m, k) (the
  // fused dbias / Gram column sums) at no extra MMA instruction.
  constexpr bool CSUM = A_MN && B_MN && OUT_F32 && CONV == 0;
  constexpr uint32_t A_BYTES = BM * BK * 2;   // 16 KB
  constexpr uint32_t B_LOAD = BN * BK * 2;    // bytes of B loaded per stage
  constexpr uint32_t B_BYTES = B_LOAD + (CSUM ? 8192 : 0);
  constexpr uint32_t STAGE_BYTES = BRES ? A_BYTES : A_BYTES + B_BYTES;
  constexpr uint32_t LOAD_BYTES = BRES ? A_BYTES : A_BYTES + B_LOAD;
  constexpr uint32_t BRES_BYTES = BRES ? 2 * B_BYTES : 0;
  constexpr uint32_t ABUF = BN + (CSUM ? 16 : 0);   // TMEM columns per accumulator buffer
  constexpr uint32_t TMEM_COLS = (2 * ABUF <= 128) ? 128 : (2 * ABUF <= 256 ? 256 : 512);
  constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  constexpr uint32_t IDESC_CS = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                                ((B_MN ? 1u : 0u) << 16) | ((uint32_t)((BN + 16) >> 3) << 17) |
                                ((uint32_t)(BM >> 4) << 24);

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bres = smem + STAGES * STAGE_BYTES;                      // BRES: 2 k-blocks of B
  uint64_t* full = reinterpret_cast<uint64_t*>(bres + BRES_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint64_t* bempty = bfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 1);
  // per-epilogue-warp staging for the TMA store: 32 rows x 128 B
  uint8_t* stage_out = bres + BRES_BYTES + 1024;                   // NEPI_ALL warps x 4 KB
  constexpr uint32_t STG_BYTES = OUT_F32 ? 0 : NEPI_ALL * 4096;              // bf16 TMA-store staging
  float* sbias_all = reinterpret_cast<float*>(stage_out + STG_BYTES);         // NEPI_ALL warps x BN floats
  float* sscale_all = sbias_all + NEPI_ALL * BN;                               // EPI: NEPI_ALL warps x BN floats


  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], (EPI == 2 && p.mask_kb >= 0) ? 1 + NEPI : 1);   // + epilogue arrivals (gating from A)
    }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], NEPI); }
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if constexpr (CSUM) {
    if (p.colsum) {   // the ones atom of every stage (never written by TMA)
      for (int st = 0; st < STAGES; ++st) {
        // ab_same: B aliases the A tile (two atoms), the ones atom follows it directly
        uint32_t* ones = reinterpret_cast<uint32_t*>(smem + st * STAGE_BYTES + A_BYTES + (p.ab_same ? 0 : B_LOAD));
        for (int i = threadIdx.x; i < 2048; i += NTHREADS) ones[i] = 0x3F803F80u;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t tiles_mn = (int64_t)p.tiles_m * p.tiles_n;
  const int64_t total = tiles_mn * p.splits * p.B;

  if (warp == 0) {
    // ============================ TMA producer ============================
    // the whole warp runs the loop (warp-uniform values in uniform registers);
    // one elected lane issues each TMA / expect_tx
    {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      int64_t bkey = -1;
      uint32_t epoch = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        int mt, nt, split, b;
        tile_coords((uint32_t)t, p, mt, nt, split, b);
        const int64_t kbeg = CONV == 2 ? 0 : (int64_t)split * p.k_chunk;
        const int64_t kend = CONV == 2 ? p.K : min(p.K, kbeg + p.k_chunk);
        const int nkb1 = (int)((kend - kbeg + BK - 1) / BK);
        const int nkb = nkb1 + (EPI == 2 ? (int)((p.K2 + BK - 1) / BK) : 0);
        const int ba = p.a_shared ? 0 : b, bb = p.b_shared ? 0 : b;
        const int m0 = mt * BM, n0 = nt * BN;
        int gn0 = 0, gy0 = 0, gx0 = 0;            // CONV 1, 2: grid position of the tile's first row
        if constexpr (CONV == 1 || CONV == 2 || CONV == 5) grid_pos((uint32_t)m0, p, gn0, gy0, gx0);
        if constexpr (BRES) {
          const int64_t key = (int64_t)bb * p.tiles_n + nt;
          if (key != bkey) {                       // new (model, n-tile): reload the resident B
            if (bkey >= 0) { mbar_wait(bempty, (epoch - 1) & 1); }
            mbar_expect_tx_w(bfull, (uint32_t)nkb * B_BYTES);
            for (int kb = 0; kb < nkb; ++kb)
              tma_load_3d_w(bres + kb * B_BYTES, &tmB, bfull, (int)(kbeg + (int64_t)kb * BK), n0, bb);
            bkey = key;
            ++epoch;
          }
        }
        // per-k-block address math without divisions (the producer thread's
        // instruction count bounds the small-N tiles): k-block kb = (tap ktap,
        // channel block kcb), advanced incrementally; a tap's image offsets are
        // recomputed only when the tap changes, per-tile invariants hoisted
        int ktap = 0, kcb = 0, tx = 0, ty = 0, ttap = 0;
        bool new_tap = true;
        int jtap[BN / 64 > 0 ? BN / 64 : 1], jci[BN / 64 > 0 ? BN / 64 : 1];
        if constexpr (CONV == 3 && !NARROW) {
#pragma unroll
          for (int j = 0; j < BN / 64; ++j) {
            const int ncol = n0 + 64 * j;
            jtap[j] = ncol / p.cg;
            jci[j] = ncol - jtap[j] * p.cg;
          }
        }
        (void)jtap; (void)jci; (void)tx; (void)ty; (void)ttap; (void)new_tap;
        for (int kb = 0; kb < nkb; ++kb) {
          if constexpr (CONV == 1 || CONV == 2 || CONV == 5) {
            if (new_tap) {
              if constexpr (CONV == 1) {
                tap_xy(p, ktap, gx0, gy0, tx, ty);
              } else if constexpr (CONV == 2) {
                int kh, oh, kw, ow;
                phase_tap(split >> 1, ktap >> 1, kh, oh);
                phase_tap(split & 1, ktap & 1, kw, ow);
                tx = gx0 + ow; ty = gy0 + oh; ttap = kh * 4 + kw;
              } else {
                tx = gx0 + ktap % 3 - 1; ty = gy0 + ktap / 3 - 1;
              }
              new_tap = false;
            }
          }
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx_w(&full[stage], (CSUM && p.ab_same) ? A_BYTES : LOAD_BYTES);
          (void)sb;
          const int k0 = (int)(kbeg + (int64_t)kb * BK);
          if constexpr (CONV == 1 && NARROW) {            // 8 taps of an 8-channel image per k-block
#pragma unroll
            for (int t8 = 0; t8 < 8; ++t8) {
              int x, y;
              tap_xy(p, kb * 8 + t8, gx0, gy0, x, y);
              tma_load_5d_w(sa + t8 * 2048, &tmA, &full[stage], 0, x, y, gn0, ba);
            }
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_3d_w(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0, bb);
            } else {
              tma_load_3d_w(sb, &tmB, &full[stage], k0, n0, bb);
            }
          } else if constexpr (CONV == 1) {               // strided gather of the input image
            const int tap = ktap, cb = kcb;
            tma_load_5d_w(sa, &tmA, &full[stage], cb * 64, tx, ty, gn0, ba);
            if constexpr (B_MN) {
              if (p.wflip) {                              // Conv dgrad (stride 1): B(n = ci, k = (t, co)) = W[co][T-1-t][ci]
#pragma unroll
                for (int j = 0; j < BN / 64; ++j)
                  tma_load_4d_w(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, p.taps - 1 - tap, cb * 64, bb);
              } else {                                    // ConvT dgrad: B(n = ci, k = (tap, co)) = Wt[tap][co][ci]
#pragma unroll
                for (int j = 0; j < BN / 64; ++j) tma_load_3d_w(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0, bb);
              }
            } else {
              tma_load_3d_w(sb, &tmB, &full[stage], k0, n0, bb);
            }
          } else if constexpr (CONV == 2) {               // sub-pixel phase `split`, tap t of 4
            const int cb = kcb, tap = ttap;
            tma_load_5d_w(sa, &tmA, &full[stage], cb * 64, tx, ty, gn0, ba);
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_4d_w(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, tap, cb * 64, bb);
            } else {
              tma_load_4d_w(sb, &tmB, &full[stage], cb * 64, n0, tap, bb);
            }
          } else if constexpr (CONV == 5) {               // shifted box (dy, dx) of 9, phase-merged weights
            tma_load_5d_w(sa, &tmA, &full[stage], kcb * 64, tx, ty, gn0, ba);
            tma_load_3d_w(sb, &tmB, &full[stage], k0, n0, bb);
          } else if constexpr (CONV == 3) {               // dY plain, B = stride-2 gather of X per (tap, ci) atom
            tma_load_3d_w(sa, &tmA, &full[stage], m0, k0, ba);
            tma_load_3d_w(sa + 8192, &tmA, &full[stage], m0 + 64, k0, ba);
            int gn, gy, gx;
            grid_pos((uint32_t)k0, p, gn, gy, gx);
            if constexpr (NARROW) {                       // 16 taps x 8 channels = one 128-column tile
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                int x, y;
                tap_xy(p, n0 / 8 + t, gx, gy, x, y);
                tma_load_5d_w(sb + t * 1024, &tmB, &full[stage], 0, x, y, gn, bb);
              }
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) {
                int x, y;
                tap_xy(p, jtap[j], gx, gy, x, y);
                tma_load_5d_w(sb + j * 8192, &tmB, &full[stage], jci[j], x, y, gn, bb);
              }
            }
          } else if constexpr (CONV == 4) {               // A = stride-2 gather of dY per (tap, co) atom, X plain
            int gn, gy, gx;
            grid_pos((uint32_t)k0, p, gn, gy, gx);
            if constexpr (NARROW) {                       // 16 taps x 8 channels = one 128-row tile
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                int x, y;
                tap_xy(p, m0 / 8 + t, gx, gy, x, y);
                tma_load_5d_w(sa + t * 1024, &tmA, &full[stage], 0, x, y, gn, ba);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int mm = m0 + 64 * j, tap = mm / p.cg, co0 = mm - tap * p.cg;
                int x, y;
                tap_xy(p, tap, gx, gy, x, y);
                tma_load_5d_w(sa + j * 8192, &tmA, &full[stage], co0, x, y, gn, ba);
              }
            }
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_3d_w(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0, bb);
          } else if (EPI == 2 && kb >= nkb1) {            // second K segment (K-major A2, B2)
            const int k2 = (kb - nkb1) * BK;
            tma_load_3d_w(sa, &tmA2, &full[stage], k2, m0, b);
            if constexpr (!BRES) tma_load_3d_w(sb, &tmB2, &full[stage], k2, n0, b);
          } else if (A_MN) {
            tma_load_3d_w(sa, &tmA, &full[stage], m0, k0, ba);
            tma_load_3d_w(sa + 8192, &tmA, &full[stage], m0 + 64, k0, ba);
          } else {
            tma_load_3d_w(sa, &tmA, &full[stage], k0, m0, ba);
          }
          if (CONV != 0 || (EPI == 2 && kb >= nkb1)) {
          } else if (CSUM && p.ab_same) {                 // Gram: the A tile is also B
          } else if constexpr (!BRES) {
            if (B_MN) {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_3d_w(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0, bb);
            } else {
              tma_load_3d_w(sb, &tmB, &full[stage], k0, n0, bb);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (++kcb == p.cblk) { kcb = 0; ++ktap; new_tap = true; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================= MMA issuer =============================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int64_t bkey = -1;
    uint32_t epoch = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      int mt_, nt_, split, b_;
      tile_coords((uint32_t)t, p, mt_, nt_, split, b_);
      (void)mt_;
      if constexpr (BRES) {
        const int bb_ = p.b_shared ? 0 : b_;
        const int64_t key = (int64_t)bb_ * p.tiles_n + nt_;
        if (key != bkey) {
          if (bkey >= 0) tc_commit_w(bempty);   // old B free once all prior MMAs retire
          __syncwarp();
          mbar_wait(bfull, epoch & 1);
          bkey = key;
          ++epoch;
        }
      }
      const int64_t kbeg = CONV == 2 ? 0 : (int64_t)split * p.k_chunk;
      const int64_t kend = CONV == 2 ? p.K : min(p.K, kbeg + p.k_chunk);
      const int nkb = (int)((kend - kbeg + BK - 1) / BK) + (EPI == 2 ? (int)((p.K2 + BK - 1) / BK) : 0);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * ABUF);
      const bool cs_tile = CSUM && p.colsum && nt_ == 0;      // column sums once per m-tile
      const uint32_t idesc = cs_tile ? IDESC_CS : IDESC;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        {
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = BRES ? smem_u32(bres + kb * B_BYTES) : ((CSUM && p.ab_same) ? sa : sa + A_BYTES);
          // NARROW image operands: SWIZZLE_NONE core matrices (K-major A of mode 1: 8-row groups
          // 128 B apart, taps 2048 B apart; MN-major: 8-k groups 128 B apart, 8-column taps 1024 B apart)
          constexpr bool NA = NARROW && (CONV == 1 || CONV == 4), NB = NARROW && CONV == 3;
          const uint64_t ad0 = NA ? (CONV == 1 ? smem_desc_nosw(sa, NOSW_K_LBO, NOSW_K_SBO)
                                               : smem_desc_nosw(sa, NOSW_MN_LBO, NOSW_MN_SBO))
                                  : (A_MN ? smem_desc(sa, 8192, 1024) : smem_desc(sa, 16, 1024));
          const uint64_t bd0 = NB ? smem_desc_nosw(sb, NOSW_MN_LBO, NOSW_MN_SBO)
                                  : (B_MN ? smem_desc(sb, 8192, 1024) : smem_desc(sb, 16, 1024));
          // per 16-element k step: SW128 K-major +32 B, SW128 MN-major +16 rows x 128 B,
          // NARROW K-major +2 taps (4096 B), NARROW MN-major +16 rows x 16 B (256 B)
          constexpr uint64_t AST = NA ? (CONV == 1 ? 256 : 16) : (A_MN ? 128 : 2);
          constexpr uint64_t BST = NB ? 16 : (B_MN ? 128 : 2);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: +32 B per 16-element k step inside the 128-B swizzle row;
            // MN-major: +16 rows x 128 B (descriptor address unit: 16 B).
            tc_mma_ss(d_tmem, ad0 + (uint64_t)k * AST, bd0 + (uint64_t)k * BST, idesc,
                      (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit_w(&empty[stage]);                  // smem slot free once these MMAs retire
          if (kb == nkb - 1) tc_commit_w(&tfull[acc]);   // accumulator ready
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (nkb == 0 && lane == 0) mbar_arrive(&tfull[acc]);   // empty K range: zero tile (not used)
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ============================== epilogue ==============================
    const int ew = warp - 2;                      // 0 .. NEPI_ALL-1
    const int grp = ew / NEPI;                    // this warp's group takes tiles of local parity grp
    const int quarter = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (ew % NEPI) >> 2;            // two warps per quarter split the 64-column steps
    const uint32_t sbias = smem_u32(sbias_all + ew * BN);
    const uint32_t sscale = smem_u32(sscale_all + ew * BN);
    constexpr int NSTEP = BN / 64;
    // sub-pixel phase tiles 64 wide (direct stores, no TMA staging): the two warps
    // of a lane quarter take one 32-column half each instead of idling one of them
    constexpr bool SPLIT_COLS = CONV == 2 && NSTEP == 1;
    constexpr bool ONE_HALF = BN == 32;           // one 32-column half: the first warp of each quarter
    const int my_steps = ONE_HALF ? (half == 0 ? 1 : 0) : (SPLIT_COLS ? 1 : (NSTEP - half + 1) / 2);
    const int acc = grp;                          // local tile parity = accumulator buffer
    uint32_t acc_phase = 0;
    int64_t cur_key = -1;
    int estage = 0;                               // stage counter mirrored from the producer (mask_kb >= 0)
    const bool mask_smem = EPI == 2 && p.mask_kb >= 0;
    int64_t li = 0;                               // local tile ordinal
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x, ++li) {
      int mt, nt, split, b;
      tile_coords((uint32_t)t, p, mt, nt, split, b);
      int tile_nkb = 0;
      if (mask_smem) {
        const int64_t kbeg_ = (int64_t)split * p.k_chunk, kend_ = min(p.K, kbeg_ + p.k_chunk);
        tile_nkb = (int)((kend_ - kbeg_ + BK - 1) / BK) + (int)((p.K2 + BK - 1) / BK);
      }
      if ((int)(li & 1) != grp) {                 // the other group's tile
        if (mask_smem) estage = (estage + tile_nkb) % STAGES;
        continue;
      }
      const int64_t m = (int64_t)mt * BM + quarter * 32 + lane;
      const bool row_ok = m < p.M;
      // per-(model, n-tile) bias / scale slices: reloaded only when the key
      // changes (BRES schedules sweep many m-tiles per key), loaded into
      // registers BEFORE the accumulator wait so the latency overlaps the MMAs
      // row-grouped bias table (seg head g.c1: one row per cloud of bias_div rows): when this
      // warp's 32 rows share one table row, that row is staged like a vector bias
      int64_t tgrp = -1;
      if (CONV == 0 && !OUT_F32 && p.bias && p.bias_div > 0) {
        const int64_t w0 = (int64_t)mt * BM + quarter * 32;
        const int64_t glo = w0 / p.bias_div, ghi = min(w0 + 31, p.M - 1) / p.bias_div;
        if (glo == ghi) tgrp = glo;
      }
      const bool vbias = p.bias && (p.bias_div == 0 || tgrp >= 0);
      const float* bsrc = p.bias ? p.bias + (int64_t)b * p.bias_bs + (tgrp >= 0 ? tgrp * p.bias_ld : 0) : nullptr;
      const int64_t key = ((tgrp + 1) * p.B + b) * p.tiles_n + nt;
      const bool reload = key != cur_key;
      float bpre[BN / 32], spre[BN / 32];
      if (reload) {
#pragma unroll
        for (int jj = 0; jj < BN / 32; ++jj) {
          const int64_t n = (int64_t)nt * BN + jj * 32 + lane;
          bpre[jj] = (vbias && n < p.N) ? bsrc[n] : 0.f;
          spre[jj] = (EPI == 1 && n < p.N) ? p.scale[(int64_t)b * p.scale_bs + n] : 0.f;
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const float* brow = nullptr;       // per-row bias table (row-grouped bias, rows of 2 groups)
      if (p.bias && p.bias_div > 0 && tgrp < 0 && row_ok)
        brow = p.bias + (int64_t)b * p.bias_bs + (m / p.bias_div) * p.bias_ld;
      if (reload) {                      // this warp's smem copies (broadcast reads later)
#pragma unroll
        for (int jj = 0; jj < BN / 32; ++jj) {
          st_shared_f32(sbias + (jj * 32 + lane) * 4, bpre[jj]);
          if (EPI == 1) st_shared_f32(sscale + (jj * 32 + lane) * 4, spre[jj]);
        }
        __syncwarp();
        cur_key = key;
      }
      if (CSUM && p.colsum && nt == 0 && half == 0) {   // fused column sums: TMEM lane = m, column 0
        uint32_t cs;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                     : "=r"(cs) : "r"(tmem_base + (uint32_t)(acc * ABUF + BN) + ((uint32_t)(quarter * 32) << 16)));
        tmem_wait_ld();
        if (row_ok) {
          const float v = __uint_as_float(cs);
          if (p.splits > 1) {
            p.colsum_part[((int64_t)split * p.B + b) * p.M + m] = v;
          } else {
            float* o = p.colsum + (int64_t)b * p.colsum_bs + m;
            *o = p.colsum_acc ? *o + v : v;
          }
        }
      }
      bool released = false;
      if (my_steps == 0) {               // nothing for this warp in this tile: release at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
#pragma unroll 1
      for (int si = 0; si < my_steps; ++si) {
        const int j = SPLIT_COLS ? 0 : half + 2 * si;   // 64-column step, processed as two 32-column halves
        const int64_t n0 = (int64_t)nt * BN + j * 64;
        const bool last = si == my_steps - 1;
        uint8_t* buf = stage_out + ew * 4096;  // bf16 staging: this warp's 32 x 64 sub-tile
        const uint32_t rowaddr = smem_u32(buf) + lane * 128;
        const uint32_t sw = (uint32_t)(lane & 7);
        if (!OUT_F32 && CONV != 2 && CONV != 5 && n0 < p.N) {   // the previous store of this warp (a tile ago) has read its staging
          if (lane == 0) tma_store_wait_read<0>();
          __syncwarp();
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if ((SPLIT_COLS && hh != half) || (ONE_HALF && hh != 0)) continue;   // warp-uniform
          uint32_t u[32];
          const uint32_t ta = tmem_base + (uint32_t)(acc * ABUF + (SPLIT_COLS ? 0 : j * 64) + hh * 32) +
                              ((uint32_t)(quarter * 32) << 16);
          tmem_ld32_nowait(ta, u);
          tmem_wait_ld();
          if (last && (SPLIT_COLS || ONE_HALF || hh == 1)) {   // this warp's last TMEM read of the tile: release it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
          }
          const int64_t c0 = n0 + hh * 32;
          // warp-uniform; the staged bf16 store is issued per 64 columns (at hh == 1), the
          // sub-pixel epilogue stores per 32
          if ((CONV == 2 ? c0 : n0) >= p.N) continue;
          float v[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(u[q]);
          if constexpr (EPI == 1) {            // fused BN apply: v = act(v * scale + shift)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 s4 = ld_shared_f4(sscale + (j * 64 + hh * 32 + 4 * q) * 4);
              const float4 t4 = ld_shared_f4(sbias + (j * 64 + hh * 32 + 4 * q) * 4);
              v[4 * q] = fmaf(v[4 * q], s4.x, t4.x); v[4 * q + 1] = fmaf(v[4 * q + 1], s4.y, t4.y);
              v[4 * q + 2] = fmaf(v[4 * q + 2], s4.z, t4.z); v[4 * q + 3] = fmaf(v[4 * q + 3], s4.w, t4.w);
            }
            if (p.act == HFTA_ACT_RELU) {
#pragma unroll
              for (int q = 0; q < 32; ++q) v[q] = fmaxf(v[q], 0.f);
            } else if (p.act == HFTA_ACT_LEAKY_RELU) {
#pragma unroll
              for (int q = 0; q < 32; ++q) v[q] = v[q] > 0.f ? v[q] : p.act_alpha * v[q];
            }
          } else {
            if (vbias) {
#pragma unroll
              for (int q = 0; q < 8; ++q) {             // smem broadcast
                const float4 t4 = ld_shared_f4(sbias + (j * 64 + hh * 32 + 4 * q) * 4);
                add_f32x2(v[4 * q], v[4 * q + 1], t4.x, t4.y);
                add_f32x2(v[4 * q + 2], v[4 * q + 3], t4.z, t4.w);
              }
            } else if (brow) {
              const float* br = brow + c0;
              if (c0 + 32 <= p.N && (reinterpret_cast<uintptr_t>(br) & 15) == 0) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {   // rows of one sample share the bias row: L1 broadcast
                  const float4 t4 = __ldg(reinterpret_cast<const float4*>(br) + q);
                  add_f32x2(v[4 * q], v[4 * q + 1], t4.x, t4.y);
                  add_f32x2(v[4 * q + 2], v[4 * q + 3], t4.z, t4.w);
                }
              } else {
#pragma unroll
                for (int q = 0; q < 32; ++q)
                  if (c0 + q < p.N) v[q] += br[q];
              }
            }
            if constexpr (CONV != 0) {           // activation of a layer without BN (D c1 LeakyReLU, G t5 Tanh)
              if (p.act == HFTA_ACT_LEAKY_RELU) {
#pragma unroll
                for (int q = 0; q < 32; ++q) v[q] = v[q] > 0.f ? v[q] : p.act_alpha * v[q];
              } else if (p.act == HFTA_ACT_TANH) {
#pragma unroll
                for (int q = 0; q < 32; ++q)             // MUFU tanh (rel. err ~2^-11 < the bf16 output rounding)
                  if (c0 + q < p.N) asm("tanh.approx.f32 %0, %1;" : "=f"(v[q]) : "f"(v[q]));
              }
            }
          }
          // gating values = this tile's A operand, still resident in smem: per
          // bf16 pair, gate = 0xFFFF where the (signed 16-bit) pattern is > 0
          // (ReLU'), from two SIMD min/max and one multiply
          uint32_t gate[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) gate[i] = 0xFFFFFFFFu;
          if (EPI == 2 && p.mask && !mask_smem && row_ok) {
            // gating tensor from global memory (a tile's k-blocks do not all fit
            // the ring, or the mask is not an operand): 32 bf16 = 4 x 16 B per row
            const uint4* gp = reinterpret_cast<const uint4*>(p.mask + (int64_t)b * p.mask_bs + m * p.mask_ld + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 raw = (c0 + 8 * q < p.N) ? __ldg(gp + q) : make_uint4(0u, 0u, 0u, 0u);
              const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                uint32_t t;
                asm("max.s16x2 %0, %1, %2;" : "=r"(t) : "r"(w4[e]), "r"(0u));
                asm("min.u16x2 %0, %1, %2;" : "=r"(t) : "r"(t), "r"(0x00010001u));
                gate[4 * q + e] = t * 0xFFFFu;
              }
            }
          }
          if (EPI == 2 && mask_smem) {
            const int st = (estage + p.mask_kb + j) % STAGES;
            const uint32_t arow = smem_u32(smem + st * STAGE_BYTES) + (uint32_t)((quarter * 32 + lane) * 128);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 raw = ld_shared_u4(arow + (((uint32_t)(hh * 4 + q) ^ sw) << 4));
              const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                uint32_t t;
                asm("max.s16x2 %0, %1, %2;" : "=r"(t) : "r"(w4[e]), "r"(0u));
                asm("min.u16x2 %0, %1, %2;" : "=r"(t) : "r"(t), "r"(0x00010001u));
                gate[4 * q + e] = t * 0xFFFFu;   // per half: 1 -> 0xFFFF, 0 -> 0
              }
            }
            if (last && hh == 1) {             // last read of this tile's A stages by this warp: release them
              __syncwarp();
              if (lane == 0)
                for (int k = 0; k < tile_nkb; ++k) mbar_arrive(&empty[(estage + k) % STAGES]);
              released = true;
            }
          }
          if constexpr (CONV == 2) {
            // sub-pixel phase: row m = (n, i, j) of the phase grid -> output pixel (n, 2i+ph, 2j+pw);
            // each thread stores its row's 32 columns (64 B) directly
            if (row_ok) {
              int gn, gy, gx;
              grid_pos((uint32_t)m, p, gn, gy, gx);
              const int64_t pix = ((int64_t)gn * p.y_h + 2 * gy + (split >> 1)) * p.y_w + 2 * gx + (split & 1);
              uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)b * p.y_bs +
                                                    pix * p.y_c + c0);
              // gated dgrad (the next layer's activation backward, e.g. D c1's LeakyReLU):
              // v *= act'(gate) with the gate tensor in the output's layout
              const uint4* gsrc = p.mask ? reinterpret_cast<const uint4*>(p.mask + (int64_t)b * p.mask_bs +
                                                                           pix * p.y_c + c0) : nullptr;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (c0 + 8 * q >= p.N) break;
                if (gsrc) {
                  const uint4 g4 = __ldg(gsrc + q);
                  const uint32_t gw[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    float g0, g1;
                    unpack_bf2(gw[e], g0, g1);
                    v[8 * q + 2 * e] *= g0 > 0.f ? 1.f : p.mask_alpha;
                    v[8 * q + 2 * e + 1] *= g1 > 0.f ? 1.f : p.mask_alpha;
                  }
                }
                uint4 w4;
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
                for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
                dst[q] = w4;
              }
            }
            if (p.colstat) {
              // BN statistics of the stored values (G's ConvT forward): the warp stages its 32
              // rows' bf16 (row = lane) and lane l sums column c0 + l; block index = (phase,
              // 32-row block of the phase grid), so the 4 phases cover the whole output
              const uint32_t srow = smem_u32(buf) + (uint32_t)lane * 128;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                uint4 w4 = make_uint4(0u, 0u, 0u, 0u);
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
                for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
                st_shared_v4(srow + (((uint32_t)q ^ (uint32_t)(lane & 7)) << 4), w4);
              }
              __syncwarp();
              const int64_t row0 = (int64_t)mt * BM + quarter * 32;
              const int nrow = (int)min((int64_t)32, p.M - row0);
              const int64_t col = c0 + lane;
              if (nrow > 0 && col < p.N) {
                const uint32_t base = smem_u32(buf) + (uint32_t)((lane & 7) * 2);
                const uint32_t qc = (uint32_t)(lane >> 3);
                float s1, s2;
                colstat_sum<CONV != 2>(base, qc, nrow, s1, s2);
                const int64_t nblk = (p.M + 31) / 32;
                float* cs = p.colstat + (int64_t)b * p.colstat_bs + ((int64_t)split * nblk + row0 / 32) * 2 * p.N + col;
                cs[0] = s1;
                cs[p.N] = s2;
              }
              __syncwarp();
            }
          } else if constexpr (CONV == 5) {
            // merged phases: column 8 q + c of row (n, i, j) -> pixel (n, 2i + (q >> 1), 2j + (q & 1)), channel c
            if (row_ok) {
              int gn, gy, gx;
              grid_pos((uint32_t)m, p, gn, gy, gx);
              __nv_bfloat16* yb = reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)b * p.y_bs;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int64_t pix = ((int64_t)gn * p.y_h + 2 * gy + (q >> 1)) * p.y_w + 2 * gx + (q & 1);
                uint4 w4;
                __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
                for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
                *reinterpret_cast<uint4*>(yb + pix * 8) = w4;
              }
            }
          } else if constexpr (!OUT_F32) {
            // bf16: 16-B chunk q of row r at chunk q ^ (r & 7) (TMA SWIZZLE_128B layout, conflict-free);
            // rows >= M and columns >= N are clipped by the tensor map
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 w4;
              __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w4);
#pragma unroll
              for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
              if (EPI == 2) {
                w4.x &= gate[4 * q]; w4.y &= gate[4 * q + 1]; w4.z &= gate[4 * q + 2]; w4.w &= gate[4 * q + 3];
              }
              st_shared_v4(rowaddr + (((uint32_t)(hh * 4 + q) ^ sw) << 4), w4);
            }
            if ((CONV == 0 || CONV == 1) && EPI == 0 && p.colstat) {
              // BN statistics of the values as stored: lane l sums column hh*32 + l over the
              // warp's 32 staged rows (row r, chunk q at q ^ (r & 7); 2-B reads, conflict-free)
              __syncwarp();
              const int64_t row0 = (int64_t)mt * BM + quarter * 32;
              const int nrow = (int)min((int64_t)32, p.M - row0);
              const int64_t col = c0 + lane;
              if (nrow > 0 && col < p.N) {
                const uint32_t base = smem_u32(buf) + (uint32_t)((lane & 7) * 2);
                const uint32_t qc = (uint32_t)(hh * 4 + (lane >> 3));
                float s1, s2;
                colstat_sum<true>(base, qc, nrow, s1, s2);
                float* cs = p.colstat + (int64_t)b * p.colstat_bs + (row0 / 32) * 2 * p.N + col;
                cs[0] = s1;
                cs[p.N] = s2;
              }
            }
            if (hh == 1) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) tma_store_3d(&tmC, buf, (int)n0, (int)(mt * BM + quarter * 32), b);
            }
          } else {
            if (!row_ok || c0 >= p.N) continue;
            const bool full_chunk = c0 + 32 <= p.N;
            float* dst = p.splits > 1 ? p.part + (((int64_t)split * p.B + b) * p.M + m) * p.N + c0
                                      : reinterpret_cast<float*>(p.C) + (int64_t)b * p.c_bs + m * p.c_ld + c0;
            const bool vec_ok = full_chunk && (p.splits > 1 ? (p.N % 4 == 0) : true);
            if (p.splits == 1 && p.accumulate) {
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (c0 + q < p.N) dst[q] += v[q];
            } else if (vec_ok) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            } else {
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (c0 + q < p.N) dst[q] = v[q];
            }
          }
        }
      }
      if (mask_smem) {                   // warps that read no mask this tile release here
        if (!released) {
          __syncwarp();
          if (lane == 0)
            for (int k = 0; k < tile_nkb; ++k) mbar_arrive(&empty[(estage + k) % STAGES]);
        }
        estage = (estage + tile_nkb) % STAGES;
      }
      acc_phase ^= 1;
    }
  }
  if (warp >= 2 && lane == 0) tma_store_wait_read<0>();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

template <bool A_MN, bool B_MN, int BN, bool OUT_F32, bool BRES, int EPI = 0>
hfta_status launch_tc(const GemmP& p, cudaStream_t s) {
  // EPI non-BRES BN=64 (the two-segment gated dgrad): 6 stages so a tile's 3
  // k-blocks can stay resident for the epilogue while the next tile loads
  // B-resident (K <= 128, HBM-bound streaming of A): 7 stages keep ~112 KB of A
  // in flight per SM (latency x per-SM share of HBM bandwidth)
  constexpr int STAGES = BRES ? (BN <= 128 ? 7 : 4) : ((BN == 256) ? 3 : ((EPI == 2 && BN == 64) ? 6 : 4));
  constexpr size_t SMEM = 1024 + (size_t)STAGES * (BM * BK * 2 + (BRES ? 0 : BN * BK * 2)) +
                          (BRES ? 2 * BN * BK * 2 : 0) + 1024 + (OUT_F32 ? 0 : NEPI_ALL * 4096) +
                          NEPI_ALL * BN * 4 * (EPI == 1 ? 2 : 1) +
                          ((A_MN && B_MN && OUT_F32) ? (size_t)STAGES * 8192 : 0);
  static_assert(SMEM <= 232448, "shared memory budget");
  if (hfta_status st = get_encode()) return st;
  CUtensorMap ta, tb;
  const int nba = p.a_bs == 0 ? 1 : p.B, nbb = p.b_bs == 0 ? 1 : p.B;
  hfta_status st;
  if (A_MN) st = make_map(&ta, p.A, p.M, p.K, p.a_ld, p.a_bs, nba, 64, BK);
  else st = make_map(&ta, p.A, p.K, p.M, p.a_ld, p.a_bs, nba, BK, BM);
  if (st) return st;
  if (B_MN) st = make_map(&tb, p.Bm, p.N, p.K, p.b_ld, p.b_bs, nbb, 64, BK);
  else st = make_map(&tb, p.Bm, p.K, p.N, p.b_ld, p.b_bs, nbb, BK, BN);
  if (st) return st;
  CUtensorMap ta2 = ta, tb2 = tb;
  if (EPI == 2 && p.K2 > 0) {
    if (hfta_status st2 = make_map(&ta2, p.A2, p.K2, p.M, p.a2_ld, p.a2_bs, p.B, BK, BM)) return st2;
    if (hfta_status st2 = make_map(&tb2, p.Bm2, p.K2, p.N, p.b2_ld, p.b2_bs, p.B, BK, BN)) return st2;
  }
  CUtensorMap tc_ = tb;
  if (!OUT_F32 && p.splits == 1) {
    cuuint64_t dims[3] = {(cuuint64_t)p.N, (cuuint64_t)p.M, (cuuint64_t)p.B};
    cuuint64_t strides[2] = {(cuuint64_t)(p.c_ld * 2), (cuuint64_t)((p.B > 1 ? p.c_bs : p.M * p.c_ld) * 2)};
    cuuint32_t box[3] = {64, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(&tc_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p.C, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HFTA_ERR_CUDA, "cuTensorMapEncodeTiled (C) failed (%d)", (int)r);
  }
  TcArgs a{};
  a.B = p.B; a.splits = p.splits; a.M = p.M; a.N = p.N; a.K = p.K; a.k_chunk = p.k_chunk;
  a.a_shared = nba == 1 && p.B > 1; a.b_shared = nbb == 1 && p.B > 1;
  a.C = p.C; a.c_bs = p.c_bs; a.c_ld = p.c_ld;
  a.bias = p.bias; a.bias_bs = p.bias_bs; a.bias_ld = p.bias_ld; a.bias_div = p.bias_div;
  a.accumulate = p.accumulate; a.part = p.part;
  a.tiles_m = (int)cdiv(p.M, BM); a.tiles_n = (int)cdiv(p.N, BN);
  a.order = (A_MN && B_MN) ? 1 : 0;
  a.scale = p.scale; a.scale_bs = p.scale_bs; a.act = p.act; a.act_alpha = p.act_alpha;
  a.mask = reinterpret_cast<const __nv_bfloat16*>(p.mask); a.mask_bs = p.mask_bs; a.mask_ld = p.mask_ld;
  a.mask_act = p.mask_act; a.mask_alpha = p.mask_alpha;
  a.K2 = EPI == 2 ? p.K2 : 0;
  a.colsum = p.colsum; a.colsum_bs = p.colsum_bs; a.colsum_acc = p.colsum_acc; a.colsum_part = p.colsum_part;
  a.colstat = OUT_F32 ? nullptr : p.colstat; a.colstat_bs = p.colstat_bs;
  a.mask_kb = -1;
  // Gram X^T X of one 128-wide tile: load the tile once, use it as both operands
  a.ab_same = (A_MN && B_MN && OUT_F32 && BN == 128 && p.A == p.Bm && p.a_ld == p.b_ld && p.a_bs == p.b_bs &&
               a.tiles_m == 1 && a.tiles_n == 1 && p.M == p.N) ? 1 : 0;
  // the gating tensor is the A operand itself (same rows, its columns = the
  // output's): read it from the resident A stage instead of global memory
  // only if every k-block of a tile fits the ring at once (else the producer
  // would wait on a stage the epilogue frees only after the accumulator is
  // ready): otherwise the epilogue reads the gate from global memory
  const bool fits = (int)(cdiv(p.K, BK) + (EPI == 2 ? cdiv(p.K2, BK) : 0)) <= STAGES;
  if (EPI == 2 && p.mask && p.splits == 1 && p.N <= BN && fits) {
    if (p.K2 > 0 && p.mask == p.A2 && p.mask_bs == p.a2_bs && p.mask_ld == p.a2_ld && p.K2 == p.N)
      a.mask_kb = (int)cdiv(p.K, BK);
    else if (p.K2 == 0 && p.mask == p.A && p.mask_bs == p.a_bs && p.mask_ld == p.a_ld && p.K == p.N && p.a_kmajor)
      a.mask_kb = 0;
  }
  auto kern = k_gemm_tc<A_MN, B_MN, BN, STAGES, OUT_F32, BRES, EPI>;
  ensure_smem(kern, SMEM);
  int64_t total = (int64_t)a.tiles_m * a.tiles_n * a.splits * a.B;
  HFTA_REQUIRE(total < ((int64_t)1 << 31), HFTA_ERR_SHAPE, "gemm_tc: %lld tiles exceed int32", (long long)total);
  int grid = (int)std::min<int64_t>(total, num_sms());
  kern<<<grid, NTHREADS, SMEM, s>>>(ta, tb, tc_, ta2, tb2, a);
  count_launches(1);
  return post_launch(s, "gemm_tc");
}

bool needs_epi(const GemmP& p) { return p.scale || p.act != HFTA_ACT_NONE || p.mask || p.K2 > 0; }
bool epi1(const GemmP& p) { return p.scale && p.bias && p.bias_div == 0 && !p.mask && p.K2 == 0; }
bool epi2(const GemmP& p) {   // bias, second K segment, gating by the A operand (or A2) itself (ReLU'), N <= 128
  if (p.scale || p.act != HFTA_ACT_NONE || p.N > 128) return false;
  if (!p.mask) return true;
  // gating by relu'(mask), mask a bf16 [B][M][N] tensor (read from the resident
  // A stage when it is the A / A2 operand and fits the ring, else from global)
  return p.mask_act == HFTA_ACT_RELU && aligned16(p.mask) && (p.mask_ld * 2) % 16 == 0 && (p.mask_bs * 2) % 16 == 0;
}

template <bool A_MN, bool B_MN, bool OUT_F32>
hfta_status dispatch_bn(const GemmP& p, cudaStream_t s) {
  if constexpr (!A_MN && !B_MN && !OUT_F32) {
    if (needs_epi(p)) {
      const bool bres = p.K2 == 0 && p.K <= 2 * BK;
      if (epi1(p)) {                              // fused BN apply (forward)
        if (p.N <= 64) return bres ? launch_tc<false, false, 64, false, true, 1>(p, s)
                                   : launch_tc<false, false, 64, false, false, 1>(p, s);
        if (p.N <= 128) return bres ? launch_tc<false, false, 128, false, true, 1>(p, s)
                                    : launch_tc<false, false, 128, false, false, 1>(p, s);
        return launch_tc<false, false, 128, false, false, 1>(p, s);
      }
      if (p.N <= 64) return bres ? launch_tc<false, false, 64, false, true, 2>(p, s)
                                 : launch_tc<false, false, 64, false, false, 2>(p, s);
      return bres ? launch_tc<false, false, 128, false, true, 2>(p, s)
                  : launch_tc<false, false, 128, false, false, 2>(p, s);
    }
    if (p.K <= 2 * BK && p.splits == 1) {        // forward with small K: B-resident schedule
      if (p.N <= 64) return launch_tc<A_MN, B_MN, 64, OUT_F32, true>(p, s);
      if (p.N <= 128) return launch_tc<A_MN, B_MN, 128, OUT_F32, true>(p, s);
      return launch_tc<A_MN, B_MN, 256, OUT_F32, true>(p, s);
    }
  }
  if (p.N <= 64) return launch_tc<A_MN, B_MN, 64, OUT_F32, false>(p, s);
  if (p.N <= 128 || OUT_F32) return launch_tc<A_MN, B_MN, 128, OUT_F32, false>(p, s);
  return launch_tc<A_MN, B_MN, 256, OUT_F32, false>(p, s);
}

// `rows` consecutive rows of a dense (n, y, x) enumeration of a gw x gh grid
// (gn images) as one box of whole grid rows / images: (bw, bh, bn)
bool grid_box(int gw, int gh, int gn, int rows, uint32_t& bw, uint32_t& bh, uint32_t& bn) {
  if (gw >= rows) {
    bw = rows; bh = 1; bn = 1;
    return gw % rows == 0;
  }
  if (rows % gw) return false;
  bw = gw;
  const int r = rows / gw;
  if (gh >= r) {
    bh = r; bn = 1;
    return gh % r == 0;
  }
  if (r % gh) return false;
  bh = gh; bn = r / gh;
  return gn % (int)bn == 0;
}

// 5-D map of the image operand {C, W, H, N, B} gathering `rows` grid rows per
// box with traversal stride `st` along W and H (2: Conv2d k4 s2 p1 windows,
// 1: the shifted ConvT / dgrad phase boxes)
hfta_status img_map(CUtensorMap* m, const ConvTcP& p, int nb, int rows, int st) {
  uint32_t bw, bh, bn;
  if (!grid_box(p.grid_w, p.grid_h, p.img_n, rows, bw, bh, bn))
    return fail(HFTA_ERR_UNSUPPORTED, "conv_tc: grid %dx%d does not tile into %d-row boxes", p.grid_w, p.grid_h, rows);
  const int64_t hw = (int64_t)p.img_h * p.img_w * p.img_c;
  const int64_t dims[5] = {p.img_c, p.img_w, p.img_h, p.img_n, nb};
  const int64_t str[5] = {1, p.img_c, (int64_t)p.img_w * p.img_c, hw, nb > 1 ? p.img_bs : (int64_t)p.img_n * hw};
  const bool narrow = p.img_c == 8;            // one 16-B row per position, SWIZZLE_NONE core matrices
  const uint32_t box[5] = {narrow ? 8u : 64u, (uint32_t)st * bw, (uint32_t)st * bh, bn, 1};
  const uint32_t es[5] = {1, (uint32_t)st, (uint32_t)st, 1, 1};
  return make_map_nd(m, p.img, 5, dims, str, box, es, !narrow);
}

template <int CONV, bool A_MN, bool B_MN, int BN, bool OUT_F32, bool NARROW = false>
hfta_status launch_conv(const ConvTcP& cp, cudaStream_t s) {
  constexpr int STAGES = (BN == 256) ? 3 : (BN == 32 ? 7 : 4);
  constexpr size_t SMEM = 1024 + (size_t)STAGES * (BM * BK * 2 + BN * BK * 2) + 1024 + (OUT_F32 ? 0 : NEPI_ALL * 4096) +
                          NEPI_ALL * BN * 4;
  static_assert(SMEM <= 232448, "shared memory budget");
  if (hfta_status st = get_encode()) return st;
  CUtensorMap ta, tb, tc_;
  const int nbi = cp.img_bs == 0 ? 1 : cp.B;
  const int nbo = cp.opd_bs == 0 ? 1 : cp.B;
  hfta_status st = HFTA_OK;
  const int ks = cp.ks > 0 ? cp.ks : 4, cs = cp.ks > 0 ? cp.cs : 2, cpd = cp.ks > 0 ? cp.cpad : 1;
  if (CONV == 1) {
    st = img_map(&ta, cp, nbi, BM, cs);
    if (!st && B_MN && cp.wflip) {   // W [Ca][taps][Cn] as {Cn, taps, Ca, B}: one tap's 64 x 64 MN-major atom
      const int64_t cn = cp.w_cn, ca = cp.w_ca, T = (int64_t)ks * ks, wbs = nbo > 1 ? cp.opd_bs : T * cn * ca;
      const int64_t dims[4] = {cn, T, ca, nbo}, str[4] = {1, cn, T * cn, wbs};
      const uint32_t box[4] = {64, 1, 64, 1}, es[4] = {1, 1, 1, 1};
      st = make_map_nd(&tb, cp.opd, 4, dims, str, box, es);
    } else if (!st) {
      st = B_MN ? make_map(&tb, cp.opd, cp.N, cp.K, cp.opd_ld, cp.opd_bs, nbo, 64, BK)
                : make_map(&tb, cp.opd, cp.K, cp.N, cp.opd_ld, cp.opd_bs, nbo, BK, BN);
    }
  } else if (CONV == 2) {
    st = img_map(&ta, cp, nbi, BM, 1);
    if (!st) {
      const int64_t cn = cp.w_cn, ca = cp.w_ca, wbs = nbo > 1 ? cp.opd_bs : 16 * cn * ca;
      if (B_MN) {        // Conv2d weights W [Ca][16][Cn] (n = ci contiguous, k = co)
        const int64_t dims[4] = {cn, 16, ca, nbo}, str[4] = {1, cn, 16 * cn, wbs};
        const uint32_t box[4] = {64, 1, 64, 1}, es[4] = {1, 1, 1, 1};
        st = make_map_nd(&tb, cp.opd, 4, dims, str, box, es);
      } else {           // ConvT2d weights Wt [16][Cn][Ca] (rows n = co, k = ci contiguous)
        const int64_t dims[4] = {ca, cn, 16, nbo}, str[4] = {1, ca, cn * ca, wbs};
        const uint32_t box[4] = {64, (uint32_t)BN, 1, 1}, es[4] = {1, 1, 1, 1};
        st = make_map_nd(&tb, cp.opd, 4, dims, str, box, es);
      }
    }
  } else if (CONV == 5) {
    st = img_map(&ta, cp, nbi, BM, 1);
    if (!st) st = make_map(&tb, cp.opd, cp.K, cp.N, cp.opd_ld, cp.opd_bs, nbo, BK, BN);
  } else if (CONV == 3) {
    st = make_map(&ta, cp.opd, cp.M, cp.K, cp.opd_ld, cp.opd_bs, nbo, 64, BK);
    if (!st) st = img_map(&tb, cp, nbi, BK, cs);
  } else {
    st = img_map(&ta, cp, nbi, BK, cs);
    if (!st) st = make_map(&tb, cp.opd, cp.N, cp.K, cp.opd_ld, cp.opd_bs, nbo, 64, BK);
  }
  if (st) return st;
  tc_ = tb;
  if (CONV == 1) {         // Y [B][M][N] bf16 through the TMA-store epilogue
    cuuint64_t dims[3] = {(cuuint64_t)cp.N, (cuuint64_t)cp.M, (cuuint64_t)cp.B};
    cuuint64_t strides[2] = {(cuuint64_t)(cp.c_ld * 2), (cuuint64_t)((cp.B > 1 ? cp.c_bs : cp.M * cp.c_ld) * 2)};
    cuuint32_t box[3] = {64, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(&tc_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, cp.C, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HFTA_ERR_CUDA, "cuTensorMapEncodeTiled (conv Y) failed (%d)", (int)r);
  }
  TcArgs a{};
  a.B = cp.B; a.M = cp.M; a.N = cp.N; a.K = cp.K;
  a.splits = CONV == 2 ? 4 : (CONV == 1 ? 1 : std::max(cp.splits, 1));     // mode 2: the 4 phases
  a.k_chunk = (CONV == 1 || CONV == 2 || cp.k_chunk <= 0) ? cp.K : cp.k_chunk;
  a.a_shared = (CONV == 1 || CONV == 2 || CONV == 4 || CONV == 5) ? (nbi == 1 && cp.B > 1) : (nbo == 1 && cp.B > 1);
  a.b_shared = (CONV == 3) ? (nbi == 1 && cp.B > 1) : (nbo == 1 && cp.B > 1);
  a.C = cp.C; a.c_bs = cp.c_bs; a.c_ld = cp.c_ld;
  a.accumulate = cp.accumulate; a.part = cp.part;
  a.tiles_m = (int)cdiv(cp.M, BM); a.tiles_n = (int)cdiv(cp.N, BN);
  a.order = (A_MN && B_MN) ? 1 : 0;
  a.mask_kb = -1;
  a.gw = cp.grid_w; a.gh = cp.grid_h; a.ghw = cp.grid_w * cp.grid_h;
  a.cblk = cp.img_c / 64;
  a.cg = cp.img_c;   // 3: C_in per tap of B; 4: C_out (the gathered dY's channels) per tap of A
  a.y_c = CONV == 5 ? 8 : (int)cp.N; a.y_h = cp.y_h; a.y_w = cp.y_w; a.y_bs = cp.c_bs;
  a.act = (CONV == 1 || CONV == 2 || CONV == 5) ? cp.act : HFTA_ACT_NONE; a.act_alpha = cp.act_alpha;
  a.ks = ks; a.cs = cs; a.cp = cpd; a.taps = ks * ks; a.wflip = cp.wflip;
  if ((CONV == 1 || CONV == 2) && !OUT_F32) {
    a.colstat = cp.colstat;
    a.colstat_bs = (CONV == 2 ? 4 : 1) * cdiv(cp.M, 32) * 2 * cp.N;   // mode 2: 4 phases of M/32 blocks
  }
  for (int t = 0; t < 64; ++t) {
    const int tt = t < a.taps ? t : 0;
    a.tkx[t] = (uint8_t)(tt % ks); a.tky[t] = (uint8_t)(tt / ks);
  }
  if (CONV == 2 && cp.gate) {        // gated dgrad: ReLU' (alpha 0) / LeakyReLU' (alpha) of the gate tensor
    a.mask = reinterpret_cast<const __nv_bfloat16*>(cp.gate); a.mask_bs = cp.gate_bs;
    a.mask_alpha = cp.gate_alpha;
  }
  auto kern = k_gemm_tc<A_MN, B_MN, BN, STAGES, OUT_F32, false, 0, CONV, NARROW>;
  ensure_smem(kern, SMEM);
  const int64_t total = (int64_t)a.tiles_m * a.tiles_n * a.splits * a.B;
  HFTA_REQUIRE(total < ((int64_t)1 << 31), HFTA_ERR_SHAPE, "conv_tc: %lld tiles exceed int32", (long long)total);
  const int grid = (int)std::min<int64_t>(total, num_sms());
  kern<<<grid, NTHREADS, SMEM, s>>>(ta, tb, tc_, ta, tb, a);
  count_launches(1);
  return post_launch(s, "conv_tc");
}

}  // namespace

bool conv_tc_supported(const ConvTcP& p) {
  const bool narrow = p.img_c == 8 && p.mode != 2 && p.mode != 5;   // 8-channel image operand (SWIZZLE_NONE boxes)
  if (p.M < 1 || p.N < 1 || p.K < 1 || (p.img_c % 64 && !narrow) || !aligned16(p.img) || !aligned16(p.opd) ||
      !aligned16(p.C))
    return false;
  if ((p.img_bs * 2) % 16 || (p.opd_bs * 2) % 16 || (p.opd_ld * 2) % 16) return false;
  uint32_t bw, bh, bn;
  const int rows = (p.mode == 1 || p.mode == 2 || p.mode == 5) ? BM : BK;
  if (!grid_box(p.grid_w, p.grid_h, p.img_n, rows, bw, bh, bn)) return false;
  const int64_t taps = p.ks > 0 ? (int64_t)p.ks * p.ks : 16;
  if (p.ks > 0 && (p.cs < 1 || p.cs > 2 || p.cpad < 0 || p.ks > 8 || (p.mode != 1 && p.mode != 3))) return false;
  if (p.wflip && (p.mode != 1 || !p.w_mn || p.cs != 1 || p.w_cn % 64 || p.w_ca % 64)) return false;
  switch (p.mode) {
    case 1: return p.K == taps * (int64_t)p.img_c && p.N % 16 == 0 && (p.c_ld * 2) % 16 == 0 &&
                   (p.c_bs * 2) % 16 == 0;
    case 2: return p.K == 4 * (int64_t)p.img_c && p.N % 8 == 0 && p.N <= 256 && p.y_h == 2 * p.grid_h &&
                   p.y_w == 2 * p.grid_w && (p.c_bs * 2) % 16 == 0;
    case 5: return p.K == 9 * (int64_t)p.img_c && p.N == 32 && p.y_h == 2 * p.grid_h && p.y_w == 2 * p.grid_w &&
                   (p.c_bs * 2) % 16 == 0 && (p.opd_ld * 2) % 16 == 0;
    case 3: return p.N == taps * (int64_t)p.img_c && p.c_ld % 4 == 0;   // narrow: 16 taps per 128-wide tile
    case 4: return p.M == 16 * (int64_t)p.img_c && p.N % 16 == 0 && p.c_ld % 4 == 0;   // narrow: M = 128
    default: return false;
  }
}

hfta_status conv_tc(const ConvTcP& p, cudaStream_t s) {
  if (!conv_tc_supported(p)) return fail(HFTA_ERR_UNSUPPORTED, "conv_tc: configuration not supported");
  if (p.img_c == 8) {        // 8-channel image operand
    switch (p.mode) {
      case 1:
        if (p.w_mn) return p.N <= 64 ? launch_conv<1, false, true, 64, false, true>(p, s)
                                     : launch_conv<1, false, true, 128, false, true>(p, s);
        return p.N <= 64 ? launch_conv<1, false, false, 64, false, true>(p, s)
                         : launch_conv<1, false, false, 128, false, true>(p, s);
      case 3: return launch_conv<3, true, true, 128, true, true>(p, s);
      default: return launch_conv<4, true, true, 128, true, true>(p, s);
    }
  }
  switch (p.mode) {
    case 1:
      if (p.w_mn) {
        if (p.N <= 64) return launch_conv<1, false, true, 64, false>(p, s);
        if (p.N <= 128) return launch_conv<1, false, true, 128, false>(p, s);
        return launch_conv<1, false, true, 256, false>(p, s);
      }
      if (p.N <= 64) return launch_conv<1, false, false, 64, false>(p, s);
      if (p.N <= 128) return launch_conv<1, false, false, 128, false>(p, s);
      return launch_conv<1, false, false, 256, false>(p, s);
    case 2:
      if (p.w_mn) {
        if (p.N <= 64) return launch_conv<2, false, true, 64, false>(p, s);
        if (p.N <= 128) return launch_conv<2, false, true, 128, false>(p, s);
        return launch_conv<2, false, true, 256, false>(p, s);
      }
      if (p.N <= 64) return launch_conv<2, false, false, 64, false>(p, s);
      if (p.N <= 128) return launch_conv<2, false, false, 128, false>(p, s);
      return launch_conv<2, false, false, 256, false>(p, s);
    case 5: return launch_conv<5, false, false, 32, false>(p, s);
    // wgrads: both operands stream per k-block, so 256-wide tiles (48 KB of
    // operands per 512 MMA cycles instead of 32 KB per 256) keep the tensor
    // pipe fed from L2
    case 3: return conv_wgrad_bn(p) == 256 ? launch_conv<3, true, true, 256, true>(p, s)
                                           : launch_conv<3, true, true, 128, true>(p, s);
    default: return conv_wgrad_bn(p) == 256 ? launch_conv<4, true, true, 256, true>(p, s)
                                            : launch_conv<4, true, true, 128, true>(p, s);
  }
}

int conv_wgrad_bn(const ConvTcP& p) {
  if (p.img_c == 8) return 128;                    // narrow: one 128-wide tile
  return (p.mode == 3 ? p.N % 256 == 0 : p.N >= 256) ? 256 : 128;
}

// ---- mode 5 operand: the phase-merged weights ----
// kernel row / column of phase `par` for input offset `off` (phase_tap's inverse), -1: unused
__device__ __forceinline__ int phase_k(int par, int off) {
  return par ? (off == 1 ? 0 : (off == 0 ? 2 : -1)) : (off == 0 ? 1 : (off == -1 ? 3 : -1));
}

__global__ void k_subpixel_w(int nb, int ca, int w_mn, const __nv_bfloat16* __restrict__ W, int64_t w_bs,
                             __nv_bfloat16* __restrict__ Wp) {
  const int64_t per = 32 * 9 * (int64_t)ca;
  const int64_t total = per * nb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / per);
    const int64_t r = i - b * per;
    const int n = (int)(r / (9 * ca)), k = (int)(r - (int64_t)n * 9 * ca);
    const int t9 = k / ca, c = k - t9 * ca, phase = n >> 3, co = n & 7;
    const int kh = phase_k(phase >> 1, t9 / 3 - 1), kw = phase_k(phase & 1, t9 % 3 - 1);
    __nv_bfloat16 v = __float2bfloat16_rn(0.f);
    if (kh >= 0 && kw >= 0) {
      const int tap = kh * 4 + kw;
      const __nv_bfloat16* wb = W + (int64_t)b * w_bs;
      v = w_mn ? wb[((int64_t)c * 16 + tap) * 8 + co] : wb[((int64_t)tap * 8 + co) * ca + c];
    }
    Wp[i] = v;
  }
}

hfta_status conv_subpixel_weights(int B, int ca, int w_mn, const void* W, int64_t w_bs, void* Wp, cudaStream_t s) {
  const int nb = w_bs == 0 ? 1 : B;
  const int64_t total = (int64_t)nb * 32 * 9 * ca;
  k_subpixel_w<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 4 * 148), 256, 0, s>>>(
      nb, ca, w_mn, reinterpret_cast<const __nv_bfloat16*>(W), w_bs, reinterpret_cast<__nv_bfloat16*>(Wp));
  count_launches(1);
  return HFTA_OK;
}

bool gemm_tc_supported(const GemmP& p, hfta_dtype dt_in, bool out_f32) {
  if (dt_in != HFTA_BF16) return false;
  if (needs_epi(p)) {
    if (out_f32 || p.splits != 1 || !p.a_kmajor || !p.b_kmajor || p.accumulate) return false;
    if (!epi1(p) && !epi2(p)) return false;
    if (p.K2 > 0 && (p.K % BK || p.K2 % BK || !aligned16(p.A2) || !aligned16(p.Bm2) || (p.a2_ld * 2) % 16 ||
                     (p.b2_ld * 2) % 16 || (p.a2_bs * 2) % 16 || (p.b2_bs * 2) % 16))
      return false;
  }
  if (p.K < 16 || p.N < 16 || p.M < 1) return false;
  if (!aligned16(p.A) || !aligned16(p.Bm)) return false;
  if ((p.a_ld * 2) % 16 || (p.b_ld * 2) % 16 || (p.a_bs * 2) % 16 || (p.b_bs * 2) % 16) return false;
  if (p.M > INT32_MAX || p.N > INT32_MAX || p.K > INT32_MAX) return false;
  if (!out_f32) {
    if (!aligned16(p.C) || (p.c_ld * 2) % 16 || (p.c_bs * 2) % 16 || p.accumulate) return false;
  } else if (p.splits == 1 && (!aligned16(p.C) || p.c_ld % 4)) {
    return false;
  }
  if (p.splits > 1 && p.k_chunk % BK) return false;
  // MN-major operands are loaded in 64-element boxes along MN; a ragged MN
  // extent leaves the tail of the last box (or a whole second box) out of
  // bounds, which TMA zero-fills (the A side only feeds rows the epilogue
  // clips; the B side stays at multiples of 16).

  if (!p.b_kmajor && (p.N % 8)) return false;     // 16-B rows; the box tail past N is zero-filled
  return true;
}

hfta_status gemm_tc(const GemmP& p, hfta_dtype dt_in, bool out_f32, cudaStream_t s) {
  (void)dt_in;
  const bool amn = !p.a_kmajor, bmn = !p.b_kmajor;
  if (out_f32) {
    if (amn && bmn) return dispatch_bn<true, true, true>(p, s);
    if (!amn && bmn) return dispatch_bn<false, true, true>(p, s);
    if (!amn && !bmn) return dispatch_bn<false, false, true>(p, s);
  } else {
    if (!amn && !bmn) return dispatch_bn<false, false, false>(p, s);
    if (!amn && bmn) return dispatch_bn<false, true, false>(p, s);
  }
  return fail(HFTA_ERR_UNSUPPORTED, "gemm_tc: operand majorness combination");
}

}  // namespace hfta
