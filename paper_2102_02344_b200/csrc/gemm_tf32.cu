// gemm_tf32.cu -- fp32-accurate model-batched GEMM on the tensor cores
// (3xTF32; SURVEY 8(b) "With HFTA_F32 ... contractions are fp32-accurate";
// reading C17/R31).  The fp32 mode of every fused Linear / Conv1d / (im2col)
// Conv contraction that the bf16 engine (gemm_tc.cu) runs in bf16.
//
// tcgen05.mma.kind::tf32 reads fp32 operands and TRUNCATES them to tf32
// (measured, tools/micro/tf32_round.cu).  With hi = trunc_tf32(x) (what the
// MMA sees for x itself) and lo = x - hi (exact in fp32, |lo| < 2^-10 |x|),
//   x . w = hi_x hi_w + hi_x lo_w + lo_x hi_w + O(2^-20 |x||w|)
// and the MMA's truncation of lo costs another 2^-11 |lo| -- ~2^-21 relative
// per product, the size of fp32's own accumulation error.  Per k-block the
// stage holds the fp32 tiles of A and B (the hi operands) and their lo tiles,
// which 4 converter warps compute in shared memory; MN-major tiles (dgrad /
// wgrad operands) are transposed by the converters into the K-major
// SWIZZLE_128B layout on the way (kind::tf32 reads MN-major only in the
// 32-B-atom swizzle, measured: tools/micro/tf32_mn.cu), so the MMA warp
// always issues K-major tf32 MMAs, 3 per k-step into one accumulator.
//
// Per CTA (persistent, 1 per SM, 448 threads): warp 0 TMA producer, warp 1
// MMA issuer, warps 2..5 lo converters, warps 6..13 epilogue (two per TMEM
// lane quarter; double-buffered accumulators).  The model index is folded
// into the tile scheduler as in gemm_tc.cu.
#include "gemm.cuh"
#include "tc_common.cuh"

namespace hfta {
namespace {

constexpr int TM = 128;       // UMMA M
constexpr int TBK = 32;       // fp32 elements per k-block = one 128-B swizzle row
constexpr int T_NCONV = 4;
constexpr int T_NEPI = 8;
constexpr int T_THREADS = (2 + T_NCONV + T_NEPI) * 32;

struct TfArgs {
  int B, splits, order;
  int64_t M, N, K, k_chunk;
  int a_shared, b_shared;
  float* C; int64_t c_bs, c_ld;
  const float* bias; int64_t bias_bs, bias_ld, bias_div;
  int accumulate;
  float* part;
  int tiles_m, tiles_n;
};

__device__ __forceinline__ void tcoords(uint32_t t, const TfArgs& p, int& mt, int& nt, int& split, int& b) {
  uint32_t r = t;
  const uint32_t tn = (uint32_t)p.tiles_n, tm = (uint32_t)p.tiles_m, sp = (uint32_t)p.splits;
  if (p.order == 0) {
    nt = (int)(r % tn); r /= tn;
    mt = (int)(r % tm); r /= tm;
  } else {
    mt = (int)(r % tm); r /= tm;
    nt = (int)(r % tn); r /= tn;
  }
  split = (int)(r % sp);
  b = (int)(r / sp);
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

template <bool A_MN, bool B_MN, int BN, int STAGES>
__global__ void __launch_bounds__(T_THREADS, 1)
k_gemm_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TfArgs p) {
  constexpr uint32_t A_BYTES = TM * TBK * 4;        // 16 KB
  constexpr uint32_t B_BYTES = BN * TBK * 4;
  constexpr uint32_t HI_BYTES = A_BYTES + B_BYTES;   // what TMA delivers per stage
  constexpr uint32_t STAGE = 2 * HI_BYTES;           // [A hi][B hi][A lo][B lo]
  constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : 256));
  // both operands K-major in shared memory (MN-major tiles are transposed by the converters)
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);     // T_NEPI warps x BN floats

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], T_NCONV);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], T_NEPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  const int64_t total = (int64_t)p.tiles_m * p.tiles_n * p.splits * p.B;

  auto krange = [&](int split, int& nkb) {
    const int64_t kbeg = (int64_t)split * p.k_chunk;
    const int64_t kend = min(p.K, kbeg + p.k_chunk);
    nkb = (int)((kend - kbeg + TBK - 1) / TBK);
    return kbeg;
  };

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        int mt, nt, split, b, nkb;
        tcoords((uint32_t)t, p, mt, nt, split, b);
        const int64_t kbeg = krange(split, nkb);
        const int ba = p.a_shared ? 0 : b, bb = p.b_shared ? 0 : b;
        const int m0 = mt * TM, n0 = nt * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full[stage], HI_BYTES);
          const int k0 = (int)(kbeg + (int64_t)kb * TBK);
          if constexpr (A_MN) {
#pragma unroll
            for (int j = 0; j < TM / 32; ++j) tma_load_3d(sa + j * 4096, &tmA, &full[stage], m0 + 32 * j, k0, ba);
          } else {
            tma_load_3d(sa, &tmA, &full[stage], k0, m0, ba);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) tma_load_3d(sb + j * 4096, &tmB, &full[stage], n0 + 32 * j, k0, bb);
          } else {
            tma_load_3d(sb, &tmB, &full[stage], k0, n0, bb);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================= MMA issuer =============================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      int mt, nt, split, b, nkb;
      tcoords((uint32_t)t, p, mt, nt, split, b);
      krange(split, nkb);
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&conv[stage], phase);            // hi landed and lo converted
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * STAGE), sb = sa + A_BYTES;
        const uint32_t la = sa + HI_BYTES, lb = sb + HI_BYTES;
        const uint64_t ah = smem_desc(sa, 16, 1024), bh = smem_desc(sb, 16, 1024);   // K-major (converted)
        const uint64_t al = smem_desc(la, 16, 1024), bl = smem_desc(lb, 16, 1024);
#pragma unroll
        for (int k = 0; k < TBK / 8; ++k) {            // +32 B per 8-element k step
          tc_mma_tf32(d_tmem, ah + k * 2, bh + k * 2, IDESC, (kb | k) != 0 ? 1u : 0u);
          tc_mma_tf32(d_tmem, ah + k * 2, bl + k * 2, IDESC, 1u);
          tc_mma_tf32(d_tmem, al + k * 2, bh + k * 2, IDESC, 1u);
        }
        tc_commit_w(&empty[stage]);
        if (kb == nkb - 1) tc_commit_w(&tfull[acc]);
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (nkb == 0 && lane == 0) mbar_arrive(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp < 2 + T_NCONV) {
    // ======================== lo = x - trunc_tf32(x) ========================
    // K-major tiles: hi = the TMA'd tile itself, lo written to the lo slot.
    // MN-major tiles (kind::tf32 reads MN-major only in a 32-B-atom swizzle
    // TMA does not produce here): the converter transposes them in place into
    // the K-major SWIZZLE_128B layout -- all 32 k of a row are read into
    // registers (column reads, conflict-free), a named barrier, then row
    // writes of hi (in place) and lo -- so the MMAs always see K-major tiles.
    const int ct = threadIdx.x - 64;               // 0 .. 127
    int stage = 0;
    uint32_t phase = 0;
    auto lo_of = [](uint32_t x) { return __float_as_uint(__uint_as_float(x) - __uint_as_float(x & 0xFFFFE000u)); };
    auto kmajor_lo = [&](uint32_t base, uint32_t bytes) {
#pragma unroll 4
      for (uint32_t c = (uint32_t)ct; c < bytes / 16; c += T_NCONV * 32) {
        const uint4 v = ld_shared_u4(base + c * 16);
        st_shared_v4(base + HI_BYTES + c * 16, make_uint4(lo_of(v.x), lo_of(v.y), lo_of(v.z), lo_of(v.w)));
      }
    };
    // MN-major tile of `rows` MN entries x 32 k: chunk j (32 MN) at j*4096, k-row at k*128,
    // entry (mn, k) at ((mn%32)/4 ^ (k&7))*16 + (mn%4)*4  ->  K-major row mn: (k/4 ^ (mn&7))*16 + (k%4)*4
    auto mn_transpose = [&](uint32_t base, int rows) {
      uint32_t v[32];
      const bool mine = ct < rows;
      const int mn = ct;
      if (mine) {
        const uint32_t cb = base + (uint32_t)((mn >> 5) * 4096 + (mn & 3) * 4);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          uint32_t x;
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x) : "r"(cb + (uint32_t)(k * 128 + ((((mn & 31) >> 2) ^ (k & 7)) << 4))));
          v[k] = x;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(T_NCONV * 32) : "memory");
      if (mine) {
        const uint32_t rb = base + (uint32_t)(mn * 128);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = (uint32_t)((q ^ (mn & 7)) << 4);
          st_shared_v4(rb + off, make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
          st_shared_v4(rb + HI_BYTES + off,
                       make_uint4(lo_of(v[4 * q]), lo_of(v[4 * q + 1]), lo_of(v[4 * q + 2]), lo_of(v[4 * q + 3])));
        }
      }
    };
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      int mt, nt, split, b, nkb;
      tcoords((uint32_t)t, p, mt, nt, split, b);
      krange(split, nkb);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        const uint32_t sa = smem_u32(smem + stage * STAGE), sb = sa + A_BYTES;
        if constexpr (A_MN) mn_transpose(sa, TM); else kmajor_lo(sa, A_BYTES);
        if constexpr (B_MN) mn_transpose(sb, BN); else kmajor_lo(sb, B_BYTES);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ============================== epilogue ==============================
    const int ew = warp - 2 - T_NCONV;             // 0 .. 7
    const int quarter = warp & 3;
    const int half = ew >> 2;                      // two warps per lane quarter take alternate 32-column chunks
    float* my_bias = sbias + ew * BN;
    int acc = 0;
    uint32_t acc_phase = 0;
    int64_t cur_key = -1;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      int mt, nt, split, b;
      tcoords((uint32_t)t, p, mt, nt, split, b);
      const int64_t m = (int64_t)mt * TM + quarter * 32 + lane;
      const bool row_ok = m < p.M;
      const bool vbias = p.bias && p.bias_div == 0 && p.splits == 1;
      const int64_t key = (int64_t)b * p.tiles_n + nt;
      if (vbias && key != cur_key) {
        for (int jj = lane; jj < BN; jj += 32) {
          const int64_t n = (int64_t)nt * BN + jj;
          my_bias[jj] = n < p.N ? p.bias[(int64_t)b * p.bias_bs + n] : 0.f;
        }
        __syncwarp();
        cur_key = key;
      }
      const float* brow = (p.bias && p.bias_div > 0 && row_ok && p.splits == 1)
                              ? p.bias + (int64_t)b * p.bias_bs + (m / p.bias_div) * p.bias_ld : nullptr;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      constexpr int NCH = BN / 32;
      const int my_n = (NCH - half + 1) / 2;
      if (my_n == 0) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      for (int si = 0; si < my_n; ++si) {
        const int j = half + 2 * si;
        uint32_t u[32];
        tmem_ld32_nowait(tmem_base + (uint32_t)(acc * BN + j * 32) + ((uint32_t)(quarter * 32) << 16), u);
        tmem_wait_ld();
        if (si == my_n - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        const int64_t c0 = (int64_t)nt * BN + j * 32;
        if (!row_ok || c0 >= p.N) continue;
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(u[q]);
        if (vbias) {
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] += my_bias[j * 32 + q];
        } else if (brow) {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (c0 + q < p.N) v[q] += brow[c0 + q];
        }
        const bool full_chunk = c0 + 32 <= p.N;
        float* dst = p.splits > 1 ? p.part + (((int64_t)split * p.B + b) * p.M + m) * p.N + c0
                                  : p.C + (int64_t)b * p.c_bs + m * p.c_ld + c0;
        const bool vec_ok = full_chunk && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
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
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// 3-D fp32 map: dim0 = contiguous extent, dim1 = rows, dim2 = models
hfta_status make_map_f32(CUtensorMap* m, const void* ptr, int64_t inner, int64_t rows, int64_t ld, int64_t bs, int nb,
                         uint32_t box_inner, uint32_t box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)nb};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)((nb > 1 ? bs : rows * ld) * 4)};
  cuuint32_t box[3] = {box_inner, box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(HFTA_ERR_CUDA, "cuTensorMapEncodeTiled (fp32) failed (%d): dims %lld x %lld x %d, ld %lld", (int)r,
                (long long)inner, (long long)rows, nb, (long long)ld);
  return HFTA_OK;
}

template <bool A_MN, bool B_MN, int BN>
hfta_status launch_tf32(const GemmP& p, cudaStream_t s) {
  constexpr int STAGES = BN <= 64 ? 4 : 3;
  constexpr size_t SMEM = 1024 + (size_t)STAGES * 2 * (TM * TBK * 4 + BN * TBK * 4) + 256 + T_NEPI * BN * 4;
  static_assert(SMEM <= 232448, "shared memory budget");
  if (hfta_status st = get_encode()) return st;
  CUtensorMap ta, tb;
  const int nba = p.a_bs == 0 ? 1 : p.B, nbb = p.b_bs == 0 ? 1 : p.B;
  hfta_status st = A_MN ? make_map_f32(&ta, p.A, p.M, p.K, p.a_ld, p.a_bs, nba, 32, TBK)
                        : make_map_f32(&ta, p.A, p.K, p.M, p.a_ld, p.a_bs, nba, TBK, TM);
  if (st) return st;
  st = B_MN ? make_map_f32(&tb, p.Bm, p.N, p.K, p.b_ld, p.b_bs, nbb, 32, TBK)
            : make_map_f32(&tb, p.Bm, p.K, p.N, p.b_ld, p.b_bs, nbb, TBK, BN);
  if (st) return st;
  TfArgs a{};
  a.B = p.B; a.splits = std::max(p.splits, 1); a.M = p.M; a.N = p.N; a.K = p.K;
  a.k_chunk = p.splits > 1 ? p.k_chunk : p.K;
  a.a_shared = nba == 1 && p.B > 1; a.b_shared = nbb == 1 && p.B > 1;
  a.C = reinterpret_cast<float*>(p.C); a.c_bs = p.c_bs; a.c_ld = p.c_ld;
  a.bias = p.bias; a.bias_bs = p.bias_bs; a.bias_ld = p.bias_ld; a.bias_div = p.bias_div;
  a.accumulate = p.accumulate; a.part = p.part;
  a.tiles_m = (int)cdiv(p.M, TM); a.tiles_n = (int)cdiv(p.N, BN);
  a.order = (A_MN && B_MN) ? 1 : 0;
  auto kern = k_gemm_tf32x3<A_MN, B_MN, BN, STAGES>;
  ensure_smem(kern, SMEM);
  const int64_t total = (int64_t)a.tiles_m * a.tiles_n * a.splits * a.B;
  HFTA_REQUIRE(total < ((int64_t)1 << 31), HFTA_ERR_SHAPE, "gemm_tf32: %lld tiles exceed int32", (long long)total);
  const int grid = (int)std::min<int64_t>(total, num_sms());
  kern<<<grid, T_THREADS, SMEM, s>>>(ta, tb, a);
  count_launches(1);
  return post_launch(s, "gemm_tf32x3");
}

}  // namespace

bool gemm_tf32_supported(const GemmP& p) {
  if (p.scale || p.act != HFTA_ACT_NONE || p.mask || p.K2 > 0 || p.colsum) return false;
  if (p.K < 8 || p.N < 16 || p.M < 1) return false;
  if (!aligned16(p.A) || !aligned16(p.Bm)) return false;
  if (p.a_ld % 4 || p.b_ld % 4 || p.a_bs % 4 || p.b_bs % 4) return false;
  if (p.M > INT32_MAX || p.N > INT32_MAX || p.K > INT32_MAX) return false;
  if (p.splits > 1 && p.k_chunk % TBK) return false;
  return true;
}

hfta_status gemm_tf32(const GemmP& p, cudaStream_t s) {
  const bool amn = !p.a_kmajor, bmn = !p.b_kmajor;
  const bool small_n = p.N <= 64;
  if (!amn && !bmn) return small_n ? launch_tf32<false, false, 64>(p, s) : launch_tf32<false, false, 128>(p, s);
  if (!amn && bmn) return small_n ? launch_tf32<false, true, 64>(p, s) : launch_tf32<false, true, 128>(p, s);
  if (amn && bmn) return small_n ? launch_tf32<true, true, 64>(p, s) : launch_tf32<true, true, 128>(p, s);
  return launch_tf32<true, false, 128>(p, s);
}

}  // namespace hfta
