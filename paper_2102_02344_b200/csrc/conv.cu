// conv.cu -- fused Conv2d / ConvTranspose2d for B models (K3/K4/K5).
// App. B rows Conv2d and ConvT2d: B same-shape
// (de)convolutions fused into one launch, model index in the tile scheduler.
//
// Tensor-core paths (bf16), no patch matrix in HBM:
//  * k4 s2 p1 with 64-multiple channels: implicit GEMM on the tcgen05 engine
//    (gemm_tc.cu CONV modes) -- TMA gathers the stride-2 windows straight into
//    the swizzled shared-memory ring (Conv2d fwd, ConvT2d dgrad, both wgrads);
//    ConvT2d fwd and Conv2d dgrad run as 4 sub-pixel phases of dense 2x2
//    stride-1 convolutions whose epilogue interleaves the phase outputs.
//  * 1x1 input, stride 1, pad 0 (DCGAN t1) and a window covering the whole
//    input (D c5): the (de)convolution IS a dense GEMM in NHWC (no gather).
// Fallback (fp32, and the 8-channel image layers D c1 fwd/wgrad, G t5
// dgrad/wgrad): explicit patch matrix through the caller's workspace:
//   im2col : col[(n,sy,sx)][(ky,kx,c)] = img[n, sy*s-p+ky, sx*s-p+kx, c]   (0 outside)
//   col2im : img[n, by, bx, c] = sum_{ky,kx: sy=(by+p-ky)/s integral, in range} col[(n,sy,sx)][(ky,kx,c)]
// ("big" grid = conv input / convT output, "small" grid = conv output / convT input).
//   conv  fwd : Y  = im2col(X) W^T                       W [Co][(ky,kx,ci)]
//   conv  bwd : dW = dY^T im2col(X) ; dX = col2im(dY W)
//   convT fwd : Y  = col2im(X Wt^T)                      Wt [(ky,kx,co)][ci]
//   convT bwd : dWt = im2col(dY)^T X ; dX = im2col(dY) Wt
// col2im is a deterministic gather (no atomics).
#include "gemm.cuh"

namespace hfta {
void wgrad_split_rows(int B, int64_t rows, int64_t N, int64_t K, int* splits, int64_t* chunk, int bn = 128);
hfta_status colsum_impl(int B, int64_t rows, int64_t C, int64_t group, hfta_dtype dt, hfta_in X, float* S,
                        int64_t S_bstride, int accumulate, void* ws, size_t ws_bytes, cudaStream_t s);
size_t colsum_ws(int B, int64_t rows, int64_t C, int64_t group);

namespace {

struct Geo2 {
  int64_t N, Hb, Wb, Hs, Ws, C;   // big / small grids, channels of the gathered image
  int kh, kw, stride, pad;
};

template <typename T, int VEC>
__global__ void k_im2col(Geo2 g, const T* __restrict__ img, int64_t ibs, T* __restrict__ col, int64_t cbs) {
  const int b = blockIdx.y;
  const int64_t cv = g.C / VEC;
  const int64_t K = (int64_t)g.kh * g.kw * g.C;
  const int64_t total = g.N * g.Hs * g.Ws * g.kh * g.kw * cv;
  const T* I = img + (int64_t)b * ibs;
  T* O = col + (int64_t)b * cbs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t t = (uint32_t)i;                    // 32-bit index math (host guarantees total < 2^31)
    const int64_t c = (int64_t)(t % (uint32_t)cv) * VEC; t /= (uint32_t)cv;
    const int kx = (int)(t % (uint32_t)g.kw); t /= (uint32_t)g.kw;
    const int ky = (int)(t % (uint32_t)g.kh); t /= (uint32_t)g.kh;
    const int64_t m = t;                         // (n, sy, sx)
    const int sx = (int)(t % (uint32_t)g.Ws); t /= (uint32_t)g.Ws;
    const int sy = (int)(t % (uint32_t)g.Hs);
    const int64_t n = t / (uint32_t)g.Hs;
    const int by = sy * g.stride - g.pad + ky, bx = sx * g.stride - g.pad + kx;
    float v[VEC];
    if (by >= 0 && by < g.Hb && bx >= 0 && bx < g.Wb) {
      ld_vec<T, VEC>(I + ((n * g.Hb + by) * g.Wb + bx) * g.C + c, v);
    } else {
#pragma unroll
      for (int q = 0; q < VEC; ++q) v[q] = 0.f;
    }
    st_vec<T, VEC>(O + m * K + ((int64_t)ky * g.kw + kx) * g.C + c, v);
  }
}

template <typename T, int VEC>
__global__ void k_col2im(Geo2 g, const T* __restrict__ col, int64_t cbs, int64_t cld, T* __restrict__ img,
                         int64_t ibs) {
  const int b = blockIdx.y;
  const int64_t cv = g.C / VEC;
  const int64_t total = g.N * g.Hb * g.Wb * cv;
  const T* Cm = col + (int64_t)b * cbs;
  T* O = img + (int64_t)b * ibs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t t = (uint32_t)i;                    // 32-bit index math (host guarantees total < 2^31)
    const int64_t c = (int64_t)(t % (uint32_t)cv) * VEC; t /= (uint32_t)cv;
    const int bx = (int)(t % (uint32_t)g.Wb); t /= (uint32_t)g.Wb;
    const int by = (int)(t % (uint32_t)g.Hb);
    const int64_t n = t / (uint32_t)g.Hb;
    float acc[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc[q] = 0.f;
    // only the taps with (b + pad - k) % stride == 0 contribute: start at that
    // residue and step by the stride (same ascending order: deterministic)
    const int ky0 = (by + g.pad) % g.stride, kx0 = (bx + g.pad) % g.stride;
    for (int ky = ky0; ky < g.kh; ky += g.stride) {
      const int ty = by + g.pad - ky;
      if (ty < 0) break;                              // ty decreases with ky
      const int sy = ty / g.stride;
      if (sy >= g.Hs) continue;
      for (int kx = kx0; kx < g.kw; kx += g.stride) {
        const int tx = bx + g.pad - kx;
        if (tx < 0) break;
        const int sx = tx / g.stride;
        if (sx >= g.Ws) continue;
        float v[VEC];
        ld_vec<T, VEC>(Cm + ((n * g.Hs + sy) * g.Ws + sx) * cld + ((int64_t)ky * g.kw + kx) * g.C + c, v);
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] += v[q];
      }
    }
    st_vec<T, VEC>(O + ((n * g.Hb + by) * g.Wb + bx) * g.C + c, acc);
  }
}

template <typename T>
void launch_im2col(const Geo2& g, const void* img, int64_t ibs, void* col, int64_t cbs, int B, cudaStream_t s) {
  const int vec = (g.C % (16 / (int)sizeof(T)) == 0) ? 16 / (int)sizeof(T) : 1;
  int64_t total = g.N * g.Hs * g.Ws * g.kh * g.kw * (g.C / vec);
  dim3 grid((unsigned)std::min<int64_t>(cdiv(total, 256), 8192), B);
  if (vec == 8) k_im2col<T, 8><<<grid, 256, 0, s>>>(g, (const T*)img, ibs, (T*)col, cbs);
  else if (vec == 4) k_im2col<T, 4><<<grid, 256, 0, s>>>(g, (const T*)img, ibs, (T*)col, cbs);
  else k_im2col<T, 1><<<grid, 256, 0, s>>>(g, (const T*)img, ibs, (T*)col, cbs);
}

template <typename T>
void launch_col2im(const Geo2& g, const void* col, int64_t cbs, int64_t cld, void* img, int64_t ibs, int B,
                   cudaStream_t s) {
  const int vec = (g.C % (16 / (int)sizeof(T)) == 0 && cld % (16 / (int)sizeof(T)) == 0) ? 16 / (int)sizeof(T) : 1;
  int64_t total = g.N * g.Hb * g.Wb * (g.C / vec);
  dim3 grid((unsigned)std::min<int64_t>(cdiv(total, 256), 8192), B);
  if (vec == 8) k_col2im<T, 8><<<grid, 256, 0, s>>>(g, (const T*)col, cbs, cld, (T*)img, ibs);
  else if (vec == 4) k_col2im<T, 4><<<grid, 256, 0, s>>>(g, (const T*)col, cbs, cld, (T*)img, ibs);
  else k_col2im<T, 1><<<grid, 256, 0, s>>>(g, (const T*)col, cbs, cld, (T*)img, ibs);
}

void im2col(hfta_dtype dt, const Geo2& g, const void* img, int64_t ibs, void* col, int64_t cbs, int B,
            cudaStream_t s) {
  if (dt == HFTA_F32) launch_im2col<float>(g, img, ibs, col, cbs, B, s);
  else launch_im2col<__nv_bfloat16>(g, img, ibs, col, cbs, B, s);
  count_launches(1);
}
void col2im(hfta_dtype dt, const Geo2& g, const void* col, int64_t cbs, int64_t cld, void* img, int64_t ibs, int B,
            cudaStream_t s) {
  if (dt == HFTA_F32) launch_col2im<float>(g, col, cbs, cld, img, ibs, B, s);
  else launch_col2im<__nv_bfloat16>(g, col, cbs, cld, img, ibs, B, s);
  count_launches(1);
}

// Shape bookkeeping of one (de)convolution.
struct Shape {
  Geo2 g;             // gather geometry
  int64_t Ho, Wo;     // output spatial dims
  int64_t Ms;         // small-grid rows N*Hs*Ws (GEMM M)
  int64_t Kc;         // im2col width kh*kw*C (C = gathered image channels)
  int64_t Ci, Co;
  bool transposed;
};

hfta_status make_shape(const hfta_conv_desc* d, Shape* sh) {
  HFTA_REQUIRE(d, HFTA_ERR_INVALID_VALUE, "conv: desc is NULL");
  HFTA_REQUIRE(d->N >= 1 && d->H >= 1 && d->W >= 1 && d->C_in >= 1 && d->C_out >= 1 && d->kh >= 1 && d->kw >= 1 &&
                   d->stride >= 1 && d->pad >= 0,
               HFTA_ERR_SHAPE, "conv: bad descriptor (N %d H %d W %d Ci %d Co %d k %dx%d s %d p %d)", d->N, d->H, d->W,
               d->C_in, d->C_out, d->kh, d->kw, d->stride, d->pad);
  Shape s{};
  s.Ci = d->C_in; s.Co = d->C_out; s.transposed = d->transposed != 0;
  if (!s.transposed) {
    s.Ho = ((int64_t)d->H + 2 * d->pad - d->kh) / d->stride + 1;
    s.Wo = ((int64_t)d->W + 2 * d->pad - d->kw) / d->stride + 1;
    HFTA_REQUIRE(s.Ho >= 1 && s.Wo >= 1, HFTA_ERR_SHAPE, "conv: empty output");
    s.g = Geo2{d->N, d->H, d->W, s.Ho, s.Wo, d->C_in, d->kh, d->kw, d->stride, d->pad};
    s.Kc = (int64_t)d->kh * d->kw * d->C_in;
  } else {
    s.Ho = ((int64_t)d->H - 1) * d->stride - 2 * d->pad + d->kh;
    s.Wo = ((int64_t)d->W - 1) * d->stride - 2 * d->pad + d->kw;
    HFTA_REQUIRE(s.Ho >= 1 && s.Wo >= 1, HFTA_ERR_SHAPE, "convT: empty output");
    s.g = Geo2{d->N, s.Ho, s.Wo, d->H, d->W, d->C_out, d->kh, d->kw, d->stride, d->pad};
    s.Kc = (int64_t)d->kh * d->kw * d->C_out;
  }
  s.Ms = (int64_t)d->N * s.g.Hs * s.g.Ws;
  // im2col / col2im index arithmetic is 32-bit per model
  HFTA_REQUIRE(s.Ms * s.Kc < ((int64_t)1 << 31) && (int64_t)d->N * s.g.Hb * s.g.Wb * s.g.C < ((int64_t)1 << 31),
               HFTA_ERR_SHAPE, "conv: %lld x %lld patch matrix per model exceeds 2^31 elements", (long long)s.Ms,
               (long long)s.Kc);
  *sh = s;
  return HFTA_OK;
}

bool k4s2p1(const hfta_conv_desc* d) { return d->kh == 4 && d->kw == 4 && d->stride == 2 && d->pad == 1; }
// Conv2d (not transposed) the gather modes take: square kernel, stride 1 or 2
bool gather_conv(const hfta_conv_desc* d) {
  return !d->transposed && d->kh == d->kw && (d->stride == 1 || d->stride == 2) && d->kh <= 15;
}
bool tc_geometry(const hfta_conv_desc* d) { return k4s2p1(d) || gather_conv(d); }

// 1x1 input, stride 1, pad 0 (ConvT) / window = whole input, pad 0 (Conv): a dense GEMM in NHWC
bool dense_convT(const hfta_conv_desc* d) { return d->transposed && d->H == 1 && d->W == 1 && d->stride == 1 && d->pad == 0; }
bool dense_conv(const hfta_conv_desc* d) { return !d->transposed && d->kh == d->H && d->kw == d->W && d->pad == 0; }

// dense model-major NHWC image operand: elements per model
int64_t img_elems(int N, int64_t H, int64_t W, int64_t C) { return (int64_t)N * H * W * C; }

ConvTcP img_op(int B, const void* ptr, int64_t bs, int N, int H, int W, int C) {
  ConvTcP p{};
  p.B = B; p.img = ptr; p.img_bs = bs; p.img_n = N; p.img_h = H; p.img_w = W; p.img_c = C;
  return p;
}

// Implicit-GEMM descriptors of the three contractions of a k4 s2 p1 layer
// (model strides: x_bs / y_bs / w_bs; dense NHWC images).
ConvTcP fwd_cp(int B, const hfta_conv_desc* d, const Shape& sh, const void* X, int64_t x_bs, const void* W,
               int64_t w_bs, int64_t w_ld, void* Y, int64_t y_bs) {
  ConvTcP cp = img_op(B, X, x_bs, d->N, d->H, d->W, d->C_in);
  cp.opd = W; cp.opd_bs = w_bs;
  const int64_t ye = img_elems(d->N, sh.Ho, sh.Wo, d->C_out);
  if (!sh.transposed) {          // strided gather of X
    cp.mode = 1; cp.M = (int64_t)d->N * sh.Ho * sh.Wo; cp.N = d->C_out;
    cp.K = (int64_t)d->kh * d->kw * d->C_in;
    cp.ks = d->kh; cp.cs = d->stride; cp.cpad = d->pad;
    cp.grid_w = (int)sh.Wo; cp.grid_h = (int)sh.Ho; cp.opd_ld = w_ld;
    cp.C = Y; cp.c_bs = y_bs; cp.c_ld = d->C_out;
  } else {                       // 4 sub-pixel phases of X against the ConvT taps
    cp.mode = 2; cp.M = (int64_t)d->N * d->H * d->W; cp.N = d->C_out; cp.K = 4 * (int64_t)d->C_in;
    cp.grid_w = d->W; cp.grid_h = d->H; cp.w_mn = 0; cp.w_cn = d->C_out; cp.w_ca = d->C_in;
    cp.C = Y; cp.c_bs = B > 1 ? y_bs : ye; cp.y_h = (int)sh.Ho; cp.y_w = (int)sh.Wo;
  }
  return cp;
}
ConvTcP wgrad_cp(int B, const hfta_conv_desc* d, const Shape& sh, const void* dY, int64_t dy_bs, const void* X,
                 int64_t x_bs) {
  ConvTcP cp;
  if (!sh.transposed) {          // dW[co][(kh,kw,ci)] = sum_(n,oy,ox) dY (x) strided gather of X
    cp = img_op(B, X, x_bs, d->N, d->H, d->W, d->C_in);
    cp.mode = 3; cp.M = d->C_out; cp.N = (int64_t)d->kh * d->kw * d->C_in;
    cp.ks = d->kh; cp.cs = d->stride; cp.cpad = d->pad;
    cp.grid_w = (int)sh.Wo; cp.grid_h = (int)sh.Ho;
    cp.opd = dY; cp.opd_bs = dy_bs; cp.opd_ld = d->C_out;
    cp.K = (int64_t)d->N * sh.Ho * sh.Wo;
  } else {                       // dWt[(kh,kw,co)][ci] = sum_(n,i,j) stride-2 gather of dY (x) X
    cp = img_op(B, dY, dy_bs, d->N, (int)sh.Ho, (int)sh.Wo, d->C_out);
    cp.mode = 4; cp.M = 16 * (int64_t)d->C_out; cp.N = d->C_in;
    cp.grid_w = d->W; cp.grid_h = d->H;
    cp.opd = X; cp.opd_bs = x_bs; cp.opd_ld = d->C_in;
    cp.K = (int64_t)d->N * d->H * d->W;
  }
  return cp;
}
ConvTcP dgrad_cp(int B, const hfta_conv_desc* d, const Shape& sh, const void* dY, int64_t dy_bs, const void* W,
                 int64_t w_bs, int64_t w_ld, void* dX, int64_t dx_bs) {
  ConvTcP cp = img_op(B, dY, dy_bs, d->N, (int)sh.Ho, (int)sh.Wo, d->C_out);
  cp.opd = W; cp.opd_bs = w_bs;
  const int64_t xe = img_elems(d->N, d->H, d->W, d->C_in);
  if (!sh.transposed && d->stride == 1) {
    // stride 1: dX = Conv2d(dY, W flipped and transposed) with pad k-1-p -- the
    // gather mode over dY, B read from W [Co][taps][Ci] at the flipped tap
    cp.mode = 1; cp.M = (int64_t)d->N * d->H * d->W; cp.N = d->C_in; cp.K = (int64_t)d->kh * d->kw * d->C_out;
    cp.ks = d->kh; cp.cs = 1; cp.cpad = d->kh - 1 - d->pad;
    cp.w_mn = 1; cp.wflip = 1; cp.w_cn = d->C_in; cp.w_ca = d->C_out;
    cp.grid_w = d->W; cp.grid_h = d->H; cp.opd_ld = w_ld;
    cp.C = dX; cp.c_bs = B > 1 ? dx_bs : xe; cp.c_ld = d->C_in;
  } else if (!sh.transposed && !k4s2p1(d)) {
    cp.mode = 0;                 // other strided Conv2d dgrads: the patch-matrix path
  } else if (!sh.transposed) {   // 4 sub-pixel phases of dY against the (adjoint) Conv taps
    cp.mode = 2; cp.M = (int64_t)d->N * sh.Ho * sh.Wo; cp.N = d->C_in; cp.K = 4 * (int64_t)d->C_out;
    cp.grid_w = (int)sh.Wo; cp.grid_h = (int)sh.Ho; cp.w_mn = 1; cp.w_cn = d->C_in; cp.w_ca = d->C_out;
    cp.C = dX; cp.c_bs = B > 1 ? dx_bs : xe; cp.y_h = d->H; cp.y_w = d->W;
  } else {                       // Conv2d(dY, Wt): stride-2 gather of dY, B = Wt MN-major
    cp.mode = 1; cp.w_mn = 1; cp.M = (int64_t)d->N * d->H * d->W; cp.N = d->C_in; cp.K = 16 * (int64_t)d->C_out;
    cp.grid_w = d->W; cp.grid_h = d->H; cp.opd_ld = w_ld;
    cp.C = dX; cp.c_bs = dx_bs; cp.c_ld = d->C_in;
  }
  return cp;
}

// Which contractions of the layer the implicit-GEMM path takes for dense,
// aligned, model-major operands (the runtime re-checks the real pointers).
void plan(int B, const hfta_conv_desc* d, hfta_dtype dt, const Shape& sh, bool& f, bool& g, bool& w) {
  f = g = w = false;
  if (dt != HFTA_BF16 || !tc_geometry(d)) return;
  char* a = reinterpret_cast<char*>(256);       // any 16-B aligned address: only eligibility is evaluated
  const int64_t xe = img_elems(d->N, d->H, d->W, d->C_in), ye = img_elems(d->N, sh.Ho, sh.Wo, d->C_out);
  const int64_t we = (int64_t)d->kh * d->kw * d->C_in * d->C_out;
  const int64_t wld = sh.transposed ? d->C_in : (int64_t)d->kh * d->kw * d->C_in;
  f = conv_tc_supported(fwd_cp(B, d, sh, a, xe, a, we, wld, a, ye));
  g = conv_tc_supported(dgrad_cp(B, d, sh, a, ye, a, we, wld, a, xe));
  w = conv_tc_supported(wgrad_cp(B, d, sh, a, ye, a, xe));
}

// the explicit patch matrix only where a fallback path runs: fp32, or an
// 8-channel image on the gathered side (D c1 fwd / wgrad, G t5 dgrad / wgrad)
size_t col_bytes(int B, const hfta_conv_desc* d, hfta_dtype dt, const Shape& sh) {
  if (dense_conv(d) || dense_convT(d)) return 0;
  bool f, g, w;
  plan(B, d, dt, sh, f, g, w);
  return (f && g && w) ? 0 : align_up((size_t)B * sh.Ms * sh.Kc * dsize(dt), 256);
}

// Mode 5 (phase-merged sub-pixel GEMM) for a mode-2 contraction with 8
// output channels (G t5 fwd, D c1 dgrad): the 4 phases x 8 channels fill one
// 32-wide tile instead of four 8-of-64-wide ones.  Its weight operand is
// rebuilt per call into the workspace.
bool merged_phases(const ConvTcP& cp) { return cp.mode == 2 && cp.w_cn == 8 && cp.w_ca % 64 == 0; }
size_t merged_w_bytes(int B, const ConvTcP& cp) {
  return merged_phases(cp) ? align_up((size_t)(cp.opd_bs == 0 ? 1 : B) * 32 * 9 * cp.w_ca * 2, 256) : 0;
}
ConvTcP as_merged(const ConvTcP& cp, void* wp) {
  ConvTcP m = cp;
  m.mode = 5; m.N = 32; m.K = 9 * (int64_t)cp.w_ca;
  m.opd = wp; m.opd_ld = m.K; m.opd_bs = cp.opd_bs == 0 ? 0 : 32 * m.K;
  return m;
}
// run a mode-2 contraction, merged when eligible (wp: >= merged_w_bytes of workspace)
// *gated: whether the kernel applied cp.gate (mode 2 only; the merged mode does not)
hfta_status run_phases(const ConvTcP& cp, void* wp, size_t wpb, cudaStream_t s, bool* gated = nullptr) {
  if (gated) *gated = false;
  if (merged_phases(cp) && wp && wpb >= merged_w_bytes(cp.B, cp)) {
    ConvTcP m = as_merged(cp, wp);
    m.gate = nullptr;
    if (conv_tc_supported(m)) {
      if (hfta_status st = conv_subpixel_weights(cp.B, cp.w_ca, cp.w_mn, cp.opd, cp.opd_bs, wp, s)) return st;
      return conv_tc(m, s);
    }
  }
  if (gated) *gated = cp.mode == 2 && cp.gate != nullptr;
  return conv_tc(cp, s);
}

// split-K partials of a tensor-core conv wgrad (modes 3, 4)
size_t conv_wgrad_part(int B, int64_t rows, int64_t M, int64_t N) {
  size_t r = 0;
  for (int bn : {128, 256}) {            // either tile width conv_wgrad_bn picks
    int sp; int64_t ch;
    wgrad_split_rows(B, rows, M, N, &sp, &ch, bn);
    r = std::max(r, sp > 1 ? (size_t)sp * B * M * N * sizeof(float) : (size_t)0);
  }
  return r;
}

hfta_status conv_wgrad_tc(ConvTcP& cp, int64_t rows, float* dW, int64_t dW_bstride, int64_t ld, int accumulate,
                          char* lws, size_t lwsb, cudaStream_t s) {
  int sp; int64_t ch;
  wgrad_split_rows(cp.B, rows, cp.M, cp.N, &sp, &ch, conv_wgrad_bn(cp));
  cp.K = rows; cp.splits = sp; cp.k_chunk = ch;
  cp.C = dW; cp.c_bs = dW_bstride; cp.c_ld = ld; cp.accumulate = accumulate;
  cp.part = nullptr;
  if (sp > 1) {
    HFTA_REQUIRE(lwsb >= (size_t)sp * cp.B * cp.M * cp.N * sizeof(float), HFTA_ERR_WORKSPACE,
                 "conv wgrad: split-K workspace too small");
    cp.part = reinterpret_cast<float*>(lws);
  }
  if (hfta_status st = conv_tc(cp, s)) return st;
  if (sp > 1) {
    GemmP g{};
    g.B = cp.B; g.M = cp.M; g.N = cp.N; g.splits = sp; g.part = cp.part; g.C = dW; g.c_bs = dW_bstride;
    g.c_ld = ld; g.accumulate = accumulate;
    if (hfta_status st = splitk_reduce(g, s)) return st;
  }
  return HFTA_OK;
}

}  // namespace
}  // namespace hfta

using namespace hfta;

extern "C" {

size_t hfta_fused_conv_workspace(int B, const hfta_conv_desc* d, hfta_dtype dt) {
  Shape sh;
  if (B < 1 || make_shape(d, &sh) != HFTA_OK) return 0;
  const size_t col = col_bytes(B, d, dt, sh);
  // weight-gradient GEMM (split-K partials) of either orientation
  const int64_t M = sh.Ms;
  size_t lin = std::max(hfta_fused_linear_bwd_workspace(B, M, sh.Co, sh.Kc, dt),
                        hfta_fused_linear_bwd_workspace(B, M, sh.Kc, sh.Ci, dt));
  lin = std::max(lin, std::max(conv_wgrad_part(B, M, sh.Co, sh.Kc), conv_wgrad_part(B, M, sh.Kc, sh.Ci)));
  if (dt == HFTA_BF16 && k4s2p1(d)) {          // phase-merged weights (fwd of a ConvT, dgrad of a Conv)
    char* a = reinterpret_cast<char*>(256);
    const int64_t xe = img_elems(d->N, d->H, d->W, d->C_in), ye = img_elems(d->N, sh.Ho, sh.Wo, d->C_out);
    const int64_t we = (int64_t)d->kh * d->kw * d->C_in * d->C_out;
    const int64_t wld = sh.transposed ? d->C_in : (int64_t)d->kh * d->kw * d->C_in;
    lin = std::max(lin, merged_w_bytes(B, fwd_cp(B, d, sh, a, xe, a, we, wld, a, ye)));
    lin = std::max(lin, merged_w_bytes(B, dgrad_cp(B, d, sh, a, ye, a, we, wld, a, xe)));
  }
  return col + align_up(lin, 256);
}

static hfta_status conv_fwd_impl(int B, const hfta_conv_desc* d, hfta_dtype dt, hfta_in X, hfta_in W, hfta_out Y,
                                 hfta_act act, float act_alpha, float* colstat, void* ws, size_t ws_bytes,
                                 hfta_stream stream);

hfta_status hfta_fused_conv_fwd(int B, const hfta_conv_desc* d, hfta_dtype dt, hfta_in X, hfta_in W, hfta_out Y,
                                hfta_act act, float act_alpha, void* ws, size_t ws_bytes, hfta_stream stream) {
  return conv_fwd_impl(B, d, dt, X, W, Y, act, act_alpha, nullptr, ws, ws_bytes, stream);
}

hfta_status hfta_fused_conv_fwd_stats(int B, const hfta_conv_desc* d, hfta_dtype dt, hfta_in X, hfta_in W,
                                      hfta_out Y, float* colstat, void* ws, size_t ws_bytes, hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_REQUIRE(colstat, HFTA_ERR_INVALID_VALUE, "conv_fwd_stats: colstat is required");
  return conv_fwd_impl(B, d, dt, X, W, Y, HFTA_ACT_NONE, 0.f, colstat, ws, ws_bytes, stream);
}

static hfta_status conv_fwd_impl(int B, const hfta_conv_desc* d, hfta_dtype dt, hfta_in X, hfta_in W, hfta_out Y,
                                 hfta_act act, float act_alpha, float* colstat, void* ws, size_t ws_bytes,
                                 hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_CHECK_B(B);
  Shape sh;
  if (hfta_status st = make_shape(d, &sh)) return st;
  HFTA_REQUIRE(X.ptr && W.ptr && Y.ptr && (Y.bstride > 0 || B == 1), HFTA_ERR_INVALID_VALUE, "conv_fwd: bad args");
  size_t need = hfta_fused_conv_workspace(B, d, dt);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "conv_fwd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  char* col = reinterpret_cast<char*>(ws);
  GemmP p{};
  p.B = B; p.splits = 1;
  HFTA_REQUIRE(X.ld == d->C_in && Y.ld == d->C_out, HFTA_ERR_SHAPE,
               "conv_fwd: images must be dense NHWC (X.ld %lld vs C_in %d, Y.ld %lld vs C_out %d)", (long long)X.ld,
               d->C_in, (long long)Y.ld, d->C_out);
  const int64_t xe = img_elems(d->N, d->H, d->W, d->C_in), ye = img_elems(d->N, sh.Ho, sh.Wo, d->C_out);
  HFTA_REQUIRE(act == HFTA_ACT_NONE || act == HFTA_ACT_LEAKY_RELU || act == HFTA_ACT_TANH || act == HFTA_ACT_RELU,
               HFTA_ERR_UNSUPPORTED, "conv_fwd: activation %d", (int)act);
  if (dt == HFTA_BF16 && tc_geometry(d) && (X.bstride == 0 || X.bstride == xe) && (Y.bstride == ye || B == 1) &&
      act != HFTA_ACT_RELU) {
    ConvTcP cp = fwd_cp(B, d, sh, X.ptr, X.bstride, W.ptr, W.bstride, W.ld, Y.ptr, Y.bstride);
    cp.act = act; cp.act_alpha = act_alpha;      // fused into the epilogue
    if (conv_tc_supported(cp)) {
      const size_t colb = col_bytes(B, d, dt, sh);
      // statistics from the epilogue: Conv2d (TMA store) and the sub-pixel phases (4 phases x M/32
      // blocks = the output's 32-row blocks when M % 32 == 0; not the merged 8-channel mode)
      const bool epi_stats = cp.mode == 1 || (cp.mode == 2 && cp.M % 32 == 0 && !merged_phases(cp));
      if (epi_stats) cp.colstat = colstat;
      if (hfta_status st = run_phases(cp, col + colb, ws_bytes - colb, s)) return st;
      if (colstat && !epi_stats)
        if (hfta_status st = colstat_rows(B, (int64_t)d->N * sh.Ho * sh.Wo, d->C_out, dt,
                                          hfta_in{Y.ptr, Y.bstride, Y.ld}, colstat, s))
          return st;
      return post_launch(s, "hfta_fused_conv_fwd");
    }
  }
  // other paths: the activation as a separate in-place pass at the end
  const auto finish = [&]() -> hfta_status {
    if (act != HFTA_ACT_NONE)
      if (hfta_status st = hfta_act_fwd(B, (int64_t)d->N * sh.Ho * sh.Wo, d->C_out, dt, act, act_alpha,
                                        hfta_in{Y.ptr, Y.bstride, Y.ld}, Y, stream))
        return st;
    if (colstat)          // statistics of the stored Y (the paths without the epilogue statistics)
      if (hfta_status st = colstat_rows(B, (int64_t)d->N * sh.Ho * sh.Wo, d->C_out, dt,
                                        hfta_in{Y.ptr, Y.bstride, Y.ld}, colstat, s))
        return st;
    return post_launch(s, "hfta_fused_conv_fwd");
  };
  if (dense_convT(d) || dense_conv(d)) {
    // t1: Y[n][(kh,kw,co)] = X[n] Wt^T ; c5: Y[n][co] = X[n][(h,w,ci)] W^T -- plain GEMMs in NHWC
    p.M = d->N; p.N = dense_convT(d) ? sh.Kc : d->C_out; p.K = dense_convT(d) ? d->C_in : sh.Kc;
    p.A = X.ptr; p.a_bs = X.bstride; p.a_ld = p.K; p.a_kmajor = 1;
    p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 1;
    p.C = Y.ptr; p.c_bs = Y.bstride; p.c_ld = p.N;
    p.k_chunk = p.K;
    if (hfta_status st = run_gemm(p, dt, false, s)) return st;
    return finish();
  }
  HFTA_REQUIRE(col_bytes(B, d, dt, sh) > 0, HFTA_ERR_UNSUPPORTED, "conv_fwd: operands not eligible for the "
               "implicit-GEMM path (alignment / model strides) and no patch-matrix workspace for this configuration");
  if (!sh.transposed) {
    // Y[(n,oy,ox)][co] = im2col(X) W^T ; a shared input image gives a shared col (bstride 0)
    const int nb = X.bstride == 0 ? 1 : B;
    im2col(dt, sh.g, X.ptr, X.bstride, col, sh.Ms * sh.Kc, nb, s);
    p.M = sh.Ms; p.N = sh.Co; p.K = sh.Kc;
    p.A = col; p.a_bs = X.bstride == 0 ? 0 : sh.Ms * sh.Kc; p.a_ld = sh.Kc; p.a_kmajor = 1;
    p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 1;
    p.C = Y.ptr; p.c_bs = Y.bstride; p.c_ld = Y.ld;
    p.k_chunk = sh.Kc;
    if (hfta_status st = run_gemm(p, dt, false, s)) return st;
  } else {
    // col[(n,iy,ix)][(ky,kx,co)] = X Wt^T, then Y = col2im(col)
    p.M = sh.Ms; p.N = sh.Kc; p.K = sh.Ci;
    p.A = X.ptr; p.a_bs = X.bstride; p.a_ld = X.ld; p.a_kmajor = 1;
    p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 1;
    p.C = col; p.c_bs = sh.Ms * sh.Kc; p.c_ld = sh.Kc;
    p.k_chunk = sh.Ci;
    if (hfta_status st = run_gemm(p, dt, false, s)) return st;
    col2im(dt, sh.g, col, sh.Ms * sh.Kc, sh.Kc, Y.ptr, Y.bstride, B, s);
  }
  return finish();
}

hfta_status hfta_fused_conv_bwd(int B, const hfta_conv_desc* d, hfta_dtype dt, hfta_in dY, hfta_in X, hfta_in W,
                                hfta_out dX, float* dW, int64_t dW_bstride, int accumulate, void* ws, size_t ws_bytes,
                                hfta_stream stream) {
  return hfta_fused_conv_bwd_gated(B, d, dt, dY, X, W, dX, dW, dW_bstride, accumulate, HFTA_ACT_NONE, 0.f,
                                   hfta_in{nullptr, 0, 1}, ws, ws_bytes, stream);
}

hfta_status hfta_fused_conv_bwd_gated(int B, const hfta_conv_desc* d, hfta_dtype dt, hfta_in dY, hfta_in X,
                                      hfta_in W, hfta_out dX, float* dW, int64_t dW_bstride, int accumulate,
                                      hfta_act dX_act, float dX_alpha, hfta_in dX_gate, void* ws, size_t ws_bytes,
                                      hfta_stream stream) {
  if (hfta_status st = check_init()) return st;
  HFTA_REQUIRE(dX_act == HFTA_ACT_NONE || dX_act == HFTA_ACT_RELU || dX_act == HFTA_ACT_LEAKY_RELU,
               HFTA_ERR_UNSUPPORTED, "conv_bwd: dX activation %d (ReLU / LeakyReLU gates only)", (int)dX_act);
  HFTA_REQUIRE(dX_act == HFTA_ACT_NONE || (dX.ptr && dX_gate.ptr && dX_gate.ld == d->C_in), HFTA_ERR_INVALID_VALUE,
               "conv_bwd: a dX activation needs dX and a dense gate tensor (ld == C_in)");
  // the activation backward of the layer that consumed X, applied to dX: in the
  // sub-pixel dgrad epilogue when that path runs, else as one pass at the end
  bool gate_done = dX_act == HFTA_ACT_NONE;
  const auto finish = [&]() -> hfta_status {
    if (!gate_done)
      if (hfta_status st = hfta_act_bwd(B, (int64_t)d->N * d->H * d->W, d->C_in, dt, dX_act, dX_alpha, dX_gate,
                                        hfta_in{dX.ptr, dX.bstride, dX.ld}, dX, stream))
        return st;
    return post_launch((cudaStream_t)stream, "hfta_fused_conv_bwd");
  };
  HFTA_CHECK_B(B);
  Shape sh;
  if (hfta_status st = make_shape(d, &sh)) return st;
  HFTA_REQUIRE(dY.ptr && X.ptr && W.ptr, HFTA_ERR_INVALID_VALUE, "conv_bwd: dY, X, W are required");
  size_t need = hfta_fused_conv_workspace(B, d, dt);
  HFTA_REQUIRE(ws && ws_bytes >= need, HFTA_ERR_WORKSPACE, "conv_bwd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  char* col = reinterpret_cast<char*>(ws);
  const size_t colb = col_bytes(B, d, dt, sh);
  char* lws = col + colb;
  const size_t lwsb = ws_bytes - colb;
  HFTA_REQUIRE(dY.ld == d->C_out && X.ld == d->C_in && (!dX.ptr || dX.ld == d->C_in), HFTA_ERR_SHAPE,
               "conv_bwd: images must be dense NHWC (dY.ld %lld, X.ld %lld, dX.ld %lld; C_in %d, C_out %d)",
               (long long)dY.ld, (long long)X.ld, (long long)dX.ld, d->C_in, d->C_out);
  const int64_t xe = img_elems(d->N, d->H, d->W, d->C_in), ye = img_elems(d->N, sh.Ho, sh.Wo, d->C_out);
  if (dense_convT(d) || dense_conv(d)) {
    // t1 / c5 are plain Linear layers in NHWC: dgrad + wgrad of the GEMM
    const int64_t Mg = d->N, Ng = dense_convT(d) ? sh.Kc : d->C_out, Kg = dense_convT(d) ? d->C_in : sh.Kc;
    if (hfta_status st = hfta_fused_linear_bwd(B, Mg, Ng, Kg, dt, hfta_in{dY.ptr, dY.bstride, Ng},
                                               hfta_in{X.ptr, X.bstride, Kg}, W,
                                               dX.ptr ? hfta_out{dX.ptr, dX.bstride, Kg} : hfta_out{nullptr, 0, 1}, dW,
                                               dW_bstride, Kg, nullptr, 0, accumulate, lws, lwsb, stream))
      return st;
    return finish();
  }
  const bool tc = dt == HFTA_BF16 && tc_geometry(d) && (X.bstride == 0 || X.bstride == xe) &&
                  (dY.bstride == ye || B == 1) && (!dX.ptr || dX.bstride == xe || B == 1);
  bool need_dW = dW != nullptr, need_dX = dX.ptr != nullptr;
  if (tc && need_dW) {
    ConvTcP cp = wgrad_cp(B, d, sh, dY.ptr, dY.bstride, X.ptr, X.bstride);
    if (conv_tc_supported(cp)) {
      if (hfta_status st = conv_wgrad_tc(cp, cp.K, dW, dW_bstride, cp.N, accumulate, lws, lwsb, s)) return st;
      need_dW = false;
    }
  }
  if (tc && need_dX) {
    ConvTcP cp = dgrad_cp(B, d, sh, dY.ptr, dY.bstride, W.ptr, W.bstride, W.ld, dX.ptr, dX.bstride);
    if (!gate_done && dX_gate.bstride == xe) {
      cp.gate = dX_gate.ptr; cp.gate_bs = dX_gate.bstride;
      cp.gate_alpha = dX_act == HFTA_ACT_LEAKY_RELU ? dX_alpha : 0.f;
    }
    if (conv_tc_supported(cp)) {
      bool gated = false;
      if (hfta_status st = run_phases(cp, lws, lwsb, s, &gated)) return st;     // after the wgrad's use of lws
      gate_done = gate_done || gated;
      need_dX = false;
    }
  }
  if (!need_dW && !need_dX) return finish();
  HFTA_REQUIRE(colb > 0, HFTA_ERR_UNSUPPORTED, "conv_bwd: operands not eligible for the implicit-GEMM path "
               "(alignment / model strides) and no patch-matrix workspace for this configuration");
  if (!need_dW) dW = nullptr;
  if (!need_dX) dX.ptr = nullptr;
  if (!sh.transposed) {
    const int nb = X.bstride == 0 ? 1 : B;
    const int64_t cbs = X.bstride == 0 ? 0 : sh.Ms * sh.Kc;
    if (dW) {
      im2col(dt, sh.g, X.ptr, X.bstride, col, sh.Ms * sh.Kc, nb, s);
      // dW[co][k] = sum_m dY[m][co] col[m][k]
      if (hfta_status st = hfta_fused_linear_bwd(B, sh.Ms, sh.Co, sh.Kc, dt, dY, hfta_in{col, cbs, sh.Kc},
                                                 W, hfta_out{nullptr, 0, 1}, dW, dW_bstride, sh.Kc, nullptr, 0,
                                                 accumulate, lws, lwsb, stream))
        return st;
    }
    if (dX.ptr) {
      // dcol[m][k] = sum_co dY[m][co] W[co][k] ; dX = col2im(dcol)
      GemmP p{};
      p.B = B; p.splits = 1; p.M = sh.Ms; p.N = sh.Kc; p.K = sh.Co; p.k_chunk = sh.Co;
      p.A = dY.ptr; p.a_bs = dY.bstride; p.a_ld = dY.ld; p.a_kmajor = 1;
      p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 0;
      p.C = col; p.c_bs = sh.Ms * sh.Kc; p.c_ld = sh.Kc;
      if (hfta_status st = run_gemm(p, dt, false, s)) return st;
      col2im(dt, sh.g, col, sh.Ms * sh.Kc, sh.Kc, dX.ptr, dX.bstride, B, s);
    }
  } else {
    // dcol = im2col(dY) over the input grid
    im2col(dt, sh.g, dY.ptr, dY.bstride, col, sh.Ms * sh.Kc, B, s);
    const hfta_in dcol{col, sh.Ms * sh.Kc, sh.Kc};
    if (dW) {
      // dWt[(ky,kx,co)][ci] = sum_m dcol[m][(ky,kx,co)] X[m][ci]
      if (hfta_status st = hfta_fused_linear_bwd(B, sh.Ms, sh.Kc, sh.Ci, dt, dcol, X, W, hfta_out{nullptr, 0, 1}, dW,
                                                 dW_bstride, sh.Ci, nullptr, 0, accumulate, lws, lwsb, stream))
        return st;
    }
    if (dX.ptr) {
      // dX[m][ci] = sum_k dcol[m][k] Wt[k][ci]
      GemmP p{};
      p.B = B; p.splits = 1; p.M = sh.Ms; p.N = sh.Ci; p.K = sh.Kc; p.k_chunk = sh.Kc;
      p.A = col; p.a_bs = sh.Ms * sh.Kc; p.a_ld = sh.Kc; p.a_kmajor = 1;
      p.Bm = W.ptr; p.b_bs = W.bstride; p.b_ld = W.ld; p.b_kmajor = 0;
      p.C = dX.ptr; p.c_bs = dX.bstride; p.c_ld = dX.ld;
      if (hfta_status st = run_gemm(p, dt, false, s)) return st;
    }
  }
  return finish();
}

}  // extern "C"
