// gemm.cuh -- the model-batched contraction engine behind the fused Linear /
// Conv1d(k=1) layers (App. B rows Linear->baddbmm P:L1271-1272 and Conv1d
// P:L1265-1266).  One launch computes, for every model b in [0, B):
//   C_b[m][n] (+)= sum_k A_b(m,k) * B_b(n,k)  (+ bias_b(m,n))
// A_b(m,k) = A[b*a_bs + m*a_ld + k]   (a_kmajor)   or  A[b*a_bs + k*a_ld + m]
// B_b(n,k) = B[b*b_bs + n*b_ld + k]   (b_kmajor)   or  B[b*b_bs + k*b_ld + n]
// fwd: A = X (K-major), B = W (K-major); dgrad: A = dY (K-major), B = W
// (MN-major); wgrad: A = dY (MN-major), B = X (MN-major), fp32 out, split-K.
#pragma once
#include "common.cuh"

namespace hfta {

struct GemmP {
  int B;
  int64_t M, N, K;
  const void* A; int64_t a_bs, a_ld; int a_kmajor;
  const void* Bm; int64_t b_bs, b_ld; int b_kmajor;
  void* C; int64_t c_bs, c_ld;
  const float* bias; int64_t bias_bs, bias_ld, bias_div;  // bias(b,m,n) = bias[b*bs + (m/div)*ld + n]
  int accumulate;   // C += result (fp32 output only)
  int splits;       // split-K chunks (>= 1); > 1 needs `part`
  int64_t k_chunk;  // reduction rows per split (multiple of the K tile)
  float* part;      // [splits][B][M][N] fp32 partials
  // ---- epilogue / operand extensions (tensor-core path, bf16 output) ----
  // v = act(v * scale[b][n] + bias) then v *= act'(mask[b][m][n]) where the
  // mask is the activation output that fed this layer (ReLU: mask > 0).
  const float* scale; int64_t scale_bs;          // NULL: no scale
  int act; float act_alpha;                      // hfta_act after the affine
  const void* mask; int64_t mask_bs, mask_ld;    // NULL: no mask
  int mask_act; float mask_alpha;
  // second K segment: C += sum_k A2(m,k) B2(n,k), k < K2 (both K-major, K2 % 64 == 0)
  const void* A2; int64_t a2_bs, a2_ld;
  const void* Bm2; int64_t b2_bs, b2_ld;
  int64_t K2;
  // fused column sums of A over the reduction (wgrad: colsum[b][m] = sum_k A(m,k)
  // = the dbias / Gram column-sum vector), computed on the tensor cores with a
  // constant ones operand (MN-major A, fp32-output tcgen05 path only)
  float* colsum; int64_t colsum_bs; int colsum_acc;   // colsum_acc: add into colsum
  float* colsum_part;                                 // [splits][B][M] when splits > 1
  // BatchNorm statistics of the bf16 OUTPUT C (tcgen05 path, plain epilogue):
  // colstat[b][blk][0|1][n] = sum / sum of squares of the stored C[b][32 blk ..
  // 32 blk + 31][n] (32-row blocks, fp32)
  float* colstat; int64_t colstat_bs;
};

// dt_in: operand dtype; out_f32: C is fp32 (else dt_in).
hfta_status gemm_simt(const GemmP& p, hfta_dtype dt_in, bool out_f32, cudaStream_t s);
hfta_status splitk_reduce(const GemmP& p, cudaStream_t s);   // C (+)= sum_s part[s]
hfta_status colsum_reduce(const GemmP& p, cudaStream_t s);   // colsum (+)= sum_s colsum_part[s]

// tcgen05 / TMA path; returns HFTA_ERR_UNSUPPORTED if the shape/alignment
// does not qualify (caller then uses gemm_simt).
hfta_status gemm_tc(const GemmP& p, hfta_dtype dt_in, bool out_f32, cudaStream_t s);
bool gemm_tc_supported(const GemmP& p, hfta_dtype dt_in, bool out_f32);

// fp32-accurate contraction on the tensor cores (3xTF32, gemm_tf32.cu): fp32
// operands / output, plain epilogue (bias, row-grouped bias, accumulate, split-K).
bool gemm_tf32_supported(const GemmP& p);
hfta_status gemm_tf32(const GemmP& p, cudaStream_t s);

// Implicit-GEMM convolution on the tcgen05 engine (kernel 4x4, stride 2, pad 1;
// gemm_tc.cu CONV modes; no im2col / col2im buffer).  Image tensors are dense
// NHWC per model [B][n][h][w][c] with c % 64 == 0 (bstride 0 = shared).
struct ConvTcP {
  int mode;                 // 1 Conv2d fwd / ConvT2d dgrad, 2 sub-pixel phases (ConvT2d fwd / Conv2d dgrad),
                            // 3 Conv2d wgrad, 4 ConvT2d wgrad, 5 merged sub-pixel phases for 8 output
                            // channels (opd = the [32][9 x C] phase-merged weights of conv_subpixel_weights)
  int B;
  int64_t M, N, K;          // GEMM extents (mode 2: per phase)
  const void* img; int64_t img_bs; int img_n, img_h, img_w, img_c;   // the gathered / shifted image operand
  int grid_w, grid_h;       // grid the GEMM rows (1, 2) / reduction rows (3, 4) enumerate
  const void* opd; int64_t opd_bs, opd_ld;   // 1: W [N][K] (K-major) or Wt [K][N] (w_mn); 2: weights;
                                             // 3: dY [K][M] (ld M); 4: X [K][N] (ld N)
  int w_mn;                 // 1: B MN-major (ConvT dgrad); 2: Conv2d weights [Ca][16][Cn] (else ConvT [16][Cn][Ca])
  int w_cn, w_ca;           // mode 2 weight dims
  void* C; int64_t c_bs, c_ld;   // 1: Y [B][M][N] bf16; 2: Y image (c_bs = model stride); 3, 4: dW fp32 (ld c_ld)
  int y_h, y_w;             // mode 2: output image size
  int accumulate; int splits; int64_t k_chunk; float* part;   // 3, 4: split-K over the reduction rows
  int act; float act_alpha;        // 1, 2 (forward): activation applied in the epilogue (layers without BN)
  float* colstat;                   // mode 1: BN statistics of the stored Y per 32-row block (gemm.cuh GemmP)
  int ks, cs, cpad;         // modes 1, 3, 4: kernel size, stride, pad of the gather (0 = DCGAN's 4, 2, 1)
  int wflip;                // mode 1, w_mn: B = W [Ca][taps][Cn] read flipped (stride-1 Conv2d dgrad)
  const void* gate; int64_t gate_bs; float gate_alpha;   // mode 2: output *= (gate > 0 ? 1 : gate_alpha)
};
bool conv_tc_supported(const ConvTcP& p);
// mode 5 operand: Wp[b][(ph,pw,co)][(dy,dx,ca)] (32 x 9 Ca, K-major bf16) from mode-2 weights
// (w_mn: Conv2d W [Ca][16][8], else ConvT2d Wt [16][8][Ca]); zeros where phase (ph,pw) does not use tap (dy,dx)
hfta_status conv_subpixel_weights(int B, int ca, int w_mn, const void* W, int64_t w_bs, void* Wp, cudaStream_t s);
hfta_status conv_tc(const ConvTcP& p, cudaStream_t s);
// tile width along N of the wgrad modes (3, 4) conv_tc launches for p (split-K policy input)
int conv_wgrad_bn(const ConvTcP& p);

// colstat[b][blk][0|1][n] of a stored [B][M][N] activation (ld N, model stride
// Y.bstride), 32-row blocks: the fallback of the epilogue statistics (bn.cu).
hfta_status colstat_rows(int B, int64_t M, int64_t N, hfta_dtype dt, hfta_in Y, float* colstat, cudaStream_t s);

// Dispatch: skinny -> tcgen05 -> SIMT (EPI features: skinny / tcgen05 only).
hfta_status run_gemm(GemmP& p, hfta_dtype dt, bool out_f32, cudaStream_t s, void* ws = nullptr, size_t wsb = 0);

// HBM-bound skinny contractions (K <= 8 fwd, N-out <= 8 dgrad, K-out <= 3 wgrad).
bool skinny_fwd_ok(const GemmP& p);
bool skinny_dgrad_ok(const GemmP& p);
bool skinny_wgrad_ok(const GemmP& p);
bool skinny_wgrad_ok_base(const GemmP& p);
size_t skinny_wgrad_ws(int B, int64_t rows, int64_t N, int64_t Ko);
hfta_status gemm_skinny(const GemmP& p, hfta_dtype dt, void* ws, size_t ws_bytes, cudaStream_t s);

}  // namespace hfta
