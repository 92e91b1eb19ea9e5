/*
 * hfta.h -- C ABI of libhfta, the B200 (sm_100a) hot path of HFTA
 * ("Horizontally Fused Training Array", arXiv 2102.02344).
 *
 * One horizontally fused training step of B same-architecture models that
 * differ only in hyper-parameters (paper §3).  Every call below
 * runs ONE set of kernel launches for all B models ("the horizontal fusion of
 * many ... operators"); the model index b is folded into the
 * launch grid / tile scheduler.  Citations: P:Lnnn = PAPER.md line nnn.
 *
 * ---------------------------------------------------------------------------
 * Conventions (apply to every entry point)
 * ---------------------------------------------------------------------------
 * Layout.  Model-major: element (b, i, j) of a per-model matrix lives at
 *   ptr[b*bstride + i*ld + j]  (elements, not bytes).
 *   This replaces the paper's channel-folded [N, B*C, ...] layout (App. B,
 *   P:L1262-1293); the two are a bijection.  bstride == 0 on an INPUT means
 *   "shared by all models" (the same data batch, reading R5).  Outputs must
 *   have bstride > 0 (or B == 1) and must not alias inputs.
 * Dtype.  HFTA_F32: every activation/operand is fp32 and contractions are
 *   fp32-accurate.  HFTA_BF16 (bf16-AMP, reading R16): activations and GEMM
 *   operands are bf16, accumulation fp32; weight gradients, BN statistics,
 *   BN affine parameters, biases, losses and optimizer state are always fp32.
 *   HFTA_BF16_F32 (hfta_fused_linear_fwd/bwd only, reading R16b): bf16 GEMM
 *   operands X, W, dY with fp32 outputs Y, dX -- the bf16-AMP contraction of
 *   a layer whose activations are kept fp32 (the per-sample FC head).
 * Ownership.  The caller owns every buffer (allocated with cudaMalloc or by
 *   PyTorch).  The library never allocates device memory, never frees, and
 *   keeps no pointer beyond the stream-ordered completion of the call.
 *   Scratch memory is passed as (ws, ws_bytes); query the size first with the
 *   matching *_workspace() function.
 * Streams.  `stream` is a cudaStream_t (NULL = legacy default stream).  All
 *   calls only enqueue work and return; hyper-parameter vectors and the step
 *   counter are DEVICE arrays so a whole step can be captured in a CUDA graph.
 * Errors.  Arguments are validated before anything is enqueued; on error
 *   nothing is launched and a status != HFTA_OK is returned;
 *   hfta_last_error() (thread-local) names the argument and shapes.  Kernel
 *   faults surface asynchronously; with env HFTA_SYNC=1 every call
 *   synchronizes its stream and reports HFTA_ERR_CUDA.
 * Device.  hfta_init() must succeed first; it requires compute capability
 *   10.0 (B200, sm_100a).  There is no fallback for any other device and no
 *   CPU path.
 * Determinism.  For fixed inputs all outputs are bitwise reproducible
 *   (fixed-order reductions, no floating-point atomics).
 */
#ifndef HFTA_H_
#define HFTA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int hfta_status;
enum {
  HFTA_OK = 0,
  HFTA_ERR_INVALID_VALUE = 1, /* null required pointer, B < 1, bad scalar   */
  HFTA_ERR_SHAPE = 2,         /* inconsistent dims/strides                   */
  HFTA_ERR_ALIGNMENT = 3,     /* pointer/stride not aligned as required      */
  HFTA_ERR_UNSUPPORTED = 4,   /* dtype / configuration not implemented       */
  HFTA_ERR_ARCH = 5,          /* device is not compute capability 10.0       */
  HFTA_ERR_WORKSPACE = 6,     /* ws too small                                */
  HFTA_ERR_CUDA = 7,          /* CUDA launch error (message has the string)  */
  HFTA_ERR_NOT_INITIALIZED = 8
};

typedef enum { HFTA_F32 = 0, HFTA_BF16 = 1, HFTA_BF16_F32 = 2 } hfta_dtype;
typedef enum {
  HFTA_ACT_NONE = 0, HFTA_ACT_RELU = 1, HFTA_ACT_LEAKY_RELU = 2,
  HFTA_ACT_TANH = 3, HFTA_ACT_SIGMOID = 4      /* standalone hfta_act_* only */
} hfta_act;

typedef struct { const void* ptr; int64_t bstride; int64_t ld; } hfta_in;
typedef struct { void* ptr; int64_t bstride; int64_t ld; } hfta_out;
typedef void* hfta_stream; /* cudaStream_t */

/* ---------------------------------------------------------------- setup -- */

/* Select `device`, check CC 10.0, cache SM count.  HFTA_ERR_ARCH otherwise. */
hfta_status hfta_init(int device);
/* Thread-local message of the last failing call ("" if none). */
const char* hfta_last_error(void);
/* Library version string. */
const char* hfta_version(void);
/* Number of kernels this library launched (process-wide counter). */
uint64_t hfta_launch_count(void);

/* ------------------------------------------------ fused Linear / Conv1d -- */
/*
 * Fused Linear and Conv1d(kernel=1): App. B rows "Linear -> baddbmm"
 * and "Conv1d", grouped with G = B.
 * For each b in [0, B):
 *   Y_b[M,N] = X_b[M,K] * W_b[N,K]^T + bias_b       (Linear, PyTorch [out,in])
 * X: [B][M][K] (bstride 0 = shared input), W: [B][N][K], Y: [B][M][N],
 * all of dtype dt; bias fp32 or NULL.  The bias is a 2-D table:
 *   bias element for (b, m, n) = bias[b*bias_bstride + (m / bias_row_div)*bias_ld + n]
 * (bias_row_div = 0 or bias_ld = 0 means a plain per-model [N] bias).  The
 * row-grouped form is the exact split-weight rewrite of PointNet-seg's
 * concat(global, point) layer.
 * Alignment: for the tensor-core path, X/W/Y pointers 16-B aligned and
 * ld*sizeof(dt), bstride*sizeof(dt) multiples of 16; other shapes run a SIMT
 * kernel (no alignment requirement).  M, N, K >= 1.
 */
hfta_status hfta_fused_linear_fwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt,
                                  hfta_in X, hfta_in W,
                                  const float* bias, int64_t bias_bstride, int64_t bias_ld,
                                  int64_t bias_row_div, hfta_out Y, hfta_stream stream);

/* Scratch bytes for hfta_fused_linear_bwd with these sizes. */
size_t hfta_fused_linear_bwd_workspace(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt);

/*
 * Backward of hfta_fused_linear_fwd (same dims).  For each b:
 *   dX_b[M,K] = dY_b[M,N] * W_b[N,K]           (dX.ptr == NULL: skipped)
 *   dW_b[N,K] (+)= dY_b^T * X_b   fp32 at dW + b*dW_bstride + n*dW_ld + k (dW_ld >= K;
 *                               a column slice of a wider weight, e.g. the split
 *                               weight of PointNet-seg's concat layer, has dW_ld > K)
 *   dbias_b[N] (+)= sum_m dY_b[m,:]   fp32 (dbias == NULL: skipped)
 * accumulate != 0 adds into dW/dbias instead of overwriting (D(real)+D(fake)
 * accumulation of the DCGAN step).  The reduction over M is split in a fixed
 * number of chunks reduced in fixed order (deterministic).
 */
hfta_status hfta_fused_linear_bwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt,
                                  hfta_in dY, hfta_in X, hfta_in W, hfta_out dX,
                                  float* dW, int64_t dW_bstride, int64_t dW_ld,
                                  float* dbias, int64_t dbias_bstride, int accumulate,
                                  void* ws, size_t ws_bytes, hfta_stream stream);

/* -------------------------------------------- fused Conv2d / ConvT2d -- */
/*
 * Fused Conv2d / ConvTranspose2d (App. B rows P:L1262-1263, P:L1268-1269;
 * grouped convolution with G = B, Fig. 3), NHWC per model.
 * desc: N images of H x W x C_in (the layer INPUT), C_out channels, kernel
 * kh x kw, stride, pad; transposed = 1 selects ConvTranspose2d (output size
 * (H-1)*stride - 2*pad + kh), else output (H + 2 pad - kh)/stride + 1.
 * Layouts (elements): X [B][N][H][W][C_in] (bstride 0 = shared images),
 * Y [B][N][Ho][Wo][C_out];
 * Conv2d weight W [B][C_out][kh][kw][C_in]   (PyTorch [Co][Ci][kh][kw] permuted),
 * ConvT2d weight W [B][kh][kw][C_out][C_in]  (PyTorch [Ci][Co][kh][kw] permuted).
 * dW fp32 in the same layout at dW + b*dW_bstride (accumulate != 0 adds: the
 * D(real) + D(fake) gradient accumulation of the DCGAN step).  dX.ptr NULL /
 * dW NULL skip that output.  No bias (the DCGAN convolutions have none).
 * act (fwd): an activation of a layer without BatchNorm (D c1 LeakyReLU
 * act_alpha, G t5 Tanh) applied to Y -- in the implicit-GEMM epilogue on the
 * tensor-core path (its backward gates on the stored output: y > 0 <=> act(y) > 0).
 * Paths: bf16 k4 s2 p1 with 8 or 64-multiple channels: implicit GEMM (TMA
 * gathers / sub-pixel phases, no patch matrix); 1x1-input / whole-window
 * layers: dense GEMMs; fp32: patch matrix + 3xTF32 GEMMs.  Images are dense
 * NHWC per model (X.ld == C_in, Y.ld == C_out).
 */
typedef struct {
  int N, H, W, C_in, C_out, kh, kw, stride, pad, transposed;
} hfta_conv_desc;
size_t hfta_fused_conv_workspace(int B, const hfta_conv_desc* desc, hfta_dtype dt);
hfta_status hfta_fused_conv_fwd(int B, const hfta_conv_desc* desc, hfta_dtype dt, hfta_in X, hfta_in W,
                                hfta_out Y, hfta_act act, float act_alpha, void* ws, size_t ws_bytes,
                                hfta_stream stream);
hfta_status hfta_fused_conv_bwd(int B, const hfta_conv_desc* desc, hfta_dtype dt, hfta_in dY, hfta_in X,
                                hfta_in W, hfta_out dX, float* dW, int64_t dW_bstride, int accumulate,
                                void* ws, size_t ws_bytes, hfta_stream stream);
/*
 * hfta_fused_conv_fwd (no activation) that also writes the BatchNorm
 * statistics of the stored Y, colstat [B][ceil(R/32)][2][C_out] with
 * R = N*Ho*Wo (layout of hfta_fused_linear_fwd_stats; size
 * hfta_linear_colstat_size(B, R, C_out)): from the implicit-GEMM epilogues
 * (Conv2d: block k = output rows 32k..32k+31; ConvT2d sub-pixel phases: the
 * blocks partition the rows phase by phase), from one pass over Y elsewhere.
 * Feed to hfta_fused_bn_fwd_colstat (which only needs the block totals).
 */
hfta_status hfta_fused_conv_fwd_stats(int B, const hfta_conv_desc* desc, hfta_dtype dt, hfta_in X, hfta_in W,
                                      hfta_out Y, float* colstat, void* ws, size_t ws_bytes, hfta_stream stream);
/*
 * As hfta_fused_conv_bwd, and dX additionally multiplied by the backward of
 * the activation that consumed X: dX *= act'(gate) with gate the activation's
 * output (or input: same sign) in dX's layout, act in {NONE, ReLU (0),
 * LeakyReLU (dX_alpha)} -- e.g. D c2's dgrad through D c1's LeakyReLU(0.2).
 * Fused into the sub-pixel dgrad epilogue (bf16 k4 s2 p1, dense gate with
 * the dX model stride); other paths apply it as one pass after the dgrad.
 */
hfta_status hfta_fused_conv_bwd_gated(int B, const hfta_conv_desc* desc, hfta_dtype dt, hfta_in dY, hfta_in X,
                                      hfta_in W, hfta_out dX, float* dW, int64_t dW_bstride, int accumulate,
                                      hfta_act dX_act, float dX_alpha, hfta_in dX_gate, void* ws, size_t ws_bytes,
                                      hfta_stream stream);

/*
 * hfta_fused_linear_fwd on the bf16 tensor-core path (X, W bf16, Y bf16; not
 * the skinny shapes) that also writes the BatchNorm statistics of the STORED
 * Y from its epilogue (the §8(b) `bn_partials`): colstat fp32
 * [B][ceil(M/32)][2][N], block k = rows 32k..32k+31, [0] = sum, [1] = sum of
 * squares (fp32 over <= 32 rows).  Size: hfta_linear_colstat_size.  Returns
 * HFTA_ERR_UNSUPPORTED where the shape does not take that path.
 */
size_t hfta_linear_colstat_size(int B, int64_t M, int64_t N);
hfta_status hfta_fused_linear_fwd_stats(int B, int64_t M, int64_t N, int64_t K, hfta_in X, hfta_in W,
                                        const float* bias, int64_t bias_bstride, int64_t bias_ld,
                                        int64_t bias_row_div, hfta_out Y, float* colstat, hfta_stream stream);

/* ------------------------------------------------------- fused BatchNorm -- */
/*
 * Fused BatchNorm1d/2d (App. B rows P:L1274-1278): statistics per (model b,
 * channel c) over the R rows of model b (reading R13); PyTorch training-mode
 * semantics (reading R6): biased variance normalises, unbiased variance
 * (R/(R-1)) enters running_var; running <- (1-momentum)*running + momentum*stat.
 * X: [B][R][C] dtype dt (R = rows, e.g. N*L points or N*H*W pixels, C contiguous).
 * gamma, beta: fp32, element (b,c) at gamma[b*gb_bstride + c].
 * running_mean/var, save_mean/save_invstd: fp32 [B][C] contiguous.
 * Y = act(gamma * (X - mean) * invstd + beta), act in {none, ReLU,
 * LeakyReLU(act_alpha)}; Y.ptr == NULL computes statistics only (the max-over-
 * points path applies BN inside hfta_bn_max_fwd).  running_* may be NULL.
 * R >= 2.
 */
size_t hfta_fused_bn_workspace(int B, int64_t R, int64_t C);
hfta_status hfta_fused_bn_fwd(int B, int64_t R, int64_t C, hfta_dtype dt, hfta_in X,
                              const float* gamma, const float* beta, int64_t gb_bstride,
                              float* running_mean, float* running_var, float momentum, float eps,
                              hfta_act act, float act_alpha, hfta_out Y,
                              float* save_mean, float* save_invstd,
                              void* ws, size_t ws_bytes, hfta_stream stream);
/*
 * Backward: dY is the gradient w.r.t. the activation output; act' is
 * recomputed from X and the saved statistics.  With z = act input:
 *   dbeta = sum_r dz, dgamma = sum_r dz*xhat,
 *   dX = gamma*invstd/R * (R*dz - dbeta - xhat*dgamma).
 * dgamma/dbeta fp32 at [b*gb_bstride + c] (accumulate != 0 adds).
 */
/*
 * hfta_fused_bn_fwd with the statistics taken from colstat (written by
 * hfta_fused_linear_fwd_stats for the same X, R rows): per (b, c) the block
 * sums are merged in a fixed order in fp64, mean = S1/R, biased variance =
 * S2/R - mean^2 (clamped at 0), running statistics and save_mean /
 * save_invstd as hfta_fused_bn_fwd; then the same apply (+ act) into Y.
 */
hfta_status hfta_fused_bn_fwd_colstat(int B, int64_t R, int64_t C, hfta_dtype dt, hfta_in X, const float* gamma,
                                      const float* beta, int64_t gb_bstride, float* running_mean, float* running_var,
                                      float momentum, float eps, hfta_act act, float act_alpha, hfta_out Y,
                                      float* save_mean, float* save_invstd, const float* colstat,
                                      hfta_stream stream);
hfta_status hfta_fused_bn_bwd(int B, int64_t R, int64_t C, hfta_dtype dt, hfta_in dY, hfta_in X,
                              const float* gamma, const float* beta, int64_t gb_bstride,
                              const float* save_mean, const float* save_invstd,
                              hfta_act act, float act_alpha, hfta_out dX,
                              float* dgamma, float* dbeta, int accumulate,
                              void* ws, size_t ws_bytes, hfta_stream stream);

/* ------------------------------------------------- PointNet glue (K8) -- */
/*
 * BN-apply + activation + max over points, fused (the max-pool of PointNet,
 * App. B row MaxPool family P:L1286-1287 as used by the cited model):
 *   out[b][n][c] = max_l act(gamma*(X[b][n*L+l][c]-mean)*invstd + beta)
 *   argmax[b][n][c] = first l attaining it (reading R15), int32.
 * X [B][N*L][C] dtype dt; out [B][N][C] fp32 (ld = out.ld).  Per-sample
 * tensors ([N] rows: pooled features, the FC head, the 3x3 transform) are
 * fp32 in both precision modes.
 */
hfta_status hfta_bn_max_fwd(int B, int64_t N, int64_t L, int64_t C, hfta_dtype dt, hfta_in X,
                            const float* gamma, const float* beta, int64_t gb_bstride,
                            const float* save_mean, const float* save_invstd,
                            hfta_act act, float act_alpha, hfta_out out, int32_t* argmax,
                            hfta_stream stream);
/*
 * Backward of hfta_bn_max_fwd followed by the BN backward: dG [B][N][C]
 * (fp32) is scattered to the argmax rows, passed through act' and BN
 * backward; writes dX [B][N*L][C] (dtype dt) and dgamma/dbeta.
 * Workspace: hfta_bn_max_bwd_workspace().
 */
size_t hfta_bn_max_bwd_workspace(int B, int64_t N, int64_t C);
hfta_status hfta_bn_max_bwd(int B, int64_t N, int64_t L, int64_t C, hfta_dtype dt,
                            hfta_in dG, hfta_in X, const int32_t* argmax,
                            const float* gamma, const float* beta, int64_t gb_bstride,
                            const float* save_mean, const float* save_invstd,
                            hfta_act act, float act_alpha, hfta_out dX,
                            float* dgamma, float* dbeta, void* ws, size_t ws_bytes,
                            hfta_stream stream);
/* ------------------------------ fused Linear -> BN -> max block (K10) -- */
/*
 * The PointNet point-feature block as ONE fused operation per pass (App. B
 * rows Conv1d P:L1265-1266, BatchNorm1d P:L1280-1281, MaxPool P:L1286-1287,
 * composed as in the cited PointNetfeat/STN3d, reading R1):
 *   Y[b][r][c] = sum_k X[b][r][k] W[b][c][k] + bias[b][c]      r = n*L + l
 *   mean/var over the R = N*L rows (biased var normalises, unbiased var
 *   enters running_var, reading R6), xhat = (Y - mean)*invstd,
 *   G[b][n][c] = max_l act(gamma*xhat + beta), argmax[b][n][c] = first l
 *   attaining it (reading R15), ext[b][n][c] = Y at that row.
 * The [B][R][C] tensor Y is never written: the forward reduces only its
 * per-cloud max out of tensor memory and takes the statistics from the Gram
 * of the layer input (reading R27):
 *   gram = X^T X [K][K], xsum = X^T 1 [K]  (fp32 outputs, caller-owned,
 *   contiguous [B][K][K] / [B][K]; inputs of the backward),
 *   mean_c = W_c xsum/R + bias_c,  var_c = W_c (gram - xsum xsum^T/R) W_c^T / R
 * (centred in fp64 before the fp32 quadratic form); the backward works in
 * the same Gram form (K10).  Precision: bf16 X/W (dt must be
 * HFTA_BF16), fp32 accumulation.  Layouts: X [B][R][K] (bstride 0 =
 * shared), W [B][C][K] (hfta_in), per-channel vectors at [b*bstride + c];
 * G, ext fp32 [B][N][C] (hfta_out), argmax int32 contiguous [B][N][C].
 * Constraints (else HFTA_ERR_UNSUPPORTED): K in {64, 128}, C % 128 == 0,
 * 16-B aligned X/W/dX with 16-B row strides.  Workspace:
 * hfta_fused_linear_bn_max_workspace() bytes, caller-owned, shared by fwd
 * and bwd (no state carried in it between the two calls).
 */
size_t hfta_fused_linear_bn_max_workspace(int B, int64_t N, int64_t L, int64_t C, int64_t K);
hfta_status hfta_fused_linear_bn_max_fwd(int B, int64_t N, int64_t L, int64_t C, int64_t K,
                                         hfta_dtype dt, hfta_in X, hfta_in W,
                                         const float* bias, int64_t bias_bstride,
                                         const float* gamma, const float* beta, int64_t gb_bstride,
                                         float* running_mean, float* running_var,
                                         float momentum, float eps, hfta_act act, float act_alpha,
                                         hfta_out G, int32_t* argmax, hfta_out ext,
                                         float* save_mean, float* save_invstd,
                                         float* gram, float* xsum,
                                         void* ws, size_t ws_bytes, hfta_stream stream);
/*
 * Backward: dG fp32 [B][N][C] -> dZ at the argmax rows (act' at the pooled
 * pre-activation), BN backward dY = gamma*invstd/R*(R*dZ - dbeta - xhat*dgamma),
 * dX = dY W (bf16, skipped if dX.ptr is NULL), dW = dY^T X (fp32 at
 * dW[b*dW_bstride + c*dW_ld + k]), dgamma/dbeta fp32, dbias (may be NULL)
 * written as exact zeros (BN-absorbed).  dY = bx*Y + cc + S (S:
 * one nonzero per cloud and channel) is never formed: dX = X M + 1 v^T + S W
 * and dW = diag(bx) W G + cc s^T + S^T X with M = W^T diag(bx) W (rounded to
 * bf16), v = W^T cc, G = X^T X, s = X^T 1 (K10).  accumulate != 0
 * adds to dW/dgamma/dbeta instead of overwriting.  ext, argmax, save_mean,
 * save_invstd, gram (= G) and xsum (= s) are the forward's outputs.
 * dX_act != NONE multiplies dX by act'(X) (X being the previous layer's
 * activation output), so dX is that layer's dZ.  C <= 1024.
 */
hfta_status hfta_fused_linear_bn_max_bwd(int B, int64_t N, int64_t L, int64_t C, int64_t K,
                                         hfta_dtype dt, hfta_in dG, hfta_in X, hfta_in W,
                                         const int32_t* argmax, hfta_in ext,
                                         const float* bias, int64_t bias_bstride,
                                         const float* gamma, const float* beta, int64_t gb_bstride,
                                         const float* save_mean, const float* save_invstd,
                                         const float* gram, const float* xsum,
                                         hfta_act act, float act_alpha, hfta_out dX,
                                         hfta_act dX_act, float dX_alpha,
                                         float* dW, int64_t dW_bstride, int64_t dW_ld,
                                         float* dbias, int64_t dbias_bstride,
                                         float* dgamma, float* dbeta, int accumulate,
                                         void* ws, size_t ws_bytes, hfta_stream stream);

/* ------------------------- fused Linear -> BN -> act, Gram form (K11) -- */
/*
 * Conv1d(k=1)/Linear -> training-mode BatchNorm -> act for all B models
 * (App. B rows P:L1265-1266; R6 conventions) with the batch
 * statistics taken from the Gram of the layer input instead of a pass over
 * the [M][N] pre-BN tensor (which is never written):
 *   G = X^T X [K][K], s = X^T 1 [K]   (fp32, outputs: kept for the backward)
 *   mean_n = (W_n . s)/M + bias_n,  var_n = W_n G W_n^T / M - ((W_n . s)/M)^2
 *   A = act(gamma*(X W^T + bias - mean)*invstd + beta)     (bf16 [B][M][N])
 * (fp64 from the fp32 G, s).  K <= 8 (streaming kernels) or K in {64, 128}
 * (tensor cores), N <= 512 (N <= 128 for K >= 64), dt must be HFTA_BF16.
 * Workspace: hfta_fused_linear_bn_workspace(B, M, N, K), shared by fwd/bwd.
 */
size_t hfta_fused_linear_bn_workspace(int B, int64_t M, int64_t N, int64_t K);
hfta_status hfta_fused_linear_bn_fwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt,
                                     hfta_in X, hfta_in W, const float* bias, int64_t bias_bstride,
                                     const float* gamma, const float* beta, int64_t gb_bstride,
                                     float* running_mean, float* running_var, float momentum, float eps,
                                     hfta_act act, float act_alpha, hfta_out A,
                                     float* save_mean, float* save_invstd, float* G, float* s,
                                     void* ws, size_t ws_bytes, hfta_stream stream);
/*
 * Backward from dZ = dL/dz (the gradient at BN's output BEFORE act, i.e. the
 * consumer already multiplied by act'): dbeta = 1^T dZ, Zm = dZ^T X,
 * dgamma = invstd*(W.Zm - mean'*dbeta), and with a = gamma*invstd,
 * bx = -a*invstd*dgamma/M, cc = -a*dbeta/M - bx*mean' (mean' = mean - bias):
 *   dW = diag(a) Zm + diag(bx) W G + cc s^T                (fp32, accumulate adds)
 *   dX = (dZ diag(a) W + X W^T diag(bx) W + 1 (W^T cc)^T) * act'(X)   (bf16)
 * where act'(X) is dX_act's derivative evaluated on X (X = the previous
 * layer's activation output; HFTA_ACT_NONE: no gating) -- so dX is the
 * previous layer's dZ.  dbias (may be NULL) = exact zeros (BN-absorbed).
 * dX.ptr NULL skips dX.  G, s: the forward's outputs.
 */
hfta_status hfta_fused_linear_bn_bwd(int B, int64_t M, int64_t N, int64_t K, hfta_dtype dt,
                                     hfta_in dZ, hfta_in X, hfta_in W, const float* bias,
                                     int64_t bias_bstride, const float* gamma, int64_t gb_bstride,
                                     const float* save_mean, const float* save_invstd,
                                     const float* G, const float* s, hfta_out dX, hfta_act dX_act,
                                     float dX_alpha, float* dW, int64_t dW_bstride, int64_t dW_ld,
                                     float* dbias, int64_t dbias_bstride, float* dgamma, float* dbeta,
                                     int accumulate, void* ws, size_t ws_bytes, hfta_stream stream);
/*
 * PointNet input transform (STN): T_b,n = F_b[n] viewed as 3x3 row-major
 * (+ I3 if add_identity), x'_b[n*L+l][:] = x[n*L+l][:] * T_b,n.
 * X fp32 [B][N*L][3] (bstride 0 = shared), F fp32 [B][N][9] (ld >= 9),
 * Xout dtype dt [B][N*L][3] (ld >= 3).
 */
hfta_status hfta_transform_points_fwd(int B, int64_t N, int64_t L, hfta_dtype dt, hfta_in X,
                                      hfta_in F, int add_identity, hfta_out Xout,
                                      hfta_stream stream);
/* dF_b[n] = sum_l x[n*L+l]^T dXout_b[n*L+l]   (fp32 [B][N][9]; dX not needed). */
hfta_status hfta_transform_points_bwd(int B, int64_t N, int64_t L, hfta_dtype dt, hfta_in X,
                                      hfta_in dXout, hfta_out dF, hfta_stream stream);
/*
 * Dropout (App. B row Dropout) with a counter-based mask
 * (reading R14): element i of model b is kept iff
 * Philox4x32-10(ctr=(i/4, b, step, layer), key=(seed lo, seed hi))[i%4]
 * >= floor(p*2^32); kept values are scaled by 1/(1-p).  i = row*cols + col.
 * step_ptr (device int64, may be NULL): when given, the counter's step is
 * *step_ptr + step, read at kernel time -- so a captured CUDA graph of the
 * training step draws a fresh mask on every replay.  b in the counter is the
 * GLOBAL model index model_offset + (local b): a model-array shard draws the
 * masks its models draw in an unsharded run (the rank's first model index);
 * model_ids (device int32 [B], nullable) overrides it with explicit per-model
 * ids (an HFHT partition of non-contiguous hyper-parameter sets draws each
 * set's own masks, whatever partition it lands in).
 * X/Y [B][rows][cols] dtype dt.  bwd: same mask applied to dY.
 */
hfta_status hfta_dropout_fwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_in X,
                             hfta_out Y, uint64_t seed, int64_t step, const int64_t* step_ptr,
                             int32_t layer, float p, int32_t model_offset, const int32_t* model_ids,
                             hfta_stream stream);
hfta_status hfta_dropout_bwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_in dY,
                             hfta_out dX, uint64_t seed, int64_t step, const int64_t* step_ptr,
                             int32_t layer, float p, int32_t model_offset, const int32_t* model_ids,
                             hfta_stream stream);
/*
 * Segmented column sums: S[b][g][c] = sum_{r in group g} X[b][r][c] with
 * groups of `group` consecutive rows (group = rows: plain column sum).
 * S fp32 at S + b*S_bstride + g*C + c.  accumulate != 0 adds.
 */
size_t hfta_colsum_workspace(int B, int64_t rows, int64_t C, int64_t group);
hfta_status hfta_colsum(int B, int64_t rows, int64_t C, int64_t group, hfta_dtype dt, hfta_in X,
                        float* S, int64_t S_bstride, int accumulate, void* ws, size_t ws_bytes,
                        hfta_stream stream);

/* ---------------------------------------------------- fused loss (K8d) -- */
/*
 * Per-model losses l_b and d l_b / d logits (App. C: the per-model gradients
 * equal B * dL/d(theta_b) for the mean-reduced fused loss L = (1/B) sum_b l_b,
 * Eq. 1-3; computed analytically, reading R9).
 * NLL: logits [B][rows][K] dtype dt, labels int32 [rows] (labels_bstride 0 =
 * shared) ; l_b = -(1/rows) sum_r log_softmax(z_r)[y_r]; dlogits dtype dt.
 * loss: fp32 [B]; mean_loss (nullable) fp32 scalar = (1/B) sum_b l_b.
 */
size_t hfta_loss_workspace(int B, int64_t rows);
hfta_status hfta_loss_nll(int B, int64_t rows, int64_t K, hfta_dtype dt, hfta_in logits,
                          const int32_t* labels, int64_t labels_bstride, float* loss,
                          float* mean_loss, hfta_out dlogits, void* ws, size_t ws_bytes,
                          hfta_stream stream);
/*
 * Sigmoid + BCE (DCGAN discriminator output, PyTorch BCELoss with its log clamp
 * at -100; reading R29): p = sigmoid(z),
 * l_b = -(1/rows) sum_r [y max(log p, -100) + (1-y) max(log(1-p), -100)] with
 * log p = -softplus(-z), log(1-p) = -softplus(z);
 * dz = (p - y) q / max(q, 1e-12) / rows, q = p(1-p) = sigmoid(z) sigmoid(-z)
 * (the BCELoss backward (p-y)/max(p(1-p),1e-12) times sigmoid' p(1-p)),
 * evaluated from z so saturated logits keep their exact value.
 * Z, dZ dtype dt [B][rows] (ld = row stride); y scalar.
 */
hfta_status hfta_loss_bce_logits(int B, int64_t rows, hfta_dtype dt, hfta_in Z, float target, float* loss,
                                 float* mean_loss, hfta_out dZ, void* ws, size_t ws_bytes,
                                 hfta_stream stream);
/* MSE (mean over rows*C): A [B][rows][C] dtype dt vs T fp32 [rows][C] (T_bstride 0 = shared). */
hfta_status hfta_loss_mse(int B, int64_t rows, int64_t C, hfta_dtype dt, hfta_in A,
                          const float* T, int64_t T_bstride, int64_t T_ld, float* loss,
                          float* mean_loss, hfta_out dA, void* ws, size_t ws_bytes,
                          hfta_stream stream);

/* ------------------------------------------------------ fused Adam (K7) -- */
/*
 * Fused Adam ("scalar-vector operations ... replaced by
 * broadcasted vector-vector operations"), PyTorch-1.6 form (reading R7).
 * For every element j of model b (param/grad/exp_avg/exp_avg_sq fp32 at
 * [b*bstride + j], j < P):
 *   g = grad + wd[b]*p ; m = beta1[b]*m + (1-beta1[b])*g ;
 *   v = beta2[b]*v + (1-beta2[b])*g^2 ;
 *   p -= lr[b]/(1-beta1[b]^t) * m / (sqrt(v)/sqrt(1-beta2[b]^t) + eps[b])
 * lr, beta1, beta2, eps, wd: device fp32 [B]; step: device int64 scalar t>=1
 * (shared, read at kernel time so graphs can replay).  param_bf16 (nullable):
 * bf16 shadow [b*bf16_bstride + j] written with round-to-nearest-even.
 */
hfta_status hfta_fused_adam(int B, int64_t P, float* param, const float* grad,
                            float* exp_avg, float* exp_avg_sq, int64_t bstride,
                            const float* lr, const float* beta1, const float* beta2,
                            const float* eps, const float* weight_decay, const int64_t* step,
                            void* param_bf16, int64_t bf16_bstride, hfta_stream stream);

/*
 * Standalone activations over [B][rows][cols] (dtype dt): act in {ReLU,
 * LeakyReLU(alpha), Tanh, Sigmoid} (App. B rows P:L1298-1311).  Backward:
 * dX = dY * act'(.), where act' is evaluated from the INPUT X for ReLU /
 * LeakyReLU and from the OUTPUT Y for Tanh (1 - y^2) / Sigmoid (y(1-y));
 * XY is that tensor.
 */
hfta_status hfta_act_fwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_act act, float alpha,
                         hfta_in X, hfta_out Y, hfta_stream stream);
hfta_status hfta_act_bwd(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_act act, float alpha,
                         hfta_in XY, hfta_in dY, hfta_out dX, hfta_stream stream);

/*
 * Fused SGD (BJ north_star "fused Adam/SGD step"; P:L910-911 tunes momentum),
 * PyTorch-1.6 form: d = grad + wd[b]*p; with momentum[b] != 0:
 * buf = (t == 1) ? d : momentum[b]*buf + (1-dampening[b])*d,
 * d = nesterov ? d + momentum[b]*buf : buf;  p -= lr[b]*d.
 * momentum_buf [b*bstride + j] (may be NULL if every momentum is 0);
 * hyper-parameters device fp32 [B]; step device int64 (shared t).
 */
hfta_status hfta_fused_sgd(int B, int64_t P, float* param, const float* grad, float* momentum_buf,
                           int64_t bstride, const float* lr, const float* momentum,
                           const float* dampening, const float* weight_decay, int nesterov,
                           const int64_t* step, void* param_bf16, int64_t bf16_bstride,
                           hfta_stream stream);
/*
 * Fused Adadelta ("Adam and Adadelta"), PyTorch-1.6 form:
 * g = grad + wd[b]*p; sq = rho*sq + (1-rho) g^2; delta = sqrt(acc+eps)/sqrt(sq+eps)*g;
 * acc = rho*acc + (1-rho) delta^2; p -= lr[b]*delta.
 */
hfta_status hfta_fused_adadelta(int B, int64_t P, float* param, const float* grad, float* square_avg,
                                float* acc_delta, int64_t bstride, const float* lr, const float* rho,
                                const float* eps, const float* weight_decay, void* param_bf16,
                                int64_t bf16_bstride, hfta_stream stream);
/*
 * Fused StepLR (per-model "Factor/Period of Learning Rate Decay",
 * P:L978-979): lr[b] = lr0[b] * gamma[b]^floor(epoch / period[b]),
 * device arrays [B]; a graph-capturable per-epoch update of the lr vector.
 */
hfta_status hfta_steplr(int B, const float* lr0, const float* gamma, const int32_t* period, int64_t epoch,
                        float* lr, hfta_stream stream);

/* ------------------------------------------- PointNet feature transform -- */
/*
 * The STNkd feature transform ("Feature Transformation" of the
 * PointNet tuning space; reading R30).  F3: fp32 [B][N][K*K] (the STNkd fc3
 * output, model stride f_bstride), K <= 64.
 * _make: Tt[b][n][j][i] = F3[b][n][i*K + j] + (i == j), dtype dt, i.e. the
 *   TRANSPOSED transform (T + I)^T, the K-major weight operand with which the
 *   per-cloud product x' = x (T + I) runs as hfta_fused_linear_fwd over B*N
 *   models (X [L][K] per cloud, W = Tt, no bias).
 * _reg: with T = F3 + I, A = T T^T - I, f = ||A||_F per (b, n):
 *   dF3[b][n][i*K + j] = dTt[b][n][j][i] + weight * 2 (A T)[i][j] / (N f)
 *   (dTt: fp32 [B][N][K][K], the weight gradient of that per-cloud Linear),
 *   loss[b] += weight * (1/N) sum_n f (fixed order), and mean_loss (nullable)
 *   = (1/B) sum_b loss[b].  Workspace: hfta_feature_transform_reg_workspace.
 */
hfta_status hfta_feature_transform_make(int B, int64_t N, int64_t K, hfta_dtype dt, const float* F3,
                                        int64_t f_bstride, hfta_out Tt, hfta_stream stream);
size_t hfta_feature_transform_reg_workspace(int B, int64_t N);
hfta_status hfta_feature_transform_reg(int B, int64_t N, int64_t K, const float* F3, int64_t f_bstride,
                                       const float* dTt, int64_t dt_bstride, float weight, float* dF3,
                                       int64_t df_bstride, float* loss, float* mean_loss, void* ws,
                                       size_t ws_bytes, hfta_stream stream);

/* ------------------------------------------ pooling (ResNet-18, NEXT-4) -- */
/*
 * Fused MaxPool2d (App. B row MaxPool2d): every (model b,
 * channel c) pooled on its own.  X [B][N][H][W][C] dense NHWC per model
 * (X.ld = C, X.bstride elements per model, 0 = shared); Y [B][N][Ho][Wo][C]
 * with Ho = (H + 2 pad - k) / stride + 1; argmax uint8 [B][N][Ho][Wo][C]
 * (model stride am_bstride) = the winning tap ky * k + kx.  Padded positions
 * take no part (PyTorch: -inf padding, requires 2 pad <= k); the first tap
 * in (ky, kx) order wins exact ties (reading R32).  k <= 15.
 * _bwd: dX[n][iy][ix][c] = sum of dY over the windows whose argmax is
 * (iy, ix) -- a gather in ascending (oy, ox) order (deterministic); dX is
 * overwritten.  Errors: HFTA_ERR_SHAPE (bad geometry, ld != C),
 * HFTA_ERR_INVALID_VALUE (null pointers).
 */
hfta_status hfta_maxpool2d_fwd(int B, int N, int H, int W, int C, int k, int stride, int pad, hfta_dtype dt,
                               hfta_in X, hfta_out Y, uint8_t* argmax, int64_t am_bstride, hfta_stream stream);
hfta_status hfta_maxpool2d_bwd(int B, int N, int H, int W, int C, int k, int stride, int pad, hfta_dtype dt,
                               hfta_in dY, const uint8_t* argmax, int64_t am_bstride, hfta_out dX,
                               hfta_stream stream);
/*
 * Fused AdaptiveAvgPool2d((1, 1)) (App. B row AdaptiveAvgPool2d,
 * P:L1289-1290): Y[b][n][c] = (1/HW) sum_q X[b][n][q][c] over the HW pixels
 * of image n (fp32 sum in pixel order); _bwd: dX[b][n][q][c] = dY[b][n][c] / HW.
 * Layouts dense ([N][HW][C] and [N][C], ld = C).
 */
hfta_status hfta_avgpool2d_fwd(int B, int64_t N, int64_t HW, int64_t C, hfta_dtype dt, hfta_in X, hfta_out Y,
                               hfta_stream stream);
hfta_status hfta_avgpool2d_bwd(int B, int64_t N, int64_t HW, int64_t C, hfta_dtype dt, hfta_in dY, hfta_out dX,
                               hfta_stream stream);

/* ------------------------------------------------------------- utility -- */
/* Y = X1 + X2 elementwise over [B][rows][cols] (dtype dt): sums the two
 * gradient paths into a shared activation (PointNet-seg's point feature). */
hfta_status hfta_add(int B, int64_t rows, int64_t cols, hfta_dtype dt, hfta_in X1, hfta_in X2,
                     hfta_out Y, hfta_stream stream);
/* n fp32 -> bf16 (RNE); used to initialise the bf16 weight shadow. */
hfta_status hfta_cast_f32_bf16(int64_t n, const float* src, void* dst, hfta_stream stream);
/* *step += 1 on device (graph-capturable step counter). */
hfta_status hfta_step_increment(int64_t* step, hfta_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* HFTA_H_ */
