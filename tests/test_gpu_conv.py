"""Per-layer parity of the fused (de)convolution (hfta_fused_conv_fwd/bwd,
App. B rows Conv2d P:L1262-1263 / ConvT2d P:L1268-1269, Fig. 3)
against oracle.layers.conv2d_* / convT2d_* at every DCGAN layer shape of the
benched batch (N = 128 images of 64 x 64, BJ configs[3]), B in {1, 3}, shared
input images (bstride 0, as D(real) sees them) and per-model ones.

Paths covered: the implicit-GEMM tcgen05 modes (stride-2 TMA gather:
D c1-c4 fwd and wgrad, G t2-t5 dgrad; sub-pixel phases: G t2-t5 fwd, D c1-c4
dgrad; ConvT wgrad: G t2-t5; the 8-channel images of D c1 / G t5 through
SWIZZLE_NONE core-matrix boxes), the dense-GEMM layers (G t1, D c5); fp32 runs
the patch-matrix path with 3xTF32 GEMMs.

Inputs are rounded to the operand dtype before the oracle sees them, so the
oracle and the kernel contract the same values (reading R16).  Gates
(normwise per model, reading R20): bf16 outputs 1e-2 (their own bf16
rounding ~2e-3); fp32 (3xTF32 tensor cores, whose fp32 accumulation over
K up to 8192 reaches ~1.5e-5) and every dW: the north_star's 1e-4.
"""
import numpy as np
import pytest
import torch

from oracle import layers as OL
from tests._cmp import assert_close

pytestmark = pytest.mark.gpu

H = None
DEV = "cuda"

#         name  transposed  H   C_in C_out  k  s  p
LAYERS = [("D.c1", 0, 64, 8, 64, 4, 2, 1),
          ("D.c2", 0, 32, 64, 128, 4, 2, 1),
          ("D.c3", 0, 16, 128, 256, 4, 2, 1),
          ("D.c4", 0, 8, 256, 512, 4, 2, 1),
          ("D.c5", 0, 4, 512, 1, 4, 1, 0),
          ("G.t1", 1, 1, 104, 512, 4, 1, 0),
          ("G.t2", 1, 4, 512, 256, 4, 2, 1),
          ("G.t3", 1, 8, 256, 128, 4, 2, 1),
          ("G.t4", 1, 16, 128, 64, 4, 2, 1),
          ("G.t5", 1, 32, 64, 8, 4, 2, 1)]


@pytest.fixture(scope="module", autouse=True)
def _init():
    global H
    import paper_2102_02344_b200.hfta as hfta
    hfta.hfta_init(0)
    H = hfta


def s():
    return torch.cuda.current_stream().cuda_stream


def rnd(a, tdt):
    return torch.tensor(a).to(tdt).double().numpy()


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def run_layer(layer, B, N, dtype, shared, seed=0, act=0, alpha=0.0):
    name, tr, Hs, Ci, Co, k, st, pd = layer
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    code = 1 if dtype == "bf16" else 0
    rng = np.random.default_rng(seed)
    Ho = (Hs - 1) * st - 2 * pd + k if tr else (Hs + 2 * pd - k) // st + 1
    nb = 1 if shared else B
    X = rnd(rng.standard_normal((nb, N, Hs, Hs, Ci)), tdt)                       # NHWC
    if tr:    # ConvT weight, arena layout [kh][kw][Co][Ci]; torch [Ci][Co][kh][kw]
        Wg = rnd(rng.standard_normal((B, k, k, Co, Ci)) / np.sqrt(Ci), tdt)
        Wt = Wg.transpose(0, 4, 3, 1, 2)
        wld = Ci
    else:     # Conv weight, arena layout [Co][kh][kw][Ci]; torch [Co][Ci][kh][kw]
        Wg = rnd(rng.standard_normal((B, Co, k, k, Ci)) / np.sqrt(k * k * Ci), tdt)
        Wt = Wg.transpose(0, 1, 4, 2, 3)
        wld = k * k * Ci
    dY = rnd(rng.standard_normal((B, N, Ho, Ho, Co)), tdt)
    dW0 = rng.standard_normal(Wg.shape).astype(np.float32).astype(np.float64)

    d = H.hfta_conv_desc()
    d.N, d.H, d.W, d.C_in, d.C_out, d.kh, d.kw, d.stride, d.pad, d.transposed = N, Hs, Hs, Ci, Co, k, k, st, pd, tr
    dev = lambda a: torch.tensor(a).to(tdt).to(DEV).contiguous()
    Xd, Wd, dYd = dev(X), dev(Wg), dev(dY)
    Y = torch.empty(B, N, Ho, Ho, Co, dtype=tdt, device=DEV)
    dX = torch.empty(B, N, Hs, Hs, Ci, dtype=tdt, device=DEV)
    dW = torch.tensor(dW0, dtype=torch.float32, device=DEV).contiguous()
    ws = torch.empty(max(H.hfta_fused_conv_workspace(B, d, code), 256), dtype=torch.uint8, device=DEV)
    xbs = 0 if shared else N * Hs * Hs * Ci
    wbs = int(np.prod(Wg.shape[1:]))
    H.hfta_fused_conv_fwd(B, d, code, H.tin(Xd, xbs, Ci), H.tin(Wd, wbs, wld), H.tout(Y, N * Ho * Ho * Co, Co),
                          act, alpha, H.ptr(ws), ws.numel(), s())
    H.hfta_fused_conv_bwd(B, d, code, H.tin(dYd, N * Ho * Ho * Co, Co), H.tin(Xd, xbs, Ci), H.tin(Wd, wbs, wld),
                          H.tout(dX, N * Hs * Hs * Ci, Ci), H.ptr(dW), wbs, 1, H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    return dict(X=X, Wt=Wt, dY=dY, dW0=dW0, Y=host(Y), dX=host(dX), dW=host(dW), Ho=Ho)


def check(layer, B, N, dtype, shared, act=0, alpha=0.0):
    name, tr, Hs, Ci, Co, k, st, pd = layer
    r = run_layer(layer, B, N, dtype, shared, act=act, alpha=alpha)
    tol_o = 1e-2 if dtype == "bf16" else 1e-4
    tol_w = 1e-4
    for b in range(B):
        xb = r["X"][0 if shared else b].transpose(0, 3, 1, 2)          # NCHW
        dyb = r["dY"][b].transpose(0, 3, 1, 2)
        Wt = r["Wt"][b]
        if tr:
            y = OL.convT2d_fwd(xb, Wt, st, pd)
            dx, dw = OL.convT2d_bwd(dyb, xb, Wt, st, pd)
            dw_g = dw.transpose(2, 3, 1, 0)                            # [Ci][Co][kh][kw] -> [kh][kw][Co][Ci]
        else:
            y = OL.conv2d_fwd(xb, Wt, st, pd)
            dx, dw = OL.conv2d_bwd(dyb, xb, Wt, st, pd)
            dw_g = dw.transpose(0, 2, 3, 1)                            # [Co][Ci][kh][kw] -> [Co][kh][kw][Ci]
        if act == H.ACT_LEAKY_RELU:
            y = OL.leaky_relu(y, alpha)
        elif act == H.ACT_TANH:
            y = OL.tanh(y)
        assert_close(r["Y"][b], y.transpose(0, 2, 3, 1), tol_o, "%s model %d Y" % (name, b))
        assert_close(r["dX"][b], dx.transpose(0, 2, 3, 1), tol_o, "%s model %d dX" % (name, b))
        assert_close(r["dW"][b], r["dW0"][b] + dw_g, tol_w, "%s model %d dW (accumulate)" % (name, b))


@pytest.mark.parametrize("layer", LAYERS, ids=[l[0] for l in LAYERS])
@pytest.mark.parametrize("B", [1, 3])
def test_conv_layer_bf16_full_batch(layer, B):
    """Every DCGAN layer at N = 128 (the bench's batch); D layers with the
    shared input image when B = 3."""
    check(layer, B, 128, "bf16", shared=(B == 3 and layer[0].startswith("D")))


@pytest.mark.parametrize("layer", LAYERS, ids=[l[0] for l in LAYERS])
def test_conv_layer_f32(layer):
    """fp32 (patch-matrix path), N = 8, B = 2, per-model inputs."""
    check(layer, 2, 8, "f32", shared=False)


def test_conv_layer_bf16_per_model_inputs():
    """Implicit-GEMM modes with per-model (non-shared) images, B = 2, N = 32."""
    for layer in LAYERS:
        if layer[0] in ("D.c2", "D.c3", "D.c4", "G.t2", "G.t3", "G.t4", "G.t5"):
            check(layer, 2, 32, "bf16", shared=False)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_conv_fused_activation(dtype):
    """The activation of a layer without BN applied by hfta_fused_conv_fwd:
    D c1 -> LeakyReLU(0.2), G t5 -> Tanh (in the implicit-GEMM epilogue in
    bf16, a separate pass in fp32), N = 32, B = 2."""
    check(LAYERS[0], 2, 32, dtype, shared=False, act=H.ACT_LEAKY_RELU, alpha=0.2)
    check(LAYERS[9], 2, 32, dtype, shared=False, act=H.ACT_TANH, alpha=0.0)


# ResNet-18 family (NEXT-4) layers at the bench's batch (N = 128 images of
# 32 x 32): the general gather modes (kernel 7 / 3 / 1, stride 1 / 2, pad 3 /
# 1 / 0), the flipped-weight stride-1 dgrad, the patch-matrix dgrads of the
# strided 3x3 / 1x1 layers, the 8-channel stem.
RESNET = [("R.stem", 0, 32, 8, 64, 7, 2, 3),
          ("R.l1", 0, 8, 64, 64, 3, 1, 1),
          ("R.l2a", 0, 8, 64, 128, 3, 2, 1),
          ("R.l2d", 0, 8, 64, 128, 1, 2, 0),
          ("R.l3", 0, 2, 256, 256, 3, 1, 1),
          ("R.l4", 0, 1, 512, 512, 3, 1, 1)]


@pytest.mark.parametrize("layer", RESNET, ids=[l[0] for l in RESNET])
@pytest.mark.parametrize("B", [1, 3])
def test_resnet_conv_bf16(layer, B):
    check(layer, B, 128, "bf16", shared=(B == 3 and layer[0] == "R.stem"))


@pytest.mark.parametrize("layer", RESNET, ids=[l[0] for l in RESNET])
def test_resnet_conv_f32(layer):
    check(layer, 2, 8, "f32", shared=False)


@pytest.mark.parametrize("layer,act,alpha", [(LAYERS[1], "leaky", 0.2), (RESNET[1], "relu", 0.0),
                                             (LAYERS[2], "relu", 0.0)], ids=["D.c2-leaky", "R.l1-relu", "D.c3-relu"])
def test_conv_bwd_gated(layer, act, alpha):
    """hfta_fused_conv_bwd_gated: dX *= act'(gate) -- fused into the sub-pixel
    dgrad epilogue (D c2 / c3), a separate pass on the other paths (R.l1)."""
    name, tr, Hs, Ci, Co, k, st, pd = layer
    B, N = 2, 32
    code = H.ACT_LEAKY_RELU if act == "leaky" else H.ACT_RELU
    rng = np.random.default_rng(11)
    Ho = (Hs + 2 * pd - k) // st + 1
    X = rnd(rng.standard_normal((B, N, Hs, Hs, Ci)), torch.bfloat16)
    Wg = rnd(rng.standard_normal((B, Co, k, k, Ci)) / np.sqrt(k * k * Ci), torch.bfloat16)
    dY = rnd(rng.standard_normal((B, N, Ho, Ho, Co)), torch.bfloat16)
    G = rnd(rng.standard_normal((B, N, Hs, Hs, Ci)), torch.bfloat16)
    d = H.hfta_conv_desc()
    d.N, d.H, d.W, d.C_in, d.C_out, d.kh, d.kw, d.stride, d.pad, d.transposed = N, Hs, Hs, Ci, Co, k, k, st, pd, tr
    dev = lambda a: torch.tensor(a).to(torch.bfloat16).to(DEV).contiguous()
    Xd, Wd, dYd, Gd = dev(X), dev(Wg), dev(dY), dev(G)
    dX = torch.empty(B, N, Hs, Hs, Ci, dtype=torch.bfloat16, device=DEV)
    ws = torch.empty(max(H.hfta_fused_conv_workspace(B, d, 1), 256), dtype=torch.uint8, device=DEV)
    xe = N * Hs * Hs * Ci
    wbs = int(np.prod(Wg.shape[1:]))
    H.hfta_fused_conv_bwd_gated(B, d, 1, H.tin(dYd, N * Ho * Ho * Co, Co), H.tin(Xd, xe, Ci),
                                H.tin(Wd, wbs, k * k * Ci), H.tout(dX, xe, Ci), None, wbs, 0, code, alpha,
                                H.tin(Gd, xe, Ci), H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    for b in range(B):
        dx, _ = OL.conv2d_bwd(dY[b].transpose(0, 3, 1, 2), X[b].transpose(0, 3, 1, 2), Wg[b].transpose(0, 3, 1, 2),
                              st, pd)
        ref = dx.transpose(0, 2, 3, 1) * np.where(G[b] > 0, 1.0, alpha)
        assert_close(host(dX)[b], ref, 1e-2, "%s gated dX model %d" % (name, b))


@pytest.mark.parametrize("layer", [LAYERS[2], RESNET[2], RESNET[1], LAYERS[7], LAYERS[6], LAYERS[5], RESNET[0]],
                         ids=["D.c3", "R.l2a", "R.l1", "G.t3-phases", "G.t2-phases", "G.t1-dense", "R.stem-narrow"])
def test_conv_fwd_stats(layer):
    """hfta_fused_conv_fwd_stats: the same Y as hfta_fused_conv_fwd and the
    per-32-row column sums / sums of squares of the stored Y (from the
    implicit-GEMM epilogue, or one pass over Y on the other paths)."""
    name, tr, Hs, Ci, Co, k, st, pd = layer
    B, N = 2, 32
    rng = np.random.default_rng(5)
    Ho = (Hs - 1) * st - 2 * pd + k if tr else (Hs + 2 * pd - k) // st + 1
    X = rnd(rng.standard_normal((B, N, Hs, Hs, Ci)), torch.bfloat16)
    shp = (B, k, k, Co, Ci) if tr else (B, Co, k, k, Ci)
    Wg = rnd(rng.standard_normal(shp) / np.sqrt(k * k * Ci), torch.bfloat16)
    d = H.hfta_conv_desc()
    d.N, d.H, d.W, d.C_in, d.C_out, d.kh, d.kw, d.stride, d.pad, d.transposed = N, Hs, Hs, Ci, Co, k, k, st, pd, tr
    dev = lambda a: torch.tensor(a).to(torch.bfloat16).to(DEV).contiguous()
    Xd, Wd = dev(X), dev(Wg)
    Y1 = torch.empty(B, N, Ho, Ho, Co, dtype=torch.bfloat16, device=DEV)
    Y2 = torch.empty_like(Y1)
    ws = torch.empty(max(H.hfta_fused_conv_workspace(B, d, 1), 256), dtype=torch.uint8, device=DEV)
    R = N * Ho * Ho
    cs = torch.empty(H.hfta_linear_colstat_size(B, R, Co) // 4, dtype=torch.float32, device=DEV)
    wbs, wld = int(np.prod(Wg.shape[1:])), (Ci if tr else k * k * Ci)
    xe = N * Hs * Hs * Ci
    H.hfta_fused_conv_fwd(B, d, 1, H.tin(Xd, xe, Ci), H.tin(Wd, wbs, wld), H.tout(Y1, R * Co, Co), 0, 0.0,
                          H.ptr(ws), ws.numel(), s())
    H.hfta_fused_conv_fwd_stats(B, d, 1, H.tin(Xd, xe, Ci), H.tin(Wd, wbs, wld), H.tout(Y2, R * Co, Co), H.ptr(cs),
                                H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    y = host(Y2).reshape(B, R, Co)
    nblk = (R + 31) // 32
    c = cs.view(B, nblk, 2, Co).double().cpu().numpy()
    for b in range(B):
        # the blocks partition the R rows (the sub-pixel phases order them by phase): totals
        np.testing.assert_allclose(c[b, :, 0].sum(0), y[b].sum(0), rtol=1e-5, atol=1e-3)
        np.testing.assert_allclose(c[b, :, 1].sum(0), (y[b] * y[b]).sum(0), rtol=1e-5, atol=1e-3)
        if not tr:       # Conv2d / fallback: block k = output rows 32k .. 32k + 31
            for kb in (0, nblk // 3, nblk - 1):
                rows = y[b, 32 * kb:min(R, 32 * kb + 32)]
                np.testing.assert_allclose(c[b, kb, 0], rows.sum(0), rtol=1e-5, atol=1e-4)
                np.testing.assert_allclose(c[b, kb, 1], (rows * rows).sum(0), rtol=1e-5, atol=1e-4)
