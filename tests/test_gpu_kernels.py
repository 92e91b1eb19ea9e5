"""Per-kernel parity of libhfta (through the C ABI) against the oracle's layer
definitions on the same seeded inputs.  Sizes span several tiles with a
ragged tail; B in {1, 3}; shared inputs use bstride 0."""
import numpy as np
import pytest
import torch

from oracle import layers as OL
from oracle.adam import adam_step
from oracle.philox import dropout_keep_mask
from tests._cmp import assert_close, relerr

pytestmark = pytest.mark.gpu

H = None
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _init():
    global H
    import paper_2102_02344_b200.hfta as hfta
    hfta.hfta_init(0)
    H = hfta


R = np.random.default_rng(2024)
DT = {"f32": (0, torch.float32), "bf16": (1, torch.bfloat16)}


def dev(a, tdt=torch.float32):
    return torch.tensor(np.asarray(a), dtype=torch.float64).to(tdt).to(DEV).contiguous()


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def rounded(a, tdt):
    """The value the device sees after storing a in tdt."""
    return torch.tensor(a).to(tdt).double().numpy()


def s():
    return torch.cuda.current_stream().cuda_stream


# ----------------------------------------------------------------- linear ----
# (M, N, K): K < 16 / N < 16 / unaligned shapes take the SIMT kernel; the rest
# (bf16) the tcgen05 kernel, including ragged M / N tails and MN-major operands.
SHAPES = [(300, 64, 3), (1000, 128, 64), (257, 200, 136), (32, 9, 256), (37, 40, 256), (130, 3, 64),
          (2000, 1024, 128), (1500, 128, 1024), (640, 256, 512), (999, 64, 128),
          (2000, 48, 64), (1000, 64, 48), (700, 16, 80),       # ragged MN-major extents (TMA OOB boxes)
          (300, 1, 2048), (200, 2, 5), (130, 7, 300)]          # tiny N: GEMV fwd, small-K dgrad, small-M wgrad


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("B,shared", [(1, False), (3, False), (3, True)])
def test_linear_fwd_bwd(dt, M, N, K, B, shared):
    code, tdt = DT[dt]
    X = rounded(R.standard_normal((1 if shared else B, M, K)), tdt)
    W = rounded(R.standard_normal((B, N, K)) / np.sqrt(K), tdt)
    bias = R.standard_normal((B, N)).astype(np.float32).astype(np.float64)
    dY = rounded(R.standard_normal((B, M, N)), tdt)
    Xd, Wd, bd, dYd = dev(X, tdt), dev(W, tdt), dev(bias), dev(dY, tdt)
    Y = torch.empty(B, M, N, dtype=tdt, device=DEV)
    xbs = 0 if shared else M * K
    H.hfta_fused_linear_fwd(B, M, N, K, code, H.tin(Xd, xbs, K), H.tin(Wd, N * K, K), H.ptr(bd), N, 0, 0,
                            H.tout(Y, M * N, N), s())
    dX = torch.empty(B, M, K, dtype=tdt, device=DEV)
    dW = torch.empty(B, N, K, device=DEV)
    db = torch.empty(B, N, device=DEV)
    ws = torch.empty(max(H.hfta_fused_linear_bwd_workspace(B, M, N, K, code), 1), dtype=torch.uint8, device=DEV)
    H.hfta_fused_linear_bwd(B, M, N, K, code, H.tin(dYd, M * N, N), H.tin(Xd, xbs, K), H.tin(Wd, N * K, K),
                            H.tout(dX, M * K, K), H.ptr(dW), N * K, K, H.ptr(db), N, 0, H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    tol = 1e-5 if dt == "f32" else 1e-2
    for b in range(B):
        xb = X[0 if shared else b]
        y = OL.linear_fwd(xb, W[b], bias[b])
        dx, dw, dbb = OL.linear_bwd(dY[b], xb, W[b])
        assert_close(host(Y[b]), y, tol, "Y")
        assert_close(host(dX[b]), dx, tol, "dX")
        # fp32 wgrad reduces over M (up to 2000 rows here) in the tensor cores' fp32
        # accumulator (3xTF32): ~1.5e-5 at M = 2000, gated at the north_star's 1e-4
        assert_close(host(dW[b]), dw, 1e-4, "dW")
        assert_close(host(db[b]), dbb, 1e-5, "dbias")


@pytest.mark.parametrize("M,N,K,B", [(32, 512, 1024, 3), (32, 40, 256, 2), (32, 9, 256, 2), (77, 64, 96, 2)])
def test_linear_bf16_f32(M, N, K, B):
    """HFTA_BF16_F32 (reading R16b): bf16 X, W, dY operands, fp32 Y and dX --
    the per-sample FC head's contraction in bf16 mode (tensor cores where
    N, K >= 16, SIMT otherwise).  Outputs are compared with the oracle on
    the same bf16-rounded operands at fp32-accumulation tolerance."""
    X = rounded(R.standard_normal((B, M, K)), torch.bfloat16)
    W = rounded(R.standard_normal((B, N, K)) / np.sqrt(K), torch.bfloat16)
    bias = R.standard_normal((B, N)).astype(np.float32).astype(np.float64)
    dY = rounded(R.standard_normal((B, M, N)), torch.bfloat16)
    Xd, Wd, bd, dYd = dev(X, torch.bfloat16), dev(W, torch.bfloat16), dev(bias), dev(dY, torch.bfloat16)
    Y = torch.empty(B, M, N, device=DEV)
    H.hfta_fused_linear_fwd(B, M, N, K, H.HFTA_BF16_F32, H.tin(Xd, M * K, K), H.tin(Wd, N * K, K), H.ptr(bd), N, 0, 0,
                            H.tout(Y, M * N, N), s())
    dX = torch.empty(B, M, K, device=DEV)
    dW = torch.empty(B, N, K, device=DEV)
    db = torch.empty(B, N, device=DEV)
    code = H.HFTA_BF16_F32
    ws = torch.empty(max(H.hfta_fused_linear_bwd_workspace(B, M, N, K, code), 1), dtype=torch.uint8, device=DEV)
    H.hfta_fused_linear_bwd(B, M, N, K, code, H.tin(dYd, M * N, N), H.tin(Xd, M * K, K), H.tin(Wd, N * K, K),
                            H.tout(dX, M * K, K), H.ptr(dW), N * K, K, H.ptr(db), N, 0, H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    assert Y.dtype == torch.float32 and dX.dtype == torch.float32
    for b in range(B):
        y = OL.linear_fwd(X[b], W[b], bias[b])
        dx, dw, dbb = OL.linear_bwd(dY[b], X[b], W[b])
        assert_close(host(Y[b]), y, 1e-5, "Y (fp32 out)")
        assert_close(host(dX[b]), dx, 1e-5, "dX (fp32 out)")
        assert_close(host(dW[b]), dw, 1e-5, "dW")
        assert_close(host(db[b]), dbb, 1e-5, "dbias")


@pytest.mark.parametrize("N", [40, 50, 56])
def test_linear_wgrad_ragged_rows_padded_ld(N):
    """bf16 wgrad with an output-feature count that is not a multiple of 16
    (the seg classifier: k = 50) and dY rows padded to a 16-B pitch: the
    MN-major A tile of the tensor-core wgrad is partly out of bounds
    (zero-filled by TMA).  dW, dbias vs the oracle on the same operands."""
    B, M, K, ldy = 2, 3000, 128, 64
    X = rounded(R.standard_normal((B, M, K)), torch.bfloat16)
    W = rounded(R.standard_normal((B, N, K)) / np.sqrt(K), torch.bfloat16)
    dY = np.zeros((B, M, ldy))
    dY[:, :, :N] = rounded(R.standard_normal((B, M, N)), torch.bfloat16)
    Xd, Wd, dYd = dev(X, torch.bfloat16), dev(W, torch.bfloat16), dev(dY, torch.bfloat16)
    dW = torch.empty(B, N, K, device=DEV)
    db = torch.empty(B, N, device=DEV)
    ws = torch.empty(max(H.hfta_fused_linear_bwd_workspace(B, M, N, K, 1), 1), dtype=torch.uint8, device=DEV)
    H.hfta_fused_linear_bwd(B, M, N, K, 1, H.tin(dYd, M * ldy, ldy), H.tin(Xd, M * K, K), H.tin(Wd, N * K, K),
                            H.tout(None, 0, 1), H.ptr(dW), N * K, K, H.ptr(db), N, 0, H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    for b in range(B):
        _, dw, dbb = OL.linear_bwd(dY[b][:, :N], X[b], W[b])
        assert_close(host(dW[b]), dw, 1e-5, "dW")
        assert_close(host(db[b]), dbb, 1e-5, "dbias")


def test_linear_bwd_accumulate_and_rowgroup_bias():
    B, M, N, K, L = 2, 500, 48, 32, 125
    X = R.standard_normal((B, M, K)).astype(np.float32).astype(np.float64)
    W = R.standard_normal((B, N, K)).astype(np.float32).astype(np.float64)
    tab = R.standard_normal((B, M // L, N)).astype(np.float32).astype(np.float64)
    Y = torch.empty(B, M, N, device=DEV)
    Xd, Wd, tabd = dev(X), dev(W), dev(tab)      # keep references: the launch is asynchronous
    H.hfta_fused_linear_fwd(B, M, N, K, 0, H.tin(Xd, M * K, K), H.tin(Wd, N * K, K), H.ptr(tabd),
                            (M // L) * N, N, L, H.tout(Y, M * N, N), s())
    dY = R.standard_normal((B, M, N)).astype(np.float32).astype(np.float64)
    dW0 = R.standard_normal((B, N, K)).astype(np.float32).astype(np.float64)
    dW, dYd = dev(dW0), dev(dY)
    ws = torch.empty(max(H.hfta_fused_linear_bwd_workspace(B, M, N, K, 0), 1), dtype=torch.uint8, device=DEV)
    H.hfta_fused_linear_bwd(B, M, N, K, 0, H.tin(dYd, M * N, N), H.tin(Xd, M * K, K),
                            H.tin(Wd, N * K, K), H.tout(None, 0, 1), H.ptr(dW), N * K, K, None, 0, 1,
                            H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    for b in range(B):
        ref = X[b] @ W[b].T + np.repeat(tab[b], L, axis=0)
        assert_close(host(Y[b]), ref, 1e-5, "row-group bias")
        assert_close(host(dW[b]), dW0[b] + dY[b].T @ X[b], 1e-5, "accumulate")


def test_linear_errors():
    with pytest.raises(H.HftaError) as e:
        H.hfta_fused_linear_fwd(0, 4, 4, 4, 0, H.hfta_in(None, 0, 4), H.hfta_in(None, 0, 4), None, 0, 0, 0,
                                H.hfta_out(None, 0, 4), s())
    assert e.value.code == 1
    x = torch.zeros(4, 4, device=DEV)
    with pytest.raises(H.HftaError) as e:
        H.hfta_fused_linear_fwd(1, 4, 4, 8, 0, H.tin(x, 0, 4), H.tin(x, 0, 4), None, 0, 0, 0, H.tout(x, 16, 4), s())
    assert e.value.code == 2 and "ld" in str(e.value)


# -------------------------------------------------------------------- BN ----
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("Rr,C,act", [(5000, 64, 1), (1000, 1024, 0), (32, 512, 1), (777, 48, 2), (300, 9, 1)])
def test_bn_fwd_bwd(dt, Rr, C, act):
    code, tdt = DT[dt]
    B = 3
    X = rounded(R.standard_normal((B, Rr, C)) * 2 + 3, tdt)
    g = R.uniform(0.5, 1.5, (B, C)).astype(np.float32).astype(np.float64)
    be = R.uniform(-0.5, 0.5, (B, C)).astype(np.float32).astype(np.float64)
    dY = rounded(R.standard_normal((B, Rr, C)), tdt)
    rm0, rv0 = R.standard_normal((B, C)).astype(np.float32), R.uniform(0.5, 2, (B, C)).astype(np.float32)
    Xd, gd, bed = dev(X, tdt), dev(g), dev(be)
    rm, rv = dev(rm0), dev(rv0)
    Y = torch.empty(B, Rr, C, dtype=tdt, device=DEV)
    sm, si = torch.empty(B, C, device=DEV), torch.empty(B, C, device=DEV)
    ws = torch.empty(H.hfta_fused_bn_workspace(B, Rr, C), dtype=torch.uint8, device=DEV)
    H.hfta_fused_bn_fwd(B, Rr, C, code, H.tin(Xd, Rr * C, C), H.ptr(gd), H.ptr(bed), C, H.ptr(rm), H.ptr(rv), 0.1,
                        1e-5, act, 0.2, H.tout(Y, Rr * C, C), H.ptr(sm), H.ptr(si), H.ptr(ws), ws.numel(), s())
    dX = torch.empty(B, Rr, C, dtype=tdt, device=DEV)
    dg, db = torch.empty(B, C, device=DEV), torch.empty(B, C, device=DEV)
    H.hfta_fused_bn_bwd(B, Rr, C, code, H.tin(dev(dY, tdt), Rr * C, C), H.tin(Xd, Rr * C, C), H.ptr(gd), H.ptr(bed),
                        C, H.ptr(sm), H.ptr(si), act, 0.2, H.tout(dX, Rr * C, C), H.ptr(dg), H.ptr(db), 0, H.ptr(ws),
                        ws.numel(), s())
    torch.cuda.synchronize()
    actf = {0: (lambda z: z, lambda d, z: d), 1: (OL.relu, OL.relu_bwd),
            2: (lambda z: OL.leaky_relu(z, 0.2), lambda d, z: OL.leaky_relu_bwd(d, z, 0.2))}[act]
    tol = 1e-5 if dt == "f32" else 1e-2
    for b in range(B):
        z, c = OL.bn_fwd(X[b], g[b], be[b])
        assert_close(host(Y[b]), actf[0](z), tol, "Y")
        rmr, rvr = OL.bn_running(rm0[b].astype(np.float64), rv0[b].astype(np.float64), c, Rr)
        assert_close(host(rm[b]), rmr, 1e-6, "running_mean")
        assert_close(host(rv[b]), rvr, 1e-6, "running_var")
        assert_close(host(sm[b]), c["mean"], 1e-6, "save_mean")
        assert_close(host(si[b]), c["invstd"], 1e-6, "save_invstd")
        dx, dgr, dbr = OL.bn_bwd(actf[1](dY[b], z), c, g[b])
        assert_close(host(dg[b]), dgr, 1e-5 if dt == "f32" else 1e-3, "dgamma")
        assert_close(host(db[b]), dbr, 1e-5 if dt == "f32" else 1e-3, "dbeta")
        assert_close(host(dX[b]), dx, 1e-4 if dt == "f32" else 2e-2, "dX")


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("act", [0, 1])
def test_bn_max_fwd_bwd(dt, act):
    code, tdt = DT[dt]
    B, N, L, C = 2, 3, 700, 136
    Rr = N * L
    X = rounded(R.standard_normal((B, Rr, C)), tdt)
    g = R.uniform(0.5, 1.5, (B, C)).astype(np.float32).astype(np.float64)
    be = R.uniform(-0.5, 0.5, (B, C)).astype(np.float32).astype(np.float64)
    Xd, gd, bed = dev(X, tdt), dev(g), dev(be)
    sm, si = torch.empty(B, C, device=DEV), torch.empty(B, C, device=DEV)
    ws = torch.empty(max(H.hfta_fused_bn_workspace(B, Rr, C), H.hfta_bn_max_bwd_workspace(B, N, C)),
                     dtype=torch.uint8, device=DEV)
    H.hfta_fused_bn_fwd(B, Rr, C, code, H.tin(Xd, Rr * C, C), H.ptr(gd), H.ptr(bed), C, None, None, 0.1, 1e-5, act,
                        0.0, H.tout(None, 0, 1), H.ptr(sm), H.ptr(si), H.ptr(ws), ws.numel(), s())
    G = torch.empty(B, N, C, device=DEV)                   # per-sample tensors are fp32
    am = torch.empty(B, N, C, dtype=torch.int32, device=DEV)
    H.hfta_bn_max_fwd(B, N, L, C, code, H.tin(Xd, Rr * C, C), H.ptr(gd), H.ptr(bed), C, H.ptr(sm), H.ptr(si), act,
                      0.0, H.tout(G, N * C, C), H.ptr(am), s())
    dG = R.standard_normal((B, N, C)).astype(np.float32).astype(np.float64)
    dGd = dev(dG)
    dX = torch.empty(B, Rr, C, dtype=tdt, device=DEV)
    dg, db = torch.empty(B, C, device=DEV), torch.empty(B, C, device=DEV)
    H.hfta_bn_max_bwd(B, N, L, C, code, H.tin(dGd, N * C, C), H.tin(Xd, Rr * C, C), H.ptr(am), H.ptr(gd),
                      H.ptr(bed), C, H.ptr(sm), H.ptr(si), act, 0.0, H.tout(dX, Rr * C, C), H.ptr(dg), H.ptr(db),
                      H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    for b in range(B):
        z, c = OL.bn_fwd(X[b], g[b], be[b])
        a = OL.relu(z) if act else z
        gmax, idx = OL.max_over_points(a.reshape(N, L, C))
        if dt == "f32":
            assert np.array_equal(host(am[b]).astype(np.int64), idx)
        assert_close(host(G[b]), gmax, 1e-5 if dt == "f32" else 1e-3, "max")
        da = OL.max_over_points_bwd(dG[b], host(am[b]).astype(np.int64), L).reshape(Rr, C)
        dz = OL.relu_bwd(da, z) if act else da
        dx, dgr, dbr = OL.bn_bwd(dz, c, g[b])
        assert_close(host(dX[b]), dx, 1e-4 if dt == "f32" else 2e-2, "dX")
        assert_close(host(dg[b]), dgr, 1e-4 if dt == "f32" else 2e-2, "dgamma")
        assert_close(host(db[b]), dbr, 1e-4 if dt == "f32" else 2e-2, "dbeta")


# ------------------------------------------------------------------ glue ----
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_transform_points(dt):
    code, tdt = DT[dt]
    B, N, L = 3, 4, 333
    x = R.standard_normal((N, L, 3)).astype(np.float32).astype(np.float64)
    F = R.standard_normal((B, N, 9)).astype(np.float32).astype(np.float64) * 0.1
    Y = torch.empty(B, N * L, 3, dtype=tdt, device=DEV)
    xd, Fd = dev(x.reshape(N * L, 3)), dev(F)
    H.hfta_transform_points_fwd(B, N, L, code, H.tin(xd, 0, 3), H.tin(Fd, N * 9, 9), 1,
                                H.tout(Y, N * L * 3, 3), s())
    dY = rounded(R.standard_normal((B, N * L, 3)), tdt)
    dF = torch.empty(B, N, 9, device=DEV)
    H.hfta_transform_points_bwd(B, N, L, code, H.tin(xd, 0, 3), H.tin(dev(dY, tdt), N * L * 3, 3),
                                H.tout(dF, N * 9, 9), s())
    torch.cuda.synchronize()
    for b in range(B):
        T = F[b].reshape(N, 3, 3) + np.eye(3)
        assert_close(host(Y[b]).reshape(N, L, 3), OL.transform_points(x, T), 1e-6 if dt == "f32" else 1e-2, "x'")
        _, dT = OL.transform_points_bwd(dY[b].reshape(N, L, 3), x, T)
        assert_close(host(dF[b]).reshape(N, 3, 3), dT, 1e-5, "dT")


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_dropout_mask_bit_exact(dt):
    code, tdt = DT[dt]
    B, rows, cols, p = 3, 32, 257, 0.3
    X = rounded(R.standard_normal((B, rows, cols)), tdt)
    Y = torch.empty(B, rows, cols, dtype=tdt, device=DEV)
    H.hfta_dropout_fwd(B, rows, cols, code, H.tin(dev(X, tdt), rows * cols, cols), H.tout(Y, rows * cols, cols), 42,
                       5, None, 0, p, 0, None, s())
    # the same mask when the step comes from a device counter (graph-capturable form): 4 + 1
    Y2 = torch.empty_like(Y)
    stepd = torch.tensor([4], dtype=torch.int64, device=DEV)
    H.hfta_dropout_fwd(B, rows, cols, code, H.tin(dev(X, tdt), rows * cols, cols), H.tout(Y2, rows * cols, cols), 42,
                       1, H.ptr(stepd), 0, p, 0, None, s())
    torch.cuda.synchronize()
    assert torch.equal(Y, Y2)
    torch.cuda.synchronize()
    for b in range(B):
        keep = dropout_keep_mask(42, b, 5, 0, rows * cols, p).reshape(rows, cols)
        got = host(Y[b])
        assert np.array_equal(got != 0, keep & (X[b] != 0))
        assert_close(got, OL.dropout(X[b], keep, np.float32(p)), 1e-6 if dt == "f32" else 1e-2, "dropout")


def test_dropout_sharded_masks_equal_unsharded():
    """A model-array shard (ranks own contiguous model blocks)
    passes its first global model index: its masks equal the masks the same
    models draw in an unsharded run and the oracle's for the global index."""
    B, rows, cols, p = 6, 16, 100, 0.3
    X = rounded(R.standard_normal((B, rows, cols)), torch.float32)
    full = torch.empty(B, rows, cols, device=DEV)
    H.hfta_dropout_fwd(B, rows, cols, 0, H.tin(dev(X), rows * cols, cols), H.tout(full, rows * cols, cols), 42,
                       3, None, 0, p, 0, None, s())
    for lo, hi in ((0, 2), (2, 4), (4, 6)):                 # 3 "ranks"
        part = torch.empty(hi - lo, rows, cols, device=DEV)
        H.hfta_dropout_fwd(hi - lo, rows, cols, 0, H.tin(dev(X[lo:hi]), rows * cols, cols),
                           H.tout(part, rows * cols, cols), 42, 3, None, 0, p, lo, None, s())
        torch.cuda.synchronize()
        assert torch.equal(part, full[lo:hi])
        for b in range(lo, hi):
            keep = dropout_keep_mask(42, b, 3, 0, rows * cols, p).reshape(rows, cols)
            assert np.array_equal(host(part[b - lo]) != 0, keep & (X[b] != 0))


def test_dropout_explicit_model_ids():
    """Per-model ids (an HFHT partition of non-contiguous hyper-parameter
    sets): model b draws the mask of id[b]."""
    B, rows, cols, p = 3, 8, 64, 0.3
    ids = [7, 2, 11]
    X = rounded(R.standard_normal((B, rows, cols)), torch.float32)
    Y = torch.empty(B, rows, cols, device=DEV)
    idd = torch.tensor(ids, dtype=torch.int32, device=DEV)
    H.hfta_dropout_fwd(B, rows, cols, 0, H.tin(dev(X), rows * cols, cols), H.tout(Y, rows * cols, cols), 42,
                       2, None, 0, p, 0, H.ptr(idd), s())
    torch.cuda.synchronize()
    for b in range(B):
        keep = dropout_keep_mask(42, ids[b], 2, 0, rows * cols, p).reshape(rows, cols)
        assert np.array_equal(host(Y[b]) != 0, keep & (X[b] != 0))


@pytest.mark.parametrize("K", [50, 40, 7])
def test_loss_nll_padded_rows(K):
    """bf16 NLL with 16-B padded rows (the seg classifier's layout, ld = 64):
    the thread-per-row kernel; loss, mean and dlogits vs the oracle."""
    B, rows, ld = 3, 1000, 64
    Z = np.zeros((B, rows, ld))
    Z[:, :, :K] = rounded(R.standard_normal((B, rows, K)) * 3, torch.bfloat16)
    y = R.integers(0, K, rows)
    loss, ml = torch.empty(B, device=DEV), torch.empty(1, device=DEV)
    dZ = torch.zeros(B, rows, ld, dtype=torch.bfloat16, device=DEV)
    ws = torch.empty(H.hfta_loss_workspace(B, rows), dtype=torch.uint8, device=DEV)
    Zd, yd = dev(Z, torch.bfloat16), dev(y, torch.int32)
    H.hfta_loss_nll(B, rows, K, 1, H.tin(Zd, rows * ld, ld), H.ptr(yd), 0, H.ptr(loss),
                    H.ptr(ml), H.tout(dZ, rows * ld, ld), H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    refs = []
    for b in range(B):
        l, dz = OL.nll_mean(Z[b][:, :K], y)
        refs.append(l)
        assert abs(host(loss)[b] - l) <= 1e-5 * abs(l)
        assert_close(host(dZ[b])[:, :K], dz, 1e-2, "dlogits")
    assert abs(host(ml)[0] - np.mean(refs)) <= 1e-5 * abs(np.mean(refs))


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_loss_nll_mse(dt):
    code, tdt = DT[dt]
    B, rows, K = 3, 300, 50
    Z = rounded(R.standard_normal((B, rows, K)) * 3, tdt)
    y = R.integers(0, K, rows)
    loss, ml = torch.empty(B, device=DEV), torch.empty(1, device=DEV)
    dZ = torch.empty(B, rows, K, dtype=tdt, device=DEV)
    ws = torch.empty(H.hfta_loss_workspace(B, rows), dtype=torch.uint8, device=DEV)
    Zd, yd = dev(Z, tdt), dev(y, torch.int32)
    H.hfta_loss_nll(B, rows, K, code, H.tin(Zd, rows * K, K), H.ptr(yd), 0, H.ptr(loss),
                    H.ptr(ml), H.tout(dZ, rows * K, K), H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    refs = []
    for b in range(B):
        l, dz = OL.nll_mean(Z[b], y)
        refs.append(l)
        assert abs(host(loss)[b] - l) <= 1e-5 * abs(l)
        assert_close(host(dZ[b]), dz, 1e-5 if dt == "f32" else 1e-2, "dlogits")
    assert abs(host(ml)[0] - np.mean(refs)) <= 1e-5 * abs(np.mean(refs))      # App. C Eq. 1
    A = rounded(R.standard_normal((B, rows, 64)), tdt)
    T = R.standard_normal((rows, 64)).astype(np.float32).astype(np.float64)
    dA = torch.empty(B, rows, 64, dtype=tdt, device=DEV)
    Ad, Td = dev(A, tdt), dev(T)
    H.hfta_loss_mse(B, rows, 64, code, H.tin(Ad, rows * 64, 64), H.ptr(Td), 0, 64, H.ptr(loss),
                    H.ptr(ml), H.tout(dA, rows * 64, 64), H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    for b in range(B):
        l, da = OL.mse_mean(A[b], T)
        assert abs(host(loss)[b] - l) <= 1e-5 * abs(l)
        assert_close(host(dA[b]), da, 1e-5 if dt == "f32" else 1e-2, "dA")


@pytest.mark.parametrize("target", [1.0, 0.0])
def test_loss_bce_saturated(target):
    """Sigmoid + BCE on the logit (reading R29) vs oracle.layers.bce_sigmoid_mean,
    including saturated logits (|z| = 20..150: q = p(1-p) below the 1e-12
    BCELoss floor, log clamp at -100) and ordinary ones; fp32 in and out."""
    B, rows = 3, 257
    Z = (R.standard_normal((B, rows)) * 4).astype(np.float32).astype(np.float64)
    sat = np.array([20.0, -20.0, 27.0, -27.0, 30.0, -30.0, 40.0, -40.0, 99.0, -101.0, 150.0, -150.0])
    Z[:, :sat.size] = sat
    loss, ml = torch.empty(B, device=DEV), torch.empty(1, device=DEV)
    dZ = torch.empty(B, rows, device=DEV)
    ws = torch.empty(H.hfta_loss_workspace(B, rows), dtype=torch.uint8, device=DEV)
    Zd = dev(Z)
    H.hfta_loss_bce_logits(B, rows, 0, H.tin(Zd, rows, 1), target, H.ptr(loss), H.ptr(ml),
                           H.tout(dZ, rows, 1), H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    for b in range(B):
        l, dz = OL.bce_sigmoid_mean(Z[b], np.full(rows, target))
        assert abs(host(loss)[b] - l) <= 1e-5 * abs(l), (b, host(loss)[b], l)
        g = host(dZ[b])
        assert_close(g, dz, 1e-5, "dz")
        # the saturated entries one by one (relative, elementwise)
        for i in range(sat.size):
            assert abs(g[i] - dz[i]) <= 1e-5 * abs(dz[i]) + 1e-30, (Z[b, i], g[i], dz[i])


@pytest.mark.parametrize("P,shadow", [(4672, True), (1001, False)])
def test_fused_adam(P, shadow):
    B, T = 3, 4
    hp = dict(lr=np.float32([1e-3, 3e-3, 1e-2]), beta1=np.float32([0.9, 0.8, 0.5]),
              beta2=np.float32([0.999, 0.99, 0.9]), eps=np.float32([1e-8, 1e-6, 1e-4]),
              wd=np.float32([0.0, 1e-2, 0.3]))
    p0 = R.standard_normal((B, P)).astype(np.float32)
    pd, gd = dev(p0), torch.empty(B, P, device=DEV)
    md, vd = torch.zeros(B, P, device=DEV), torch.zeros(B, P, device=DEV)
    sh = torch.empty(B, P, dtype=torch.bfloat16, device=DEV) if shadow else None
    hv = {k: dev(v) for k, v in hp.items()}
    step = torch.zeros(1, dtype=torch.int64, device=DEV)
    ps = [p0[b].astype(np.float64) for b in range(B)]
    ms = [np.zeros(P) for _ in range(B)]
    vs = [np.zeros(P) for _ in range(B)]
    for t in range(1, T + 1):
        g = R.standard_normal((B, P)).astype(np.float32)
        gd.copy_(torch.from_numpy(g))
        H.hfta_step_increment(H.ptr(step), s())
        H.hfta_fused_adam(B, P, H.ptr(pd), H.ptr(gd), H.ptr(md), H.ptr(vd), P, H.ptr(hv["lr"]), H.ptr(hv["beta1"]),
                          H.ptr(hv["beta2"]), H.ptr(hv["eps"]), H.ptr(hv["wd"]), H.ptr(step), H.ptr(sh), P, s())
        for b in range(B):
            ps[b], ms[b], vs[b] = adam_step(ps[b], g[b].astype(np.float64), ms[b], vs[b], t,
                                            *(float(hp[k][b]) for k in ("lr", "beta1", "beta2", "eps", "wd")))
    torch.cuda.synchronize()
    for b in range(B):
        assert_close(host(pd[b]), ps[b], 1e-6, "param")
        assert_close(host(md[b]), ms[b], 1e-6, "m")
        assert_close(host(vd[b]), vs[b], 1e-6, "v")
        if shadow:
            assert np.array_equal(host(sh[b]), rounded(host(pd[b]), torch.bfloat16))


@pytest.mark.parametrize("nesterov", [0, 1])
def test_fused_sgd(nesterov):
    from oracle.optim import sgd_step
    B, P, T = 3, 1000, 4
    hp = dict(lr=np.float32([1e-2, 5e-2, 1e-3]), mom=np.float32([0.9, 0.5, 0.0]), damp=np.float32([0.0, 0.1, 0.0]),
              wd=np.float32([0.0, 1e-2, 3e-2]))
    p0 = R.standard_normal((B, P)).astype(np.float32)
    pd, gd, bd = dev(p0), torch.empty(B, P, device=DEV), torch.zeros(B, P, device=DEV)
    hv = {k: dev(v) for k, v in hp.items()}
    step = torch.zeros(1, dtype=torch.int64, device=DEV)
    ps = [p0[b].astype(np.float64) for b in range(B)]
    bufs = [None] * B
    for t in range(1, T + 1):
        g = R.standard_normal((B, P)).astype(np.float32)
        gd.copy_(torch.from_numpy(g))
        H.hfta_step_increment(H.ptr(step), s())
        H.hfta_fused_sgd(B, P, H.ptr(pd), H.ptr(gd), H.ptr(bd), P, H.ptr(hv["lr"]), H.ptr(hv["mom"]),
                         H.ptr(hv["damp"]), H.ptr(hv["wd"]), nesterov, H.ptr(step), None, P, s())
        for b in range(B):
            ps[b], bufs[b] = sgd_step(ps[b], g[b].astype(np.float64), bufs[b], t, *(float(hp[k][b]) for k in
                                      ("lr", "mom", "damp", "wd")), bool(nesterov))
    torch.cuda.synchronize()
    for b in range(B):
        assert_close(host(pd[b]), ps[b], 1e-6, "sgd param")


def test_fused_adadelta_and_steplr():
    from oracle.optim import adadelta_step, steplr
    B, P, T = 2, 999, 3
    hp = dict(lr=np.float32([1.0, 0.5]), rho=np.float32([0.9, 0.5]), eps=np.float32([1e-6, 1e-4]),
              wd=np.float32([0.0, 1e-2]))
    p0 = R.standard_normal((B, P)).astype(np.float32)
    pd, gd = dev(p0), torch.empty(B, P, device=DEV)
    sq, ac = torch.zeros(B, P, device=DEV), torch.zeros(B, P, device=DEV)
    hv = {k: dev(v) for k, v in hp.items()}
    st = [(p0[b].astype(np.float64), np.zeros(P), np.zeros(P)) for b in range(B)]
    for t in range(T):
        g = R.standard_normal((B, P)).astype(np.float32)
        gd.copy_(torch.from_numpy(g))
        H.hfta_fused_adadelta(B, P, H.ptr(pd), H.ptr(gd), H.ptr(sq), H.ptr(ac), P, H.ptr(hv["lr"]), H.ptr(hv["rho"]),
                              H.ptr(hv["eps"]), H.ptr(hv["wd"]), None, P, s())
        for b in range(B):
            st[b] = adadelta_step(st[b][0], g[b].astype(np.float64), st[b][1], st[b][2],
                                  *(float(hp[k][b]) for k in ("lr", "rho", "eps", "wd")))
    torch.cuda.synchronize()
    for b in range(B):
        assert_close(host(pd[b]), st[b][0], 1e-6, "adadelta param")
    lr0, gam, per = dev([0.1, 1e-3]), dev([0.5, 0.9]), torch.tensor([10, 3], dtype=torch.int32, device=DEV)
    out = torch.empty(2, device=DEV)
    for ep in (0, 9, 10, 25):
        H.hfta_steplr(2, H.ptr(lr0), H.ptr(gam), H.ptr(per), ep, H.ptr(out), s())
        torch.cuda.synchronize()
        ref = [steplr(float(np.float32(0.1)), float(np.float32(0.5)), 10, ep),
               steplr(float(np.float32(1e-3)), float(np.float32(0.9)), 3, ep)]
        assert np.allclose(host(out), ref, rtol=1e-6)


@pytest.mark.parametrize("M,N,K,B", [(5000, 256, 512, 2), (777, 128, 64, 3), (80, 512, 128, 1)])
def test_linear_fwd_stats_and_bn_from_colstat(M, N, K, B):
    """hfta_fused_linear_fwd_stats writes the same Y as hfta_fused_linear_fwd
    plus per-32-row column sums / sums of squares of the STORED bf16 Y; BN
    forward from those partials matches BN forward with its own statistics
    pass (mean / invstd 1e-5, outputs within one bf16 rounding)."""
    code, tdt = DT["bf16"]
    X = rounded(R.standard_normal((B, M, K)), tdt)
    W = rounded(R.standard_normal((B, N, K)) / np.sqrt(K), tdt)
    bias = torch.tensor(R.standard_normal((B, N)), dtype=torch.float32, device=DEV)
    Xd, Wd = dev(X, tdt), dev(W, tdt)
    Y1 = torch.empty(B, M, N, dtype=tdt, device=DEV)
    Y2 = torch.empty_like(Y1)
    cs = torch.empty(H.hfta_linear_colstat_size(B, M, N) // 4, dtype=torch.float32, device=DEV)
    H.hfta_fused_linear_fwd(B, M, N, K, code, H.tin(Xd, M * K, K), H.tin(Wd, N * K, K), H.ptr(bias), N, 0, 0,
                            H.tout(Y1, M * N, N), s())
    H.hfta_fused_linear_fwd_stats(B, M, N, K, H.tin(Xd, M * K, K), H.tin(Wd, N * K, K), H.ptr(bias), N, 0, 0,
                                  H.tout(Y2, M * N, N), H.ptr(cs), s())
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    y = host(Y2)
    nblk = (M + 31) // 32
    c = cs.view(B, nblk, 2, N).double().cpu().numpy()
    for b in range(B):
        for k in (0, nblk // 2, nblk - 1):
            rows = y[b, 32 * k:min(M, 32 * k + 32)]
            np.testing.assert_allclose(c[b, k, 0], rows.sum(0), rtol=1e-5, atol=1e-4)
            np.testing.assert_allclose(c[b, k, 1], (rows * rows).sum(0), rtol=1e-5, atol=1e-4)
    g = torch.tensor(R.uniform(0.5, 1.5, (B, N)), dtype=torch.float32, device=DEV)
    be = torch.tensor(R.uniform(-0.5, 0.5, (B, N)), dtype=torch.float32, device=DEV)
    outs = []
    for use_cs in (False, True):
        rm, rv = torch.zeros(B, N, device=DEV), torch.ones(B, N, device=DEV)
        sm, si = torch.empty(B, N, device=DEV), torch.empty(B, N, device=DEV)
        Z = torch.empty_like(Y2)
        if use_cs:
            H.hfta_fused_bn_fwd_colstat(B, M, N, code, H.tin(Y2, M * N, N), H.ptr(g), H.ptr(be), N, H.ptr(rm),
                                        H.ptr(rv), 0.1, 1e-5, 1, 0.0, H.tout(Z, M * N, N), H.ptr(sm), H.ptr(si),
                                        H.ptr(cs), s())
        else:
            ws = torch.empty(H.hfta_fused_bn_workspace(B, M, N), dtype=torch.uint8, device=DEV)
            H.hfta_fused_bn_fwd(B, M, N, code, H.tin(Y2, M * N, N), H.ptr(g), H.ptr(be), N, H.ptr(rm), H.ptr(rv),
                                0.1, 1e-5, 1, 0.0, H.tout(Z, M * N, N), H.ptr(sm), H.ptr(si), H.ptr(ws), ws.numel(),
                                s())
        torch.cuda.synchronize()
        outs.append((host(Z), host(sm), host(si), host(rm), host(rv)))
    (z0, m0, i0, rm0, rv0), (z1, m1, i1, rm1, rv1) = outs
    assert_close(m1, m0, 1e-5, "mean")
    assert_close(i1, i0, 1e-5, "invstd")
    assert_close(rv1, rv0, 1e-5, "running var")
    assert_close(z1, z0, 4e-3, "BN output")
