"""Parity of the fused Linear -> BN -> act -> max block (K10,
hfta_fused_linear_bn_max_fwd/bwd) against the oracle's composition of the
layer definitions (oracle.layers: linear, bn (training), act, max over points
and their backward), element by element, on bf16-rounded inputs.

Shapes: ragged clouds (L not a multiple of the 64/128-point tiles), tiles
spanning many tiny clouds, channel counts leaving a partial channel group
(C = 640), K = 64 and 128, shared input (bstride 0), gamma of both signs (the
min-side of the pooled maximum), accumulate, split and unsplit wgrad."""
import numpy as np
import pytest
import torch

from oracle import layers as OL
from tests._cmp import assert_close

pytestmark = pytest.mark.gpu

H = None
DEV = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _init():
    global H
    import paper_2102_02344_b200.hfta as hfta
    hfta.hfta_init(0)
    H = hfta


def s():
    return torch.cuda.current_stream().cuda_stream


def bf(a):
    return torch.tensor(a).to(torch.bfloat16).double().numpy()


def dev(a, tdt=torch.float32):
    return torch.tensor(np.asarray(a), dtype=torch.float64).to(tdt).to(DEV).contiguous()


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


ACT = {0: (lambda z: z, lambda d, z: d), 1: (OL.relu, OL.relu_bwd)}


def run_block(B, N, L, C, K, act, shared=False, seed=0, accumulate=0, neg_gamma=True, dx_act=0):
    rng = np.random.default_rng(seed)
    R = N * L
    X = bf(np.maximum(rng.standard_normal((1 if shared else B, R, K)), 0) + 0.1 * rng.standard_normal((1 if shared else B, R, K)))
    W = bf(rng.standard_normal((B, C, K)) / np.sqrt(K))
    bias = rng.uniform(-0.2, 0.2, (B, C)).astype(np.float32).astype(np.float64)
    g = rng.uniform(0.75, 1.25, (B, C))
    if neg_gamma:
        g *= np.where(rng.random((B, C)) < 0.3, -1.0, 1.0)
    g = g.astype(np.float32).astype(np.float64)
    be = rng.uniform(-0.1, 0.1, (B, C)).astype(np.float32).astype(np.float64)
    rm0 = rng.standard_normal((B, C)).astype(np.float32).astype(np.float64) * 0.1
    rv0 = rng.uniform(0.5, 2, (B, C)).astype(np.float32).astype(np.float64)
    dG = rng.standard_normal((B, N, C)).astype(np.float32).astype(np.float64)
    dW0 = rng.standard_normal((B, C, K)).astype(np.float32).astype(np.float64)
    dg0 = rng.standard_normal((B, C)).astype(np.float32).astype(np.float64)

    Xd, Wd = dev(X, torch.bfloat16), dev(W, torch.bfloat16)
    bd, gd, bed, rm, rv, dGd = dev(bias), dev(g), dev(be), dev(rm0), dev(rv0), dev(dG)
    G = torch.empty(B, N, C, device=DEV)
    ext = torch.empty(B, N, C, device=DEV)
    am = torch.empty(B, N, C, dtype=torch.int32, device=DEV)
    sm, si = torch.empty(B, C, device=DEV), torch.empty(B, C, device=DEV)
    gram, xsum = torch.empty(B, K, K, device=DEV), torch.empty(B, K, device=DEV)
    ws = torch.empty(H.hfta_fused_linear_bn_max_workspace(B, N, L, C, K), dtype=torch.uint8, device=DEV)
    xbs = 0 if shared else R * K
    H.hfta_fused_linear_bn_max_fwd(B, N, L, C, K, 1, H.tin(Xd, xbs, K), H.tin(Wd, C * K, K), H.ptr(bd), C, H.ptr(gd),
                                   H.ptr(bed), C, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, act, 0.0, H.tout(G, N * C, C),
                                   H.ptr(am), H.tout(ext, N * C, C), H.ptr(sm), H.ptr(si), H.ptr(gram), H.ptr(xsum),
                                   H.ptr(ws), ws.numel(), s())
    dX = torch.empty(B, R, K, dtype=torch.bfloat16, device=DEV)
    dW = dev(dW0) if accumulate else torch.empty(B, C, K, device=DEV)
    dgam = dev(dg0) if accumulate else torch.empty(B, C, device=DEV)
    dbet = dev(dg0) if accumulate else torch.empty(B, C, device=DEV)
    dbias = torch.full((B, C), 7.0, device=DEV)
    H.hfta_fused_linear_bn_max_bwd(B, N, L, C, K, 1, H.tin(dGd, N * C, C), H.tin(Xd, xbs, K), H.tin(Wd, C * K, K),
                                   H.ptr(am), H.tin(ext, N * C, C), H.ptr(bd), C, H.ptr(gd), H.ptr(bed), C, H.ptr(sm),
                                   H.ptr(si), H.ptr(gram), H.ptr(xsum), act, 0.0, H.tout(dX, R * K, K), dx_act, 0.0, H.ptr(dW), C * K, K, H.ptr(dbias), C,
                                   H.ptr(dgam), H.ptr(dbet), accumulate, H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    out = dict(G=host(G), ext=host(ext), am=am.cpu().numpy().astype(np.int64), sm=host(sm), si=host(si),
               rm=host(rm), rv=host(rv), gram=host(gram), xsum=host(xsum), dX=host(dX), dW=host(dW), dg=host(dgam),
               db=host(dbet), dbias=host(dbias))
    inp = dict(X=X, W=W, bias=bias, g=g, be=be, rm0=rm0, rv0=rv0, dG=dG, dW0=dW0, dg0=dg0)
    return out, inp


def test_linear_bn_max_gated_dx():
    """dX_act = ReLU: dX is multiplied by act'(X) (X > 0), the previous layer's dZ."""
    B, N, L, C, K, act = 2, 3, 700, 256, 128, 1
    out, inp = run_block(B, N, L, C, K, act, seed=11, dx_act=1)
    for b in range(B):
        o = oracle_block(inp, b, N, L, act, False)
        assert_close(out["dX"][b], o["dX"] * (inp["X"][b] > 0), 2e-2, "gated dX")


def oracle_block(inp, b, N, L, act, shared):
    """The block as the paper's layers compose it, fp64 (oracle.layers)."""
    X = inp["X"][0 if shared else b]
    y = OL.linear_fwd(X, inp["W"][b], inp["bias"][b])
    z, cache = OL.bn_fwd(y, inp["g"][b], inp["be"][b])
    a = ACT[act][0](z)
    C = y.shape[1]
    gmax, idx = OL.max_over_points(a.reshape(N, L, C))
    rm, rv = OL.bn_running(inp["rm0"][b], inp["rv0"][b], cache, N * L)
    da = OL.max_over_points_bwd(inp["dG"][b], idx, L).reshape(N * L, C)
    dz = ACT[act][1](da, z)
    dy, dgam, dbet = OL.bn_bwd(dz, cache, inp["g"][b])
    dx, dw, _ = OL.linear_bwd(dy, X, inp["W"][b])
    return dict(y=y, z=z, G=gmax, idx=idx, mean=cache["mean"], invstd=cache["invstd"], rm=rm, rv=rv, dX=dx, dW=dw,
                dg=dgam, db=dbet)


CASES = [  # B, N, L, C, K, act, shared
    (2, 3, 700, 256, 128, 1, False),     # ragged clouds, tiles straddling clouds, STN-style ReLU
    (2, 2, 1000, 640, 128, 0, False),    # partial channel group (5 blocks), feat-style no act
    (3, 40, 5, 128, 64, 1, True),        # tiny clouds: one tile spans many; shared input; K = 64
    (1, 1, 100, 128, 128, 0, False),     # a single partial chunk; unsplit wgrad
    (4, 8, 333, 384, 128, 1, False),
    (2, 3, 700, 512, 128, 1, False),
    (2, 2, 1000, 1024, 128, 0, False),
    (3, 40, 5, 512, 64, 1, True),
    (1, 1, 100, 1024, 128, 1, False),
]


@pytest.mark.parametrize("B,N,L,C,K,act,shared", CASES)
def test_linear_bn_max(B, N, L, C, K, act, shared):
    out, inp = run_block(B, N, L, C, K, act, shared)
    for b in range(B):
        o = oracle_block(inp, b, N, L, act, shared)
        # forward: fp32 accumulation of exact bf16 products -> fp32-level agreement
        # argmax: unique where the pooled value is not ReLU-clamped; where all
        # of a cloud's points clamp to 0 every index is a valid choice (its
        # gradient is 0) and the kernel reports the extreme of Y instead.
        live = o["G"] > 0 if act == 1 else np.ones_like(o["G"], dtype=bool)
        assert np.array_equal(out["am"][b][live], o["idx"][live]), "argmax"
        assert_close(out["G"][b], o["G"], 1e-5, "G")
        ext_ref = np.take_along_axis(o["y"].reshape(N, L, -1), out["am"][b][:, None, :], axis=1)[:, 0, :]
        assert_close(out["ext"][b], ext_ref, 1e-5, "ext")
        Xb = inp["X"][0 if shared else b]
        assert_close(out["gram"][b], Xb.T @ Xb, 1e-5, "gram = X^T X")
        assert_close(out["xsum"][b], Xb.sum(0), 1e-5, "xsum = X^T 1")
        assert_close(out["sm"][b], o["mean"], 1e-5, "save_mean")
        assert_close(out["si"][b], o["invstd"], 1e-5, "save_invstd")
        assert_close(out["rm"][b], o["rm"], 1e-5, "running_mean")
        assert_close(out["rv"][b], o["rv"], 1e-5, "running_var")
        # backward: dY enters the contractions in bf16 (the AMP precision of
        # per-point tensors, reading R16) -> the bf16 gate
        assert_close(out["dg"][b], o["dg"], 1e-4, "dgamma")
        assert_close(out["db"][b], o["db"], 1e-4, "dbeta")
        assert_close(out["dX"][b], o["dX"], 2e-2, "dX")
        assert_close(out["dW"][b], o["dW"], 2e-2, "dW")
        assert np.all(out["dbias"][b] == 0.0), "BN-absorbed bias gradient must be exactly 0"


def test_linear_bn_max_accumulate():
    B, N, L, C, K, act = 2, 3, 300, 256, 128, 1
    out, inp = run_block(B, N, L, C, K, act, accumulate=1, seed=5)
    for b in range(B):
        o = oracle_block(inp, b, N, L, act, False)
        assert_close(out["dW"][b], inp["dW0"][b] + o["dW"], 2e-2, "dW accumulate")
        assert_close(out["dg"][b], inp["dg0"][b] + o["dg"], 1e-4, "dgamma accumulate")
        assert_close(out["db"][b], inp["dg0"][b] + o["db"], 1e-4, "dbeta accumulate")


def test_linear_bn_max_deterministic():
    a, _ = run_block(2, 4, 500, 256, 128, 1, seed=9)
    b, _ = run_block(2, 4, 500, 256, 128, 1, seed=9)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_linear_bn_max_errors():
    x = torch.zeros(64, 96, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(H.HftaError) as e:      # K must be 64 or 128
        H.hfta_fused_linear_bn_max_fwd(1, 1, 64, 128, 96, 1, H.tin(x, 0, 96), H.tin(x, 0, 96), None, 0, None, None,
                                       0, None, None, 0.1, 1e-5, 0, 0.0, H.tout(x, 0, 1), None, H.tout(x, 0, 1), None,
                                       None, None, None, None, 0, s())
    assert e.value.code == 4
    with pytest.raises(H.HftaError) as e:      # fp32 operands are not this path
        H.hfta_fused_linear_bn_max_fwd(1, 1, 64, 128, 64, 0, H.tin(x, 0, 64), H.tin(x, 0, 64), None, 0, None, None,
                                       0, None, None, 0.1, 1e-5, 0, 0.0, H.tout(x, 0, 1), None, H.tout(x, 0, 1), None,
                                       None, None, None, None, 0, s())
    assert e.value.code == 4
