"""Parity of the fused Linear -> BN -> act layer in Gram form (K11,
hfta_fused_linear_bn_fwd/bwd) against the oracle's composition of
linear -> bn (training) -> relu and the backward of linear and bn
(oracle.layers), element by element on bf16-rounded inputs.

Shapes: K = 3 (the xyz layer: streaming kernels, shared input with bstride 0
as STN's first layer sees it), K = 64 and 128 (tensor cores, ragged M), with
and without the act'(X) gating of dX (X = the previous layer's ReLU output),
accumulate."""
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


def run(B, M, N, K, shared=False, gate=False, accumulate=0, seed=0):
    rng = np.random.default_rng(seed)
    nb = 1 if shared else B
    if K <= 8:
        X = bf(rng.standard_normal((nb, M, K)))
    else:   # the previous layer's ReLU output: nonnegative with exact zeros
        X = bf(np.maximum(rng.standard_normal((nb, M, K)) + 0.3, 0))
    W = bf(rng.standard_normal((B, N, K)) / np.sqrt(K))
    bias = rng.uniform(-0.2, 0.2, (B, N)).astype(np.float32).astype(np.float64)
    g = rng.uniform(0.75, 1.25, (B, N)).astype(np.float32).astype(np.float64)
    be = rng.uniform(-0.1, 0.1, (B, N)).astype(np.float32).astype(np.float64)
    rm0 = (0.1 * rng.standard_normal((B, N))).astype(np.float32).astype(np.float64)
    rv0 = rng.uniform(0.5, 2, (B, N)).astype(np.float32).astype(np.float64)
    dA = rng.standard_normal((B, M, N))
    dW0 = rng.standard_normal((B, N, K)).astype(np.float32).astype(np.float64)
    dg0 = rng.standard_normal((B, N)).astype(np.float32).astype(np.float64)

    # oracle forward (needed for dZ = dA * relu'(z), the kernel's input)
    ref = []
    for b in range(B):
        xb = X[0 if shared else b]
        y = OL.linear_fwd(xb, W[b], bias[b])
        z, cache = OL.bn_fwd(y, g[b], be[b])
        ref.append((xb, y, z, cache))
    dZ = np.stack([bf(OL.relu_bwd(dA[b], ref[b][2])) for b in range(B)])

    Xd, Wd = dev(X, torch.bfloat16), dev(W, torch.bfloat16)
    bd, gd, bed, rm, rv = dev(bias), dev(g), dev(be), dev(rm0), dev(rv0)
    A = torch.empty(B, M, N, dtype=torch.bfloat16, device=DEV)
    sm, si = torch.empty(B, N, device=DEV), torch.empty(B, N, device=DEV)
    G, sv = torch.empty(B, K, K, device=DEV), torch.empty(B, K, device=DEV)
    ws = torch.empty(H.hfta_fused_linear_bn_workspace(B, M, N, K), dtype=torch.uint8, device=DEV)
    xbs = 0 if shared else M * K
    H.hfta_fused_linear_bn_fwd(B, M, N, K, 1, H.tin(Xd, xbs, K), H.tin(Wd, N * K, K), H.ptr(bd), N, H.ptr(gd),
                               H.ptr(bed), N, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, 1, 0.0, H.tout(A, M * N, N), H.ptr(sm),
                               H.ptr(si), H.ptr(G), H.ptr(sv), H.ptr(ws), ws.numel(), s())
    dZd = dev(dZ, torch.bfloat16)
    dX = torch.empty(B, M, K, dtype=torch.bfloat16, device=DEV) if not shared else None
    dW = dev(dW0) if accumulate else torch.empty(B, N, K, device=DEV)
    dgam = dev(dg0) if accumulate else torch.empty(B, N, device=DEV)
    dbet = dev(dg0) if accumulate else torch.empty(B, N, device=DEV)
    dbias = torch.full((B, N), 5.0, device=DEV)
    H.hfta_fused_linear_bn_bwd(B, M, N, K, 1, H.tin(dZd, M * N, N), H.tin(Xd, xbs, K), H.tin(Wd, N * K, K), H.ptr(bd),
                               N, H.ptr(gd), N, H.ptr(sm), H.ptr(si), H.ptr(G), H.ptr(sv),
                               H.tout(dX, M * K, K), 1 if gate else 0, 0.0, H.ptr(dW), N * K, K, H.ptr(dbias), N,
                               H.ptr(dgam), H.ptr(dbet), accumulate, H.ptr(ws), ws.numel(), s())
    torch.cuda.synchronize()
    out = dict(A=host(A), sm=host(sm), si=host(si), rm=host(rm), rv=host(rv), G=host(G), sv=host(sv),
               dX=None if dX is None else host(dX), dW=host(dW), dg=host(dgam), db=host(dbet), dbias=host(dbias))
    return out, dict(X=X, W=W, g=g, rm0=rm0, rv0=rv0, dZ=dZ, dW0=dW0, dg0=dg0, ref=ref)


CASES = [  # B, M, N, K, shared, gate
    (3, 1000, 64, 3, True, False),       # STN c1: shared xyz input, no dX
    (2, 3000, 64, 3, False, False),      # feat c1: per-model transformed xyz, dX into xyz
    (2, 1777, 128, 3, False, False),     # K = 3 -> N = 128: the 256-B-row dX kernel (16 x 16-B loads per row)
    (2, 2500, 128, 64, False, True),     # c2: K = 64 tensor cores, dX gated by the c1 ReLU
    (2, 1111, 128, 64, False, False),    # ragged M, ungated
    (2, 777, 64, 128, False, True),      # K = 128, N = 64
    # gated two-segment dX whose tile has more k-blocks than the ring has
    # stages (4 + 2 > 4, 6 + 1 > 6): the gate is read from global memory
    # instead of the resident A stage (a hang before)
    (2, 1300, 256, 128, False, True),
    (2, 700, 384, 64, False, True),
    (1, 500, 512, 128, False, True),
]


@pytest.mark.parametrize("B,M,N,K,shared,gate", CASES)
def test_linear_bn(B, M, N, K, shared, gate):
    out, inp = run(B, M, N, K, shared, gate)
    for b in range(B):
        xb, y, z, cache = inp["ref"][b]
        assert_close(out["G"][b], xb.T @ xb, 1e-5, "G")
        assert_close(out["sv"][b], xb.sum(0), 1e-5, "s")
        assert_close(out["sm"][b], cache["mean"], 1e-4, "save_mean")
        assert_close(out["si"][b], cache["invstd"], 1e-4, "save_invstd")
        rmr, rvr = OL.bn_running(inp["rm0"][b], inp["rv0"][b], cache, M)
        assert_close(out["rm"][b], rmr, 1e-4, "running_mean")
        assert_close(out["rv"][b], rvr, 1e-4, "running_var")
        assert_close(out["A"][b], OL.relu(z), 1e-2, "A = relu(bn(x W^T + b))")
        dy, dgr, dbr = OL.bn_bwd(inp["dZ"][b], cache, inp["g"][b])
        dx, dw, _ = OL.linear_bwd(dy, xb, inp["W"][b])
        assert_close(out["dg"][b], dgr, 1e-4, "dgamma")
        assert_close(out["db"][b], dbr, 1e-4, "dbeta")
        assert_close(out["dW"][b], dw, 2e-2, "dW")
        assert np.all(out["dbias"][b] == 0.0), "BN-absorbed bias gradient must be exactly 0"
        if out["dX"] is not None:
            ref_dx = dx * (xb > 0) if gate else dx
            assert_close(out["dX"][b], ref_dx, 2e-2, "dX")


def test_linear_bn_accumulate():
    B, M, N, K = 2, 1500, 128, 64
    out, inp = run(B, M, N, K, accumulate=1, seed=3)
    for b in range(B):
        xb, y, z, cache = inp["ref"][b]
        dy, dgr, dbr = OL.bn_bwd(inp["dZ"][b], cache, inp["g"][b])
        _, dw, _ = OL.linear_bwd(dy, xb, inp["W"][b])
        assert_close(out["dW"][b], inp["dW0"][b] + dw, 2e-2, "dW accumulate")
        assert_close(out["dg"][b], inp["dg0"][b] + dgr, 1e-4, "dgamma accumulate")


def test_linear_bn_errors():
    x = torch.zeros(64, 32, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(H.HftaError) as e:      # K = 32 is neither streaming nor tensor-core width
        H.hfta_fused_linear_bn_fwd(1, 64, 32, 32, 1, H.tin(x, 0, 32), H.tin(x, 0, 32), None, 0, None, None, 0, None,
                                   None, 0.1, 1e-5, 1, 0.0, H.tout(x, 0, 32), None, None, None, None, None, 0, s())
    assert e.value.code == 4
