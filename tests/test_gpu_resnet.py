"""NEXT-4, the ResNet-18 family through the C ABI vs the oracle
(oracle/resnet.py): the pooling kernels per call, then one fused training
step (conv 7x7 / 3x3 / 1x1 at strides 1 and 2, BN2d, ReLU, residual adds,
MaxPool2d, AdaptiveAvgPool2d, Linear, cross entropy, Adadelta) of B models,
decision-matched (readings R15b/R15c/R28, tests/_decide.py) and gated per
gradient tensor at fp32 1e-4 / bf16 max(2e-2, 3 x the bf16-storage witness)."""
import numpy as np
import pytest
import torch

import synth
from oracle import layers as Lr
from oracle import resnet as OR
from tests._cmp import TOL, relerr
from tests import _decide as DE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_2102_02344_b200.hfta as H
    H.hfta_init(0)


def _dt(dtype):
    import paper_2102_02344_b200.hfta as H
    return (H.HFTA_F32, torch.float32) if dtype == "f32" else (H.HFTA_BF16, torch.bfloat16)


def _nchw(t):
    return t.detach().float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,N,Hs,C,k,s,p,shared", [
    (3, 4, 16, 64, 3, 2, 1, False),      # the ResNet stem pool
    (1, 2, 9, 24, 3, 2, 1, False),       # odd size, C not a vector multiple in bf16 (24 % 8 == 0), ragged
    (2, 3, 7, 5, 2, 2, 0, True),         # scalar path (C = 5), shared input
    (2, 2, 8, 16, 3, 1, 1, False)])      # stride 1: overlapping windows in both directions
def test_maxpool(dtype, B, N, Hs, C, k, s, p, shared):
    import paper_2102_02344_b200.hfta as H
    dt, tdt = _dt(dtype)
    g = np.random.default_rng(B * 100 + Hs)
    x = np.round(g.standard_normal((1 if shared else B, N, Hs, Hs, C)) * 4) / 4     # many exact ties
    X = torch.tensor(x, dtype=tdt, device="cuda")
    xr = X.double().cpu().numpy()                                    # the values the kernel sees
    Ho = (Hs + 2 * p - k) // s + 1
    Y = torch.empty(B, N, Ho, Ho, C, dtype=tdt, device="cuda")
    am = torch.empty(B, N, Ho, Ho, C, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    H.hfta_maxpool2d_fwd(B, N, Hs, Hs, C, k, s, p, dt, H.tin(X, 0 if shared else X[0].numel(), C),
                         H.tout(Y, Y[0].numel(), C), H.ptr(am), am[0].numel(), st)
    dy = g.standard_normal((B, N, Ho, Ho, C))
    dY = torch.tensor(dy, dtype=tdt, device="cuda")
    dyr = dY.double().cpu().numpy()
    dX = torch.empty(B, N, Hs, Hs, C, dtype=tdt, device="cuda")
    H.hfta_maxpool2d_bwd(B, N, Hs, Hs, C, k, s, p, dt, H.tin(dY, dY[0].numel(), C), H.ptr(am), am[0].numel(),
                         H.tout(dX, dX[0].numel(), C), st)
    torch.cuda.synchronize()
    for b in range(B):
        xb = xr[0 if shared else b].transpose(0, 3, 1, 2)
        y_ref, idx = Lr.maxpool2d_fwd(xb, k, s, p)
        assert np.array_equal(Y[b].double().cpu().numpy().transpose(0, 3, 1, 2), y_ref)     # exact: a selection
        assert np.array_equal(am[b].cpu().numpy().astype(np.int64), idx)                   # first tap on ties
        dx_ref = Lr.maxpool2d_bwd(dyr[b].transpose(0, 3, 1, 2), idx, xb.shape, k, s, p)
        got = dX[b].double().cpu().numpy().transpose(0, 3, 1, 2)
        # fp32 sums of at most ceil(k/s)^2 terms; bf16: one output rounding
        assert relerr(got, dx_ref) <= (1e-6 if dtype == "f32" else 4e-3)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,N,HW,C", [(3, 5, 1, 512), (2, 4, 16, 64), (1, 3, 49, 6)])
def test_avgpool(dtype, B, N, HW, C):
    import paper_2102_02344_b200.hfta as H
    dt, tdt = _dt(dtype)
    g = np.random.default_rng(HW + C)
    X = torch.tensor(g.standard_normal((B, N, HW, C)), dtype=tdt, device="cuda")
    Y = torch.empty(B, N, C, dtype=tdt, device="cuda")
    dY = torch.tensor(g.standard_normal((B, N, C)), dtype=tdt, device="cuda")
    dX = torch.empty(B, N, HW, C, dtype=tdt, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    H.hfta_avgpool2d_fwd(B, N, HW, C, dt, H.tin(X, X[0].numel(), C), H.tout(Y, Y[0].numel(), C), st)
    H.hfta_avgpool2d_bwd(B, N, HW, C, dt, H.tin(dY, dY[0].numel(), C), H.tout(dX, dX[0].numel(), C), st)
    torch.cuda.synchronize()
    tol = 1e-6 if dtype == "f32" else 4e-3
    xr, dyr = X.double().cpu().numpy(), dY.double().cpu().numpy()
    for b in range(B):
        x4 = xr[b].reshape(N, HW, 1, C).transpose(0, 3, 1, 2)
        assert relerr(Y[b].double().cpu().numpy(), Lr.avgpool_global_fwd(x4)) <= tol
        assert relerr(dX[b].double().cpu().numpy().reshape(N, HW, 1, C).transpose(0, 3, 1, 2),
                      Lr.avgpool_global_bwd(dyr[b], x4.shape)) <= tol


def run_resnet(dtype, B=2, N=8, widths=OR.STAGES, seed=0):
    from paper_2102_02344_b200.resnet import FusedResNet18
    specs = synth.param_specs("resnet18", widths=widths)
    Ps = [synth.init_params("resnet18", 1000 + b, widths=widths) for b in range(B)]
    hp = synth.hparams_resnet(3, B)
    x, labels = synth.cifar(seed, N=N)
    net = FusedResNet18(B, specs, Ps, hp, N=N, widths=widths, dtype=dtype)
    net.set_inputs(torch.tensor(x.transpose(0, 2, 3, 1), dtype=torch.float32, device="cuda"),
                   torch.tensor(labels, device="cuda"))
    loss = net.step().cpu().numpy().copy()
    torch.cuda.synchronize()
    res = []
    for b in range(B):
        gpu = {"stem.relu": _nchw(net.stem["a"][b]) > 0,
               "stem.pool": net.stem["am"][b].cpu().numpy().astype(np.int64).reshape(-1, widths[0])}
        vals = {"stem.relu": _nchw(net.stem["a"][b])}
        for blk in net.blocks:
            n = blk["name"]
            a1, h = _nchw(blk["a1"][b]), _nchw(blk["h"][b])
            gpu[n + ".relu1"], gpu[n + ".relu2"] = a1 > 0, h > 0
            vals[n + ".relu1"], vals[n + ".relu2"] = a1, h
        P64 = {k_: v.astype(np.float64) for k_, v in Ps[b].items()}
        hp_b = {k_: float(v[b]) for k_, v in hp.items()}
        step = lambda: OR.train_step(P64, {}, {}, (x.astype(np.float64), labels), hp_b, widths)
        # the GPU stores every conv / fc output (pre-BN, logits) in the compute dtype
        r, report, rw = DE.with_decisions(step, gpu, dtype, out_layers=("conv1", "l", "fc"))
        zerr = DE.decision_errors(report.pop("_ctx"), vals, report["_margins"])
        res.append(dict(ref=r, report=report, witness=rw, zerr=zerr, p0=P64, hp=hp_b))
    return net, loss, res, hp


def _check(dtype, net, loss, res, B):
    from paper_2102_02344_b200.resnet import _to_torch
    tol = TOL[dtype]
    worst = []
    for b in range(B):
        rep, ref, wit = res[b]["report"], res[b]["ref"], res[b]["witness"]
        print("\n  model %d decisions (flagged/size, flips): %s" % (b, " ".join(
            "%s:%d/%d,%d" % (k, v["flagged"], v["size"], v["flips"]) for k, v in rep.items()
            if not k.startswith("_"))))
        bad = {k: v for k, v in rep.items() if not k.startswith("_") and v["unflagged_disagree"]}
        assert not bad, "model %d: GPU decisions differ from the oracle outside the flagged band: %s" % (b, bad)
        for site, e in res[b]["zerr"].items():
            assert e <= 1.0, "model %d site %s: GPU z error is %.2f x the margin" % (b, site, e)
        assert abs(loss[b] - ref["loss"]) <= tol * abs(ref["loss"]), (b, loss[b], ref["loss"])
        G = net.grads(b)
        grad_gate = {}
        for n, r_ in ref["grads"].items():
            gt = DE.gate(tol, wit["grads"][n], wit["own"]["grads"][n])
            grad_gate[n] = gt
            e = relerr(G[n], r_)
            worst.append((e / gt, e, gt, b, n))
            assert e <= gt, "model %d %s: %.3e > %.3e" % (b, n, e, gt)
            # Adadelta state and the updated parameters (square_avg = (1 - rho) g^2 at step 1)
            sq_ref, acc_ref = ref["opt"][n]
            sq = _to_torch(n, net.arena.host_tensor("m", n)[b])
            assert relerr(sq, sq_ref) <= 2 * gt * 1.01 + 1e-6, (b, n, "square_avg")
        # the Adadelta update p1 - p0 of every tensor, gated like a gradient (its
        # step-1 map g -> delta is nonlinear: the witness's change of the
        # update itself sets the bf16 gate, reading R28)
        # Implied bound: delta = f(g') with g' = g + wd p0 and 0 <= f'(g') <= 1
        # at step 1, so ||d delta|| <= ||d g|| and an update error up to
        # gate(g) * ||g'|| / ||delta|| follows from a gradient within its gate.
        P, P0, hp_b = net.params(b), res[b]["p0"], res[b]["hp"]
        for n, p_ref in ref["params"].items():
            upd = p_ref - P0[n]
            g_eff = ref["grads"][n] + hp_b["wd"] * P0[n]
            implied = grad_gate[n] * np.linalg.norm(g_eff) * hp_b["lr"] / max(np.linalg.norm(upd), 1e-300)
            gu = max(DE.gate(tol, wit["params"][n] - P0[n], wit["own"]["params"][n] - P0[n]), implied)
            eu = relerr(P[n] - P0[n], upd)
            assert eu <= gu, (b, n, "update", eu, gu)
        rs = net.running_stats(b)
        for name, (rm, rv) in rs.items():
            for k2, got in ((".rm", rm), (".rv", rv)):
                g_ = DE.gate(tol, wit["stats"][name + k2], wit["own"]["stats"][name + k2])
                assert relerr(got, ref["stats"][name + k2]) <= g_, (b, name, k2)
    worst.sort(reverse=True)
    print("\n[%s] worst gradient errors (err / gate): %s" % (dtype, " ".join(
        "%s:%.2e/%.1e" % (n, e, g) for _, e, g, b, n in worst[:8])))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_resnet18_step_small(dtype):
    """Full-width ResNet-18 on 32 x 32 images, N = 8, B = 2."""
    net, loss, res, hp = run_resnet(dtype, B=2, N=8)
    _check(dtype, net, loss, res, 2)


@pytest.mark.parametrize("dtype", ["f32"])
def test_resnet18_step_narrow_b3(dtype):
    """Narrow widths (the fused operators at other channel counts), B = 3."""
    net, loss, res, hp = run_resnet(dtype, B=3, N=6, widths=(16, 32, 32, 64), seed=1)
    _check(dtype, net, loss, res, 3)


def test_pool_and_gated_conv_errors():
    """Validation before any launch: bad pooling geometry, non-dense layouts,
    a dgrad gate with an activation other than ReLU / LeakyReLU."""
    import paper_2102_02344_b200.hfta as H
    st = torch.cuda.current_stream().cuda_stream
    X = torch.zeros(1, 2, 8, 8, 16, dtype=torch.bfloat16, device="cuda")
    Y = torch.zeros(1, 2, 4, 4, 16, dtype=torch.bfloat16, device="cuda")
    am = torch.zeros(1, 2, 4, 4, 16, dtype=torch.uint8, device="cuda")
    with pytest.raises(H.HftaError) as e:          # pad > k / 2
        H.hfta_maxpool2d_fwd(1, 2, 8, 8, 16, 3, 2, 2, H.HFTA_BF16, H.tin(X, X[0].numel(), 16),
                             H.tout(Y, Y[0].numel(), 16), H.ptr(am), am[0].numel(), st)
    assert e.value.code == H.HFTA_ERR_SHAPE
    with pytest.raises(H.HftaError) as e:          # ld != C (not dense NHWC)
        H.hfta_maxpool2d_fwd(1, 2, 8, 8, 16, 3, 2, 1, H.HFTA_BF16, H.tin(X, X[0].numel(), 32),
                             H.tout(Y, Y[0].numel(), 16), H.ptr(am), am[0].numel(), st)
    assert e.value.code == H.HFTA_ERR_SHAPE
    with pytest.raises(H.HftaError) as e:          # B = 0
        H.hfta_avgpool2d_fwd(0, 2, 64, 16, H.HFTA_BF16, H.tin(X, 0, 16), H.tout(Y, 16, 16), st)
    assert e.value.code == H.HFTA_ERR_INVALID_VALUE
    d = H.hfta_conv_desc()
    d.N, d.H, d.W, d.C_in, d.C_out, d.kh, d.kw, d.stride, d.pad, d.transposed = 2, 8, 8, 64, 64, 3, 3, 1, 1, 0
    Xc = torch.zeros(1, 2, 8, 8, 64, dtype=torch.bfloat16, device="cuda")
    Wc = torch.zeros(1, 64, 3, 3, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(H.HftaError) as e:          # Tanh is not a gate activation
        H.hfta_fused_conv_bwd_gated(1, d, H.HFTA_BF16, H.tin(Xc, Xc[0].numel(), 64), H.tin(Xc, Xc[0].numel(), 64),
                                    H.tin(Wc, Wc[0].numel(), 576), H.tout(Xc, Xc[0].numel(), 64), None, 0, 0,
                                    H.ACT_TANH, 0.0, H.tin(Xc, Xc[0].numel(), 64), None, 0, st)
    assert e.value.code == H.HFTA_ERR_UNSUPPORTED
