"""Pins of the oracle's layer definitions against things other than itself:
worked examples, closed forms, brute-force loops, PyTorch CPU fp64 library
routines and central finite differences (h=1e-6, rel 1e-4,
abs floor 1e-7)."""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import layers as L
from oracle.adam import adam_step
from oracle.philox import dropout_keep_mask

R = np.random.default_rng(123)


def t(a):
    return torch.tensor(a, dtype=torch.float64)


def fd_check(f, x, dx_analytic, n=6, h=1e-6, rel=1e-4, floor=1e-7):
    """Central differences of scalar f at n random coordinates of x."""
    flat = x.reshape(-1)
    idx = R.choice(flat.size, size=min(n, flat.size), replace=False)
    for i in idx:
        old = flat[i]
        flat[i] = old + h
        fp = f()
        flat[i] = old - h
        fm = f()
        flat[i] = old
        num = (fp - fm) / (2 * h)
        ana = dx_analytic.reshape(-1)[i]
        assert abs(num - ana) <= max(rel * abs(num), floor), (i, num, ana)


# ---------------------------------------------------------------- linear ----

def test_linear_worked_example():
    # [[1,2],[3,4]] x [[5],[6]] = [[17],[39]]; Linear stores W as [out, in].
    y = L.linear_fwd(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0, 6.0]]))
    assert np.array_equal(y, [[17.0], [39.0]])


def test_linear_bruteforce_and_torch():
    x, W, b = R.standard_normal((5, 4)), R.standard_normal((3, 4)), R.standard_normal(3)
    y = L.linear_fwd(x, W, b)
    ref = np.zeros((5, 3))
    for r in range(5):
        for n in range(3):
            ref[r, n] = b[n] + sum(x[r, k] * W[n, k] for k in range(4))
    assert np.allclose(y, ref, rtol=1e-14, atol=1e-14)
    assert np.allclose(y, F.linear(t(x), t(W), t(b)).numpy(), rtol=1e-14, atol=1e-14)


def test_linear_bwd_fd_and_autograd():
    x, W, b = R.standard_normal((7, 5)), R.standard_normal((4, 5)), R.standard_normal(4)
    C = R.standard_normal((7, 4))
    f = lambda: float((L.linear_fwd(x, W, b) * C).sum())
    dx, dW, db = L.linear_bwd(C, x, W)
    fd_check(f, x, dx)
    fd_check(f, W, dW)
    fd_check(f, b, db)
    xt, Wt, bt = (t(a).requires_grad_() for a in (x, W, b))
    (F.linear(xt, Wt, bt) * t(C)).sum().backward()
    for a, r in ((dx, xt), (dW, Wt), (db, bt)):
        assert np.allclose(a, r.grad.numpy(), rtol=1e-13, atol=1e-13)


# ------------------------------------------------------------- batchnorm ----

def test_bn_closed_form_moments():
    x = R.standard_normal((50, 6)) * 3 + 1
    g, be = R.uniform(0.5, 1.5, 6), R.uniform(-1, 1, 6)
    y, c = L.bn_fwd(x, g, be)
    var = x.var(axis=0)
    assert np.allclose(y.mean(axis=0), be, atol=1e-12)
    assert np.allclose(y.var(axis=0), g * g * var / (var + L.BN_EPS), rtol=1e-12)


def test_bn_vs_torch_fwd_running_bwd():
    x = R.standard_normal((40, 5)) * 2 - 0.5
    g, be = R.uniform(0.5, 1.5, 5), R.uniform(-1, 1, 5)
    rm0, rv0 = R.standard_normal(5), R.uniform(0.5, 2, 5)
    y, c = L.bn_fwd(x, g, be)
    rm, rv = L.bn_running(rm0, rv0, c, 40)
    xt, gt, bt = (t(a).requires_grad_() for a in (x, g, be))
    rmt, rvt = t(rm0.copy()), t(rv0.copy())
    yt = F.batch_norm(xt, rmt, rvt, gt, bt, training=True, momentum=0.1, eps=1e-5)
    assert np.allclose(y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(rm, rmt.numpy(), rtol=1e-13) and np.allclose(rv, rvt.numpy(), rtol=1e-13)
    C = R.standard_normal((40, 5))
    (yt * t(C)).sum().backward()
    dx, dg, db = L.bn_bwd(C, c, g)
    assert np.allclose(dx, xt.grad.numpy(), rtol=1e-10, atol=1e-12)
    assert np.allclose(dg, gt.grad.numpy(), rtol=1e-12)
    assert np.allclose(db, bt.grad.numpy(), rtol=1e-12)


def test_bn_running_recurrence_k_steps():
    # after k steps on constant batches the running mean is
    # (1 - 0.9^k) * mean (start 0), a closed form of the recurrence.
    x = R.standard_normal((30, 3)) + 2.0
    rm, rv = np.zeros(3), np.ones(3)
    for _ in range(5):
        _, c = L.bn_fwd(x, np.ones(3), np.zeros(3))
        rm, rv = L.bn_running(rm, rv, c, 30)
    assert np.allclose(rm, (1 - 0.9 ** 5) * x.mean(axis=0), rtol=1e-13)
    uv = x.var(axis=0, ddof=1)
    assert np.allclose(rv, 0.9 ** 5 + (1 - 0.9 ** 5) * uv, rtol=1e-13)


def test_bn_bwd_fd():
    x = R.standard_normal((12, 3))
    g, be = R.uniform(0.5, 1.5, 3), R.uniform(-1, 1, 3)
    C = R.standard_normal((12, 3))
    f = lambda: float((L.bn_fwd(x, g, be)[0] * C).sum())
    _, c = L.bn_fwd(x, g, be)
    dx, dg, db = L.bn_bwd(C, c, g)
    fd_check(f, x, dx)
    fd_check(f, g, dg)
    fd_check(f, be, db)


def test_bn2d_vs_torch():
    x = R.standard_normal((3, 4, 5, 5))
    g, be = R.uniform(0.5, 1.5, 4), R.uniform(-1, 1, 4)
    y, c = L.bn2d_fwd(x, g, be)
    xt = t(x).requires_grad_()
    yt = F.batch_norm(xt, None, None, t(g), t(be), training=True, eps=1e-5)
    assert np.allclose(y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
    C = R.standard_normal(x.shape)
    (yt * t(C)).sum().backward()
    dx, _, _ = L.bn2d_bwd(C, c, g)
    assert np.allclose(dx, xt.grad.numpy(), rtol=1e-10, atol=1e-12)


# ----------------------------------------------------------- activations ----

def test_activations_closed_forms():
    assert np.array_equal(L.relu(np.array([-1.0, 0.0, 2.0])), [0.0, 0.0, 2.0])
    assert np.allclose(L.leaky_relu(np.array([-1.0, 3.0]), 0.2), [-0.2, 3.0])
    x = R.standard_normal(20)
    assert np.allclose(L.tanh(x), torch.tanh(t(x)).numpy(), rtol=1e-15)
    assert np.allclose(L.sigmoid(x), torch.sigmoid(t(x)).numpy(), rtol=1e-14)
    C = R.standard_normal(20)
    for fwd, bwd, use_y in ((L.tanh, L.tanh_bwd, True), (L.sigmoid, L.sigmoid_bwd, True),
                            (L.relu, L.relu_bwd, False), (L.leaky_relu, L.leaky_relu_bwd, False)):
        y = fwd(x)
        d = bwd(C, y if use_y else x)
        fd_check(lambda: float((fwd(x) * C).sum()), x, d)


# --------------------------------------------------------- PointNet glue ----

def test_max_over_points_bruteforce_first_index():
    x = R.standard_normal((3, 9, 4))
    x[1, 2, 3] = x[1, 7, 3] = 50.0            # tie: first index wins (reading R15)
    g, idx = L.max_over_points(x)
    for n in range(3):
        for c in range(4):
            best, bi = -np.inf, -1
            for l in range(9):
                if x[n, l, c] > best:
                    best, bi = x[n, l, c], l
            assert g[n, c] == best and idx[n, c] == bi
    assert idx[1, 3] == 2
    dg = R.standard_normal((3, 4))
    dx = L.max_over_points_bwd(dg, idx, 9)
    assert dx.sum() == pytest.approx(dg.sum()) and np.count_nonzero(dx) == 12


def test_transform_points_bruteforce_and_fd():
    x, T = R.standard_normal((2, 5, 3)), R.standard_normal((2, 3, 3))
    y = L.transform_points(x, T)
    for n in range(2):
        for l in range(5):
            for j in range(3):
                assert y[n, l, j] == pytest.approx(sum(x[n, l, i] * T[n, i, j] for i in range(3)), rel=1e-14)
    C = R.standard_normal(y.shape)
    dx, dT = L.transform_points_bwd(C, x, T)
    f = lambda: float((L.transform_points(x, T) * C).sum())
    fd_check(f, x, dx)
    fd_check(f, T, dT)


def test_dropout_mask_and_scale():
    keep = dropout_keep_mask(42, 1, 3, 0, 200000, 0.3)
    assert abs(keep.mean() - 0.7) < 0.005                      # distributional
    assert dropout_keep_mask(42, 1, 3, 0, 10, 0.0).all()       # p = 0 keeps everything
    assert not np.array_equal(keep[:64], dropout_keep_mask(42, 2, 3, 0, 64, 0.3))  # per-model streams
    x = R.standard_normal(10)
    k = dropout_keep_mask(7, 0, 1, 0, 10, 0.5)
    assert np.allclose(L.dropout(x, k, 0.5), np.where(k, 2 * x, 0.0))


# ---------------------------------------------------------------- losses ----

def test_loss_closed_forms():
    # uniform logits -> ln K; BCE(0.5, 1) = ln 2.
    loss, dz = L.nll_mean(np.zeros((4, 40)), np.array([0, 5, 39, 7]))
    assert loss == pytest.approx(math.log(40), rel=1e-15)
    assert np.allclose(dz.sum(axis=1), 0.0, atol=1e-16)
    loss, _ = L.bce_mean(np.array([0.5]), np.array([1.0]))
    assert loss == pytest.approx(math.log(2), rel=1e-15)
    assert L.mse_mean(np.ones(3), np.ones(3))[0] == 0.0


def test_bce_sigmoid_closed_forms_and_torch():
    """Reading R29 pins: (i) wherever fp64 sigmoid is not saturated, the
    logit form equals torch's Sigmoid -> BCELoss (fp64, autograd) -- loss and
    gradient; (ii) closed forms at saturation: BCE(sigmoid(50), 0) = softplus(50)
    = 50 + log1p(e^-50); BCE(sigmoid(150), 0) = 100 (the -100 clamp);
    the gradient below the 1e-12 floor is (p - y) q / 1e-12 with
    q = e^-|z| / (1 + e^-|z|)^2; BCE(sigmoid(0), 1) = ln 2."""
    z = R.uniform(-12, 12, 40)      # torch's 1 - sigmoid(z) loses digits beyond
    for y0 in (0.0, 1.0):
        y = np.full(z.size, y0)
        loss, dz = L.bce_sigmoid_mean(z, y)
        zt = t(z).requires_grad_()
        lt = F.binary_cross_entropy(torch.sigmoid(zt), t(y))
        lt.backward()
        assert loss == pytest.approx(lt.item(), rel=1e-10)
        assert np.allclose(dz, zt.grad.numpy(), rtol=1e-7, atol=0)
        fd_check(lambda: L.bce_sigmoid_mean(z, y)[0], z, dz)
    l, _ = L.bce_sigmoid_mean(np.array([50.0]), np.array([0.0]))
    assert l == pytest.approx(50.0 + math.log1p(math.exp(-50.0)), rel=1e-15)
    l, d = L.bce_sigmoid_mean(np.array([150.0, -150.0]), np.array([0.0, 1.0]))
    assert l == pytest.approx(100.0, rel=1e-15)
    for zz, yy in ((30.0, 0.0), (-30.0, 1.0), (40.0, 0.0), (-35.0, 0.0)):
        e = math.exp(-abs(zz))
        q = e / (1 + e) ** 2
        p = 1 / (1 + math.exp(-zz))
        sig_neg = 1 / (1 + e) if zz < 0 else e / (1 + e)      # sigmoid(-z)
        pmy = -sig_neg if yy == 1.0 else p - yy
        _, d = L.bce_sigmoid_mean(np.array([zz]), np.array([yy]))
        ref = pmy * q / max(q, 1e-12)
        assert d[0] == pytest.approx(ref, rel=1e-12), (zz, yy, d[0], ref)
    l, d = L.bce_sigmoid_mean(np.array([0.0]), np.array([1.0]))
    assert l == pytest.approx(math.log(2), rel=1e-15) and d[0] == pytest.approx(-0.5, rel=1e-15)


def test_philox_known_answers():
    """oracle/philox.py against the Random123 known-answer vectors
    (tests/golden/philox_kat.txt), the external pin of reading R14."""
    import os
    from oracle.philox import philox4x32_10
    path = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")
    n = 0
    for line in open(path):
        if not line.strip() or line.startswith("#"):
            continue
        f = line.split()
        assert f[0] == "10"
        ctr = [int(v, 16) for v in f[1:5]]
        key = [int(v, 16) for v in f[5:7]]
        want = [int(v, 16) for v in f[7:11]]
        got = [int(np.asarray(w).item()) for w in philox4x32_10(ctr, key)]
        assert got == want, (line, [hex(g) for g in got])
        n += 1
    assert n == 3


def test_losses_vs_torch_and_fd():
    z, y = R.standard_normal((6, 10)), R.integers(0, 10, 6)
    loss, dz = L.nll_mean(z, y)
    zt = t(z).requires_grad_()
    lt = F.nll_loss(F.log_softmax(zt, dim=1), torch.tensor(y))
    lt.backward()
    assert loss == pytest.approx(lt.item(), rel=1e-14)
    assert np.allclose(dz, zt.grad.numpy(), rtol=1e-12, atol=1e-15)
    fd_check(lambda: L.nll_mean(z, y)[0], z, dz)
    p, tgt = R.uniform(0.05, 0.95, 8), (R.uniform(size=8) > 0.5).astype(float)
    loss, dp = L.bce_mean(p, tgt)
    pt = t(p).requires_grad_()
    lt = F.binary_cross_entropy(pt, t(tgt))
    lt.backward()
    assert loss == pytest.approx(lt.item(), rel=1e-14)
    assert np.allclose(dp, pt.grad.numpy(), rtol=1e-12)
    a, T = R.standard_normal((4, 3)), R.standard_normal((4, 3))
    loss, da = L.mse_mean(a, T)
    assert loss == pytest.approx(F.mse_loss(t(a), t(T)).item(), rel=1e-14)
    fd_check(lambda: L.mse_mean(a, T)[0], a, da)


# ------------------------------------------------------------------ conv ----

def _conv_brute(x, W, s, p):
    N, Ci, H, Wd = x.shape
    Co, _, kh, kw = W.shape
    Ho, Wo = (H + 2 * p - kh) // s + 1, (Wd + 2 * p - kw) // s + 1
    y = np.zeros((N, Co, Ho, Wo))
    for n in range(N):
        for o in range(Co):
            for i in range(Ho):
                for j in range(Wo):
                    acc = 0.0
                    for c in range(Ci):
                        for u in range(kh):
                            for v in range(kw):
                                yy, xx = i * s - p + u, j * s - p + v
                                if 0 <= yy < H and 0 <= xx < Wd:
                                    acc += x[n, c, yy, xx] * W[o, c, u, v]
                    y[n, o, i, j] = acc
    return y


@pytest.mark.parametrize("s,p", [(2, 1), (1, 0)])
def test_conv2d_bruteforce_torch_fd(s, p):
    x, W = R.standard_normal((2, 3, 8, 8)), R.standard_normal((4, 3, 4, 4))
    y = L.conv2d_fwd(x, W, s, p)
    assert np.allclose(y, _conv_brute(x, W, s, p), rtol=1e-12, atol=1e-12)
    xt, Wt = t(x).requires_grad_(), t(W).requires_grad_()
    yt = F.conv2d(xt, Wt, stride=s, padding=p)
    assert np.allclose(y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
    C = R.standard_normal(y.shape)
    (yt * t(C)).sum().backward()
    dx, dW = L.conv2d_bwd(C, x, W, s, p)
    assert np.allclose(dx, xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(dW, Wt.grad.numpy(), rtol=1e-12, atol=1e-12)
    fd_check(lambda: float((L.conv2d_fwd(x, W, s, p) * C).sum()), W, dW)


@pytest.mark.parametrize("s,p,H", [(2, 1, 4), (1, 0, 1)])
def test_convT2d_size_adjoint_torch(s, p, H):
    x, W = R.standard_normal((2, 5, H, H)), R.standard_normal((5, 3, 4, 4))
    y = L.convT2d_fwd(x, W, s, p)
    assert y.shape[2] == (H - 1) * s - 2 * p + 4                    # S:L133 closed form
    # adjoint identity <ConvT(x), v> = <x, Conv(v)> with the same weights
    v = R.standard_normal(y.shape)
    assert float((y * v).sum()) == pytest.approx(float((x * L.conv2d_fwd(v, W, s, p)).sum()), rel=1e-12)
    xt, Wt = t(x).requires_grad_(), t(W).requires_grad_()
    yt = F.conv_transpose2d(xt, Wt, stride=s, padding=p)
    assert np.allclose(y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
    (yt * t(v)).sum().backward()
    dx, dW = L.convT2d_bwd(v, x, W, s, p)
    assert np.allclose(dx, xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    assert np.allclose(dW, Wt.grad.numpy(), rtol=1e-12, atol=1e-12)


def test_grouped_conv_equals_per_model():
    # Fig. 3 / S:L140: B=2, C_x=3, C_y=4 -> one grouped conv with
    # 6 in, 8 out channels and 2 groups equals the two serial convs.
    x = [R.standard_normal((2, 3, 6, 6)) for _ in range(2)]
    W = [R.standard_normal((4, 3, 4, 4)) for _ in range(2)]
    fused = F.conv2d(t(np.concatenate(x, 1)), t(np.concatenate(W, 0)), stride=2, padding=1, groups=2).numpy()
    assert fused.shape[1] == 8
    for b in range(2):
        assert np.allclose(fused[:, 4 * b:4 * b + 4], L.conv2d_fwd(x[b], W[b], 2, 1), rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ adam ----

def test_adam_first_step_closed_form():
    p, g = R.standard_normal(50), R.standard_normal(50)
    lr, b1, b2, eps, wd = 1e-3, 0.8, 0.99, 1e-6, 0.01
    p1, m, v = adam_step(p, g, np.zeros(50), np.zeros(50), 1, lr, b1, b2, eps, wd)
    gg = g + wd * p
    assert np.allclose(p1 - p, -lr * gg / (np.abs(gg) + eps), rtol=1e-12, atol=1e-18)
    # zero gradient, wd = 0: no change
    assert np.array_equal(adam_step(p, 0 * g, 0 * g, 0 * g, 1, lr, b1, b2, eps, 0.0)[0], p)


def test_adam_vs_torch_one_group_per_model():
    B = 3
    lr, b1, b2, eps, wd = [1e-3, 3e-3, 1e-2], [0.9, 0.8, 0.5], [0.999, 0.99, 0.9], [1e-8, 1e-6, 1e-4], [0, 1e-2, 0.3]
    p0 = R.standard_normal((B, 20))
    grads = R.standard_normal((10, B, 20))
    tp = [torch.nn.Parameter(t(p0[b].copy())) for b in range(B)]
    opt = torch.optim.Adam([dict(params=[tp[b]], lr=lr[b], betas=(b1[b], b2[b]), eps=eps[b],
                                 weight_decay=wd[b]) for b in range(B)])
    ps = [p0[b].copy() for b in range(B)]
    ms = [np.zeros(20) for _ in range(B)]
    vs = [np.zeros(20) for _ in range(B)]
    for step in range(10):
        for b in range(B):
            tp[b].grad = t(grads[step, b])
            ps[b], ms[b], vs[b] = adam_step(ps[b], grads[step, b], ms[b], vs[b], step + 1,
                                            lr[b], b1[b], b2[b], eps[b], wd[b])
        opt.step()
    for b in range(B):
        assert np.allclose(ps[b], tp[b].detach().numpy(), rtol=1e-13, atol=1e-15)


# ------------------------------------------------- SGD / Adadelta / StepLR ----

def test_sgd_vs_torch_one_group_per_model():
    from oracle.optim import sgd_step
    B = 3
    cfg = [dict(lr=1e-2, momentum=0.9, dampening=0.0, weight_decay=0.0, nesterov=False),
           dict(lr=5e-2, momentum=0.5, dampening=0.1, weight_decay=1e-2, nesterov=False),
           dict(lr=1e-3, momentum=0.8, dampening=0.0, weight_decay=3e-2, nesterov=True)]
    p0 = R.standard_normal((B, 17))
    grads = R.standard_normal((6, B, 17))
    tp = [torch.nn.Parameter(t(p0[b].copy())) for b in range(B)]
    opt = torch.optim.SGD([dict(params=[tp[b]], **cfg[b]) for b in range(B)])
    ps, bufs = [p0[b].copy() for b in range(B)], [None] * B
    for step in range(6):
        for b in range(B):
            tp[b].grad = t(grads[step, b])
            c = cfg[b]
            ps[b], bufs[b] = sgd_step(ps[b], grads[step, b], bufs[b], step + 1, c["lr"], c["momentum"],
                                      c["dampening"], c["weight_decay"], c["nesterov"])
        opt.step()
    for b in range(B):
        assert np.allclose(ps[b], tp[b].detach().numpy(), rtol=1e-13, atol=1e-15)


def test_adadelta_vs_torch_and_first_step_closed_form():
    from oracle.optim import adadelta_step
    B = 2
    cfg = [dict(lr=1.0, rho=0.9, eps=1e-6, weight_decay=0.0), dict(lr=0.5, rho=0.5, eps=1e-4, weight_decay=1e-2)]
    p0 = R.standard_normal((B, 11))
    grads = R.standard_normal((5, B, 11))
    tp = [torch.nn.Parameter(t(p0[b].copy())) for b in range(B)]
    opt = torch.optim.Adadelta([dict(params=[tp[b]], **cfg[b]) for b in range(B)])
    st = [(p0[b].copy(), np.zeros(11), np.zeros(11)) for b in range(B)]
    for step in range(5):
        for b in range(B):
            tp[b].grad = t(grads[step, b])
            c = cfg[b]
            st[b] = adadelta_step(st[b][0], grads[step, b], st[b][1], st[b][2], c["lr"], c["rho"], c["eps"],
                                  c["weight_decay"])
            if step == 0:   # |update| = lr g sqrt(eps) / sqrt(eps + (1-rho) g^2)
                g = grads[0, b] + c["weight_decay"] * p0[b]
                up = c["lr"] * g * np.sqrt(c["eps"]) / np.sqrt(c["eps"] + (1 - c["rho"]) * g * g)
                assert np.allclose(p0[b] - st[b][0], up, rtol=1e-12)
        opt.step()
    for b in range(B):
        assert np.allclose(st[b][0], tp[b].detach().numpy(), rtol=1e-12, atol=1e-15)


def test_steplr_closed_form():
    from oracle.optim import steplr
    assert steplr(0.1, 0.5, 10, 25) == pytest.approx(0.025, rel=1e-15)
    assert steplr(0.1, 1.0, 10, 25) == 0.1
    assert [steplr(1.0, 0.5, 5, e) for e in (0, 4, 5, 9, 10)] == [1.0, 1.0, 0.5, 0.5, 0.25]
