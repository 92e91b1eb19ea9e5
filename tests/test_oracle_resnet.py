"""Pins of the ResNet-18 oracle (NEXT-4, oracle/resnet.py) and its pooling
layers (oracle/layers.py) against things other than itself: brute-force
window loops, PyTorch CPU fp64 functional ops + autograd (an independent
implementation of the same network), the published parameter count."""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth
from oracle import layers as Lr
from oracle import resnet as R



def test_param_count_is_torchvision_resnet18_10_classes():
    """torchvision resnet18(num_classes=10) has 11 181 642 parameters (the
    1000-class model's 11 689 512 minus 513 x 990)."""
    n = sum(int(np.prod(s)) for _, s, _ in synth.param_specs("resnet18"))
    assert n == 11689512 - 513 * 990 == 11181642


def _maxpool_brute(x, k, s, p):
    N, C, H, W = x.shape
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    y = np.zeros((N, C, Ho, Wo))
    arg = np.zeros((N, C, Ho, Wo, 2), dtype=np.int64)
    for n, c, oy, ox in itertools.product(range(N), range(C), range(Ho), range(Wo)):
        best, bi = -np.inf, None
        for ky in range(k):
            for kx in range(k):
                iy, ix = oy * s - p + ky, ox * s - p + kx
                if 0 <= iy < H and 0 <= ix < W and x[n, c, iy, ix] > best:   # strict: first tap wins ties
                    best, bi = x[n, c, iy, ix], (iy, ix)
        y[n, c, oy, ox] = best
        arg[n, c, oy, ox] = bi
    return y, arg


@pytest.mark.parametrize("H,k,s,p", [(9, 3, 2, 1), (8, 3, 2, 1), (7, 2, 2, 0), (5, 3, 1, 1)])
def test_maxpool_brute_force_with_ties(H, k, s, p):
    g = np.random.default_rng(H * 10 + k)
    x = np.round(g.standard_normal((2, 3, H, H)) * 2) / 2         # coarse grid: many exact ties
    y, idx = Lr.maxpool2d_fwd(x, k, s, p)
    yb, arg = _maxpool_brute(x, k, s, p)
    assert np.array_equal(y, yb)
    dy = g.standard_normal(y.shape)
    dx = Lr.maxpool2d_bwd(dy, idx, x.shape, k, s, p)
    dxb = np.zeros_like(x)
    N, C, Ho, Wo = y.shape
    for n, c, oy, ox in itertools.product(range(N), range(C), range(Ho), range(Wo)):
        iy, ix = arg[n, c, oy, ox]
        dxb[n, c, iy, ix] += dy[n, c, oy, ox]
    assert np.array_equal(dx, dxb)


def test_maxpool_and_avgpool_vs_torch():
    g = np.random.default_rng(3)
    x = g.standard_normal((2, 4, 16, 16))
    dy = g.standard_normal((2, 4, 8, 8))
    tx = torch.tensor(x, requires_grad=True)
    ty = F.max_pool2d(tx, 3, 2, 1)
    ty.backward(torch.tensor(dy))
    y, idx = Lr.maxpool2d_fwd(x, 3, 2, 1)
    np.testing.assert_allclose(y, ty.detach().numpy(), rtol=0, atol=0)
    np.testing.assert_allclose(Lr.maxpool2d_bwd(dy, idx, x.shape, 3, 2, 1), tx.grad.numpy(), rtol=0, atol=1e-15)
    tx.grad = None
    ta = F.adaptive_avg_pool2d(tx, 1)
    da = g.standard_normal((2, 4))
    ta.backward(torch.tensor(da)[:, :, None, None])
    np.testing.assert_allclose(Lr.avgpool_global_fwd(x), ta.detach().numpy()[:, :, 0, 0], rtol=1e-14)
    np.testing.assert_allclose(Lr.avgpool_global_bwd(da, x.shape), tx.grad.numpy(), rtol=1e-14)


def _torch_resnet(P, x, labels, widths):
    """The same network written with torch.nn.functional (fp64, autograd)."""
    T = {n: torch.tensor(v, requires_grad=True) for n, v in P.items()}
    run = {}

    def bn(y, name):
        rm, rv = torch.zeros(y.shape[1], dtype=torch.float64), torch.ones(y.shape[1], dtype=torch.float64)
        out = F.batch_norm(y, rm, rv, T[name + ".g"], T[name + ".beta"], training=True, momentum=0.1, eps=1e-5)
        run[name] = (rm, rv)
        return out

    h = F.relu(bn(F.conv2d(torch.tensor(x), T["conv1.W"], stride=2, padding=3), "bn1"))
    h = F.max_pool2d(h, 3, 2, 1)
    for name, cin, cout, stride, down in R.block_names(widths):
        a = F.relu(bn(F.conv2d(h, T[name + ".conv1.W"], stride=stride, padding=1), name + ".bn1"))
        z = bn(F.conv2d(a, T[name + ".conv2.W"], padding=1), name + ".bn2")
        sc = bn(F.conv2d(h, T[name + ".down.W"], stride=stride), name + ".dbn") if down else h
        h = F.relu(z + sc)
    f = F.adaptive_avg_pool2d(h, 1).flatten(1)
    logits = F.linear(f, T["fc.W"], T["fc.b"])
    loss = F.cross_entropy(logits, torch.tensor(labels))
    loss.backward()
    return float(loss.detach()), {n: t.grad.numpy() for n, t in T.items()}, run


@pytest.mark.parametrize("widths", [(8, 8, 16, 16), (8, 16, 16, 32)])
def test_resnet18_oracle_vs_torch_autograd(widths):
    P = {n: v.astype(np.float64) for n, v in synth.init_params("resnet18", 1001, widths=widths).items()}
    x, labels = synth.cifar(seed=5, N=6)
    loss, G, newS, _ = R.loss_grads(P, {}, x.astype(np.float64), labels, widths)
    tl, tg, run = _torch_resnet(P, x.astype(np.float64), labels, widths)
    assert abs(loss - tl) <= 1e-12 * abs(tl)
    assert set(G) == set(tg)
    for n in tg:
        err = np.linalg.norm(G[n] - tg[n]) / max(np.linalg.norm(tg[n]), 1e-300)
        assert err < 1e-10, (n, err)
    for name, (rm, rv) in run.items():
        np.testing.assert_allclose(newS[name + ".rm"], rm.numpy(), rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(newS[name + ".rv"], rv.numpy(), rtol=1e-12, atol=1e-14)


def test_resnet18_step_vs_torch_adadelta():
    """One fused step over B = 2 models with different hyper-parameters equals
    two torch.optim.Adadelta steps (one param group per model)."""
    widths = (8, 8, 16, 16)
    hp = synth.hparams_resnet(3, 2)
    Ps = [{n: v.astype(np.float64) for n, v in synth.init_params("resnet18", 1000 + b, widths=widths).items()}
          for b in range(2)]
    x, labels = synth.cifar(seed=7, N=4)
    res, losses, mean = R.fused_step_oracle(Ps, [{}, {}], [{}, {}], (x.astype(np.float64), labels), hp, widths)
    for b in range(2):
        T = {n: torch.tensor(v, requires_grad=True) for n, v in Ps[b].items()}
        opt = torch.optim.Adadelta(list(T.values()), lr=float(hp["lr"][b]), rho=float(hp["rho"][b]),
                                   eps=float(hp["eps"][b]), weight_decay=float(hp["wd"][b]))
        for n, t in T.items():
            t.grad = torch.tensor(res[b]["grads"][n])
        opt.step()
        for n, t in T.items():
            np.testing.assert_allclose(res[b]["params"][n], t.detach().numpy(), rtol=1e-12, atol=1e-14)
    assert abs(mean - losses.mean()) == 0.0
