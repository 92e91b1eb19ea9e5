"""ResNet-18 training step for ONE model (NumPy fp64) -- the second model
family (the paper's secondary benchmark).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Architecture (reading R33): the ResNet-18 of the PyTorch examples the paper
cites (torchvision `resnet18`, BasicBlock, ImageNet stem) with 10
classes, trained on CIFAR-10-shaped 32 x 32 images: conv 7x7 s2 p3 (no
bias) -> BN -> ReLU -> MaxPool 3x3 s2 p1; four stages of two BasicBlocks
(widths 64, 128, 256, 512; the first block of stages 2-4 has stride 2 and a
1x1 s2 conv + BN shortcut); AdaptiveAvgPool2d(1); Linear 512 -> 10; cross
entropy (log_softmax + NLL, mean).  BasicBlock: conv3x3(s) -> BN -> ReLU ->
conv3x3 -> BN, + shortcut, ReLU.  Optimizer: Adadelta, PyTorch-1.6
form (oracle/optim.py), per-model lr, rho, eps, wd.

Every layer is the serial operator of its App. B fusion row (Conv2d
P:L1262-1263, BatchNorm2d P:L1277-1278, MaxPool2d / AdaptiveAvgPool2d
P:L1286-1290, ReLU, Linear P:L1271-1272); B fused models = B independent
runs of this function.  ReLU gates and max-pool argmaxes are
decision sites (oracle/decisions.py).
"""
import numpy as np

from . import layers as Lr
from . import decisions as D
from .models import _bn_state, _bn_err_scale, _conv
from .optim import adadelta_step

STAGES = (64, 128, 256, 512)


def block_names(widths=STAGES):
    """(name, C_in, C_out, stride, has_downsample) of the 8 BasicBlocks."""
    out = []
    cin = widths[0]
    for s, w in enumerate(widths):
        for b in range(2):
            stride = 2 if (s > 0 and b == 0) else 1
            out.append(("l%d.%d" % (s + 1, b), cin, w, stride, stride != 1 or cin != w))
            cin = w
    return out


def _bn2d(P, S, newS, y, bn):
    z, c = Lr.bn2d_fwd(y, P[bn + ".g"], P[bn + ".beta"])
    rm, rv = _bn_state(S, bn, y.shape[1])
    newS[bn + ".rm"], newS[bn + ".rv"] = Lr.bn_running(rm, rv, c, y.size // y.shape[1])
    return z, c, _bn_err_scale(y, c, P[bn + ".g"])


def _rms_c(x):
    return np.sqrt(np.mean(x * x, axis=(0, 2, 3)))


def forward(P, S, newS, x, widths=STAGES):
    """x [N, 3, H, W] -> logits [N, k] and the cache of the backward."""
    cache = {}
    y, hs, Ws = _conv(P, x, "conv1.W", 2, 3)
    z, c, esc = _bn2d(P, S, newS, y, "bn1")
    gate = D.relu_gate("stem.relu", z, esc)
    a = z * gate
    cache["stem"] = (hs, Ws, c, gate)
    win = Lr.maxpool2d_windows(a, 3, 2, 1)
    N, Ho, Wo, T, C = win.shape
    idx = D.max_index("stem.pool", win.reshape(N * Ho * Wo, T, C), _rms_c(a)).reshape(N, Ho, Wo, C)
    h, _ = Lr.maxpool2d_fwd(a, 3, 2, 1, idx)
    cache["pool"] = (idx, a.shape)
    for name, cin, cout, stride, down in block_names(widths):
        y1, h1s, W1s = _conv(P, h, name + ".conv1.W", stride, 1)
        z1, c1, e1 = _bn2d(P, S, newS, y1, name + ".bn1")
        g1 = D.relu_gate(name + ".relu1", z1, e1)
        a1 = z1 * g1
        y2, h2s, W2s = _conv(P, a1, name + ".conv2.W", 1, 1)
        z2, c2, e2 = _bn2d(P, S, newS, y2, name + ".bn2")
        if down:
            yd, hds, Wds = _conv(P, h, name + ".down.W", stride, 0)
            sc, cd, ed = _bn2d(P, S, newS, yd, name + ".dbn")
            dcache = (hds, Wds, cd)
            esc_sc = ed
        else:
            sc, dcache, esc_sc = h, None, _rms_c(h)
        u = z2 + sc
        g2 = D.relu_gate(name + ".relu2", u, e2 + esc_sc)
        cache[name] = (h1s, W1s, c1, g1, h2s, W2s, c2, g2, dcache, stride)
        h = u * g2
    f = Lr.avgpool_global_fwd(h)
    cache["avg"] = h.shape
    fs = D.store(f, "act", "fc")
    logits = D.store(Lr.linear_fwd(fs, D.store(P["fc.W"], "w", "fc"), P["fc.b"]), "out", "fc", f.shape[1])
    cache["fc"] = fs
    return logits, cache


def backward(P, dlogits, cache, widths=STAGES):
    G = {}
    df, G["fc.W"], G["fc.b"] = Lr.linear_bwd(D.store(dlogits, "grad"), cache["fc"], D.store(P["fc.W"], "w", "fc"))
    dh = Lr.avgpool_global_bwd(df, cache["avg"])
    for name, cin, cout, stride, down in reversed(block_names(widths)):
        h1s, W1s, c1, g1, h2s, W2s, c2, g2, dcache, stride = cache[name]
        du = dh * g2
        dy2, G[name + ".bn2.g"], G[name + ".bn2.beta"] = Lr.bn2d_bwd(du, c2, P[name + ".bn2.g"])
        da1, G[name + ".conv2.W"] = Lr.conv2d_bwd(D.store(dy2, "grad"), h2s, W2s, 1, 1)
        dy1, G[name + ".bn1.g"], G[name + ".bn1.beta"] = Lr.bn2d_bwd(da1 * g1, c1, P[name + ".bn1.g"])
        dh_new, G[name + ".conv1.W"] = Lr.conv2d_bwd(D.store(dy1, "grad"), h1s, W1s, stride, 1)
        if dcache is not None:
            hds, Wds, cd = dcache
            dyd, G[name + ".dbn.g"], G[name + ".dbn.beta"] = Lr.bn2d_bwd(du, cd, P[name + ".dbn.g"])
            dsc, G[name + ".down.W"] = Lr.conv2d_bwd(D.store(dyd, "grad"), hds, Wds, stride, 0)
        else:
            dsc = du
        dh = dh_new + dsc
    idx, a_shape = cache["pool"]
    da = Lr.maxpool2d_bwd(dh, idx, a_shape, 3, 2, 1)
    hs, Ws, c, gate = cache["stem"]
    dy, G["bn1.g"], G["bn1.beta"] = Lr.bn2d_bwd(da * gate, c, P["bn1.g"])
    _, G["conv1.W"] = Lr.conv2d_bwd(D.store(dy, "grad"), hs, Ws, 2, 3, need_dx=False)
    return G


def loss_grads(P, S, x, labels, widths=STAGES):
    newS = {}
    logits, cache = forward(P, S, newS, x, widths)
    loss, dlogits = Lr.nll_mean(logits, labels)
    G = backward(P, dlogits, cache, widths)
    return loss, G, newS, dict(logits=logits)


def adadelta_model(params, grads, state, hp_b):
    """Adadelta on every tensor of one model; state: name -> (square_avg, acc_delta)."""
    new_p, new_s = {}, {}
    for name, p in params.items():
        sq, acc = state.get(name, (np.zeros_like(p), np.zeros_like(p)))
        new_p[name], sq, acc = adadelta_step(p, grads[name], sq, acc, hp_b["lr"], hp_b["rho"], hp_b["eps"],
                                             hp_b["wd"])
        new_s[name] = (sq, acc)
    return new_p, new_s


def train_step(P, S, opt, batch, hp_b, widths=STAGES):
    """One serial step of one model: forward, backward, Adadelta."""
    x, labels = batch
    loss, G, newS, out = loss_grads(P, S, x, labels, widths)
    newP, newOpt = adadelta_model(P, G, opt, hp_b)
    return dict(loss=loss, grads=G, params=newP, opt=newOpt, stats=newS, out=out)


def fused_step_oracle(Ps, Ss, opts, batch, hp, widths=STAGES):
    """B independent serial steps and the fused loss (App. C Eq. 1)."""
    res = [train_step(Ps[b], Ss[b], opts[b], batch, {k: float(v[b]) for k, v in hp.items()}, widths)
           for b in range(len(Ps))]
    losses = np.array([r["loss"] for r in res])
    return res, losses, losses.mean()
