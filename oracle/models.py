"""Per-model training steps, each model trained ALONE (NumPy fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

HFTA's defining invariant: fusion "only" applies "mathematically equivalent
transformations" and "theoretically does not have any effect on the
models' original convergence"; per-model gradients of the fused loss
equal the serial ones (App. C Eq. 1-3, with the sum over
b = 0..B-1, reading R8).  So the oracle of a fused step over B models is B
independent serial steps: `fused_step_oracle` below is literally a Python loop
over b calling the one-model step with hp_b.

Architectures (reading R1): PointNet cls/seg as in the implementation cited at
P:L1659 (STN3d + PointNetfeat + heads; feature transform off, R2); DCGAN as in
the example cited at P:L1662 (nz=100, ngf=ndf=64, nc=3, bias-free convs).
cfg1 is BJ configs[0]: shared MLP conv 3->64->64 with BN+ReLU, MSE loss.
"""
import numpy as np

from . import layers as Lr
from .adam import adam_model
from .philox import dropout_keep_mask


# ------------------------------------------------------------- helpers ----
# Decision margins (reading R15b).  ReLU'(z) and the argmax of a max-pool are
# discontinuous decisions; an element whose decision is within rounding
# distance of the threshold may legitimately be taken either way by a
# lower-precision implementation.  When `MARGINS` is a list, every ReLU and
# max-pool of a forward pass appends its smallest relative margin:
#   ReLU: min_r,c |z| / rms(z)    max-pool: min_n,c (top1 - top2) / |top1|
MARGINS = None


def _note(kind, name, value):
    if MARGINS is not None:
        MARGINS.append((kind, name, float(value)))


def _relu_margin(name, z):
    if MARGINS is not None:
        _note("relu", name, np.min(np.abs(z)) / max(np.sqrt(np.mean(z * z)), 1e-300))


def _max_margin(name, x):
    if MARGINS is not None:
        s = np.sort(x, axis=1)
        _note("max", name, np.min((s[:, -1] - s[:, -2]) / np.maximum(np.abs(s[:, -1]), 1e-300)))


def _bn_state(state, name, C):
    return state.get(name + ".rm", np.zeros(C)), state.get(name + ".rv", np.ones(C))


def _conv_bn_act(P, S, newS, r, conv, bn, act):
    """y = r W^T + b -> BN (train) -> act; returns output and cache."""
    y = Lr.linear_fwd(r, P[conv + ".W"], P[conv + ".b"])
    z, c = Lr.bn_fwd(y, P[bn + ".g"], P[bn + ".beta"])
    rm, rv = _bn_state(S, bn, y.shape[1])
    newS[bn + ".rm"], newS[bn + ".rv"] = Lr.bn_running(rm, rv, c, y.shape[0])
    if act == "relu":
        _relu_margin(bn, z)
    a = Lr.relu(z) if act == "relu" else z
    return a, dict(r=r, z=z, bn=c, conv=conv, bnn=bn, act=act)


def _conv_bn_act_bwd(P, G, da, cache, need_dx=True):
    dz = Lr.relu_bwd(da, cache["z"]) if cache["act"] == "relu" else da
    dy, G[cache["bnn"] + ".g"], G[cache["bnn"] + ".beta"] = Lr.bn_bwd(dz, cache["bn"], P[cache["bnn"] + ".g"])
    dr, G[cache["conv"] + ".W"], G[cache["conv"] + ".b"] = Lr.linear_bwd(dy, cache["r"], P[cache["conv"] + ".W"], need_dx)
    return dr


# -------------------------------------------------------------- cfg1 ----

def mlp_cfg1_loss_grads(P, S, x, T):
    """BJ configs[0]: a = relu(bn(x W1^T + b1)); a2 = relu(bn(a W2^T + b2)); l = mse(a2, T)."""
    newS = {}
    a1, k1 = _conv_bn_act(P, S, newS, x, "c1", "bn1", "relu")
    a2, k2 = _conv_bn_act(P, S, newS, a1, "c2", "bn2", "relu")
    loss, da2 = Lr.mse_mean(a2, T)
    G = {}
    da1 = _conv_bn_act_bwd(P, G, da2, k2)
    _conv_bn_act_bwd(P, G, da1, k1, need_dx=False)
    return loss, G, newS, dict(a2=a2)


# ---------------------------------------------------------- PointNet ----

def _stn_fwd(P, S, newS, x):
    N, L, _ = x.shape
    r = x.reshape(N * L, 3)
    a1, k1 = _conv_bn_act(P, S, newS, r, "stn.c1", "stn.bn1", "relu")
    a2, k2 = _conv_bn_act(P, S, newS, a1, "stn.c2", "stn.bn2", "relu")
    a3, k3 = _conv_bn_act(P, S, newS, a2, "stn.c3", "stn.bn3", "relu")
    _max_margin("stn.max", a3.reshape(N, L, -1))
    g, idx = Lr.max_over_points(a3.reshape(N, L, -1))
    f1, k4 = _conv_bn_act(P, S, newS, g, "stn.fc1", "stn.bn4", "relu")
    f2, k5 = _conv_bn_act(P, S, newS, f1, "stn.fc2", "stn.bn5", "relu")
    f3 = Lr.linear_fwd(f2, P["stn.fc3.W"], P["stn.fc3.b"])
    T = f3.reshape(N, 3, 3) + np.eye(3)
    return T, dict(k=(k1, k2, k3, k4, k5), idx=idx, f2=f2, L=L)


def _stn_bwd(P, G, dT, c):
    N = dT.shape[0]
    df2, G["stn.fc3.W"], G["stn.fc3.b"] = Lr.linear_bwd(dT.reshape(N, 9), c["f2"], P["stn.fc3.W"])
    k1, k2, k3, k4, k5 = c["k"]
    df1 = _conv_bn_act_bwd(P, G, df2, k5)
    dg = _conv_bn_act_bwd(P, G, df1, k4)
    da3 = Lr.max_over_points_bwd(dg, c["idx"], c["L"]).reshape(-1, dg.shape[1])
    da2 = _conv_bn_act_bwd(P, G, da3, k3)
    da1 = _conv_bn_act_bwd(P, G, da2, k2)
    _conv_bn_act_bwd(P, G, da1, k1, need_dx=False)   # input points: no dgrad


def _feat_fwd(P, S, newS, x):
    N, L, _ = x.shape
    T, stn_c = _stn_fwd(P, S, newS, x)
    xt = Lr.transform_points(x, T)
    r = xt.reshape(N * L, 3)
    a1, k1 = _conv_bn_act(P, S, newS, r, "feat.c1", "feat.bn1", "relu")
    a2, k2 = _conv_bn_act(P, S, newS, a1, "feat.c2", "feat.bn2", "relu")
    z3, k3 = _conv_bn_act(P, S, newS, a2, "feat.c3", "feat.bn3", None)
    _max_margin("feat.max", z3.reshape(N, L, -1))
    g, idx = Lr.max_over_points(z3.reshape(N, L, -1))
    return g, a1, dict(T=T, stn=stn_c, x=x, k=(k1, k2, k3), idx=idx, L=L)


def _feat_bwd(P, G, dg, da1_extra, c):
    k1, k2, k3 = c["k"]
    dz3 = Lr.max_over_points_bwd(dg, c["idx"], c["L"]).reshape(-1, dg.shape[1])
    da2 = _conv_bn_act_bwd(P, G, dz3, k3)
    da1 = _conv_bn_act_bwd(P, G, da2, k2)
    if da1_extra is not None:
        da1 = da1 + da1_extra
    dr = _conv_bn_act_bwd(P, G, da1, k1)
    N, L = c["x"].shape[0], c["L"]
    _, dT = Lr.transform_points_bwd(dr.reshape(N, L, 3), c["x"], c["T"])
    _stn_bwd(P, G, dT, c["stn"])


def pointnet_cls_loss_grads(P, S, x, labels, keep, p_drop):
    """Forward + backward of PointNetCls for ONE model; keep = dropout keep mask [N, f2]."""
    newS = {}
    g, _, fc = _feat_fwd(P, S, newS, x)
    h1, k1 = _conv_bn_act(P, S, newS, g, "head.fc1", "head.bn1", "relu")
    y2 = Lr.linear_fwd(h1, P["head.fc2.W"], P["head.fc2.b"])
    d2 = Lr.dropout(y2, keep, p_drop)
    z2, bn2 = Lr.bn_fwd(d2, P["head.bn2.g"], P["head.bn2.beta"])
    rm, rv = _bn_state(S, "head.bn2", d2.shape[1])
    newS["head.bn2.rm"], newS["head.bn2.rv"] = Lr.bn_running(rm, rv, bn2, d2.shape[0])
    _relu_margin("head.bn2", z2)
    h2 = Lr.relu(z2)
    logits = Lr.linear_fwd(h2, P["head.fc3.W"], P["head.fc3.b"])
    loss, dlogits = Lr.nll_mean(logits, labels)
    G = {}
    dh2, G["head.fc3.W"], G["head.fc3.b"] = Lr.linear_bwd(dlogits, h2, P["head.fc3.W"])
    dz2 = Lr.relu_bwd(dh2, z2)
    dd2, G["head.bn2.g"], G["head.bn2.beta"] = Lr.bn_bwd(dz2, bn2, P["head.bn2.g"])
    dy2 = Lr.dropout_bwd(dd2, keep, p_drop)
    dh1, G["head.fc2.W"], G["head.fc2.b"] = Lr.linear_bwd(dy2, h1, P["head.fc2.W"])
    dg = _conv_bn_act_bwd(P, G, dh1, k1)
    _feat_bwd(P, G, dg, None, fc)
    return loss, G, newS, dict(logits=logits, T=fc["T"], g=g)


def pointnet_seg_loss_grads(P, S, x, labels):
    """Forward + backward of PointNetDenseCls for ONE model; labels [N, L]."""
    newS = {}
    N, L, _ = x.shape
    g, pointfeat, fc = _feat_fwd(P, S, newS, x)
    C3 = g.shape[1]
    h0 = np.concatenate([np.repeat(g, L, axis=0), pointfeat], axis=1)   # [N*L, C3+C1]
    h1, k1 = _conv_bn_act(P, S, newS, h0, "head.c1", "head.bn1", "relu")
    h2, k2 = _conv_bn_act(P, S, newS, h1, "head.c2", "head.bn2", "relu")
    h3, k3 = _conv_bn_act(P, S, newS, h2, "head.c3", "head.bn3", "relu")
    logits = Lr.linear_fwd(h3, P["head.c4.W"], P["head.c4.b"])
    loss, dlogits = Lr.nll_mean(logits, labels.reshape(-1))
    G = {}
    dh3, G["head.c4.W"], G["head.c4.b"] = Lr.linear_bwd(dlogits, h3, P["head.c4.W"])
    dh2 = _conv_bn_act_bwd(P, G, dh3, k3)
    dh1 = _conv_bn_act_bwd(P, G, dh2, k2)
    dh0 = _conv_bn_act_bwd(P, G, dh1, k1)
    dg = dh0[:, :C3].reshape(N, L, C3).sum(axis=1)
    _feat_bwd(P, G, dg, dh0[:, C3:], fc)
    return loss, G, newS, dict(logits=logits, T=fc["T"], g=g)


# -------------------------------------------------------------- DCGAN ----

G_LAYERS = [(1, 0), (2, 1), (2, 1), (2, 1), (2, 1)]     # (stride, pad) of t1..t5
D_LAYERS = [(2, 1), (2, 1), (2, 1), (2, 1), (1, 0)]     # c1..c5


def gen_fwd(P, S, newS, z):
    h = z.reshape(z.shape[0], -1, 1, 1)
    cache = []
    for i, (s, p) in enumerate(G_LAYERS):
        y = Lr.convT2d_fwd(h, P["t%d.W" % (i + 1)], s, p)
        if i < 4:
            bn = "bn%d" % (i + 1)
            zz, c = Lr.bn2d_fwd(y, P[bn + ".g"], P[bn + ".beta"])
            rm, rv = _bn_state(S, bn, y.shape[1])
            newS[bn + ".rm"], newS[bn + ".rv"] = Lr.bn_running(rm, rv, c, y.size // y.shape[1])
            cache.append((h, zz, c))
            h = Lr.relu(zz)
        else:
            cache.append((h, None, None))
            h = Lr.tanh(y)
    return h, cache


def gen_bwd(P, dimg, img, cache):
    G = {}
    dy = Lr.tanh_bwd(dimg, img)
    for i in range(4, -1, -1):
        s, p = G_LAYERS[i]
        h, zz, c = cache[i]
        if i < 4:
            bn = "bn%d" % (i + 1)
            dzz = Lr.relu_bwd(dy, zz)
            dy, G[bn + ".g"], G[bn + ".beta"] = Lr.bn2d_bwd(dzz, c, P[bn + ".g"])
        dh, G["t%d.W" % (i + 1)] = Lr.convT2d_bwd(dy, h, P["t%d.W" % (i + 1)], s, p, need_dx=i > 0)
        dy = dh
    return G


def disc_fwd(P, S, newS, img):
    """D forward; returns (sigmoid output [N], logit [N], cache)."""
    h = img
    cache = []
    for i, (s, p) in enumerate(D_LAYERS):
        y = Lr.conv2d_fwd(h, P["c%d.W" % (i + 1)], s, p)
        if i == 0:
            cache.append((h, y, None))
            h = Lr.leaky_relu(y)
        elif i < 4:
            bn = "bn%d" % (i + 1)
            zz, c = Lr.bn2d_fwd(y, P[bn + ".g"], P[bn + ".beta"])
            rm, rv = _bn_state(S, bn, y.shape[1])
            newS[bn + ".rm"], newS[bn + ".rv"] = Lr.bn_running(rm, rv, c, y.size // y.shape[1])
            cache.append((h, zz, c))
            h = Lr.leaky_relu(zz)
        else:
            cache.append((h, None, None))
            logit = y.reshape(-1)
            h = Lr.sigmoid(y)
    return h.reshape(-1), logit, cache


def disc_bwd(P, dlogit, cache, need_wgrad=True, need_dx=False):
    """Backward through D from d(logit) [N] (the Sigmoid -> BCE gradient,
    reading R29); returns (dimg or None, grads)."""
    G = {}
    N = dlogit.shape[0]
    dy = dlogit.reshape(N, 1, 1, 1)
    dh = None
    for i in range(4, -1, -1):
        s, p = D_LAYERS[i]
        h, zz, c = cache[i]
        if i == 0:
            dy = Lr.leaky_relu_bwd(dy, zz)
        elif i < 4:
            bn = "bn%d" % (i + 1)
            dzz = Lr.leaky_relu_bwd(dy, zz)
            dy, G[bn + ".g"], G[bn + ".beta"] = Lr.bn2d_bwd(dzz, c, P[bn + ".g"])
        dh, dW = Lr.conv2d_bwd(dy, h, P["c%d.W" % (i + 1)], s, p, need_dx=(i > 0 or need_dx))
        if need_wgrad:
            G["c%d.W" % (i + 1)] = dW
        dy = dh
    return dh, G


def dcgan_iteration(PG, PD, SG, SD, optG, optD, real, z, t, hp_b, hpD_b=None):
    """One DCGAN iteration for ONE model, in the order of the cited example
    (reading R4): D(real) backward, D(fake.detach) backward accumulating,
    Adam(D), D'(fake) backward into G, Adam(G).  hpD_b (default hp_b) lets a
    test give D its own hyper-parameters (e.g. lr 0)."""
    hpD_b = hp_b if hpD_b is None else hpD_b
    newSD1, newSD2, newSD3, newSG = {}, {}, {}, {}
    N = real.shape[0]
    ones, zeros = np.ones(N), np.zeros(N)
    out_r, zr, cr = disc_fwd(PD, SD, newSD1, real)
    errD_real, dz = Lr.bce_sigmoid_mean(zr, ones)
    _, GD_r = disc_bwd(PD, dz, cr)
    fake, cg = gen_fwd(PG, SG, newSG, z)
    out_f, zf, cf = disc_fwd(PD, newSD1, newSD2, fake)
    errD_fake, dz = Lr.bce_sigmoid_mean(zf, zeros)
    _, GD_f = disc_bwd(PD, dz, cf)
    GD = {k: GD_r[k] + GD_f[k] for k in GD_r}
    PD2, optD2 = adam_model(PD, GD, optD, t, hpD_b)
    out_g, zg, cg2 = disc_fwd(PD2, newSD2, newSD3, fake)
    errG, dz = Lr.bce_sigmoid_mean(zg, ones)
    dfake, _ = disc_bwd(PD2, dz, cg2, need_wgrad=False, need_dx=True)
    GG = gen_bwd(PG, dfake, fake, cg)
    PG2, optG2 = adam_model(PG, GG, optG, t, hp_b)
    return dict(errD_real=errD_real, errD_fake=errD_fake, errG=errG, GD=GD, GG=GG,
                PD=PD2, PG=PG2, optD=optD2, optG=optG2, SD=newSD3, SG=newSG, fake=fake,
                out_real=out_r, out_fake=out_f, out_g=out_g)


# ------------------------------------------------- the fused-step oracle ----

def hp_of(hp, b):
    return {k: float(v[b]) for k, v in hp.items()}


def train_step(arch, P, S, opt, batch, t, hp_b, b=0, dropout_seed=42, p_drop=0.3):
    """One serial training step of model b: forward, backward, Adam (t >= 1).

    Returns loss, grads (before the step), new params, new Adam state, new BN
    running stats and a few forward outputs.
    """
    if arch == "mlp_cfg1":
        loss, G, newS, out = mlp_cfg1_loss_grads(P, S, *batch)
    elif arch == "pointnet_cls":
        x, labels = batch
        f2 = P["head.fc2.W"].shape[0]
        keep = dropout_keep_mask(dropout_seed, b, t, 0, x.shape[0] * f2, p_drop).reshape(x.shape[0], f2)
        loss, G, newS, out = pointnet_cls_loss_grads(P, S, x, labels, keep, p_drop)
        out["keep"] = keep
    elif arch == "pointnet_seg":
        loss, G, newS, out = pointnet_seg_loss_grads(P, S, *batch)
    else:
        raise ValueError(arch)
    newP, newOpt = adam_model(P, G, opt, t, hp_b)
    return dict(loss=loss, grads=G, params=newP, opt=newOpt, stats=newS, out=out)


def decision_margins(arch, P, batch, t=1, b=0, **kw):
    """Smallest ReLU / max-pool margins of one model's forward (reading R15b)."""
    global MARGINS
    MARGINS = []
    try:
        train_step(arch, P, {}, {}, batch, t, dict(lr=0.0, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0), b=b, **kw)
        return list(MARGINS)
    finally:
        MARGINS = None


def fused_step_oracle(arch, Ps, Ss, opts, batch, t, hp, **kw):
    """The oracle of one fused step over B models: B independent serial steps
    (P:L923), plus the fused loss L = (1/B) sum_b l_b (App. C Eq. 1)."""
    res = [train_step(arch, Ps[b], Ss[b], opts[b], batch, t, hp_of(hp, b), b=b, **kw)
           for b in range(len(Ps))]
    losses = np.array([r["loss"] for r in res])
    return res, losses, losses.mean()
