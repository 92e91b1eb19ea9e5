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
from . import decisions as D


# ------------------------------------------------------------- helpers ----
# Decision sites (oracle/decisions.py, readings R15b/R15c): every ReLU /
# LeakyReLU gate and max-pool argmax goes through `D.relu_gate` /
# `D.max_index`, which take the oracle's own decision unless a test has
# activated a `Decisions` context with an override inside the flagged band.
# `D.store` is the identity unless a conditioning-witness run installs a
# rounding of stored operands (never used to produce a reference value).


def _bn_state(state, name, C):
    return state.get(name + ".rm", np.zeros(C)), state.get(name + ".rv", np.ones(C))


def _bn_err_scale(y, c, gamma):
    """Magnitude of an implementation's rounding error in z = BN(y) per
    channel: |gamma| rms(y) invstd (decision sites only, reading R15c)."""
    axes = tuple(i for i in range(y.ndim) if i != 1)
    return np.abs(gamma) * np.sqrt(np.mean(y * y, axis=axes)) * c["invstd"]


def _lin(P, r, name):
    """Linear layer on the operands an implementation stores (identity here)."""
    rs, Ws = D.store(r, "act", name), D.store(P[name + ".W"], "w", name)
    return D.store(Lr.linear_fwd(rs, Ws, P[name + ".b"]), "out", name, rs.shape[1]), rs, Ws


def _lin_bwd(dy, rs, Ws, need_dx=True):
    return Lr.linear_bwd(D.store(dy, "grad"), rs, Ws, need_dx)


def _conv_bn_act(P, S, newS, r, conv, bn, act):
    """y = r W^T + b -> BN (train) -> act; returns output and cache."""
    y, rs, Ws = _lin(P, r, conv)
    z, c = Lr.bn_fwd(y, P[bn + ".g"], P[bn + ".beta"])
    rm, rv = _bn_state(S, bn, y.shape[1])
    newS[bn + ".rm"], newS[bn + ".rv"] = Lr.bn_running(rm, rv, c, y.shape[0])
    esc = _bn_err_scale(y, c, P[bn + ".g"])
    gate = D.relu_gate(bn, z, esc) if act == "relu" else None
    a = z * gate if act == "relu" else z           # relu(z) with the site's decision
    return a, dict(r=rs, W=Ws, z=z, gate=gate, bn=c, conv=conv, bnn=bn, act=act, esc=esc)


def _conv_bn_act_bwd(P, G, da, cache, need_dx=True):
    dz = da * cache["gate"] if cache["act"] == "relu" else da
    dy, G[cache["bnn"] + ".g"], G[cache["bnn"] + ".beta"] = Lr.bn_bwd(dz, cache["bn"], P[cache["bnn"] + ".g"])
    dr, G[cache["conv"] + ".W"], G[cache["conv"] + ".b"] = _lin_bwd(dy, cache["r"], cache["W"], need_dx)
    return dr


def _max_pool(name, x, scale=None):
    """Max over the L points of x [N, L, C] with the site's argmax (reading R15)."""
    idx = D.max_index(name, x, scale)
    return np.take_along_axis(x, idx[:, None, :], axis=1)[:, 0, :], idx


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

def _stn_fwd(P, S, newS, x, pre="stn"):
    """STN3d (pre "stn", x = points [N, L, 3]) or STNkd (pre "fstn", x = the
    64-d point features [N, L, k]): conv k->64->128->1024 (BN, ReLU), max over
    points, fc 1024->512->256 (BN, ReLU), fc 256->k*k, + I_k (reading R1)."""
    N, L, k = x.shape
    r = x.reshape(N * L, k)
    a1, k1 = _conv_bn_act(P, S, newS, r, pre + ".c1", pre + ".bn1", "relu")
    a2, k2 = _conv_bn_act(P, S, newS, a1, pre + ".c2", pre + ".bn2", "relu")
    a3, k3 = _conv_bn_act(P, S, newS, a2, pre + ".c3", pre + ".bn3", "relu")
    g, idx = _max_pool(pre + ".max", a3.reshape(N, L, -1), k3["esc"])
    f1, k4 = _conv_bn_act(P, S, newS, g, pre + ".fc1", pre + ".bn4", "relu")
    f2, k5 = _conv_bn_act(P, S, newS, f1, pre + ".fc2", pre + ".bn5", "relu")
    f3, f2s, W3s = _lin(P, f2, pre + ".fc3")
    T = f3.reshape(N, k, k) + np.eye(k)
    return T, dict(k=(k1, k2, k3, k4, k5), idx=idx, f2=f2s, W3=W3s, L=L, pre=pre)


def _stn_bwd(P, G, dT, c, need_dx=False):
    N, k, _ = dT.shape
    pre = c["pre"]
    df2, G[pre + ".fc3.W"], G[pre + ".fc3.b"] = _lin_bwd(dT.reshape(N, k * k), c["f2"], c["W3"])
    k1, k2, k3, k4, k5 = c["k"]
    df1 = _conv_bn_act_bwd(P, G, df2, k5)
    dg = _conv_bn_act_bwd(P, G, df1, k4)
    da3 = Lr.max_over_points_bwd(dg, c["idx"], c["L"]).reshape(-1, dg.shape[1])
    da2 = _conv_bn_act_bwd(P, G, da3, k3)
    da1 = _conv_bn_act_bwd(P, G, da2, k2)
    return _conv_bn_act_bwd(P, G, da1, k1, need_dx=need_dx)   # STN3d: input points, no dgrad


FT_REG_WEIGHT = 0.001      # feature-transform regularizer weight of the cited training script (reading R30)


def feature_transform_reg(T):
    """Regularizer of the 64 x 64 feature transform (reading R30):
    l = mean_n ||T_n T_n^T - I||_F, and dl/dT_n = 2 A_n T_n / (N ||A_n||_F),
    A_n = T_n T_n^T - I (symmetric)."""
    N, k, _ = T.shape
    A = np.matmul(T, T.transpose(0, 2, 1)) - np.eye(k)
    f = np.sqrt(np.sum(A * A, axis=(1, 2)))
    dT = 2.0 * np.matmul(A, T) / (N * np.maximum(f, 1e-300))[:, None, None]
    return f.mean(), dT


def _feat_fwd(P, S, newS, x, ft=False):
    N, L, _ = x.shape
    T, stn_c = _stn_fwd(P, S, newS, x)
    xt = Lr.transform_points(x, T)
    r = xt.reshape(N * L, 3)
    a1, k1 = _conv_bn_act(P, S, newS, r, "feat.c1", "feat.bn1", "relu")
    fc = dict(T=T, stn=stn_c, x=x, L=L, ft=ft)
    if ft:     # feature transform: x' = a1 T2 per cloud, T2 from STNkd(a1) (reading R30)
        T2, fstn_c = _stn_fwd(P, S, newS, a1.reshape(N, L, -1), "fstn")
        a1t = Lr.transform_points(a1.reshape(N, L, -1), T2).reshape(N * L, -1)
        fc.update(T2=T2, fstn=fstn_c, a1=a1)
        a1 = a1t
    a2, k2 = _conv_bn_act(P, S, newS, a1, "feat.c2", "feat.bn2", "relu")
    z3, k3 = _conv_bn_act(P, S, newS, a2, "feat.c3", "feat.bn3", None)
    g, idx = _max_pool("feat.max", z3.reshape(N, L, -1), k3["esc"])
    fc.update(k=(k1, k2, k3), idx=idx)
    return g, a1, fc


def _feat_bwd(P, G, dg, da1_extra, c):
    k1, k2, k3 = c["k"]
    N, L = c["x"].shape[0], c["L"]
    dz3 = Lr.max_over_points_bwd(dg, c["idx"], c["L"]).reshape(-1, dg.shape[1])
    da2 = _conv_bn_act_bwd(P, G, dz3, k3)
    da1 = _conv_bn_act_bwd(P, G, da2, k2)
    if da1_extra is not None:
        da1 = da1 + da1_extra
    if c["ft"]:          # back through x' = a1 T2 and STNkd(a1); + the regularizer's dT2
        C1 = da1.shape[1]
        da1_, dT2 = Lr.transform_points_bwd(da1.reshape(N, L, C1), c["a1"].reshape(N, L, C1), c["T2"])
        dT2 = dT2 + FT_REG_WEIGHT * c["dT2_reg"]
        da1 = da1_.reshape(N * L, C1) + _stn_bwd(P, G, dT2, c["fstn"], need_dx=True)
    dr = _conv_bn_act_bwd(P, G, da1, k1)
    _, dT = Lr.transform_points_bwd(dr.reshape(N, L, 3), c["x"], c["T"])
    _stn_bwd(P, G, dT, c["stn"])


def _ft_loss(fc):
    """Adds the feature-transform regularizer term to the loss (and keeps its
    gradient for the backward)."""
    if not fc["ft"]:
        return 0.0
    reg, fc["dT2_reg"] = feature_transform_reg(fc["T2"])
    return FT_REG_WEIGHT * reg


def pointnet_cls_loss_grads(P, S, x, labels, keep, p_drop, ft=False):
    """Forward + backward of PointNetCls for ONE model; keep = dropout keep mask
    [N, f2]; ft: feature transform on (loss += 0.001 * regularizer)."""
    newS = {}
    g, _, fc = _feat_fwd(P, S, newS, x, ft)
    h1, k1 = _conv_bn_act(P, S, newS, g, "head.fc1", "head.bn1", "relu")
    y2, h1s, W2s = _lin(P, h1, "head.fc2")
    d2 = Lr.dropout(y2, keep, p_drop)
    z2, bn2 = Lr.bn_fwd(d2, P["head.bn2.g"], P["head.bn2.beta"])
    rm, rv = _bn_state(S, "head.bn2", d2.shape[1])
    newS["head.bn2.rm"], newS["head.bn2.rv"] = Lr.bn_running(rm, rv, bn2, d2.shape[0])
    gate2 = D.relu_gate("head.bn2", z2, _bn_err_scale(d2, bn2, P["head.bn2.g"]))
    h2 = z2 * gate2
    logits, h2s, W3s = _lin(P, h2, "head.fc3")
    loss, dlogits = Lr.nll_mean(logits, labels)
    loss = loss + _ft_loss(fc)
    G = {}
    dh2, G["head.fc3.W"], G["head.fc3.b"] = _lin_bwd(dlogits, h2s, W3s)
    dz2 = dh2 * gate2
    dd2, G["head.bn2.g"], G["head.bn2.beta"] = Lr.bn_bwd(dz2, bn2, P["head.bn2.g"])
    dy2 = Lr.dropout_bwd(dd2, keep, p_drop)
    dh1, G["head.fc2.W"], G["head.fc2.b"] = _lin_bwd(dy2, h1s, W2s)
    dg = _conv_bn_act_bwd(P, G, dh1, k1)
    _feat_bwd(P, G, dg, None, fc)
    return loss, G, newS, dict(logits=logits, T=fc["T"], g=g)


def pointnet_seg_loss_grads(P, S, x, labels, ft=False):
    """Forward + backward of PointNetDenseCls for ONE model; labels [N, L]."""
    newS = {}
    N, L, _ = x.shape
    g, pointfeat, fc = _feat_fwd(P, S, newS, x, ft)
    C3 = g.shape[1]
    h0 = np.concatenate([np.repeat(g, L, axis=0), pointfeat], axis=1)   # [N*L, C3+C1]
    h1, k1 = _conv_bn_act(P, S, newS, h0, "head.c1", "head.bn1", "relu")
    h2, k2 = _conv_bn_act(P, S, newS, h1, "head.c2", "head.bn2", "relu")
    h3, k3 = _conv_bn_act(P, S, newS, h2, "head.c3", "head.bn3", "relu")
    logits, h3s, W4s = _lin(P, h3, "head.c4")
    loss, dlogits = Lr.nll_mean(logits, labels.reshape(-1))
    loss = loss + _ft_loss(fc)
    G = {}
    dh3, G["head.c4.W"], G["head.c4.b"] = _lin_bwd(dlogits, h3s, W4s)
    dh2 = _conv_bn_act_bwd(P, G, dh3, k3)
    dh1 = _conv_bn_act_bwd(P, G, dh2, k2)
    dh0 = _conv_bn_act_bwd(P, G, dh1, k1)
    dg = dh0[:, :C3].reshape(N, L, C3).sum(axis=1)
    _feat_bwd(P, G, dg, dh0[:, C3:], fc)
    return loss, G, newS, dict(logits=logits, T=fc["T"], g=g)


# -------------------------------------------------------------- DCGAN ----

G_LAYERS = [(1, 0), (2, 1), (2, 1), (2, 1), (2, 1)]     # (stride, pad) of t1..t5
D_LAYERS = [(2, 1), (2, 1), (2, 1), (2, 1), (1, 0)]     # c1..c5


def _conv(P, h, name, s, p, transposed=False):
    hs, Ws = D.store(h, "act", name), D.store(P[name], "w", name)
    f = Lr.convT2d_fwd if transposed else Lr.conv2d_fwd
    k = Ws.shape[0] * Ws.shape[2] * Ws.shape[3] if transposed else Ws.shape[1] * Ws.shape[2] * Ws.shape[3]
    return D.store(f(hs, Ws, s, p), "out", name, k), hs, Ws


def gen_fwd(P, S, newS, z, tag="G"):
    h = z.reshape(z.shape[0], -1, 1, 1)
    cache = []
    for i, (s, p) in enumerate(G_LAYERS):
        y, hs, Ws = _conv(P, h, "t%d.W" % (i + 1), s, p, transposed=True)
        if i < 4:
            bn = "bn%d" % (i + 1)
            zz, c = Lr.bn2d_fwd(y, P[bn + ".g"], P[bn + ".beta"])
            rm, rv = _bn_state(S, bn, y.shape[1])
            newS[bn + ".rm"], newS[bn + ".rv"] = Lr.bn_running(rm, rv, c, y.size // y.shape[1])
            gate = D.relu_gate("%s.%s" % (tag, bn), zz, _bn_err_scale(y, c, P[bn + ".g"]))
            cache.append((hs, Ws, gate, c))
            h = zz * gate
        else:
            cache.append((hs, Ws, None, None))
            h = Lr.tanh(y)
    return h, cache


def gen_bwd(P, dimg, img, cache):
    G = {}
    dy = Lr.tanh_bwd(dimg, img)
    for i in range(4, -1, -1):
        s, p = G_LAYERS[i]
        hs, Ws, gate, c = cache[i]
        if i < 4:
            bn = "bn%d" % (i + 1)
            dy, G[bn + ".g"], G[bn + ".beta"] = Lr.bn2d_bwd(dy * gate, c, P[bn + ".g"])
        dh, G["t%d.W" % (i + 1)] = Lr.convT2d_bwd(D.store(dy, "grad"), hs, Ws, s, p, need_dx=i > 0)
        dy = dh
    return G


def _leaky(zz, gate, a=0.2):
    return np.where(gate, zz, a * zz)


def disc_fwd(P, S, newS, img, tag="D"):
    """D forward; returns (sigmoid output [N], logit [N], cache)."""
    h = img
    cache = []
    for i, (s, p) in enumerate(D_LAYERS):
        y, hs, Ws = _conv(P, h, "c%d.W" % (i + 1), s, p)
        if i == 0:
            gate = D.relu_gate("%s.c1" % tag, y)
            cache.append((hs, Ws, gate, None))
            h = _leaky(y, gate)
        elif i < 4:
            bn = "bn%d" % (i + 1)
            zz, c = Lr.bn2d_fwd(y, P[bn + ".g"], P[bn + ".beta"])
            rm, rv = _bn_state(S, bn, y.shape[1])
            newS[bn + ".rm"], newS[bn + ".rv"] = Lr.bn_running(rm, rv, c, y.size // y.shape[1])
            gate = D.relu_gate("%s.%s" % (tag, bn), zz, _bn_err_scale(y, c, P[bn + ".g"]))
            cache.append((hs, Ws, gate, c))
            h = _leaky(zz, gate)
        else:
            cache.append((hs, Ws, None, None))
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
        hs, Ws, gate, c = cache[i]
        if i == 0:
            dy = _leaky(dy, gate)
        elif i < 4:
            bn = "bn%d" % (i + 1)
            dy, G[bn + ".g"], G[bn + ".beta"] = Lr.bn2d_bwd(_leaky(dy, gate), c, P[bn + ".g"])
        dh, dW = Lr.conv2d_bwd(D.store(dy, "grad"), hs, Ws, s, p, need_dx=(i > 0 or need_dx))
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
    out_r, zr, cr = disc_fwd(PD, SD, newSD1, real, tag="Dr")
    errD_real, dz = Lr.bce_sigmoid_mean(zr, ones)
    _, GD_r = disc_bwd(PD, dz, cr)
    fake, cg = gen_fwd(PG, SG, newSG, z, tag="G")
    out_f, zf, cf = disc_fwd(PD, newSD1, newSD2, fake, tag="Df")
    errD_fake, dz = Lr.bce_sigmoid_mean(zf, zeros)
    _, GD_f = disc_bwd(PD, dz, cf)
    GD = {k: GD_r[k] + GD_f[k] for k in GD_r}
    PD2, optD2 = adam_model(PD, GD, optD, t, hpD_b)
    out_g, zg, cg2 = disc_fwd(PD2, newSD2, newSD3, fake, tag="Dg")
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


def train_step(arch, P, S, opt, batch, t, hp_b, b=0, dropout_seed=42, p_drop=0.3, ft=False):
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
        loss, G, newS, out = pointnet_cls_loss_grads(P, S, x, labels, keep, p_drop, ft)
        out["keep"] = keep
    elif arch == "pointnet_seg":
        loss, G, newS, out = pointnet_seg_loss_grads(P, S, *batch, ft=ft)
    else:
        raise ValueError(arch)
    newP, newOpt = adam_model(P, G, opt, t, hp_b)
    return dict(loss=loss, grads=G, params=newP, opt=newOpt, stats=newS, out=out)


def fused_step_oracle(arch, Ps, Ss, opts, batch, t, hp, **kw):
    """The oracle of one fused step over B models: B independent serial steps
    (P:L923), plus the fused loss L = (1/B) sum_b l_b (App. C Eq. 1)."""
    res = [train_step(arch, Ps[b], Ss[b], opts[b], batch, t, hp_of(hp, b), b=b, **kw)
           for b in range(len(Ps))]
    losses = np.array([r["loss"] for r in res])
    return res, losses, losses.mean()
