"""Pins of the oracle's whole-model steps: central finite differences of the
full per-model loss (SURVEY §8(c) "whole step" (v)), PyTorch autograd fp64
replicas built from torch.nn.functional (library routines), and the
fused-step invariants (B=1 degeneracy, permutation equivariance, duplicate
models)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth
from oracle import models as M
from oracle.adam import adam_model

R = np.random.default_rng(7)
TINY = (4, 8, 16, 8, 8)


def fd_params(lossf, P, G, per_tensor=2, h=1e-6, rel=1e-4, floor=1e-7, skip=()):
    for name, p in P.items():
        if name not in G or any(s in name for s in skip):
            continue
        flat = p.reshape(-1)
        for i in R.choice(flat.size, size=min(per_tensor, flat.size), replace=False):
            old = flat[i]
            flat[i] = old + h
            fp = lossf()
            flat[i] = old - h
            fm = lossf()
            flat[i] = old
            num = (fp - fm) / (2 * h)
            ana = G[name].reshape(-1)[i]
            assert abs(num - ana) <= max(rel * abs(num), floor), (name, i, num, ana)


def test_cfg1_fd():
    P = synth.init_params("mlp_cfg1", 1000)
    x, T = synth.mlp_cfg1_batch(0)
    loss, G, _, _ = M.mlp_cfg1_loss_grads(P, {}, x, T)
    fd_params(lambda: M.mlp_cfg1_loss_grads(P, {}, x, T)[0], P, G, per_tensor=4)


def test_pointnet_cls_fd_tiny():
    P = synth.init_params("pointnet_cls", 1000, k=5, widths=TINY)
    x, y = synth.points_cls(0, N=3, L=16, k=5)
    keep = R.uniform(size=(3, 8)) > 0.3
    lf = lambda: M.pointnet_cls_loss_grads(P, {}, x, y, keep, 0.3)[0]
    loss, G, _, _ = M.pointnet_cls_loss_grads(P, {}, x, y, keep, 0.3)
    assert set(G) == set(P)
    fd_params(lf, P, G)


def test_pointnet_seg_fd_tiny():
    P = synth.init_params("pointnet_seg", 1000, k=6, widths=TINY)
    x, y = synth.points_seg(0, N=2, L=16, k=6)
    lf = lambda: M.pointnet_seg_loss_grads(P, {}, x, y)[0]
    loss, G, _, _ = M.pointnet_seg_loss_grads(P, {}, x, y)
    assert set(G) == set(P)
    fd_params(lf, P, G)


# ------------------------------------------------- torch autograd replicas ----

def _tbn(x, P, n, stats, key):
    rm, rv = torch.zeros(x.shape[1], dtype=torch.float64), torch.ones(x.shape[1], dtype=torch.float64)
    y = F.batch_norm(x, rm, rv, P[n + ".g"], P[n + ".beta"], training=True, momentum=0.1, eps=1e-5)
    stats[key] = (rm, rv)
    return y


def torch_pointnet_cls(Pn, x, y, keep, p):
    """PointNetCls written with torch.nn.functional in the [N, C, L] layout of
    the cited implementation (Conv1d k=1), autograd for the backward."""
    P = {k: torch.tensor(v, requires_grad=True) for k, v in Pn.items()}
    st = {}
    xt = torch.tensor(x).transpose(1, 2)                    # [N, 3, L]
    conv = lambda h, n: F.conv1d(h, P[n + ".W"][:, :, None], P[n + ".b"])
    h = F.relu(_tbn(conv(xt, "stn.c1"), P, "stn.bn1", st, 1))
    h = F.relu(_tbn(conv(h, "stn.c2"), P, "stn.bn2", st, 2))
    h = F.relu(_tbn(conv(h, "stn.c3"), P, "stn.bn3", st, 3))
    h = torch.max(h, 2)[0]
    h = F.relu(_tbn(F.linear(h, P["stn.fc1.W"], P["stn.fc1.b"]), P, "stn.bn4", st, 4))
    h = F.relu(_tbn(F.linear(h, P["stn.fc2.W"], P["stn.fc2.b"]), P, "stn.bn5", st, 5))
    T = F.linear(h, P["stn.fc3.W"], P["stn.fc3.b"]).view(-1, 3, 3) + torch.eye(3, dtype=torch.float64)
    h = torch.bmm(xt.transpose(2, 1), T).transpose(2, 1)
    h = F.relu(_tbn(conv(h, "feat.c1"), P, "feat.bn1", st, 6))
    h = F.relu(_tbn(conv(h, "feat.c2"), P, "feat.bn2", st, 7))
    h = _tbn(conv(h, "feat.c3"), P, "feat.bn3", st, 8)
    g = torch.max(h, 2)[0]
    h = F.relu(_tbn(F.linear(g, P["head.fc1.W"], P["head.fc1.b"]), P, "head.bn1", st, 9))
    h = F.linear(h, P["head.fc2.W"], P["head.fc2.b"]) * torch.tensor(keep.astype(float)) / (1 - p)
    h = F.relu(_tbn(h, P, "head.bn2", st, 10))
    logits = F.linear(h, P["head.fc3.W"], P["head.fc3.b"])
    loss = F.nll_loss(F.log_softmax(logits, dim=1), torch.tensor(y))
    loss.backward()
    return loss.item(), {k: v.grad.numpy() for k, v in P.items()}


def test_pointnet_cls_vs_torch_autograd():
    P = synth.init_params("pointnet_cls", 1001, k=7, widths=(8, 16, 32, 16, 16))
    x, y = synth.points_cls(3, N=4, L=40, k=7)
    keep = R.uniform(size=(4, 16)) > 0.3
    loss, G, _, _ = M.pointnet_cls_loss_grads(P, {}, x, y, keep, 0.3)
    tl, tG = torch_pointnet_cls(P, x, y, keep, 0.3)
    assert loss == pytest.approx(tl, rel=1e-12)
    for k in P:
        num = np.linalg.norm(G[k] - tG[k])
        assert num <= 1e-9 * max(np.linalg.norm(tG[k]), 1e-12) + 1e-13, k


def _torch_G(P, z):
    h = z.view(z.shape[0], -1, 1, 1)
    for i, (s, p) in enumerate(M.G_LAYERS):
        h = F.conv_transpose2d(h, P["t%d.W" % (i + 1)], stride=s, padding=p)
        if i < 4:
            h = F.relu(F.batch_norm(h, None, None, P["bn%d.g" % (i + 1)], P["bn%d.beta" % (i + 1)],
                                    training=True, eps=1e-5))
    return torch.tanh(h)


def _torch_D(P, img):
    h = img
    for i, (s, p) in enumerate(M.D_LAYERS):
        h = F.conv2d(h, P["c%d.W" % (i + 1)], stride=s, padding=p)
        if 1 <= i <= 3:
            h = F.batch_norm(h, None, None, P["bn%d.g" % (i + 1)], P["bn%d.beta" % (i + 1)],
                             training=True, eps=1e-5)
        h = F.leaky_relu(h, 0.2) if i < 4 else torch.sigmoid(h)
    return h.view(-1)


def test_dcgan_iteration_vs_torch():
    """One DCGAN iteration (example order, reading R4) vs torch autograd +
    torch.optim.Adam, N=4 so it runs in seconds."""
    N, t = 4, 1
    PG, PD = synth.init_params("dcgan_g", 1000), synth.init_params("dcgan_d", 1000)
    real = synth.images(0, N=N)
    z = synth.noise(0, 0, 1, N=N)
    hp = dict(lr=2e-4, beta1=0.5, beta2=0.999, eps=1e-8, wd=0.0)
    res = M.dcgan_iteration(PG, PD, {}, {}, {}, {}, real, z, t, hp)
    tG = {k: torch.nn.Parameter(torch.tensor(v)) for k, v in PG.items()}
    tD = {k: torch.nn.Parameter(torch.tensor(v)) for k, v in PD.items()}
    oG = torch.optim.Adam(tG.values(), lr=2e-4, betas=(0.5, 0.999))
    oD = torch.optim.Adam(tD.values(), lr=2e-4, betas=(0.5, 0.999))
    ones, zeros = torch.ones(N, dtype=torch.float64), torch.zeros(N, dtype=torch.float64)
    errDr = F.binary_cross_entropy(_torch_D(tD, torch.tensor(real)), ones)
    errDr.backward()
    fake = _torch_G(tG, torch.tensor(z))
    errDf = F.binary_cross_entropy(_torch_D(tD, fake.detach()), zeros)
    errDf.backward()
    gD = {k: v.grad.numpy().copy() for k, v in tD.items()}
    oD.step()
    for v in tG.values():
        v.grad = None
    errG = F.binary_cross_entropy(_torch_D(tD, fake), ones)
    errG.backward()
    gG = {k: v.grad.numpy().copy() for k, v in tG.items()}
    oG.step()
    assert res["errD_real"] == pytest.approx(errDr.item(), rel=1e-11)
    assert res["errD_fake"] == pytest.approx(errDf.item(), rel=1e-11)
    assert res["errG"] == pytest.approx(errG.item(), rel=1e-11)
    for k in gD:
        assert np.linalg.norm(res["GD"][k] - gD[k]) <= 1e-8 * np.linalg.norm(gD[k]) + 1e-14, k
    for k in gG:
        assert np.linalg.norm(res["GG"][k] - gG[k]) <= 1e-8 * np.linalg.norm(gG[k]) + 1e-14, k
    for k in tD:
        assert np.allclose(res["PD"][k], tD[k].detach().numpy(), rtol=1e-9, atol=1e-12), k
    for k in tG:
        assert np.allclose(res["PG"][k], tG[k].detach().numpy(), rtol=1e-9, atol=1e-12), k


# ------------------------------------------------------ fused invariants ----

def _cfg1_models(B, seeds):
    return ([synth.init_params("mlp_cfg1", s) for s in seeds], [{} for _ in range(B)],
            [{} for _ in range(B)])


def test_fused_oracle_permutation_and_duplicates():
    """Permuting per-model hyper-vectors and initial parameters permutes every
    per-model output; identical models give identical slices."""
    hp = synth.hparams_pointnet(7, 3)
    batch = synth.mlp_cfg1_batch(0)
    Ps, Ss, Os = _cfg1_models(3, [1000, 1001, 1002])
    res, losses, Lf = M.fused_step_oracle("mlp_cfg1", Ps, Ss, Os, batch, 1, hp)
    assert Lf == pytest.approx(losses.mean())
    perm = [2, 0, 1]
    hp2 = {k: v[perm] for k, v in hp.items()}
    res2, losses2, _ = M.fused_step_oracle("mlp_cfg1", [Ps[i] for i in perm], Ss, Os, batch, 1, hp2)
    assert np.array_equal(losses2, losses[perm])
    for j, i in enumerate(perm):
        for k in res[i]["params"]:
            assert np.array_equal(res2[j]["params"][k], res[i]["params"][k])
    hpd = {k: np.array([v[0], v[0]]) for k, v in hp.items()}
    resd, ld, _ = M.fused_step_oracle("mlp_cfg1", [Ps[0], Ps[0]], Ss[:2], Os[:2], batch, 1, hpd)
    assert ld[0] == ld[1]


def test_loss_scaling_eq3_fused_autograd():
    """App. C Eq. 1-3 (sum over b = 0..B-1, reading R8): the
    fused loss L = (1/B) sum_b l_b, scaled by B, has per-model gradients equal
    to each model's serial gradient.  An independent fused formulation (torch
    fp64 autograd over all B cfg1 models at once, one graph) is compared with
    the oracle, which trains every model ALONE: gradients of B*L equal the
    oracle's per-model gradients, and gradients of L are 1/B of them."""
    B = 3
    Ps = [synth.init_params("mlp_cfg1", 1000 + b) for b in range(B)]
    x, T = synth.mlp_cfg1_batch(0)
    tp = [{k: torch.tensor(v, requires_grad=True) for k, v in P.items()} for P in Ps]
    xt, Tt = torch.tensor(x), torch.tensor(T)

    def model_loss(P):
        h = F.linear(xt, P["c1.W"], P["c1.b"])
        h = F.relu(F.batch_norm(h, None, None, P["bn1.g"], P["bn1.beta"], training=True, eps=1e-5))
        h = F.linear(h, P["c2.W"], P["c2.b"])
        h = F.relu(F.batch_norm(h, None, None, P["bn2.g"], P["bn2.beta"], training=True, eps=1e-5))
        return F.mse_loss(h, Tt)

    losses = torch.stack([model_loss(P) for P in tp])
    Lf = losses.mean()                                  # Eq. 1
    (B * Lf).backward()                                 # Eq. 3's scaling
    for b in range(B):
        loss, G, _, _ = M.mlp_cfg1_loss_grads(Ps[b], {}, x, T)
        assert losses[b].item() == pytest.approx(loss, rel=1e-12)
        for k in G:
            assert np.allclose(tp[b][k].grad.numpy(), G[k], rtol=1e-9, atol=1e-14), (b, k)
    for P in tp:
        for v in P.values():
            v.grad = None
    Lf2 = torch.stack([model_loss(P) for P in tp]).mean()
    Lf2.backward()                                      # unscaled: 1/B of the serial gradient (Eq. 2)
    loss, G, _, _ = M.mlp_cfg1_loss_grads(Ps[0], {}, x, T)
    for k in G:
        assert np.allclose(B * tp[0][k].grad.numpy(), G[k], rtol=1e-9, atol=1e-14), k


# ----------------------------------------------------- decision sites ----

def _cls_tiny(margin, override=None, force=False):
    from oracle import decisions as Dm
    P = synth.init_params("pointnet_cls", 1000, k=5, widths=TINY)
    x, y = synth.points_cls(0, N=3, L=16, k=5)
    keep = np.random.default_rng(3).uniform(size=(3, 8)) > 0.3
    d = Dm.Decisions(margin, override, force)
    with Dm.use(d):
        loss, G, _, _ = M.pointnet_cls_loss_grads(P, {}, x, y, keep, 0.3)
    return loss, G, d


def test_decisions_default_is_plain_definition():
    """An active context without overrides changes nothing (bitwise), and it
    records every ReLU and max-pool site with its own decision."""
    P = synth.init_params("pointnet_cls", 1000, k=5, widths=TINY)
    x, y = synth.points_cls(0, N=3, L=16, k=5)
    keep = np.random.default_rng(3).uniform(size=(3, 8)) > 0.3
    l0, G0, _, _ = M.pointnet_cls_loss_grads(P, {}, x, y, keep, 0.3)
    l1, G1, d = _cls_tiny(0.5)
    assert l0 == l1 and all(np.array_equal(G0[k], G1[k]) for k in G0)
    assert set(d.sites) == {"stn.bn1", "stn.bn2", "stn.bn3", "stn.max", "stn.bn4", "stn.bn5", "feat.bn1",
                            "feat.bn2", "feat.max", "head.bn1", "head.bn2"}
    for k, v in d.sites.items():
        assert v["flips"] == 0 and np.array_equal(v["own"], v["used"])


def test_decisions_override_inside_band_only():
    """A flip inside the flagged band is taken (and moves the gradient, as a
    different valid subgradient); a flip outside it, or an argmax override
    whose value is not within the margin of the top, raises DecisionError."""
    from oracle import decisions as Dm
    _, G0, d = _cls_tiny(0.2)
    site = d.sites["feat.bn2"]
    flagged = np.argwhere(site["flag"] & site["own"])
    unflagged = np.argwhere(~site["flag"] & site["own"])
    assert len(flagged) and len(unflagged)
    ov = site["own"].copy()
    ov[tuple(flagged[0])] = False
    _, G1, d1 = _cls_tiny(0.2, {"feat.bn2": ov})
    assert d1.sites["feat.bn2"]["flips"] == 1
    assert not np.array_equal(G1["feat.c2.W"], G0["feat.c2.W"])
    ov = site["own"].copy()
    ov[tuple(unflagged[0])] = False
    with pytest.raises(Dm.DecisionError):
        _cls_tiny(0.2, {"feat.bn2": ov})
    _, _, dd = _cls_tiny(0.2, {"feat.bn2": ov}, force=True)       # witness mode: no validation
    assert dd.sites["feat.bn2"]["flips"] == 1
    # argmax: any index holding a value within the margin of the top is valid
    m = d.sites["feat.max"]
    own = m["own"]
    ov = (own + 1) % 16
    with pytest.raises(Dm.DecisionError):
        _cls_tiny(0.2, {"feat.max": ov})
    _, _, d2 = _cls_tiny(1e6, {"feat.max": ov})                   # huge margin: everything is a tie
    assert d2.sites["feat.max"]["flips"] == own.size


def test_decisions_max_ties_flagged_exactly():
    """Brute force on a tiny tensor: the max site flags exactly the (cloud,
    channel) pairs whose top-2 gap is within margin * rms, and exact ties
    (e.g. an all-zero ReLU output) are always flagged."""
    from oracle import decisions as Dm
    x = np.array([[[1.0, 0.0], [0.9, 0.0], [0.2, 0.0]],
                  [[0.0, 3.0], [0.5, 1.0], [0.49, 2.9]]])       # [N=2, L=3, C=2]
    d = Dm.Decisions(0.05)
    with Dm.use(d):
        idx = Dm.max_index("m", x)
    rms = np.sqrt(np.mean(x * x, axis=(0, 1)))
    want = np.zeros((2, 2), bool)
    for n in range(2):
        for c in range(2):
            v = np.sort(x[n, :, c])
            want[n, c] = v[-1] - v[-2] <= 0.05 * rms[c]
    assert np.array_equal(d.sites["m"]["flag"], want)
    assert want[0, 1] and idx[0, 1] == 0                          # all-zero channel: tie, first index
    assert np.array_equal(idx, np.argmax(x, axis=1))


# --------------------------------------------------- feature transform ----

def test_feature_transform_reg_closed_forms():
    """Reading R30: ||T T^T - I||_F is 0 for orthogonal T (rotations), and for
    T = c I it is |c^2 - 1| sqrt(k) with gradient 2 c sign(c^2 - 1) I / (N sqrt(k))."""
    k, N = 5, 3
    Q, _ = np.linalg.qr(R.standard_normal((k, k)))
    l, dT = M.feature_transform_reg(np.stack([Q] * N))
    assert l < 1e-12
    for c in (0.5, 1.7):
        l, dT = M.feature_transform_reg(np.stack([c * np.eye(k)] * N))
        assert l == pytest.approx(abs(c * c - 1) * np.sqrt(k), rel=1e-12)
        assert np.allclose(dT, 2 * c * np.sign(c * c - 1) / (N * np.sqrt(k)) * np.eye(k)[None], rtol=1e-12)


def test_pointnet_cls_feature_transform_fd_tiny():
    P = synth.init_params("pointnet_cls", 1000, k=5, widths=TINY, ft=True)
    assert "fstn.fc3.W" in P and P["fstn.fc3.W"].shape == (TINY[0] ** 2, TINY[4])
    x, y = synth.points_cls(0, N=3, L=16, k=5)
    keep = R.uniform(size=(3, 8)) > 0.3
    lf = lambda: M.pointnet_cls_loss_grads(P, {}, x, y, keep, 0.3, ft=True)[0]
    loss, G, _, _ = M.pointnet_cls_loss_grads(P, {}, x, y, keep, 0.3, ft=True)
    assert set(G) == set(P)
    fd_params(lf, P, G)


def test_pointnet_seg_feature_transform_fd_tiny():
    P = synth.init_params("pointnet_seg", 1000, k=6, widths=TINY, ft=True)
    x, y = synth.points_seg(0, N=2, L=16, k=6)
    lf = lambda: M.pointnet_seg_loss_grads(P, {}, x, y, ft=True)[0]
    loss, G, _, _ = M.pointnet_seg_loss_grads(P, {}, x, y, ft=True)
    assert set(G) == set(P)
    fd_params(lf, P, G)


def test_pointnet_cls_feature_transform_vs_torch_autograd():
    """PointNetCls(feature_transform=True) of the cited implementation in
    torch.nn.functional (STNkd, bmm, feature_transform_regularizer * 0.001),
    fp64 autograd, vs the oracle's hand-written backward."""
    W = (8, 16, 32, 16, 16)
    Pn = synth.init_params("pointnet_cls", 1003, k=7, widths=W, ft=True)
    x, y = synth.points_cls(2, N=4, L=20, k=7)
    keep = R.uniform(size=(4, W[4])) > 0.3
    P = {k: torch.tensor(v, requires_grad=True) for k, v in Pn.items()}
    st = {}
    conv = lambda h, n: F.conv1d(h, P[n + ".W"][:, :, None], P[n + ".b"])

    def stn(h, pre, k):
        h = F.relu(_tbn(conv(h, pre + ".c1"), P, pre + ".bn1", st, pre + "1"))
        h = F.relu(_tbn(conv(h, pre + ".c2"), P, pre + ".bn2", st, pre + "2"))
        h = F.relu(_tbn(conv(h, pre + ".c3"), P, pre + ".bn3", st, pre + "3"))
        h = torch.max(h, 2)[0]
        h = F.relu(_tbn(F.linear(h, P[pre + ".fc1.W"], P[pre + ".fc1.b"]), P, pre + ".bn4", st, pre + "4"))
        h = F.relu(_tbn(F.linear(h, P[pre + ".fc2.W"], P[pre + ".fc2.b"]), P, pre + ".bn5", st, pre + "5"))
        return F.linear(h, P[pre + ".fc3.W"], P[pre + ".fc3.b"]).view(-1, k, k) + torch.eye(k, dtype=torch.float64)

    xt = torch.tensor(x).transpose(1, 2)
    T = stn(xt, "stn", 3)
    h = torch.bmm(xt.transpose(2, 1), T).transpose(2, 1)
    h = F.relu(_tbn(conv(h, "feat.c1"), P, "feat.bn1", st, "f1"))
    T2 = stn(h, "fstn", W[0])
    h = torch.bmm(h.transpose(2, 1), T2).transpose(2, 1)
    h = F.relu(_tbn(conv(h, "feat.c2"), P, "feat.bn2", st, "f2"))
    g = torch.max(_tbn(conv(h, "feat.c3"), P, "feat.bn3", st, "f3"), 2)[0]
    h = F.relu(_tbn(F.linear(g, P["head.fc1.W"], P["head.fc1.b"]), P, "head.bn1", st, "h1"))
    h = F.linear(h, P["head.fc2.W"], P["head.fc2.b"]) * torch.tensor(keep.astype(float)) / 0.7
    h = F.relu(_tbn(h, P, "head.bn2", st, "h2"))
    logits = F.linear(h, P["head.fc3.W"], P["head.fc3.b"])
    I = torch.eye(W[0], dtype=torch.float64)[None]
    reg = torch.mean(torch.norm(torch.bmm(T2, T2.transpose(2, 1)) - I, dim=(1, 2)))
    loss = F.nll_loss(F.log_softmax(logits, dim=1), torch.tensor(y)) + 0.001 * reg
    loss.backward()
    l0, G, _, _ = M.pointnet_cls_loss_grads(Pn, {}, x, y, keep, 0.3, ft=True)
    assert l0 == pytest.approx(loss.item(), rel=1e-12)
    for k in G:
        assert np.allclose(G[k], P[k].grad.numpy(), rtol=1e-8, atol=1e-12), k
