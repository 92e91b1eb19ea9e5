"""Whole-step parity: one fused PointNet training step of B models on the GPU
(through the C ABI) against the oracle that trains each model alone
(App. C Eq. 3).  Gradients are gated before the Adam step, updated
parameters / Adam moments normwise per model (readings R20, R21)."""
import numpy as np
import pytest
import torch

import synth
from oracle import models as OM
from tests._cmp import TOL, relerr

pytestmark = pytest.mark.gpu

# Biases of layers followed by BatchNorm have an analytically zero gradient
# (BN removes any per-channel shift); their computed values are rounding
# noise on both sides, so they are checked as ~0 instead of normwise.
BN_ABSORBED = ("stn.c1.b", "stn.c2.b", "stn.c3.b", "stn.fc1.b", "stn.fc2.b", "feat.c1.b", "feat.c2.b",
               "feat.c3.b", "head.fc1.b", "head.fc2.b", "head.c1.b", "head.c2.b", "head.c3.b")


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_2102_02344_b200.hfta as H
    H.hfta_init(0)


def run_pair(task, dtype, B, N, L, k, steps=1, widths=None, seed=0):
    from paper_2102_02344_b200.pointnet import FusedPointNet
    arch = "pointnet_" + task
    specs = [(n, s) for n, s, _ in synth.param_specs(arch, k, widths)]
    Ps = [synth.init_params(arch, 1000 + b, k, widths) for b in range(B)]
    hp = synth.hparams_pointnet(7, B)
    x, y = (synth.points_cls if task == "cls" else synth.points_seg)(seed, N=N, L=L, k=k)
    net = FusedPointNet(B, specs, Ps, hp, task=task, dtype=dtype, N=N, L=L, k=k)
    xd = torch.tensor(x.reshape(N * L, 3), dtype=torch.float32, device="cuda")
    yd = torch.tensor(y, dtype=torch.int32, device="cuda")
    S = [{} for _ in range(B)]
    O = [{} for _ in range(B)]
    P = list(Ps)
    out = []
    for t in range(1, steps + 1):
        loss = net.step(xd, yd).detach().cpu().numpy().copy()
        res, losses, _ = OM.fused_step_oracle(arch, P, S, O, (x, y), t, hp)
        out.append((loss, losses, [net.grads(b) for b in range(B)], res))
        P = [r["params"] for r in res]
        S = [r["stats"] for r in res]
        O = [r["opt"] for r in res]
    torch.cuda.synchronize()
    return net, out


def check_step(net, loss, ref_losses, grads, res, tol, B):
    for b in range(B):
        assert abs(loss[b] - ref_losses[b]) <= tol * abs(ref_losses[b]), (b, loss[b], ref_losses[b])
        G = grads[b]
        R = res[b]["grads"]
        for n in R:
            if n in BN_ABSORBED:
                wn = np.linalg.norm(R[n.replace(".b", ".W")])
                assert np.linalg.norm(G[n]) <= max(10 * tol, 1e-3) * wn + 1e-6, n
                continue
            e = relerr(G[n], R[n])
            assert e <= tol, "model %d grad %s: %.3e" % (b, n, e)
        # after the Adam step: whole-model normwise (reading R21)
        p = np.concatenate([net.params(b)[n].ravel() for n in R])
        pr = np.concatenate([res[b]["params"][n].ravel() for n in R])
        assert relerr(p, pr) <= tol, "model %d params after step: %.3e" % (b, relerr(p, pr))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_cls_step_small(dtype):
    B, N, L, k = 3, 4, 300, 40
    net, out = run_pair("cls", dtype, B, N, L, k)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, TOL[dtype], B)
    # BN running statistics of every layer
    for b in range(B):
        for name in net.bn_names:
            rm = net.running[name][0][b].cpu().numpy()
            assert relerr(rm, res[b]["stats"][name + ".rm"]) <= TOL[dtype], name


def test_pointnet_cls_two_steps_f32():
    B, N, L, k = 2, 4, 200, 10
    net, out = run_pair("cls", "f32", B, N, L, k, steps=2)
    for loss, ref, grads, res in out:
        for b in range(B):
            assert abs(loss[b] - ref[b]) <= 1e-4 * abs(ref[b])
    loss, ref, grads, res = out[-1]
    check_step(net, loss, ref, grads, res, TOL["f32"], B)


def test_pointnet_cls_duplicate_models_bitwise():
    """Identical hyper-parameters and initial parameters -> bitwise-identical
    slices (SURVEY §8(c) whole step (iv)); catches model-index bugs."""
    from paper_2102_02344_b200.pointnet import FusedPointNet
    B, N, L, k = 3, 4, 300, 40
    specs = [(n, s) for n, s, _ in synth.param_specs("pointnet_cls", k)]
    P0 = synth.init_params("pointnet_cls", 1000, k)
    hp1 = synth.hparams_pointnet(7, 1)
    hp = {kk: np.repeat(v, B) for kk, v in hp1.items()}
    net = FusedPointNet(B, specs, [P0] * B, hp, task="cls", dtype="f32", N=N, L=L, k=k, p_drop=0.0)
    x, y = synth.points_cls(0, N=N, L=L, k=k)
    net.step(torch.tensor(x.reshape(-1, 3), dtype=torch.float32, device="cuda"),
             torch.tensor(y, dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    g = net.arena.g.cpu().numpy()
    p = net.arena.p.cpu().numpy()
    for b in range(1, B):
        assert np.array_equal(g[b], g[0]) and np.array_equal(p[b], p[0])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_cls_step_full_size(dtype):
    """BJ configs[1] shapes (N=32, L=2500, k=40) with B=2; the oracle takes
    ~25 s per model."""
    B, N, L, k = 2, 32, 2500, 40
    net, out = run_pair("cls", dtype, B, N, L, k)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, TOL[dtype], B)
