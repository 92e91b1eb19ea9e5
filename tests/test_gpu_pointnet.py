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
from tests import _decide as DE

pytestmark = pytest.mark.gpu

# Several gradients are analytically ZERO: biases of layers followed by
# BatchNorm (BN removes any per-channel shift), and the BN shift of the layer
# whose max-pooled output feeds Linear -> BN (the shift moves every sample's
# pooled feature equally).  Their computed values are rounding noise on both
# sides (oracle ~1e-16, fp32 ~1e-9 relative), so a tensor whose oracle norm is
# below 1e-9 of the model's largest gradient norm is checked as ~0 instead of
# normwise.
ZERO_REL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_2102_02344_b200.hfta as H
    H.hfta_init(0)


def run_pair(task, dtype, B, N, L, k, steps=1, widths=None, seed=0, witness=None, ft=False):
    """GPU fused step(s) and, per model, the oracle re-run with the GPU's
    decisions inside the oracle's own flagged band (tests/_decide.py).  The
    bf16 witness (reading R28) is computed on the first step."""
    from paper_2102_02344_b200.pointnet import FusedPointNet
    arch = "pointnet_" + task
    witness = (dtype == "bf16") if witness is None else witness
    specs = [(n, s) for n, s, _ in synth.param_specs(arch, k, widths, ft)]
    Ps = [synth.init_params(arch, 1000 + b, k, widths, ft) for b in range(B)]
    hp = synth.hparams_pointnet(7, B)
    x, y = (synth.points_cls if task == "cls" else synth.points_seg)(seed, N=N, L=L, k=k)
    net = FusedPointNet(B, specs, Ps, hp, task=task, dtype=dtype, N=N, L=L, k=k, feature_transform=ft)
    xd = torch.tensor(x.reshape(N * L, 3), dtype=torch.float32, device="cuda")
    yd = torch.tensor(y, dtype=torch.int32, device="cuda")
    S = [{} for _ in range(B)]
    O = [{} for _ in range(B)]
    P = list(Ps)
    out = []
    for t in range(1, steps + 1):
        loss = net.step(xd, yd).detach().cpu().numpy().copy()
        torch.cuda.synchronize()
        res = []
        for b in range(B):
            gpu = DE.pointnet_gpu_decisions(net, b)
            r, report, rw = DE.oracle_with_decisions(arch, P[b], S[b], O[b], (x, y), t, OM.hp_of(hp, b), b, gpu,
                                                     dtype, L=L, ft=ft)
            if r is None and t > 1:
                # after a step the trajectories may differ by O(lr) where the step-1 update was
                # sign-decided (reading R21): later steps compare against the oracle's own decisions
                r = OM.train_step(arch, P[b], S[b], O[b], (x, y), t, OM.hp_of(hp, b), b=b, ft=ft)
            r = r if r is not None else {"loss": np.nan, "params": P[b], "stats": S[b], "opt": O[b], "grads": {}}
            r["p_before"] = P[b]
            r["report"] = report
            r["zerr"] = DE.decision_errors(report["_ctx"], DE.pointnet_gpu_values(net, b), report["_margins"])
            r["witness"] = rw
            report.pop("_ctx")                    # the per-site arrays (GBs at full size)
            # the GPU state after this step (later steps overwrite the net)
            r["gpu_after"] = dict(
                params=net.params(b),
                m={n: net.arena.host_tensor("m", n)[b] for n, _ in net.arena.specs},
                v={n: net.arena.host_tensor("v", n)[b] for n, _ in net.arena.specs},
                running={n: tuple(t_[b].cpu().numpy() for t_ in net.running[n]) for n in net.bn_names})
            res.append(r)
        out.append((loss, np.array([r["loss"] for r in res]), [net.grads(b) for b in range(B)], res))
        P = [r["params"] for r in res]
        S = [r["stats"] for r in res]
        O = [r["opt"] for r in res]
    return net, out


def check_step(net, loss, ref_losses, grads, res, dtype, B):
    """Every per-model quantity of the step vs the decision-matched oracle:
    loss; every gradient tensor and BN running statistic at max(north_star
    tolerance -- fp32 1e-4, bf16 2e-2 -- , 3 x the conditioning witness of that
    quantity at the path's precision, reading R28); BN running mean and
    variance of every layer; Adam m and v; the update on the elements whose
    sign the oracle alone decides (reading R21)."""
    tol = TOL[dtype]
    worst = []
    for b in range(B):
        rep = {k: v for k, v in res[b]["report"].items() if not k.startswith("_")}
        print("\n  model %d decisions (flagged/size, flips, unflagged disagreements, max dist/margin, margin): %s" % (
            b, " ".join("%s:%d/%d,%d,%d,%.2f,%.1e" % (k, v["flagged"], v["size"], v["flips"], v["unflagged_disagree"],
                                                      v["max_dist"], v["margin"]) for k, v in rep.items())))
        print("  model %d max z error / margin: %s" % (b, " ".join(
            "%s:%.2f" % (k, e) for k, e in res[b]["zerr"].items())))
    for b in range(B):
        r = res[b]
        bad = {k: v for k, v in r["report"].items() if not k.startswith("_") and v["unflagged_disagree"]}
        assert not bad, "model %d: GPU decisions differ from the oracle outside the flagged band: %s" % (b, bad)
        for site, e in r["zerr"].items():      # the margin covers the GPU's decision-variable error
            assert e <= 1.0, "model %d site %s: GPU z error is %.2f x the margin" % (b, site, e)
        assert abs(loss[b] - ref_losses[b]) <= tol * abs(ref_losses[b]), (b, loss[b], ref_losses[b])
        G, Rg = grads[b], r["grads"]
        gmax = max(np.linalg.norm(v) for v in Rg.values())
        gtol = {}
        for n in Rg:
            if np.linalg.norm(Rg[n]) < ZERO_REL * gmax:
                assert np.linalg.norm(G[n]) <= 1e-1 * tol * gmax, "model %d grad %s not ~0" % (b, n)
                continue
            gtol[n] = DE.gate(tol, r["witness"]["grads"][n], r["witness"]["own"]["grads"][n])
            e = relerr(G[n], Rg[n])
            worst.append((e / gtol[n], e, gtol[n], b, n))
            assert e <= gtol[n], "model %d grad %s: %.3e > %.3e" % (b, n, e, gtol[n])
        ga = r["gpu_after"]
        ws_, os_ = r["witness"]["stats"], r["witness"]["own"]["stats"]
        for name in net.bn_names:
            rm, rv = ga["running"][name]
            for key, got in ((".rm", rm), (".rv", rv)):
                g_ = DE.gate(tol, ws_[name + key], os_[name + key])
                assert relerr(got, r["stats"][name + key]) <= g_, (b, name, key, relerr(got, r["stats"][name + key]), g_)
        m_gpu, v_gpu = ga["m"], ga["v"]
        for n in gtol:
            m_ref, v_ref = r["opt"][n]
            assert relerr(m_gpu[n], m_ref) <= gtol[n] * 1.01 + 1e-6, (b, n, "exp_avg")
            assert relerr(v_gpu[n], v_ref) <= 2.0 * gtol[n] * 1.01 + 1e-6, (b, n, "exp_avg_sq")
        pb, p0 = ga["params"], r["p_before"]
        wd = float(net.hv.t["wd"][b].item())
        for n in gtol:
            g = Rg[n] + wd * p0[n]            # what Adam normalises (coupled L2 decay)
            rms = np.sqrt(np.mean(g * g))
            mask = np.abs(g) > (1e-1 if dtype == "f32" else 5e-1) * rms
            if not mask.any():
                continue
            e = relerr((pb[n] - p0[n])[mask], (r["params"][n] - p0[n])[mask])
            assert e <= gtol[n], "model %d update of %s: %.3e" % (b, n, e)
    worst.sort(reverse=True)
    print("\n[%s] worst gradient errors (err / gate): %s" % (dtype, " ".join(
        "%s:%.2e/%.1e" % (n, e, g) for _, e, g, b, n in worst[:6])))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_cls_step_small(dtype):
    B, N, L, k = 3, 32, 50, 40
    net, out = run_pair("cls", dtype, B, N, L, k)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, dtype, B)


def test_pointnet_cls_two_steps_f32():
    """Two steps: step 1 is gated as usual; after one Adam step the two
    trajectories may separate by O(lr) in elements whose step-1 gradient is
    below rounding noise (reading R21), so step 2 is gated on the loss only."""
    B, N, L, k = 2, 32, 50, 10
    net, out = run_pair("cls", "f32", B, N, L, k, steps=2)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, "f32", B)
    loss, ref, grads, res = out[1]
    for b in range(B):
        assert abs(loss[b] - ref[b]) <= 1e-3 * abs(ref[b])


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
    ~10-20 s per model and pass."""
    B, N, L, k = 2, 32, 2500, 40
    net, out = run_pair("cls", dtype, B, N, L, k)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, dtype, B)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_seg_step_small(dtype):
    """PointNet-seg (BJ configs[2] architecture, k = 50) with the split-weight
    concat layer, N=8 clouds x L=300 points, B=3."""
    B, N, L, k = 3, 8, 300, 50
    net, out = run_pair("seg", dtype, B, N, L, k)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, dtype, B)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_seg_step_full_size(dtype):
    """seg at BJ configs[2] shapes (N = 32, L = 2500, k = 50), B = 2."""
    B, N, L, k = 2, 32, 2500, 50
    net, out = run_pair("seg", dtype, B, N, L, k)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, dtype, B)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_cls_feature_transform_small(dtype):
    """Feature transform on (STNkd 64 x 64 + 0.001 regularizer, P:L981,
    reading R30): N = 8 clouds x L = 300 points, B = 3."""
    B, N, L, k = 3, 8, 300, 40
    net, out = run_pair("cls", dtype, B, N, L, k, ft=True)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, dtype, B)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_pointnet_cls_feature_transform_full_size(dtype):
    """Feature transform at BJ configs[1] shapes (N = 32, L = 2500), B = 2."""
    B, N, L, k = 2, 32, 2500, 40
    net, out = run_pair("cls", dtype, B, N, L, k, ft=True)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, dtype, B)


def test_pointnet_seg_feature_transform_small_f32():
    """seg with the feature transform (the head's point feature is x' = a1 T2)."""
    B, N, L, k = 2, 4, 500, 50
    net, out = run_pair("seg", "f32", B, N, L, k, ft=True)
    loss, ref, grads, res = out[0]
    check_step(net, loss, ref, grads, res, "f32", B)
