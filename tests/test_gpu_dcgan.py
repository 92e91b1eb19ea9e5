"""One fused DCGAN iteration (BJ configs[3] architecture: 64x64 G + D,
ConvT2d/Conv2d/BN2d, LeakyReLU/ReLU/Tanh/Sigmoid+BCE, per-model Adam on
both nets) through the C ABI vs the oracle that runs each model's iteration
alone in the order of the cited example (reading R4).  Small batch (N=4) so
the fp64 oracle finishes in seconds; the kernels are the full-size ones
(every layer of the 64x64 models)."""
import numpy as np
import pytest
import torch

import synth
from oracle import models as OM
from tests._cmp import TOL, relerr
from tests import _decide as DE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _init():
    import paper_2102_02344_b200.hfta as H
    H.hfta_init(0)


def _nchw(t):
    return t.detach().float().cpu().numpy().astype(np.float64).transpose(0, 3, 1, 2)


def run_dcgan(dtype, B=2, N=4, seed=0, d_lr_zero=False):
    """One fused DCGAN iteration on the GPU (with the D activations of each of
    its three D passes snapshotted for their ReLU / LeakyReLU decisions), then
    per model the oracle iteration with the GPU's decisions inside the
    oracle's flagged bands (tests/_decide.py)."""
    from paper_2102_02344_b200.dcgan import FusedDCGAN, NC
    gs = [(n, s) for n, s, _ in synth.param_specs("dcgan_g")]
    ds = [(n, s) for n, s, _ in synth.param_specs("dcgan_d")]
    PG = [synth.init_params("dcgan_g", 1000 + b) for b in range(B)]
    PD = [synth.init_params("dcgan_d", 2000 + b) for b in range(B)]
    hp = synth.hparams_dcgan(3, B)
    real = synth.images(seed, N=N)                            # NCHW
    zs = np.stack([synth.noise(seed, b, 1, N=N) for b in range(B)])
    net = FusedDCGAN(B, gs, ds, PG, PD, hp, N=N, dtype=dtype)
    hpD = dict(hp)
    if d_lr_zero:
        hpD["lr"] = np.zeros(B)
        net.hvD.set("lr", hpD["lr"])
    snaps = []
    orig_bce = net._bce

    def bce_snap(target, out_loss, s):       # D forward of this pass is done: keep its activations
        snaps.append([t.clone() for t in net.dh])
        orig_bce(target, out_loss, s)
    net._bce = bce_snap
    net.set_inputs(torch.tensor(real.transpose(0, 2, 3, 1), dtype=torch.float32, device="cuda"),
                   torch.tensor(zs, dtype=torch.float32, device="cuda"))
    errs = [e.cpu().numpy().copy() for e in net.step()]
    torch.cuda.synchronize()
    assert len(snaps) == 3
    res = []
    for b in range(B):
        gpu, vals = {}, {}
        for i in range(4):
            a = _nchw(net.gh[i][b])
            gpu["G.bn%d" % (i + 1)], vals["G.bn%d" % (i + 1)] = a > 0, a
        for tag, sn in zip(("Dr", "Df", "Dg"), snaps):
            for i in range(4):
                site = "%s.c1" % tag if i == 0 else "%s.bn%d" % (tag, i + 1)
                a = _nchw(sn[i][b])
                gpu[site], vals[site] = a > 0, a
        step = lambda: OM.dcgan_iteration(PG[b], PD[b], {}, {}, {}, {}, real, zs[b], 1, OM.hp_of(hp, b),
                                          OM.hp_of(hpD, b))
        # the GPU stores every conv output (pre-BN / pre-activation) in the compute dtype
        # Dg: the third D pass runs through D', whose t = 1 Adam update is
        # sign-decided where D's gradient is rounding noise (reading R21): with
        # D's lr > 0 its decision variables differ by more than rounding, so
        # it keeps the oracle's decisions (G's gradients, its only consumers,
        # are gated in the D-lr-0 test where D' = D exactly)
        skip = () if d_lr_zero else ("Dg.",)
        r, report, rw = DE.with_decisions(step, gpu, dtype, out_layers=("c", "t"), skip=skip)
        zerr = DE.decision_errors(report.pop("_ctx"), {k: v for k, v in vals.items() if not k.startswith(skip or "@")},
                                  report["_margins"])
        res.append(dict(ref=r, report=report, witness=rw, zerr=zerr))
    return net, errs, res, hp


def _gates(dtype, ref, wit, key):
    tol = TOL[dtype]
    g = {}
    for n, v in ref[key].items():
        g[n] = DE.gate(tol, wit[key][n], wit["own"][key][n])
    return g


def _check(dtype, net, errs, res, hp, B, gate_g):
    """Losses; every D gradient tensor (fp32 1e-4, bf16 max(2e-2, 3 x the
    bf16-storage witness), reading R28); G gradients the same when D's update
    is exact (gate_g: D lr 0 -- otherwise G's gradients flow through D' whose
    t = 1 Adam update is sign-decided where D's gradient is rounding noise,
    reading R21); BN running statistics of both nets; Adam moments."""
    tol = TOL[dtype]
    worst = []
    for b in range(B):
        rep = res[b]["report"]
        print("\n  model %d decisions (flagged/size, flips, max dist/margin, margin): %s" % (b, " ".join(
            "%s:%d/%d,%d,%.2f,%.1e" % (k, v["flagged"], v["size"], v["flips"], v["max_dist"], v["margin"])
            for k, v in rep.items() if not k.startswith("_"))))
        print("  model %d max z error / margin: %s" % (b, " ".join("%s:%.2f" % kv for kv in res[b]["zerr"].items())))
    for b in range(B):
        rep, ref, wit = res[b]["report"], res[b]["ref"], res[b]["witness"]
        bad = {k: v for k, v in rep.items() if not k.startswith("_") and v["unflagged_disagree"]}
        assert not bad, "model %d: GPU decisions differ from the oracle outside the flagged band: %s" % (b, bad)
        for site, e in res[b]["zerr"].items():
            assert e <= 1.0, "model %d site %s: GPU z error is %.2f x the margin" % (b, site, e)
        for i, k in enumerate(("errD_real", "errD_fake", "errG")):
            assert abs(errs[i][b] - ref[k]) <= tol * abs(ref[k]), (b, k, errs[i][b], ref[k])
        GD, GG = net.D.grads(b), net.G.grads(b)
        for half, G, key, gate in (("D", GD, "GD", True), ("G", GG, "GG", gate_g)):
            gt = _gates(dtype, ref, wit, key)
            for n, r_ in ref[key].items():
                e = relerr(G[n], r_)
                worst.append((e / gt[n], e, gt[n], b, half + "." + n, gate))
                if gate:
                    assert e <= gt[n], "model %d %s.%s: %.3e > %.3e" % (b, half, n, e, gt[n])
            if gate:
                arena = (net.D if half == "D" else net.G).arena
                from paper_2102_02344_b200.dcgan import _to_torch
                opt = ref["optD" if half == "D" else "optG"]
                for n in ref[key]:
                    m_ref, v_ref = opt[n]
                    m = _to_torch(n, arena.host_tensor("m", n)[b])
                    v = _to_torch(n, arena.host_tensor("v", n)[b])
                    assert relerr(m, m_ref) <= gt[n] * 1.01 + 1e-6, (b, half, n, "exp_avg")
                    assert relerr(v, v_ref) <= 2 * gt[n] * 1.01 + 1e-6, (b, half, n, "exp_avg_sq")
        for half, key in (("D", "SD"), ("G", "SG")):
            h = net.D if half == "D" else net.G
            st, ws_, os_ = ref[key], wit[key], wit["own"][key]
            for name in h.bn:
                rm, rv = (t[b].cpu().numpy() for t in h.running[name])
                for k2, got in ((".rm", rm), (".rv", rv)):
                    g_ = DE.gate(tol, ws_[name + k2], os_[name + k2])
                    assert relerr(got, st[name + k2]) <= g_, (b, half, name, k2, relerr(got, st[name + k2]), g_)
    worst.sort(reverse=True)
    print("\n[%s] worst gradient errors (err / gate, gated): %s" % (dtype, " ".join(
        "%s:%.2e/%.1e%s" % (n, e, g, "" if gd else "(ungated)") for _, e, g, b, n, gd in worst[:8])))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dcgan_iteration_small(dtype):
    """Full iteration, small batch (N = 4), B = 3 models."""
    net, errs, res, hp = run_dcgan(dtype, 3, N=4)
    _check(dtype, net, errs, res, hp, 3, gate_g=False)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dcgan_iteration_full_batch(dtype):
    """BJ configs[3] shapes: N = 128 images of 64 x 64, B = 2 (the 32-bit
    index guards and the bench's tile counts)."""
    net, errs, res, hp = run_dcgan(dtype, 2, N=128)
    _check(dtype, net, errs, res, hp, 2, gate_g=False)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dcgan_generator_gradients(dtype):
    """D's learning rate 0 (so D' = D exactly on both sides): every generator
    gradient tensor gated as the discriminator's (fp32 1e-4; bf16 the
    witness gate), at N = 32."""
    net, errs, res, hp = run_dcgan(dtype, 2, N=32, d_lr_zero=True)
    _check(dtype, net, errs, res, hp, 2, gate_g=True)
