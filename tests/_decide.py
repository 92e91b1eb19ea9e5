"""Whole-step parity with decision overrides (readings R15b, R15c, R28).

Test infrastructure: reads the GPU step's own decisions (ReLU gates from its
stored activations, max-pool argmaxes from its argmax buffers), checks that
they equal the oracle's at every position the oracle did NOT flag as within
its rounding band, then re-runs the oracle with the GPU's choices at the
flagged positions only (the oracle itself rejects anything else, see
oracle/decisions.py), so every gradient can be compared against ONE valid
subgradient instead of a result a rounding-level decision flip moves.

No method arithmetic here: decisions are booleans / indices read from the GPU
buffers; all values come from the oracle.
"""
import numpy as np
import torch

from oracle import decisions as Dm
from oracle import models as OM

# Decision margins relative to the per-channel rms of the decision variable
# (reading R15c).  They are >= 8x the largest decision-variable error the GPU
# path shows (measured by `decision_errors` on positive ReLU outputs, where
# the stored activation IS the GPU's pre-activation value).
MARGIN = {"f32": 2.0 ** -14, "bf16": 2.0 ** -5}


def _h(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def pointnet_gpu_decisions(net, b):
    """Decisions of the fused PointNet step for model b, keyed by oracle site."""
    S = net.S
    d = {}
    for p in ("stn", "feat"):
        for i in (1, 2):
            d["%s.bn%d" % (p, i)] = _h(S["%s.a%d" % (p, i)][b]) > 0
        d[p + ".max"] = S[p + ".amax"][b].cpu().numpy().astype(np.int64)
    d["_stn.pooled_on"] = _h(S["stn.g"][b]) > 0           # ReLU gate of stn.bn3 at the argmax rows
    d["stn.bn4"] = _h(S["stn.h4"][b]) > 0
    d["stn.bn5"] = _h(S["stn.h5"][b]) > 0
    if net.task == "cls":
        d["head.bn1"] = _h(S["head.h1"][b]) > 0
        d["head.bn2"] = _h(S["head.h2"][b]) > 0
    else:
        for i in (1, 2, 3):
            d["head.bn%d" % i] = _h(S["seg.h%d" % i][b]) > 0
    return d


def pointnet_gpu_values(net, b):
    """GPU activations at the ReLU sites (positive entries = its z)."""
    S = net.S
    v = {"stn.bn1": S["stn.a1"][b], "stn.bn2": S["stn.a2"][b], "feat.bn1": S["feat.a1"][b],
         "feat.bn2": S["feat.a2"][b], "stn.bn4": S["stn.h4"][b], "stn.bn5": S["stn.h5"][b]}
    if net.task == "cls":
        v.update({"head.bn1": S["head.h1"][b], "head.bn2": S["head.h2"][b]})
    else:
        v.update({"head.bn%d" % i: S["seg.h%d" % i][b] for i in (1, 2, 3)})
    return {k: _h(t) for k, t in v.items()}


def decision_errors(ctx, gpu_vals):
    """max |z_gpu - z_oracle| / rms_c(z) over positions near the threshold
    (0 < z_oracle <= rms_c, GPU output > 0: there the stored ReLU output is the
    GPU's z, up to its storage rounding) -- the margin must exceed it."""
    out = {}
    for site, a in gpu_vals.items():
        if site not in ctx.sites:
            continue
        z = ctx.sites[site]["z"]
        a = a.reshape(z.shape)
        axes = tuple(i for i in range(z.ndim) if i != 1)
        rms = np.expand_dims(np.sqrt(np.mean(z * z, axis=axes)), axes)
        sel = (a > 0) & (z > 0) & (z <= rms)
        out[site] = float(np.max(np.abs(a - z)[sel] / np.broadcast_to(rms, z.shape)[sel])) if sel.any() else 0.0
    return out


def build_override(own_ctx, gpu, L=None):
    """Override map from the GPU decisions + a per-site agreement report.
    Raises AssertionError naming the site if the GPU disagrees with the oracle
    at an unflagged position."""
    override, report = {}, {}
    for site, v in own_ctx.sites.items():
        own, flag = v["own"], v["flag"]
        if site == "stn.bn3":
            # only the argmax rows' gates are observable (and used by the backward)
            ov = own.copy()
            amax = gpu["stn.max"]
            N, C = amax.shape
            rows = np.arange(N)[:, None] * L + amax
            ov[rows, np.arange(C)[None, :]] = gpu["_stn.pooled_on"]
            g = ov
        elif site in gpu:
            g = np.asarray(gpu[site]).reshape(own.shape)
        else:
            continue
        diff = g != own
        bad = diff & ~flag          # (a flagged argmax change is value-checked by the oracle itself)
        report[site] = dict(flagged=int(flag.sum()), size=int(flag.size), flips=int(diff.sum()),
                            unflagged_disagree=int(bad.sum()))
        assert not bad.any(), "GPU decision differs from the oracle outside the flagged band at %s: %s" % (
            site, report[site])
        override[site] = g
    return override, report


def bf16_round(x, what):
    return torch.tensor(np.asarray(x, dtype=np.float64)).to(torch.bfloat16).double().numpy()


def oracle_with_decisions(arch, P, S, O, batch, t, hp_b, b, gpu, margin, L=None, witness=False, **kw):
    """(oracle result with the GPU's flagged-band decisions, agreement report,
    witness result or None).  The witness re-runs the SAME decisions with
    bf16 rounding of every stored operand (reading R28): the size of the
    gradient change bf16-AMP storage alone causes on this step."""
    d1 = Dm.Decisions(margin)
    with Dm.use(d1):
        OM.train_step(arch, P, S, O, batch, t, hp_b, b=b, **kw)
    override, report = build_override(d1, gpu, L)
    report["_ctx"] = d1
    d2 = Dm.Decisions(margin, override)
    with Dm.use(d2):
        res = OM.train_step(arch, P, S, O, batch, t, hp_b, b=b, **kw)
    res_w = None
    if witness:
        used = {k: v["used"] for k, v in d2.sites.items()}
        d3 = Dm.Decisions(margin, used, force=True, store=bf16_round)
        with Dm.use(d3):
            res_w = OM.train_step(arch, P, S, O, batch, t, hp_b, b=b, **kw)
    return res, report, res_w
