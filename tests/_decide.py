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
import zlib

import numpy as np
import torch

from oracle import decisions as Dm
from oracle import models as OM

# Decision margins, in units of each site's error scale (reading R15c).
# fp32: fixed, >= 5x the largest decision-variable error the GPU path shows
# (`decision_errors`, measured on the box: <= 1.3 x 2^-14).  bf16: calibrated
# per site from the bf16-storage witness -- WITNESS_SAFETY x the largest
# change of the site's decision variable that bf16 rounding of the stored
# operands causes in the oracle itself (at least BF16_FLOOR).
MARGIN_F32 = 2.0 ** -14       # floor of the fp32 margins (the witness calibrates them per site)
# bf16 gradient gate per tensor: max(2e-2, WITNESS_GATE x the witness's
# normwise change of that gradient).  The GPU rounds at a few points the
# witness does not model (dZ stored in bf16 between kernels, the K10 M matrix
# in bf16), measured GPU error / witness <= 1.7 on the box (reading R28).
WITNESS_GATE = 3.0
WITNESS_SAFETY = 3.0
BF16_FLOOR = 2.0 ** -8
MARGIN = {"f32": MARGIN_F32, "bf16": BF16_FLOOR}


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
    if getattr(net, "ft", False):          # STNkd of the feature transform
        for i in (1, 2):
            d["fstn.bn%d" % i] = _h(S["fstn.a%d" % i][b]) > 0
        d["fstn.max"] = S["fstn.amax"][b].cpu().numpy().astype(np.int64)
        d["_fstn.pooled_on"] = _h(S["fstn.g"][b]) > 0
        d["fstn.bn4"] = _h(S["fstn.h4"][b]) > 0
        d["fstn.bn5"] = _h(S["fstn.h5"][b]) > 0
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
    if getattr(net, "ft", False):
        v.update({"fstn.bn1": S["fstn.a1"][b], "fstn.bn2": S["fstn.a2"][b], "fstn.bn4": S["fstn.h4"][b],
                  "fstn.bn5": S["fstn.h5"][b]})
    if net.task == "cls":
        v.update({"head.bn1": S["head.h1"][b], "head.bn2": S["head.h2"][b]})
    else:
        v.update({"head.bn%d" % i: S["seg.h%d" % i][b] for i in (1, 2, 3)})
    return {k: _h(t) for k, t in v.items()}


def decision_errors(ctx, gpu_vals, margins):
    """max |z_gpu - z_oracle| / (scale_c * margin) over positions near the
    threshold (0 < z_oracle <= rms_c(z), GPU output > 0: there the stored ReLU
    output is the GPU's z, up to its storage rounding), scale_c the site's
    error scale (oracle/decisions.py) -- must stay below 1."""
    out = {}
    for site, a in gpu_vals.items():
        if site not in ctx.sites:
            continue
        z = ctx.sites[site]["z"]
        a = a.reshape(z.shape)
        axes = tuple(i for i in range(z.ndim) if i != 1)
        rms = np.expand_dims(np.sqrt(np.mean(z * z, axis=axes)), axes)
        sel = (a > 0) & (z > 0) & (z <= rms)
        sc = np.broadcast_to(ctx.sites[site]["scale"], z.shape)
        out[site] = float(np.max(np.abs(a - z)[sel] / sc[sel])) / margins[site] if sel.any() else 0.0
    return out


def witness_margins(own, wit, floor=None):
    """Per-site margins from the witness (same decisions): WITNESS_SAFETY x
    the largest |change| of the decision variable over its error scale."""
    floor = BF16_FLOOR if floor is None else floor
    m = {}
    for site, v in own.sites.items():
        w = wit.sites[site]
        key = "z" if v["kind"] == "relu" else "x"
        sc = v["scale"] if v["kind"] == "relu" else v["scale"][:, None, :]
        fin = np.isfinite(w[key]) & np.isfinite(v[key])      # -inf: padded max-pool window taps
        err = float(np.max(np.abs(np.where(fin, w[key] - v[key], 0.0)) / sc))
        m[site] = max(floor, WITNESS_SAFETY * err)
    return m


def build_override(own_ctx, gpu, margins, L=None, skip=()):
    """Override map from the GPU decisions + a per-site agreement report:
    flagged count, flips, disagreements outside the flagged band and the
    largest normalised distance of any disagreement from the threshold
    (|z| / scale for a gate, (top - chosen) / scale for an argmax, in units
    of the site's margin: <= 1 for every valid override)."""
    override, report = {}, {}
    for site, v in own_ctx.sites.items():
        if any(site.startswith(p) for p in skip):
            continue
        own = v["own"]
        flag = Dm.flags(v, margins[site])
        if site in ("stn.bn3", "fstn.bn3"):
            # only the argmax rows' gates are observable (and used by the backward)
            pre = site.split(".")[0]
            ov = own.copy()
            amax = gpu[pre + ".max"]
            N, C = amax.shape
            rows = np.arange(N)[:, None] * L + amax
            ov[rows, np.arange(C)[None, :]] = gpu["_%s.pooled_on" % pre]
            g = ov
        elif site in gpu:
            g = np.asarray(gpu[site]).reshape(own.shape)
        else:
            continue
        diff = g != own
        bad = diff & ~flag          # (a flagged argmax change is value-checked by the oracle itself)
        dist = 0.0
        if diff.any():
            if v["kind"] == "relu":
                sc = np.broadcast_to(v["scale"], v["z"].shape)
                dist = float(np.max(np.abs(v["z"])[diff] / sc[diff]))
            else:
                val = np.take_along_axis(v["x"], np.clip(g, 0, v["x"].shape[1] - 1)[:, None, :], axis=1)[:, 0, :]
                sc = np.broadcast_to(v["scale"], v["top"].shape)
                dist = float(np.max((v["top"] - val)[diff] / sc[diff]))
        report[site] = dict(flagged=int(flag.sum()), size=int(flag.size), flips=int(diff.sum()),
                            unflagged_disagree=int(bad.sum()), max_dist=dist / margins[site],
                            margin=margins[site])
        override[site] = g
    return override, report


def _rb(x):
    return torch.tensor(np.asarray(x, dtype=np.float64)).to(torch.bfloat16).double().numpy()


def bf16_store(out_layers=()):
    """Witness rounding at the bf16-AMP storage points: every contraction's
    inputs, weights and incoming gradients; its output only for the layers
    whose pre-activation the GPU path stores in bf16 (`out_layers`)."""
    def f(x, what, name, k=None):
        if what == "out" and (name is None or not any(name.startswith(p) for p in out_layers)):
            return x
        return _rb(x)
    return f


def f32_store():
    """fp32 witness: every stored operand rounded to fp32, and every
    contraction output perturbed by relative noise of the size fp32
    accumulation leaves (2^-24 sqrt(k), k the contraction length; seeded per
    layer, so the witness is deterministic)."""
    def f(x, what, name, k=None):
        x = np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)
        if what == "out" and k:
            g = np.random.default_rng(zlib.crc32(repr((name, x.shape)).encode()))
            x = x * (1.0 + 2.0 ** -24 * np.sqrt(k) * g.standard_normal(x.shape))
        return x
    return f


# PointNet: K10/K11 keep y in fp32 (never stored); the seg head stores y1..y3 in bf16
POINTNET_OUT = ("head.c1", "head.c2", "head.c3")


def oracle_with_decisions(arch, P, S, O, batch, t, hp_b, b, gpu, dtype, L=None, witness=False, **kw):
    """(oracle result with the GPU's flagged-band decisions, agreement report,
    witness result or None).

    pass 1: the oracle's own decisions and decision variables;
    witness (bf16): the same decisions with bf16 rounding of every stored
      operand (reading R28) -- per-site margins (bf16) and the per-tensor
      gradient sensitivity to bf16 storage;
    pass 2: the GPU's decisions inside the flagged bands (validated by the
      oracle), the reference every GPU quantity is compared with."""
    step = lambda: OM.train_step(arch, P, S, O, batch, t, hp_b, b=b, **kw)
    return with_decisions(step, gpu, dtype, L=L, witness=witness, out_layers=POINTNET_OUT)


def with_decisions(step, gpu, dtype, L=None, witness=False, out_layers=(), skip=()):
    """The three-pass flow above for any oracle step callable `step()`.
    Sites whose name starts with a prefix in `skip` keep the oracle's own
    decisions and are not compared.  The witness runs in both precisions
    (bf16: storage rounding; fp32: storage rounding + accumulation-size
    noise, reading R28) and calibrates the per-site margins and the
    per-tensor gates."""
    d1 = Dm.Decisions()
    with Dm.use(d1):
        res1 = step()
    own = {k: v["own"] for k, v in d1.sites.items()}
    dw = Dm.Decisions(0.0, own, force=True, store=bf16_store(out_layers) if dtype == "bf16" else f32_store())
    with Dm.use(dw):
        res_w = step()
    res_w["own"] = res1                 # the same decisions without the rounding
    margins = witness_margins(d1, dw, BF16_FLOOR if dtype == "bf16" else MARGIN_F32)
    override, report = build_override(d1, gpu, margins, L, skip)
    report["_ctx"] = d1
    report["_margins"] = margins
    if any(v["unflagged_disagree"] for k, v in report.items() if not k.startswith("_")):
        return None, report, res_w          # the caller reports and fails
    d2 = Dm.Decisions(0.0, override, margins=margins)
    with Dm.use(d2):
        res = step()
    return res, report, res_w


def gate(tol, wit, own, ref_shape_ok=True):
    """Per-quantity gate of reading R28: max(north_star tolerance,
    WITNESS_GATE x the witness's normwise change of that quantity)."""
    from tests._cmp import relerr
    return max(tol, WITNESS_GATE * relerr(wit, own))
