"""Decision sites of a forward pass: ReLU / LeakyReLU gates and max-pool argmaxes.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Why (readings R15b, R15c in DESIGN.md): a training step is piecewise smooth.
ReLU'(z) = [z > 0] and the argmax of a max-pool are discontinuous decisions;
an implementation that reaches z (or the pooled values) with a rounding error
e may take a decision whose oracle value lies within e of its threshold
either way, and BOTH choices are valid subgradients of the same step (the
paper's equivalence, holds up to floating-point reordering,
P:L1380-1381).  Outside that band the decision is unique.

A `Decisions` context, when active (`with use(d): ...`), makes every site of
the oracle's forward pass
  * record its own decision (`own`) and the set of positions within the
    margin of the threshold (`flag`):
      ReLU   flag = |z| <= margin_rel * scale_c            (per channel c)
      max    flag = top1 - top2 <= margin_rel * scale_c    (per (cloud, channel))
    where scale_c is the magnitude the rounding error of z is proportional
    to: for z = BN(y) = gamma (y - mu) / sigma + beta it is
    |gamma| rms_c(y) / sigma (an error relative to |y| is amplified by
    rms(y) / sigma when BN removes a large mean), else rms_c(z)
  * take an OVERRIDE decision if one is given for the site -- but only where
    the oracle itself flagged the position: an override that disagrees with
    the oracle's own decision outside the flagged set raises DecisionError
    (for the max, the overriding index must hold a value within the margin of
    the top), so an override can never move the oracle off the set of valid
    results.
  * `force=True` (witness runs only) takes the override without validation.

The margin of a site is a multiple of its error scale: a fixed one (fp32) or
one calibrated per site from a conditioning witness (bf16: the oracle re-run
with bf16 rounding of every stored operand, tests/_decide.py; reading R15c).

With no active context (the default) every site takes its own decision, the
plain definition (first index on exact max ties, reading R15).
"""
import contextlib

import numpy as np

ACTIVE = None


class DecisionError(AssertionError):
    pass


class Decisions:
    """margin_rel: default margin of every site; margins: per-site margins
    (relative to the site's error scale) overriding it."""

    def __init__(self, margin_rel=0.0, override=None, force=False, store=None, margins=None):
        self.margin_rel = float(margin_rel)
        self.margins = dict(margins or {})
        self.override = dict(override or {})
        self.force = force
        self.store = store          # witness runs only: rounding applied to stored operands
        self.sites = {}

    def margin(self, name):
        return float(self.margins.get(name, self.margin_rel))


@contextlib.contextmanager
def use(d):
    global ACTIVE
    prev, ACTIVE = ACTIVE, d
    try:
        yield d
    finally:
        ACTIVE = prev


def _rms_c(x, axes):
    return np.sqrt(np.mean(x * x, axis=axes))


def flags(rec, margin):
    """Positions of a recorded site within `margin` (x its error scale) of the
    decision threshold: |z| for a gate, top1 - top2 for an argmax."""
    if rec["kind"] == "relu":
        return np.abs(rec["z"]) <= margin * rec["scale"]
    return rec["gap"] <= margin * rec["scale"]


def relu_gate(name, z, scale=None):
    """Gate [z > 0] of a ReLU / LeakyReLU on z [rows, C] or [N, C, H, W]
    (channel axis 1).  scale [C]: the magnitude an implementation's rounding
    error in z is proportional to (default rms_c(z))."""
    own = z > 0.0
    d = ACTIVE
    if d is None:
        return own
    axes = tuple(i for i in range(z.ndim) if i != 1)
    scale = np.expand_dims(_rms_c(z, axes) if scale is None else np.asarray(scale), axes)
    rec = dict(kind="relu", own=own, z=z, scale=scale)
    flag = flags(rec, d.margin(name))
    used = own
    flips = 0
    if name in d.override:
        ov = np.asarray(d.override[name], dtype=bool).reshape(z.shape)
        diff = ov != own
        if not d.force:
            bad = diff & ~flag
            if bad.any():
                i = np.argwhere(bad)[0]
                raise DecisionError("%s: override flips %d unflagged gate(s), e.g. at %s (z = %.6g)"
                                    % (name, int(bad.sum()), tuple(i), z[tuple(i)]))
        flips = int(diff.sum())
        used = ov
    rec.update(flag=flag, used=used, flips=flips)
    d.sites[name] = rec
    return used


def max_index(name, x, scale=None):
    """argmax over axis 1 of x [N, L, C] (first index on exact ties); scale [C]
    as for relu_gate (default rms_c(x))."""
    own = np.argmax(x, axis=1)
    d = ACTIVE
    if d is None:
        return own
    top = np.take_along_axis(x, own[:, None, :], axis=1)[:, 0, :]
    srt = np.sort(x, axis=1)
    gap = srt[:, -1, :] - srt[:, -2, :] if x.shape[1] > 1 else np.full(top.shape, np.inf)
    scale = (_rms_c(x, (0, 1)) if scale is None else np.asarray(scale))[None, :]
    rec = dict(kind="max", own=own, x=x, top=top, gap=gap, scale=scale)
    m = d.margin(name)
    flag = flags(rec, m)
    used = own
    flips = 0
    if name in d.override:
        ov = np.asarray(d.override[name], dtype=np.int64).reshape(own.shape)
        diff = ov != own
        if not d.force:
            if ((ov < 0) | (ov >= x.shape[1])).any():
                raise DecisionError("%s: override index out of range" % name)
            val = np.take_along_axis(x, ov[:, None, :], axis=1)[:, 0, :]
            bad = diff & ~(flag & (val >= top - m * scale))
            if bad.any():
                i = tuple(np.argwhere(bad)[0])
                raise DecisionError("%s: override argmax at %d unflagged position(s), e.g. %s (top %.6g, chosen %.6g, "
                                    "gap %.3g)" % (name, int(bad.sum()), i, top[i], val[i], gap[i]))
        flips = int(diff.sum())
        used = ov
    rec.update(flag=flag, used=used, flips=flips)
    d.sites[name] = rec
    return used


def store(x, what, name=None, k=None):
    """Witness runs only: the rounding an implementation applies to a stored
    operand ("act", "w", "out", "grad") of layer `name` (k: the contraction
    length of an "out"); identity otherwise."""
    d = ACTIVE
    if d is None or d.store is None:
        return x
    return d.store(x, what, name, k)
