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
      ReLU   flag = |z| <= margin_rel * rms_c(z)         (per channel c)
      max    flag = top1 - top2 <= margin_rel * rms_c(x) (per (cloud, channel))
  * take an OVERRIDE decision if one is given for the site -- but only where
    the oracle itself flagged the position: an override that disagrees with
    the oracle's own decision outside the flagged set raises DecisionError
    (for the max, the overriding index must hold a value within the margin of
    the top), so an override can never move the oracle off the set of valid
    results.
  * `force=True` (witness runs only) takes the override without validation.

With no active context (the default) every site takes its own decision, the
plain definition (first index on exact max ties, reading R15).
"""
import contextlib

import numpy as np

ACTIVE = None


class DecisionError(AssertionError):
    pass


class Decisions:
    def __init__(self, margin_rel=0.0, override=None, force=False, store=None):
        self.margin_rel = float(margin_rel)
        self.override = dict(override or {})
        self.force = force
        self.store = store          # witness runs only: rounding applied to stored operands
        self.sites = {}

    def summary(self):
        return {k: (v["kind"], int(v["flag"].sum()), int(v["flag"].size), int(v.get("flips", 0)))
                for k, v in self.sites.items()}


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


def relu_gate(name, z):
    """Gate [z > 0] of a ReLU / LeakyReLU on z [rows, C] or [N, C, H, W] (channel axis 1)."""
    own = z > 0.0
    d = ACTIVE
    if d is None:
        return own
    axes = tuple(i for i in range(z.ndim) if i != 1)
    scale = np.expand_dims(_rms_c(z, axes), axes)
    flag = np.abs(z) <= d.margin_rel * scale
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
    d.sites[name] = dict(kind="relu", own=own, flag=flag, used=used, flips=flips, z=z)
    return used


def max_index(name, x):
    """argmax over axis 1 of x [N, L, C] (first index on exact ties)."""
    own = np.argmax(x, axis=1)
    d = ACTIVE
    if d is None:
        return own
    top = np.take_along_axis(x, own[:, None, :], axis=1)[:, 0, :]
    s = np.sort(x, axis=1)
    gap = s[:, -1, :] - s[:, -2, :] if x.shape[1] > 1 else np.full(top.shape, np.inf)
    margin = d.margin_rel * _rms_c(x, (0, 1))[None, :]
    flag = gap <= margin
    used = own
    flips = 0
    if name in d.override:
        ov = np.asarray(d.override[name], dtype=np.int64).reshape(own.shape)
        diff = ov != own
        if not d.force:
            if ((ov < 0) | (ov >= x.shape[1])).any():
                raise DecisionError("%s: override index out of range" % name)
            val = np.take_along_axis(x, ov[:, None, :], axis=1)[:, 0, :]
            bad = diff & ~(flag & (val >= top - margin))
            if bad.any():
                i = tuple(np.argwhere(bad)[0])
                raise DecisionError("%s: override argmax at %d unflagged position(s), e.g. %s (top %.6g, chosen %.6g, "
                                    "gap %.3g, margin %.3g)" % (name, int(bad.sum()), i, top[i], val[i], gap[i],
                                                                margin[0, i[1]]))
        flips = int(diff.sum())
        used = ov
    d.sites[name] = dict(kind="max", own=own, flag=flag, used=used, flips=flips)
    return used


def store(x, what):
    """Witness runs only: the rounding an implementation applies to a stored
    operand ("act", "w", "grad"); identity otherwise."""
    d = ACTIVE
    if d is None or d.store is None:
        return x
    return d.store(x, what)
