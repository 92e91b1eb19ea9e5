"""Comparison helpers shared by the GPU parity tests (no method arithmetic).

Tolerance metric (reading R20): normwise per (tensor, model)
  ||a - r||_2 / max(||r||_2, 1e-30)
fp32 path: 1e-4; bf16-AMP path: 2e-2 (BJ north_star).
"""
import numpy as np

TOL = {"f32": 1e-4, "bf16": 2e-2}


def relerr(a, r):
    a = np.asarray(a, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    return float(np.linalg.norm((a - r).ravel()) / max(np.linalg.norm(r.ravel()), 1e-30))


def assert_close(a, r, tol, what=""):
    e = relerr(a, r)
    assert e <= tol, "%s: normwise rel err %.3e > %.1e" % (what, e, tol)
    return e
