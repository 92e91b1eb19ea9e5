"""Serial Adam for ONE model with its own scalar hyper-parameters, NumPy fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper: fused optimizers replace "scalar-vector operations (e.g.
multiplying a learning rate under tuning with the gradients)" by "broadcasted
vector-vector operations".  The serial operation each model runs
is therefore plain Adam with its own (lr, beta1, beta2, eps, wd).  Form
(reading R7): PyTorch 1.6 Adam, coupled L2 weight decay, eps added after
sqrt(v)/sqrt(1 - beta2^t), bias corrections with the shared step t.
"""
import numpy as np


def adam_step(p, g, m, v, t, lr, beta1, beta2, eps, wd):
    """One Adam step on arrays of one parameter tensor; returns (p, m, v)."""
    g = g + wd * p
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    denom = np.sqrt(v) / np.sqrt(bc2) + eps
    p = p - (lr / bc1) * m / denom
    return p, m, v


def adam_model(params, grads, state, t, hp_b):
    """Apply adam_step to every tensor of one model. state: name -> (m, v)."""
    new_p, new_s = {}, {}
    for name, p in params.items():
        if name not in grads:
            new_p[name] = p
            continue
        m, v = state.get(name, (np.zeros_like(p), np.zeros_like(p)))
        new_p[name], m, v = adam_step(p, grads[name], m, v, t, hp_b["lr"], hp_b["beta1"],
                                      hp_b["beta2"], hp_b["eps"], hp_b["wd"])
        new_s[name] = (m, v)
    return new_p, new_s
