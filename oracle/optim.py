"""Serial SGD(+momentum/Nesterov), Adadelta and StepLR for ONE model with its
own scalar hyper-parameters, NumPy fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper names fused optimizers "e.g., Adam and Adadelta" and "learning rate
schedulers (e.g., StepLR)", tunes momentum and the
"Factor/Period of Learning Rate Decay"; BJ north_star names a
fused "Adam/SGD step".  The serial operations each model runs are the
PyTorch-1.6 forms (reading R7 extended): coupled L2 weight decay, SGD
momentum buffer initialised to the first d_p (no dampening on step 1).
"""
import math

import numpy as np


def sgd_step(p, g, buf, t, lr, momentum, dampening, wd, nesterov):
    d = g + wd * p
    if momentum != 0.0:
        buf = d.copy() if t == 1 else momentum * buf + (1.0 - dampening) * d
        d = d + momentum * buf if nesterov else buf
    return p - lr * d, buf


def adadelta_step(p, g, sq, acc, lr, rho, eps, wd):
    g = g + wd * p
    sq = rho * sq + (1.0 - rho) * g * g
    std = np.sqrt(sq + eps)
    delta = np.sqrt(acc + eps) / std * g
    acc = rho * acc + (1.0 - rho) * delta * delta
    return p - lr * delta, sq, acc


def steplr(lr0, gamma, period, epoch):
    """lr(epoch) = lr0 * gamma ** floor(epoch / period)."""
    return lr0 * gamma ** math.floor(epoch / period)
