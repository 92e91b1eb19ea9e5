"""Serial (one model) layer definitions with hand-written backward, NumPy fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Each function is the plain definition of the PyTorch operator that one row of
the paper's fusion-rule table (App. B) fuses; the paper fuses
them but never changes what they compute ("mathematically equivalent
transformations").  Layouts are PyTorch's: Linear weight
[out, in]; Conv2d NCHW with weight [Co, Ci, kh, kw]; ConvTranspose2d weight
[Ci, Co, kh, kw].  Conv1d with kernel 1 (PointNet) is the per-point Linear,
written on [rows, C] matrices.  Library primitives used as single steps:
matmul / tensordot, sum, max, argmax, exp, log.
"""
import numpy as np

BN_EPS = 1e-5        # reading R6 (PyTorch BatchNorm default)
BN_MOMENTUM = 0.1


# -------------------------------------------------------------- Linear ----
# App. B row Linear -> baddbmm; Conv1d row.

def linear_fwd(x, W, b=None):
    """y[r, n] = sum_k x[r, k] W[n, k] + b[n]."""
    y = x @ W.T
    if b is not None:
        y = y + b
    return y


def linear_bwd(dy, x, W, need_dx=True):
    """dx = dy W ; dW = dy^T x ; db = sum_r dy."""
    dx = dy @ W if need_dx else None
    return dx, dy.T @ x, dy.sum(axis=0)


# ----------------------------------------------------------- BatchNorm ----
# App. B rows BatchNorm1d/2d: statistics per channel over all
# rows of ONE model (reading R13), PyTorch training-mode semantics (R6).

def bn_fwd(x, gamma, beta, eps=BN_EPS):
    """x [R, C] -> y, cache.  Biased variance normalises."""
    mean = x.mean(axis=0)
    var = ((x - mean) ** 2).mean(axis=0)
    invstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mean) * invstd
    return gamma * xhat + beta, dict(mean=mean, var=var, invstd=invstd, xhat=xhat)


def bn_running(rm, rv, cache, R, momentum=BN_MOMENTUM):
    """running stats: unbiased variance R/(R-1) for the running estimate (R6)."""
    rm = (1.0 - momentum) * rm + momentum * cache["mean"]
    rv = (1.0 - momentum) * rv + momentum * cache["var"] * R / (R - 1.0)
    return rm, rv


def bn_bwd(dy, cache, gamma):
    """Standard BN backward: dbeta = sum dy, dgamma = sum dy*xhat,
    dx = gamma*invstd/R * (R dy - dbeta - xhat dgamma)."""
    R = dy.shape[0]
    xhat = cache["xhat"]
    dbeta = dy.sum(axis=0)
    dgamma = (dy * xhat).sum(axis=0)
    dx = gamma * cache["invstd"] / R * (R * dy - dbeta - xhat * dgamma)
    return dx, dgamma, dbeta


def nchw_to_rows(x):
    """[N, C, H, W] -> [N*H*W, C] (BatchNorm2d statistics over N, H, W)."""
    N, C, H, W = x.shape
    return x.transpose(0, 2, 3, 1).reshape(N * H * W, C)


def rows_to_nchw(r, shape):
    N, C, H, W = shape
    return r.reshape(N, H, W, C).transpose(0, 3, 1, 2)


def bn2d_fwd(x, gamma, beta, eps=BN_EPS):
    y, c = bn_fwd(nchw_to_rows(x), gamma, beta, eps)
    return rows_to_nchw(y, x.shape), c


def bn2d_bwd(dy, cache, gamma):
    dx, dg, db = bn_bwd(nchw_to_rows(dy), cache, gamma)
    return rows_to_nchw(dx, dy.shape), dg, db


# --------------------------------------------------------- activations ----
# App. B rows ReLU, LeakyReLU, Tanh; Sigmoid (DCGAN D output).

def relu(x):
    return np.maximum(x, 0.0)


def relu_bwd(dy, x):
    return dy * (x > 0.0)


def leaky_relu(x, a=0.2):
    return np.where(x > 0.0, x, a * x)


def leaky_relu_bwd(dy, x, a=0.2):
    return np.where(x > 0.0, dy, a * dy)


def tanh(x):
    return np.tanh(x)


def tanh_bwd(dy, y):
    return dy * (1.0 - y * y)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def sigmoid_bwd(dy, y):
    return dy * y * (1.0 - y)


# -------------------------------------------------- PointNet glue ops ----

def max_over_points(x):
    """x [N, L, C] -> max over L and first argmax (reading R15)."""
    idx = np.argmax(x, axis=1)
    return np.take_along_axis(x, idx[:, None, :], axis=1)[:, 0, :], idx


def max_over_points_bwd(dg, idx, L):
    N, C = dg.shape
    dx = np.zeros((N, L, C))
    np.put_along_axis(dx, idx[:, None, :], dg[:, None, :], axis=1)
    return dx


def transform_points(x, T):
    """x'[n] = x[n] @ T[n] (bmm of [L,3] by [3,3]); PointNet STN transform."""
    return np.matmul(x, T)


def transform_points_bwd(dxp, x, T):
    return np.matmul(dxp, T.transpose(0, 2, 1)), np.matmul(x.transpose(0, 2, 1), dxp)


def dropout(x, keep, p):
    """App. B row Dropout: y = x * keep / (1 - p)."""
    return x * keep / (1.0 - p)


def dropout_bwd(dy, keep, p):
    return dy * keep / (1.0 - p)


# -------------------------------------------------------------- losses ----
# Per-model losses l_b (App. C: "no assumption is made on the
# exact formula of l_beta").  Mean reduction, as in the cited models.

def log_softmax(z):
    m = z.max(axis=-1, keepdims=True)
    return z - m - np.log(np.exp(z - m).sum(axis=-1, keepdims=True))


def nll_mean(z, y):
    """l = -1/N sum_n log_softmax(z)[n, y_n]; dz = (softmax - onehot)/N."""
    N = z.shape[0]
    ls = log_softmax(z)
    loss = -ls[np.arange(N), y].mean()
    dz = np.exp(ls)
    dz[np.arange(N), y] -= 1.0
    return loss, dz / N


def mse_mean(a, T):
    d = a - T
    return (d * d).mean(), 2.0 * d / d.size


def bce_mean(p, y):
    """PyTorch BCELoss (mean) with its log clamp at -100; dp as its backward."""
    lp = np.maximum(np.log(p), -100.0)
    l1p = np.maximum(np.log(1.0 - p), -100.0)
    loss = -(y * lp + (1.0 - y) * l1p).mean()
    dp = (p - y) / np.maximum(p * (1.0 - p), 1e-12) / p.size
    return loss, dp


def softplus(z):
    """log(1 + e^z), written without overflow: max(z, 0) + log1p(e^-|z|)."""
    return np.maximum(z, 0.0) + np.log1p(np.exp(-np.abs(z)))


def bce_sigmoid_mean(z, y):
    """The discriminator's Sigmoid -> BCELoss(mean) as a function of its
    logit z (reading R29): with p = sigmoid(z), log p = -softplus(-z) and
    log(1 - p) = -softplus(z) (identities), so

      l = -mean(y * max(-softplus(-z), -100) + (1 - y) * max(-softplus(z), -100))

    and, chaining BCELoss's backward dp = (p - y) / max(p (1 - p), 1e-12) with
    sigmoid's dz = dp p (1 - p), dz = (p - y) q / max(q, 1e-12) / n with
    q = p (1 - p) = sigmoid(z) sigmoid(-z).  Evaluated from z, the value is
    the exact one for every z (computing p first saturates p to 1 at
    z > ~37 in fp64)."""
    sp_pos, sp_neg = softplus(z), softplus(-z)
    loss = -(y * np.maximum(-sp_neg, -100.0) + (1.0 - y) * np.maximum(-sp_pos, -100.0)).mean()
    p, pn = np.exp(-sp_neg), np.exp(-sp_pos)          # sigmoid(z), sigmoid(-z)
    q = p * pn
    pmy = np.where(y == 1.0, -pn, p - y)              # p - y, written as -sigmoid(-z) when y = 1
    dz = pmy * q / np.maximum(q, 1e-12) / z.size
    return loss, dz


# ---------------------------------------------------------- Conv2d ----
# App. B row Conv2d; Fig. 3.  Definition written as a
# sum over kernel taps, each tap one tensordot over input channels.

def _out(H, k, s, p):
    return (H + 2 * p - k) // s + 1


def conv2d_fwd(x, W, s, p):
    N, Ci, H, Wd = x.shape
    Co, _, kh, kw = W.shape
    Ho, Wo = _out(H, kh, s, p), _out(Wd, kw, s, p)
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    y = np.zeros((N, Co, Ho, Wo))
    for ky in range(kh):
        for kx in range(kw):
            patch = xp[:, :, ky:ky + s * (Ho - 1) + 1:s, kx:kx + s * (Wo - 1) + 1:s]
            y += np.tensordot(patch, W[:, :, ky, kx], axes=([1], [1])).transpose(0, 3, 1, 2)
    return y


def conv2d_bwd(dy, x, W, s, p, need_dx=True):
    N, Ci, H, Wd = x.shape
    Co, _, kh, kw = W.shape
    _, _, Ho, Wo = dy.shape
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    dxp = np.zeros_like(xp) if need_dx else None
    dW = np.zeros_like(W)
    for ky in range(kh):
        for kx in range(kw):
            sl = (slice(None), slice(None), slice(ky, ky + s * (Ho - 1) + 1, s),
                  slice(kx, kx + s * (Wo - 1) + 1, s))
            dW[:, :, ky, kx] = np.tensordot(dy, xp[sl], axes=([0, 2, 3], [0, 2, 3]))
            if need_dx:
                dxp[sl] += np.tensordot(dy, W[:, :, ky, kx], axes=([1], [0])).transpose(0, 3, 1, 2)
    dx = dxp[:, :, p:p + H, p:p + Wd] if need_dx else None
    return dx, dW


# ------------------------------------------------- ConvTranspose2d ----
# App. B row ConvT2d.  Definition: every input pixel scatters
# W[ci, :, ky, kx] * x to output position (iy*s - p + ky, ix*s - p + kx);
# output size (H-1)*s - 2p + k.

def convT2d_fwd(x, W, s, p):
    N, Ci, H, Wd = x.shape
    _, Co, kh, kw = W.shape
    Hf, Wf = (H - 1) * s + kh, (Wd - 1) * s + kw
    full = np.zeros((N, Co, Hf, Wf))
    for ky in range(kh):
        for kx in range(kw):
            full[:, :, ky:ky + s * (H - 1) + 1:s, kx:kx + s * (Wd - 1) + 1:s] += \
                np.tensordot(x, W[:, :, ky, kx], axes=([1], [0])).transpose(0, 3, 1, 2)
    return full[:, :, p:Hf - p, p:Wf - p]


def convT2d_bwd(dy, x, W, s, p, need_dx=True):
    N, Ci, H, Wd = x.shape
    _, Co, kh, kw = W.shape
    Hf, Wf = (H - 1) * s + kh, (Wd - 1) * s + kw
    dfull = np.zeros((N, Co, Hf, Wf))
    dfull[:, :, p:Hf - p, p:Wf - p] = dy
    dx = np.zeros_like(x) if need_dx else None
    dW = np.zeros_like(W)
    for ky in range(kh):
        for kx in range(kw):
            g = dfull[:, :, ky:ky + s * (H - 1) + 1:s, kx:kx + s * (Wd - 1) + 1:s]
            dW[:, :, ky, kx] = np.tensordot(x, g, axes=([0, 2, 3], [0, 2, 3]))
            if need_dx:
                dx += np.tensordot(g, W[:, :, ky, kx], axes=([1], [1])).transpose(0, 3, 1, 2)
    return dx, dW


# ------------------------------------------------------ pooling (NEXT-4) ----
# App. B rows MaxPool2d and AdaptiveAvgPool2d: the fused
# operator pools each of the B x C channels independently, i.e. the serial
# operator per model.  PyTorch semantics: padding takes no part in the max
# (padded positions are -inf), the first window tap wins exact ties (reading
# R32), the output size is floor((H + 2p - k) / s) + 1.

def maxpool2d_windows(x, k, s, p):
    """x [N, C, H, W] -> windows [N, Ho, Wo, k*k, C], tap t = ky*k + kx, -inf outside."""
    N, C, H, W = x.shape
    Ho, Wo = _out(H, k, s, p), _out(W, k, s, p)
    xp = np.full((N, C, H + 2 * p, W + 2 * p), -np.inf)
    xp[:, :, p:p + H, p:p + W] = x
    win = np.empty((N, Ho, Wo, k * k, C))
    for ky in range(k):
        for kx in range(k):
            win[:, :, :, ky * k + kx, :] = xp[:, :, ky:ky + s * (Ho - 1) + 1:s,
                                              kx:kx + s * (Wo - 1) + 1:s].transpose(0, 2, 3, 1)
    return win


def maxpool2d_fwd(x, k, s, p, idx=None):
    """y [N, C, Ho, Wo] = max over each window; idx [N, Ho, Wo, C] the tap
    (first on ties) -- or the given idx (a decision taken elsewhere)."""
    win = maxpool2d_windows(x, k, s, p)
    if idx is None:
        idx = np.argmax(win, axis=3)
    y = np.take_along_axis(win, idx[:, :, :, None, :], axis=3)[:, :, :, 0, :]
    return y.transpose(0, 3, 1, 2), idx


def maxpool2d_bwd(dy, idx, x_shape, k, s, p):
    """dx: each output gradient routed to the input pixel of its window's argmax."""
    N, C, H, W = x_shape
    _, _, Ho, Wo = dy.shape
    dxp = np.zeros((N, C, H + 2 * p, W + 2 * p))
    n, oy, ox, c = np.meshgrid(np.arange(N), np.arange(Ho), np.arange(Wo), np.arange(C), indexing="ij")
    iy = oy * s + idx // k
    ix = ox * s + idx % k
    np.add.at(dxp, (n, c, iy, ix), dy.transpose(0, 2, 3, 1))
    return dxp[:, :, p:p + H, p:p + W]


def avgpool_global_fwd(x):
    """AdaptiveAvgPool2d((1, 1)): y [N, C] = mean over H, W."""
    return x.mean(axis=(2, 3))


def avgpool_global_bwd(dy, x_shape):
    N, C, H, W = x_shape
    return np.broadcast_to(dy[:, :, None, None] / (H * W), x_shape).copy()
