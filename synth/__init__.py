"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no layer, loss or optimizer
math).  It only draws random numbers with NumPy's PCG64 and lays them out:
data batches, per-model noise, per-model hyper-parameter vectors and
per-model initial parameters.  Both `oracle/` and the CUDA-path tests import
it; neither side imports the other.

Every array is produced in float64, rounded to float32 and returned as
float64, so that the fp64 oracle and the fp32/bf16 device path start from
bit-identical values.

Recipes:
  * PointNet points: per sample an anisotropic Gaussian blob whose axis scales
    depend on the class, centred and scaled into the unit sphere, rotated
    about y by a random angle, plus N(0, 0.02) jitter (the preprocessing style
    of the PointNet implementation the paper cites).
  * Segmentation labels: per point, a part index fixed by the octant of the
    point and the sample's class, so the task is learnable.
  * DCGAN real images: U(-1, 1) (the tanh range), NCHW [N, 3, 64, 64].
  * DCGAN noise: N(0, 1), one independent draw per (seed, model b, step).
  * Hyper-parameters: the tuning ranges of P:L973-977 (lr log-uniform,
    beta1/beta2 uniform, weight decay uniform).
  * Initial parameters: PyTorch defaults for PointNet (uniform
    +-1/sqrt(fan_in)); BN affine perturbed (gamma ~ U(0.75, 1.25),
    beta ~ U(-0.1, 0.1)) so the affine path is exercised; DCGAN N(0, 0.02)
    conv and N(1, 0.02)/0 BN (the cited DCGAN example).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "f32", "rng", "points_cls", "points_seg", "images", "noise",
    "hparams_cfg1", "hparams_pointnet", "hparams_dcgan",
    "param_specs", "init_params", "mlp_cfg1_batch",
]


def f32(a):
    """Round to float32 and return as float64 (bit-identical start values)."""
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def rng(*seed_words):
    return np.random.Generator(np.random.PCG64(list(int(s) for s in seed_words)))


# ---------------------------------------------------------------- data ----

def _blobs(g, N, L, k):
    labels = g.integers(0, k, size=N)
    pts = np.empty((N, L, 3))
    for n in range(N):
        c = int(labels[n])
        scales = np.array([0.3 + 0.7 * ((c * 7) % 11) / 10.0,
                           0.3 + 0.7 * ((c * 5) % 13) / 12.0,
                           0.3 + 0.7 * ((c * 3) % 7) / 6.0])
        p = g.standard_normal((L, 3)) * scales
        p -= p.mean(axis=0)
        p /= np.max(np.linalg.norm(p, axis=1))
        th = g.uniform(0.0, 2.0 * np.pi)
        rot = np.array([[np.cos(th), 0.0, -np.sin(th)],
                        [0.0, 1.0, 0.0],
                        [np.sin(th), 0.0, np.cos(th)]])
        p = p @ rot + g.normal(0.0, 0.02, size=(L, 3))
        pts[n] = p
    return pts, labels


def points_cls(seed=0, N=32, L=2500, k=40):
    """ModelNet40-shaped point clouds [N, L, 3] and class labels [N] (BJ cfg2)."""
    pts, labels = _blobs(rng(seed, 1), N, L, k)
    return f32(pts), labels.astype(np.int64)


def points_seg(seed=0, N=32, L=2500, k=50):
    """ShapeNet-part-shaped point clouds [N, L, 3] and part labels [N, L] (BJ cfg3)."""
    pts, cls = _blobs(rng(seed, 2), N, L, 16)
    octant = ((pts[..., 0] > 0).astype(np.int64) + 2 * (pts[..., 1] > 0)
              + 4 * (pts[..., 2] > 0))
    labels = (cls[:, None] * 3 + octant) % k
    return f32(pts), labels.astype(np.int64)


def images(seed=0, N=128, C=3, H=64, W=64):
    """Real images NCHW in the tanh range (BJ cfg4)."""
    return f32(rng(seed, 3).uniform(-1.0, 1.0, size=(N, C, H, W)))


def noise(seed, b, step, N=128, nz=100):
    """Per-model generator noise z_b ~ N(0,1) [N, nz] for (seed, b, step)."""
    return f32(rng(seed, 4, b, step).standard_normal((N, nz)))


def cifar(seed=0, N=128, k=10, H=32, W=32):
    """CIFAR-10-shaped batch (ResNet-18 family, NEXT-4): images NCHW ~ N(0,1)
    (the normalised-pixel range) and labels uniform in [0, k)."""
    g = rng(seed, 9)
    return f32(g.standard_normal((N, 3, H, W))), g.integers(0, k, size=N).astype(np.int64)


def mlp_cfg1_batch(seed=0, N=2, L=128, C_out=64):
    """BJ cfg1: shared points [N*L, 3] ~ U(-1,1) and target [N*L, C_out] ~ N(0,1)."""
    g = rng(seed, 5)
    x = g.uniform(-1.0, 1.0, size=(N * L, 3))
    T = g.standard_normal((N * L, C_out))
    return f32(x), f32(T)


# ------------------------------------------------------ hyper-parameters ----

def hparams_cfg1():
    """BJ cfg1 per-model vectors (cfg 1 row)."""
    return dict(lr=f32([1e-3, 3e-3]), beta1=f32([0.9, 0.8]),
                beta2=f32([0.999, 0.99]), eps=f32([1e-8, 1e-6]),
                wd=f32([0.0, 1e-2]))


def hparams_pointnet(seed, B):
    """Per-model vectors drawn from the tuning ranges of P:L973-977."""
    g = rng(seed, 6)
    return dict(lr=f32(10.0 ** g.uniform(-4.0, -2.0, size=B)),
                beta1=f32(g.uniform(0.001, 0.999, size=B)),
                beta2=f32(g.uniform(0.001, 0.999, size=B)),
                eps=f32(np.full(B, 1e-8)),
                wd=f32(g.uniform(0.0, 0.5, size=B)))


def hparams_dcgan(seed, B):
    g = rng(seed, 7)
    return dict(lr=f32(10.0 ** g.uniform(np.log10(5e-5), -3.0, size=B)),
                beta1=f32(g.uniform(0.3, 0.9, size=B)),
                beta2=f32(np.full(B, 0.999)),
                eps=f32(np.full(B, 1e-8)),
                wd=f32(np.zeros(B)))


def hparams_resnet(seed, B):
    """Per-model Adadelta vectors (ranges: reading R33)."""
    g = rng(seed, 10)
    return dict(lr=f32(10.0 ** g.uniform(-1.0, 0.5, size=B)),
                rho=f32(g.uniform(0.8, 0.95, size=B)),
                eps=f32(np.full(B, 1e-6)),
                wd=f32(g.uniform(0.0, 1e-3, size=B)))


# ------------------------------------------------------------ parameters ----
# A spec entry is (name, shape, init) with PyTorch layouts: Linear/Conv1d(k=1)
# weight [out, in]; Conv2d weight [Co, Ci, kh, kw]; ConvTranspose2d weight
# [Ci, Co, kh, kw].  init in {"u:<fan_in>", "bn_w", "bn_b", "n002", "bn_w_gan",
# "zero"}.

def _lin(prefix, fin, fout, bias=True):
    s = [(prefix + ".W", (fout, fin), "u:%d" % fin)]
    if bias:
        s.append((prefix + ".b", (fout,), "u:%d" % fin))
    return s


def _bn(prefix, c, gan=False):
    return [(prefix + ".g", (c,), "bn_w_gan" if gan else "bn_w"),
            (prefix + ".beta", (c,), "zero" if gan else "bn_b")]


POINTNET_WIDTHS = (64, 128, 1024, 512, 256)
SEG_HEAD_WIDTHS = (512, 256, 128)


def param_specs(arch, k=None, widths=None, ft=False):
    """Parameter list of an architecture (shapes only; Appendix A of SURVEY).

    `widths` = (c1, c2, c3, f1, f2) narrows PointNet for tiny finite-difference
    cases; the seg head then uses (f1, f2, c2).  Default: the paper's model.
    """
    if arch == "mlp_cfg1":
        return (_lin("c1", 3, 64) + _bn("bn1", 64) + _lin("c2", 64, 64)
                + _bn("bn2", 64))
    if arch in ("pointnet_cls", "pointnet_seg"):
        c1, c2, c3, f1, f2 = POINTNET_WIDTHS if widths is None else widths
        s = []
        # STN3d
        s += _lin("stn.c1", 3, c1) + _lin("stn.c2", c1, c2) + _lin("stn.c3", c2, c3)
        s += _lin("stn.fc1", c3, f1) + _lin("stn.fc2", f1, f2) + _lin("stn.fc3", f2, 9)
        s += _bn("stn.bn1", c1) + _bn("stn.bn2", c2) + _bn("stn.bn3", c3)
        s += _bn("stn.bn4", f1) + _bn("stn.bn5", f2)
        # PointNetfeat
        s += _lin("feat.c1", 3, c1) + _lin("feat.c2", c1, c2) + _lin("feat.c3", c2, c3)
        s += _bn("feat.bn1", c1) + _bn("feat.bn2", c2) + _bn("feat.bn3", c3)
        if ft:     # STNkd on the c1 features (feature transform, k = c1)
            s += _lin("fstn.c1", c1, c1) + _lin("fstn.c2", c1, c2) + _lin("fstn.c3", c2, c3)
            s += _lin("fstn.fc1", c3, f1) + _lin("fstn.fc2", f1, f2) + _lin("fstn.fc3", f2, c1 * c1)
            s += _bn("fstn.bn1", c1) + _bn("fstn.bn2", c2) + _bn("fstn.bn3", c3)
            s += _bn("fstn.bn4", f1) + _bn("fstn.bn5", f2)
        if arch == "pointnet_cls":
            k = 40 if k is None else k
            s += _lin("head.fc1", c3, f1) + _lin("head.fc2", f1, f2) + _lin("head.fc3", f2, k)
            s += _bn("head.bn1", f1) + _bn("head.bn2", f2)
        else:
            k = 50 if k is None else k
            h1, h2, h3 = SEG_HEAD_WIDTHS if widths is None else (f1, f2, c2)
            s += _lin("head.c1", c3 + c1, h1) + _lin("head.c2", h1, h2)
            s += _lin("head.c3", h2, h3) + _lin("head.c4", h3, k)
            s += _bn("head.bn1", h1) + _bn("head.bn2", h2) + _bn("head.bn3", h3)
        return s
    if arch == "dcgan_g":
        nz, ngf, nc = 100, 64, 3
        ch = [nz, ngf * 8, ngf * 4, ngf * 2, ngf, nc]
        s = []
        for i in range(5):
            s.append(("t%d.W" % (i + 1), (ch[i], ch[i + 1], 4, 4), "n002"))
            if i < 4:
                s += _bn("bn%d" % (i + 1), ch[i + 1], gan=True)
        return s
    if arch == "dcgan_d":
        ndf, nc = 64, 3
        ch = [nc, ndf, ndf * 2, ndf * 4, ndf * 8, 1]
        s = []
        for i in range(5):
            s.append(("c%d.W" % (i + 1), (ch[i + 1], ch[i], 4, 4), "n002"))
            if 1 <= i <= 3:
                s += _bn("bn%d" % (i + 1), ch[i + 1], gan=True)
        return s
    if arch == "resnet18":
        k = 10 if k is None else k
        w = (64, 128, 256, 512) if widths is None else widths
        s = [("conv1.W", (w[0], 3, 7, 7), "u:%d" % (3 * 49))] + _bn("bn1", w[0])
        cin = w[0]
        for si, c in enumerate(w):
            for b in range(2):
                stride = 2 if (si > 0 and b == 0) else 1
                n = "l%d.%d" % (si + 1, b)
                s += [(n + ".conv1.W", (c, cin, 3, 3), "u:%d" % (9 * cin))] + _bn(n + ".bn1", c)
                s += [(n + ".conv2.W", (c, c, 3, 3), "u:%d" % (9 * c))] + _bn(n + ".bn2", c)
                if stride != 1 or cin != c:
                    s += [(n + ".down.W", (c, cin, 1, 1), "u:%d" % cin)] + _bn(n + ".dbn", c)
                cin = c
        return s + _lin("fc", w[-1], k)
    raise ValueError("unknown arch %r" % (arch,))


def init_params(arch, seed, k=None, widths=None, ft=False):
    """Initial parameters of one model (seed = 1000 + b by convention)."""
    g = rng(seed, 8)
    out = {}
    for name, shape, init in param_specs(arch, k, widths, ft):
        if init.startswith("u:"):
            bound = 1.0 / np.sqrt(int(init[2:]))
            v = g.uniform(-bound, bound, size=shape)
        elif init == "bn_w":
            v = g.uniform(0.75, 1.25, size=shape)
        elif init == "bn_b":
            v = g.uniform(-0.1, 0.1, size=shape)
        elif init == "n002":
            v = g.normal(0.0, 0.02, size=shape)
        elif init == "bn_w_gan":
            v = g.normal(1.0, 0.02, size=shape)
        elif init == "zero":
            v = np.zeros(shape)
        else:
            raise ValueError(init)
        out[name] = f32(v)
    return out
