"""Conditioning witness for bf16-AMP parity of the PointNet-cls step (CPU only).

Runs the cited PointNet-cls model (torch.nn.functional, float64 autograd) at
BJ cfg2 shapes, once in plain fp64 and then with bf16 round-to-nearest-even
inserted at the points an AMP implementation stores bf16 (conv weights,
conv inputs, conv outputs, and the gradients flowing through them), and
reports the normwise relative error of every parameter gradient against fp64.
A second pair of AMP runs differ only by 1e-7 relative perturbations before
each rounding (what fp32-vs-fp64 accumulation order does), measuring how
chaotic the rounding is.  Results are recorded in DESIGN.md ("bf16 parity").

usage: python tools/amp_conditioning.py [N L [bf16|f32]]   (f32: the same
witness with float32 storage rounding, i.e. the fp32 path's floor)
"""
import sys

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
import synth  # noqa: E402

NOISE = [0.0]
RDT = [torch.bfloat16]


class Round(torch.autograd.Function):
    """bf16 RNE in forward and backward (fp64 carrier)."""
    @staticmethod
    def forward(ctx, t, on):
        ctx.on = on
        return _rb(t) if on else t

    @staticmethod
    def backward(ctx, g):
        return (_rb(g) if ctx.on else g), None


def _rb(t):
    if NOISE[0]:
        t = t * (1 + NOISE[0] * torch.randn_like(t))
    return t.to(RDT[0]).double()


def run(Pn, x, y, keep, p, rw=False, ri=False, ro=False):
    P = {k: torch.tensor(v, requires_grad=True) for k, v in Pn.items()}

    def bn(h, n):
        return F.batch_norm(h, None, None, P[n + ".g"], P[n + ".beta"], training=True, eps=1e-5)

    def conv(h, n):
        out = F.conv1d(Round.apply(h, ri), Round.apply(P[n + ".W"], rw)[:, :, None], P[n + ".b"])
        return Round.apply(out, ro)

    def lin(h, n):
        return F.linear(h, P[n + ".W"], P[n + ".b"])

    xt = torch.tensor(x).transpose(1, 2)
    h = F.relu(bn(conv(xt, "stn.c1"), "stn.bn1"))
    h = F.relu(bn(conv(h, "stn.c2"), "stn.bn2"))
    h = F.relu(bn(conv(h, "stn.c3"), "stn.bn3"))
    h = torch.max(h, 2)[0]
    h = F.relu(bn(lin(h, "stn.fc1"), "stn.bn4"))
    h = F.relu(bn(lin(h, "stn.fc2"), "stn.bn5"))
    T = lin(h, "stn.fc3").view(-1, 3, 3) + torch.eye(3, dtype=torch.float64)
    h = torch.bmm(xt.transpose(2, 1), T).transpose(2, 1)
    h = F.relu(bn(conv(h, "feat.c1"), "feat.bn1"))
    h = F.relu(bn(conv(h, "feat.c2"), "feat.bn2"))
    g = torch.max(bn(conv(h, "feat.c3"), "feat.bn3"), 2)[0]
    h = F.relu(bn(lin(g, "head.fc1"), "head.bn1"))
    h = lin(h, "head.fc2") * torch.tensor(keep.astype(float)) / (1 - p)
    logits = lin(F.relu(bn(h, "head.bn2")), "head.fc3")
    loss = F.nll_loss(F.log_softmax(logits, 1), torch.tensor(y))
    loss.backward()
    return loss.item(), {k: v.grad.numpy() for k, v in P.items()}


def main():
    N, L = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (32, 2500)
    if len(sys.argv) > 3 and sys.argv[3] == "f32":
        RDT[0] = torch.float32
    print("rounding dtype:", RDT[0])
    P = synth.init_params("pointnet_cls", 1000)
    x, y = synth.points_cls(0, N=N, L=L)
    keep = np.random.default_rng(0).uniform(size=(N, 256)) > 0.3
    l0, g0 = run(P, x, y, keep, 0.3)
    gmax = max(np.linalg.norm(v) for v in g0.values())
    live = [k for k in g0 if np.linalg.norm(g0[k]) > 1e-9 * gmax]   # skip analytically-zero grads
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    for name, kw in [("weights only", dict(rw=True)), ("inputs only", dict(ri=True)),
                     ("outputs only", dict(ro=True)), ("all (AMP)", dict(rw=True, ri=True, ro=True))]:
        l, g = run(P, x, y, keep, 0.3, **kw)
        e = [rel(g[k], g0[k]) for k in live]
        worst = sorted(zip(e, live), reverse=True)[:4]
        whole = rel(np.concatenate([g[k].ravel() for k in live]), np.concatenate([g0[k].ravel() for k in live]))
        print("%-13s loss rel %.1e | whole-model grad rel %.2e | per tensor: median %.2e max %.2e | worst %s" %
              (name, abs(l - l0) / l0, whole, np.median(e), max(e),
               " ".join("%s:%.1e" % (k, v) for v, k in worst)))
    l1, g1 = run(P, x, y, keep, 0.3, rw=True, ri=True, ro=True)
    NOISE[0] = 1e-7
    torch.manual_seed(1)
    l2, g2 = run(P, x, y, keep, 0.3, rw=True, ri=True, ro=True)
    e = [rel(g2[k], g1[k]) for k in live]
    print("AMP vs AMP with 1e-7 pre-rounding noise: loss rel %.1e | grad median %.2e max %.2e" %
          (abs(l1 - l2) / l1, np.median(e), max(e)))


if __name__ == "__main__":
    main()
