"""Conditioning witness for BJ configs[0] (shared MLP) in bf16-AMP: fp64
autograd with bf16 RNE rounding at the tensors the fused step stores in bf16
(x, W, y1, a1, y2, a2 and the gradients flowing through them), vs fp64.
Records the attainable normwise gradient error per tensor."""
import sys

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
import synth  # noqa: E402



class Round(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t):
        return t.to(torch.bfloat16).double()

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).double()


def run(P, x, T, rb):
    Pt = {k: torch.tensor(v, requires_grad=True) for k, v in P.items()}
    r = Round.apply if rb else (lambda t: t)
    h = r(torch.tensor(x))
    for i in (1, 2):
        y = r(F.linear(h, r(Pt["c%d.W" % i]), Pt["c%d.b" % i]))
        h = r(F.relu(F.batch_norm(y, None, None, Pt["bn%d.g" % i], Pt["bn%d.beta" % i], training=True, eps=1e-5)))
    loss = F.mse_loss(h, torch.tensor(T))
    loss.backward()
    return {k: v.grad.numpy() for k, v in Pt.items()}


if __name__ == "__main__":
    P = synth.init_params("mlp_cfg1", 1000)
    x, T = synth.mlp_cfg1_batch(0)
    g0, g1 = run(P, x, T, False), run(P, x, T, True)
    for k in g0:
        if np.linalg.norm(g0[k]) > 1e-9:
            print("%-8s bf16-AMP normwise rel err %.3e" % (k, np.linalg.norm(g1[k] - g0[k]) / np.linalg.norm(g0[k])))
