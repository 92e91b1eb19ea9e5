"""Unfused serial baselines for bench.py (SURVEY §8(d) "Beside it" 2).

(a) PyTorch eager, one model after another ("each training job is executed
    on a single accelerator", the paper's Serial baseline):
    stock torch.nn PointNet-cls (the cited implementation's layers, reading
    R1), cuDNN/cuBLAS kernels, bf16 autocast for AMP (TF32 off for fp32),
    torch.optim.Adam.  Not part of the product path.
(b) libhfta at B = 1 looped: the same fused kernels with one model per
    launch -- the fusion gain on identical kernels.
Both report model-samples/s of a serial loop (independent of how many models
the loop visits, so a few models are timed).
"""
import time

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F


class _STN3d(nn.Module):
    def __init__(self):
        super().__init__()
        self.c1, self.c2, self.c3 = nn.Conv1d(3, 64, 1), nn.Conv1d(64, 128, 1), nn.Conv1d(128, 1024, 1)
        self.fc1, self.fc2, self.fc3 = nn.Linear(1024, 512), nn.Linear(512, 256), nn.Linear(256, 9)
        self.b1, self.b2, self.b3 = nn.BatchNorm1d(64), nn.BatchNorm1d(128), nn.BatchNorm1d(1024)
        self.b4, self.b5 = nn.BatchNorm1d(512), nn.BatchNorm1d(256)

    def forward(self, x):
        x = F.relu(self.b1(self.c1(x)))
        x = F.relu(self.b2(self.c2(x)))
        x = F.relu(self.b3(self.c3(x)))
        x = torch.max(x, 2)[0]
        x = F.relu(self.b4(self.fc1(x)))
        x = F.relu(self.b5(self.fc2(x)))
        return self.fc3(x).view(-1, 3, 3) + torch.eye(3, device=x.device, dtype=x.dtype)


class PointNetCls(nn.Module):
    def __init__(self, k=40):
        super().__init__()
        self.stn = _STN3d()
        self.c1, self.c2, self.c3 = nn.Conv1d(3, 64, 1), nn.Conv1d(64, 128, 1), nn.Conv1d(128, 1024, 1)
        self.b1, self.b2, self.b3 = nn.BatchNorm1d(64), nn.BatchNorm1d(128), nn.BatchNorm1d(1024)
        self.fc1, self.fc2, self.fc3 = nn.Linear(1024, 512), nn.Linear(512, 256), nn.Linear(256, k)
        self.bn1, self.bn2 = nn.BatchNorm1d(512), nn.BatchNorm1d(256)
        self.drop = nn.Dropout(0.3)

    def forward(self, x):                      # x [N, 3, L]
        T = self.stn(x)
        x = torch.bmm(x.transpose(2, 1), T).transpose(2, 1)
        x = F.relu(self.b1(self.c1(x)))
        x = F.relu(self.b2(self.c2(x)))
        x = self.b3(self.c3(x))
        x = torch.max(x, 2)[0]
        x = F.relu(self.bn1(self.fc1(x)))
        x = F.relu(self.bn2(self.drop(self.fc2(x))))
        return F.log_softmax(self.fc3(x), dim=1)


def serial_pytorch(x_nl3, labels, n_models=4, steps=3, warmup=2, dtype="bf16", device="cuda"):
    """Model-samples/s of the eager per-model loop (each model: fwd, bwd, Adam)."""
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    models = [PointNetCls().to(device) for _ in range(n_models)]
    opts = [torch.optim.Adam(m.parameters(), lr=1e-3) for m in models]
    x = x_nl3.transpose(1, 2).contiguous()
    y = labels.long()
    N = x.shape[0]

    def one_round():
        for m, o in zip(models, opts):
            o.zero_grad(set_to_none=True)
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=(dtype == "bf16")):
                out = m(x)
                loss = F.nll_loss(out.float(), y)
            loss.backward()
            o.step()

    for _ in range(warmup):
        one_round()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one_round()
    e1.record()
    torch.cuda.synchronize()
    return n_models * N * steps / (e0.elapsed_time(e1) / 1e3)


def serial_libhfta_b1(net_b1, steps=3, warmup=2):
    """Model-samples/s of libhfta with ONE model per launch (net built with B=1)."""
    for _ in range(warmup):
        net_b1.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        net_b1.step()
    e1.record()
    torch.cuda.synchronize()
    return net_b1.N * steps / (e0.elapsed_time(e1) / 1e3)
