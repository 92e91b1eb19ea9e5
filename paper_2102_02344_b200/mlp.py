"""Fused shared-MLP training step: BJ configs[0] (B = 2 PointNet-style shared
MLPs, Conv1d k=1 3 -> 64 -> 64 with BN + ReLU, MSE against a shared target,
one fused Adam step with per-model hyper-parameters).  The smallest whole
step of the hot path; every layer is one C-ABI call for all B models.
"""
import torch

from . import hfta as H
from .fused import Workspace
from .net import FusedNet, _Acts, _in, _out, A_RELU


class FusedMLP(FusedNet):
    bn_followed = frozenset({"c1", "c2"})

    def __init__(self, B, param_specs, params, hp, rows=256, dtype="f32", device="cuda"):
        self._base_init(B, param_specs, params, hp, dtype, device)
        self.R = rows
        sh = self.arena.shape
        self.c1, self.c2 = sh["c1.W"][0], sh["c2.W"][0]
        a = _Acts(B, self.tdt, self.device)
        R = rows
        self.x_dt = torch.empty(R, 3, dtype=self.tdt, device=self.device)
        self.S = dict(y1=a(R, self.c1), a1=a(R, self.c1), y2=a(R, self.c2), a2=a(R, self.c2),
                      da2=a(R, self.c2), dy2=a(R, self.c2), da1=a(R, self.c1), dy1=a(R, self.c1))
        self.loss = torch.zeros(B, dtype=torch.float32, device=self.device)
        self.mean_loss = torch.zeros(1, dtype=torch.float32, device=self.device)
        ws = Workspace(self.device)
        for (M, Nn, K) in [(R, self.c1, 3), (R, self.c2, self.c1)]:
            ws.reserve(H.hfta_fused_linear_bwd_workspace(B, M, Nn, K, self.dt))
        for C in (self.c1, self.c2):
            ws.reserve(H.hfta_fused_bn_workspace(B, R, C))
        ws.reserve(H.hfta_loss_workspace(B, R))
        ws.alloc()
        self.ws = ws

    def step(self, x, target, stream=None):
        """x: device fp32 [rows, 3] shared; target: device fp32 [rows, c2] shared."""
        s = H.stream_ptr(stream)
        S, R, B = self.S, self.R, self.B
        self.t += 1
        if self.dt == H.HFTA_F32:
            self.x_dt = x
        else:
            H.hfta_cast_f32_bf16(R * 3, H.ptr(x), H.ptr(self.x_dt), s)
        xin = H.tin(self.x_dt, 0, 3)
        self._lin_fwd(xin, R, "c1", S["y1"], s)
        self._bn_fwd(S["y1"], "bn1", A_RELU, S["a1"], s)
        self._lin_fwd(_in(S["a1"]), R, "c2", S["y2"], s)
        self._bn_fwd(S["y2"], "bn2", A_RELU, S["a2"], s)
        H.hfta_loss_mse(B, R, self.c2, self.dt, _in(S["a2"]), H.ptr(target), 0, self.c2, H.ptr(self.loss),
                        H.ptr(self.mean_loss), _out(S["da2"]), self.ws.ptr, self.ws.nbytes, s)
        self._bn_bwd(S["da2"], S["y2"], "bn2", A_RELU, S["dy2"], s)
        self._lin_bwd(S["dy2"], _in(S["a1"]), R, "c2", S["da1"], s)
        self._bn_bwd(S["da1"], S["y1"], "bn1", A_RELU, S["dy1"], s)
        self._lin_bwd(S["dy1"], xin, R, "c1", None, s)
        self.adam(s)
        return self.loss
