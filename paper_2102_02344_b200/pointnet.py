"""Fused PointNet training step (BJ configs[1..2]; the PointNet the paper
benchmarks, model of the implementation it cites, reading R1).

`FusedPointNet(B, ...)` holds B PointNet models that share an architecture
and a data batch but have their own parameters and hyper-parameters
(P:L851-857).  `step(x, labels)` runs ONE horizontally fused training step
(forward, backward, fused Adam) for all B models through libhfta's C ABI:
every layer is one set of launches for all B models.  Activations are kept
model-major [B][rows][C] with C contiguous (rows = N*L points).

Per-model results are unfused with `params(b)` / `arena.host_tensor`.
"""
import os

import numpy as np
import torch

from . import hfta as H
from .fused import Workspace
from .net import FusedNet, _Acts, _in, _out, A_RELU, A_NONE

# Layers whose output feeds a training-mode BatchNorm directly: the gradient
# of their bias is identically zero (BN's input gradient sums to zero over the
# rows: sum_r dx_r = gamma*invstd*(sum dz - dbeta - dgamma*sum(xhat)/R) = 0
# since sum(xhat) = 0), so the fused step writes exact zeros instead of
# reducing a rounding-noise column sum.
BN_FOLLOWED = {"stn.c1", "stn.c2", "stn.c3", "stn.fc1", "stn.fc2", "feat.c1", "feat.c2", "feat.c3",
               "head.fc1", "head.c1", "head.c2", "head.c3",
               "fstn.c1", "fstn.c2", "fstn.c3", "fstn.fc1", "fstn.fc2"}


class FusedPointNet(FusedNet):
    """B fused PointNet models (task 'cls' or 'seg')."""

    bn_followed = BN_FOLLOWED

    def __init__(self, B, param_specs, params, hp, task="cls", dtype="f32", N=32, L=2500, k=40,
                 p_drop=0.3, dropout_seed=42, device="cuda", feature_transform=False, ft_weight=0.001, model_offset=0,
                 model_ids=None):
        assert task in ("cls", "seg")
        self._base_init(B, param_specs, params, hp, dtype, device)
        self.task, self.N, self.L, self.k = task, N, L, k
        self.R = N * L
        self.p_drop, self.dropout_seed = p_drop, dropout_seed
        self.model_offset = int(model_offset)     # global index of model 0 (model-array sharding: dropout masks)
        # explicit per-model dropout ids (HFHT partitions of non-contiguous sets), else model_offset + b
        self.model_ids = (torch.tensor(np.asarray(model_ids, dtype=np.int32), device=device)
                          if model_ids is not None else None)
        sh = self.arena.shape
        self.c1, self.c2, self.c3 = sh["stn.c1.W"][0], sh["stn.c2.W"][0], sh["stn.c3.W"][0]
        self.f1, self.f2 = sh["stn.fc1.W"][0], sh["stn.fc2.W"][0]
        # bf16: c3 -> bn3 -> max runs as the fused tensor-core block (K10);
        # the [R][1024] pre-BN activation is never materialised.
        self.fuse_lbm = self.dt == H.HFTA_BF16 and self.c3 % 128 == 0 and self.c3 <= 1024 and self.c2 in (64, 128)
        # bf16: c1 -> bn1 -> relu and c2 -> bn2 -> relu run in Gram form (K11):
        # statistics from G = X^T X, BN apply in the GEMM epilogue, backward
        # without forming dY; the pre-BN y1 / y2 are never stored.
        self.fuse_bn = self.fuse_lbm and self.c1 in (64, 128) and self.c2 <= 128
        # feature transform (reading R30): STNkd on the c1 features, x' = a1 T2 per cloud
        self.ft, self.ft_weight = bool(feature_transform), float(ft_weight)
        self.pf_key = "feat.a1t" if self.ft else "feat.a1"        # the point feature c2 / the seg head consume
        self._alloc()

    # ------------------------------------------------------------ buffers --
    def _alloc(self):
        B, N, R = self.B, self.N, self.R
        c1, c2, c3, f1, f2 = self.c1, self.c2, self.c3, self.f1, self.f2
        a = _Acts(B, self.tdt, self.device)          # per-point tensors: dt
        f = _Acts(B, torch.float32, self.device)     # per-sample tensors: fp32 in both modes
        self.x_dt = torch.empty(R, 3, dtype=self.tdt, device=self.device)
        S = {}
        for p in ("stn", "feat") + (("fstn",) if self.ft else ()):
            kin = c1 if p == "fstn" else 3                              # input channels of the block's c1
            if self.fuse_bn:
                S[p + ".a1"], S[p + ".a2"] = a(R, c1), a(R, c2)
                S[p + ".G1"], S[p + ".s1"] = f(kin, kin), f(1, kin)    # Gram / column sums of the layer inputs
                S[p + ".G2"], S[p + ".s2"] = f(c1, c1), f(1, c1)
            else:
                S[p + ".y1"], S[p + ".a1"] = a(R, c1), a(R, c1)
                S[p + ".y2"], S[p + ".a2"] = a(R, c2), a(R, c2)
            if self.fuse_lbm:
                S[p + ".ext"] = f(N, c3)            # Y at the argmax rows (the block's saved tensor)
                S[p + ".G3"], S[p + ".s3"] = f(c2, c2), f(1, c2)     # Gram / column sums of the c3 input
            else:
                S[p + ".y3"] = a(R, c3)
            S[p + ".g"] = f(N, c3)
            S[p + ".amax"] = torch.empty(B, N, c3, dtype=torch.int32, device=self.device)
        S["stn.f1"], S["stn.h4"] = f(N, f1), f(N, f1)
        S["stn.f2"], S["stn.h5"] = f(N, f2), f(N, f2)
        S["stn.f3"] = f(N, 9)
        S["feat.xt"] = a(R, 3)
        if self.ft:
            S["fstn.f1"], S["fstn.h4"] = f(N, f1), f(N, f1)
            S["fstn.f2"], S["fstn.h5"] = f(N, f2), f(N, f2)
            S["fstn.f3"], S["d.ff3"] = f(N, c1 * c1), f(N, c1 * c1)
            S["ft.Tt"] = a(N * c1, c1)                  # (T2 + I)^T per cloud: [B][N][c1][c1]
            S["ft.dTt"] = f(N * c1, c1)
            S["feat.a1t"] = a(R, c1)                    # x' = a1 T2
            S["d.a1p"], S["d.a1q"] = a(R, c1), a(R, c1)
        if self.task == "cls":
            S["head.y1"], S["head.h1"] = f(N, f1), f(N, f1)
            S["head.y2"], S["head.d2"], S["head.h2"] = f(N, f2), f(N, f2), f(N, f2)
            S["head.logits"] = f(N, self.k)
            S["d.logits"] = f(N, self.k)
            S["d.f2a"], S["d.f2b"] = f(N, f2), f(N, f2)
            S["d.f1a"], S["d.f1b"] = f(N, f1), f(N, f1)
        if self.task == "seg":
            sh = self.arena.shape
            h1, h2, h3 = sh["head.c1.W"][0], sh["head.c2.W"][0], sh["head.c3.W"][0]
            self.h1w, self.h2w, self.h3w = h1, h2, h3
            kpad = (self.k + 15) // 16 * 16          # logits ld: 16-element aligned rows
            S["seg.u"] = f(N, h1)                   # g Wg^T + b: per-sample bias table of the split weight
            S["seg.y1"], S["seg.h1"] = a(R, h1), a(R, h1)
            # BN statistics from the head GEMMs' epilogues (bf16; HFTA_SEG_COLSTAT=0 disables)
            self._colstat = (torch.empty(H.hfta_linear_colstat_size(B, R, max(h1, h2, h3)) // 4, dtype=torch.float32,
                                         device=self.device)
                             if self.dt == H.HFTA_BF16 and os.environ.get("HFTA_SEG_COLSTAT", "1") != "0" else None)
            S["seg.y2"], S["seg.h2"] = a(R, h2), a(R, h2)
            S["seg.y3"], S["seg.h3"] = a(R, h3), a(R, h3)
            S["seg.logits"], S["d.logits"] = a(R, kpad), a(R, kpad)
            S["d.s1a"], S["d.s1b"] = a(R, h1), a(R, h1)
            S["d.s2a"], S["d.s2b"] = a(R, h2), a(R, h2)
            S["d.s3a"], S["d.s3b"] = a(R, h3), a(R, h3)
            S["seg.S"] = f(N, h1)                   # per-sample row sums of dy1
            S["d.pf"] = a(R, c1)                    # gradient reaching the point feature from the head
        if not self.fuse_lbm:
            S["d.big"] = a(R, c3)
        if self.fuse_bn:
            S["d.c2a"], S["d.c1a"] = a(R, c2), a(R, c1)
        else:
            S["d.c2a"], S["d.c2b"] = a(R, c2), a(R, c2)
            S["d.c1a"], S["d.c1b"] = a(R, c1), a(R, c1)
        S["d.g"] = f(N, c3)
        S["d.xt"] = a(R, 3)
        S["d.f3"] = f(N, 9)
        S["d.sf1a"], S["d.sf1b"] = f(N, f1), f(N, f1)
        S["d.sf2a"], S["d.sf2b"] = f(N, f2), f(N, f2)
        self.S = S
        self.loss = torch.zeros(B, dtype=torch.float32, device=self.device)
        self.mean_loss = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.labels = torch.zeros(N if self.task == "cls" else R, dtype=torch.int32, device=self.device)
        ws = Workspace(self.device)
        for (M, Nn, K) in [(R, c1, 3), (R, c2, c1), (R, c3, c2), (N, f1, c3), (N, f2, f1), (N, 9, f2),
                           (N, self.k, f2)]:
            for dt in (self.dt, H.HFTA_F32):
                ws.reserve(H.hfta_fused_linear_bwd_workspace(B, M, Nn, K, dt))
        for (Rr, Cc) in [(R, c1), (R, c2), (R, c3), (N, f1), (N, f2)]:
            ws.reserve(H.hfta_fused_bn_workspace(B, Rr, Cc))
        ws.reserve(H.hfta_bn_max_bwd_workspace(B, N, c3))
        if self.fuse_lbm:
            ws.reserve(H.hfta_fused_linear_bn_max_workspace(B, N, self.L, c3, c2))
        if self.fuse_bn:
            ws.reserve(H.hfta_fused_linear_bn_workspace(B, R, c1, 3))
            ws.reserve(H.hfta_fused_linear_bn_workspace(B, R, c2, c1))
            ws.reserve(H.hfta_fused_linear_bn_workspace(B, R, c1, c1))
        if self.ft:
            for dt in (self.dt, H.HFTA_F32):
                ws.reserve(H.hfta_fused_linear_bwd_workspace(B * N, self.L, c1, c1, dt))
                ws.reserve(H.hfta_fused_linear_bwd_workspace(B, N, c1 * c1, f2, dt))
                ws.reserve(H.hfta_fused_linear_bwd_workspace(B, R, c1, c1, dt))
            ws.reserve(H.hfta_feature_transform_reg_workspace(B, N))
        if self.task == "seg":
            for (M, Nn, K) in [(R, self.h1w, c1), (N, self.h1w, c3), (R, self.h2w, self.h1w), (R, self.h3w, self.h2w),
                               (R, self.k, self.h3w)]:
                for dt in (self.dt, H.HFTA_F32):
                    ws.reserve(H.hfta_fused_linear_bwd_workspace(B, M, Nn, K, dt))
            for Cc in (self.h1w, self.h2w, self.h3w):
                ws.reserve(H.hfta_fused_bn_workspace(B, R, Cc))
            ws.reserve(H.hfta_colsum_workspace(B, R, self.h1w, self.L))
        ws.reserve(H.hfta_loss_workspace(B, N if self.task == "cls" else R))
        ws.alloc()
        self.ws = ws

    # -------------------------------------------------------------- step --
    def probe_roofline(self, name, ms, peaks, path="simt"):
        """Roofline of the fused c3 block (K10), timed as ONE block (Gram,
        sign flip, k_lbm_fwd, statistics, pooled outputs: the call the C ABI
        exposes; k_lbm_fwd's own share comes from the ncu launch list).
        Algorithmic work = the method's contraction only (2 B R C K flops in
        forward; dgrad + wgrad = 2x that in backward) -- the Gram X^T X the
        Gram-form statistics add is NOT counted.  Arithmetic intensity ~C
        flop/B >> the ridge: tensor-bound against the sustained bf16 peak."""
        layer, kind = name.split(":")
        if not (self.fuse_lbm and layer.endswith(".c3")):
            return super().probe_roofline(name, ms, peaks, path)
        B, R, C, K, N = self.B, self.R, self.c3, self.c2, self.N
        if kind == "fwd":
            flops = 2.0 * B * R * C * K
            nbytes = B * (R * K * 2 + C * K * 2 + N * C * 12 + C * 16)
        else:
            flops = 2.0 * 2.0 * B * R * C * K
            nbytes = B * (2 * R * K * 2 + C * K * 2 + C * K * 4 + N * C * 12 + C * 16)
        t = float(np.mean(ms)) / 1e3 if ms else float("nan")
        ach = flops / t / 1e12
        return {"bound": "tensor", "achieved": ach, "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                "frac": ach / peaks["bf16_tflops_sustained"], "traffic": None,
                "kernel": name + " (fused c3->bn3->max block: 5 launches timed together)",
                "launches_timed": len(ms), "ms_per_launch": t * 1e3,
                "algorithmic": {"flops": flops, "bytes": nbytes, "note": "method flops 2BRCK (Gram term excluded)"},
                "peak_source": peaks["source"]}

    def _block_fwd(self, p, act, s):
        """c3 -> bn3 -> act -> max over points (STN: ReLU, feat: none)."""
        S, R = self.S, self.R
        if not self.fuse_lbm:
            self._lin_fwd(_in(S[p + ".a2"]), R, p + ".c3", S[p + ".y3"], s)
            self._bn_fwd(S[p + ".y3"], p + ".bn3", act, None, s)
            self._bn_max_fwd(S[p + ".y3"], p + ".bn3", act, S[p + ".g"], S[p + ".amax"], s)
            return
        ar, P, bn = self.arena, self.arena.P, p + ".bn3"
        rm, rv = self.running[bn]
        sm, si = self.saved[bn]
        e0 = self._pbegin(p + ".c3:fwd", s)
        H.hfta_fused_linear_bn_max_fwd(self.B, self.N, self.L, self.c3, self.c2, self.dt, _in(S[p + ".a2"]),
                                       ar.w_in(p + ".c3.W", self.dt), ar.fptr("p", p + ".c3.b"), P,
                                       ar.fptr("p", bn + ".g"), ar.fptr("p", bn + ".beta"), P, H.ptr(rm), H.ptr(rv),
                                       0.1, 1e-5, act, self.act_alpha, _out(S[p + ".g"]), H.ptr(S[p + ".amax"]),
                                       _out(S[p + ".ext"]), H.ptr(sm), H.ptr(si), H.ptr(S[p + ".G3"]),
                                       H.ptr(S[p + ".s3"]), self.ws.ptr, self.ws.nbytes, s)
        self._pend(e0)

    def _block_bwd(self, p, act, s, dx_act=A_NONE):
        """Backward of _block_fwd from d.g; writes d.c2a (grad of a2, times act'(a2) when dx_act is
        set, i.e. the c2 layer's dZ) and the c3/bn3 gradients."""
        S, R = self.S, self.R
        if not self.fuse_lbm:
            self._bn_max_bwd(S["d.g"], S[p + ".y3"], S[p + ".amax"], p + ".bn3", act, S["d.big"], s)
            self._lin_bwd(S["d.big"], _in(S[p + ".a2"]), R, p + ".c3", S["d.c2a"], s)
            return
        ar, P, bn = self.arena, self.arena.P, p + ".bn3"
        sm, si = self.saved[bn]
        e0 = self._pbegin(p + ".c3:bwd", s)
        H.hfta_fused_linear_bn_max_bwd(self.B, self.N, self.L, self.c3, self.c2, self.dt, _in(S["d.g"]),
                                       _in(S[p + ".a2"]), ar.w_in(p + ".c3.W", self.dt), H.ptr(S[p + ".amax"]),
                                       _in(S[p + ".ext"]), ar.fptr("p", p + ".c3.b"), P, ar.fptr("p", bn + ".g"),
                                       ar.fptr("p", bn + ".beta"), P, H.ptr(sm), H.ptr(si), H.ptr(S[p + ".G3"]),
                                       H.ptr(S[p + ".s3"]), act, self.act_alpha,
                                       _out(S["d.c2a"]), dx_act, self.act_alpha, ar.fptr("g", p + ".c3.W"), P, self.c2,
                                       ar.fptr("g", p + ".c3.b"), P, ar.fptr("g", bn + ".g"), ar.fptr("g", bn + ".beta"),
                                       0, self.ws.ptr, self.ws.nbytes, s)
        self._pend(e0)

    def _lbn_fwd(self, p, i, X, K, s):
        """Fused c{i} -> bn{i} -> relu of branch p (Gram form).  X: hfta_in of the layer input."""
        S, ar, P = self.S, self.arena, self.arena.P
        lin, bn = "%s.c%d" % (p, i), "%s.bn%d" % (p, i)
        Nn = self.arena.shape[lin + ".W"][0]
        rm, rv = self.running[bn]
        sm, si = self.saved[bn]
        H.hfta_fused_linear_bn_fwd(self.B, self.R, Nn, K, self.dt, X, ar.w_in(lin + ".W", self.dt),
                                   ar.fptr("p", lin + ".b"), P, ar.fptr("p", bn + ".g"), ar.fptr("p", bn + ".beta"), P,
                                   H.ptr(rm), H.ptr(rv), 0.1, 1e-5, A_RELU, self.act_alpha,
                                   _out(S["%s.a%d" % (p, i)]), H.ptr(sm), H.ptr(si), H.ptr(S["%s.G%d" % (p, i)]),
                                   H.ptr(S["%s.s%d" % (p, i)]), self.ws.ptr, self.ws.nbytes, s)

    def _lbn_bwd(self, p, i, dZ, X, K, dX, dx_act, s):
        """Backward of _lbn_fwd from dZ (gradient at bn{i}'s output, relu' applied)."""
        S, ar, P = self.S, self.arena, self.arena.P
        lin, bn = "%s.c%d" % (p, i), "%s.bn%d" % (p, i)
        Nn = self.arena.shape[lin + ".W"][0]
        sm, si = self.saved[bn]
        H.hfta_fused_linear_bn_bwd(self.B, self.R, Nn, K, self.dt, _in(dZ), X, ar.w_in(lin + ".W", self.dt),
                                   ar.fptr("p", lin + ".b"), P, ar.fptr("p", bn + ".g"), P, H.ptr(sm), H.ptr(si),
                                   H.ptr(S["%s.G%d" % (p, i)]), H.ptr(S["%s.s%d" % (p, i)]),
                                   _out(dX) if dX is not None else H.tout(None, 0, 1), dx_act, self.act_alpha,
                                   ar.fptr("g", lin + ".W"), P, K, ar.fptr("g", lin + ".b"), P,
                                   ar.fptr("g", bn + ".g"), ar.fptr("g", bn + ".beta"), 0, self.ws.ptr,
                                   self.ws.nbytes, s)

    def _stn_feat_fwd_fused(self, x, s):
        S = self.S
        self._lbn_fwd("stn", 1, H.tin(self.x_dt, 0, 3), 3, s)
        self._lbn_fwd("stn", 2, _in(S["stn.a1"]), self.c1, s)
        self._block_fwd("stn", A_RELU, s)
        self._stn_head_fwd(s)
        H.hfta_transform_points_fwd(self.B, self.N, self.L, self.dt, H.tin(x, 0, 3), _in(S["stn.f3"]), 1,
                                    _out(S["feat.xt"]), s)
        self._lbn_fwd("feat", 1, _in(S["feat.xt"]), 3, s)
        if self.ft:
            self._lbn_fwd("fstn", 1, _in(S["feat.a1"]), self.c1, s)
            self._lbn_fwd("fstn", 2, _in(S["fstn.a1"]), self.c1, s)
            self._block_fwd("fstn", A_RELU, s)
            self._stn_head_fwd(s, "fstn")
            self._ft_apply(s)
        self._lbn_fwd("feat", 2, _in(S[self.pf_key]), self.c1, s)
        self._block_fwd("feat", A_NONE, s)

    def _stn_feat_bwd_fused(self, x, s):
        S, R, N = self.S, self.R, self.N
        seg = self.task == "seg"
        # feat: K10 bwd -> dZ2 (gated by relu'(a2)); c2 -> dZ1 (gated by relu'(a1), after the
        # seg head's gradient is added for seg); c1 -> d xt
        self._block_bwd("feat", A_NONE, s, dx_act=A_RELU)
        gate_now = not seg and not self.ft        # the c2 input is a1 itself (a ReLU output): gate in the GEMM
        self._lbn_bwd("feat", 2, S["d.c2a"], _in(S[self.pf_key]), self.c1, S["d.c1a"], A_RELU if gate_now else A_NONE,
                      s)
        if seg:      # the point feature also feeds the seg head: add its gradient
            H.hfta_add(self.B, R, self.c1, self.dt, _in(S["d.c1a"]), _in(S["d.pf"]), _out(S["d.c1a"]), s)
        if self.ft:  # back through x' = a1 T2 (+ regularizer) and STNkd(a1): d.c1a = d(a1), not yet gated
            self._ft_bwd(s, fused=True)
        if not gate_now:
            H.hfta_act_bwd(self.B, R, self.c1, self.dt, A_RELU, self.act_alpha, _in(S["feat.a1"]), _in(S["d.c1a"]),
                           _out(S["d.c1a"]), s)
        self._lbn_bwd("feat", 1, S["d.c1a"], _in(S["feat.xt"]), 3, S["d.xt"], A_NONE, s)
        H.hfta_transform_points_bwd(self.B, N, self.L, self.dt, H.tin(x, 0, 3), _in(S["d.xt"]), _out(S["d.f3"]), s)
        self._stn_head_bwd(s)
        self._block_bwd("stn", A_RELU, s, dx_act=A_RELU)
        self._lbn_bwd("stn", 2, S["d.c2a"], _in(S["stn.a1"]), self.c1, S["d.c1a"], A_RELU, s)
        self._lbn_bwd("stn", 1, S["d.c1a"], H.tin(self.x_dt, 0, 3), 3, None, A_NONE, s)

    def _stn_head_fwd(self, s, p="stn"):
        S = self.S
        self._lin_fwd(_in(S[p + ".g"]), self.N, p + ".fc1", S[p + ".f1"], s)
        self._bn_fwd(S[p + ".f1"], p + ".bn4", A_RELU, S[p + ".h4"], s)
        self._lin_fwd(_in(S[p + ".h4"]), self.N, p + ".fc2", S[p + ".f2"], s)
        self._bn_fwd(S[p + ".f2"], p + ".bn5", A_RELU, S[p + ".h5"], s)
        self._lin_fwd(_in(S[p + ".h5"]), self.N, p + ".fc3", S[p + ".f3"], s)

    def _stn_head_bwd(self, s, p="stn"):
        """From d(f3) (S["d.f3"] / S["d.ff3"]) to the pooled feature's gradient S["d.g"]."""
        S, N = self.S, self.N
        self._lin_bwd(S["d.f3" if p == "stn" else "d.ff3"], _in(S[p + ".h5"]), N, p + ".fc3", S["d.sf2a"], s)
        self._bn_bwd(S["d.sf2a"], S[p + ".f2"], p + ".bn5", A_RELU, S["d.sf2b"], s)
        self._lin_bwd(S["d.sf2b"], _in(S[p + ".h4"]), N, p + ".fc2", S["d.sf1a"], s)
        self._bn_bwd(S["d.sf1a"], S[p + ".f1"], p + ".bn4", A_RELU, S["d.sf1b"], s)
        self._lin_bwd(S["d.sf1b"], _in(S[p + ".g"]), N, p + ".fc1", S["d.g"], s)

    # ------------------------------------------------ feature transform --
    def _ft_views(self):
        """The per-cloud operands as B*N fused 'models': a1 / x' [B*N][L][c1], Tt [B*N][c1][c1]."""
        S, L, c1 = self.S, self.L, self.c1
        return (H.tin(S["feat.a1"], L * c1, c1), H.tin(S["ft.Tt"], c1 * c1, c1), H.tout(S["feat.a1t"], L * c1, c1))

    def _ft_apply(self, s):
        """T2 = STNkd fc3 + I (transposed, compute dtype) and x' = a1 T2 per cloud (reading R30)."""
        S, N, c1 = self.S, self.N, self.c1
        H.hfta_feature_transform_make(self.B, N, c1, self.dt, H.ptr(S["fstn.f3"]), N * c1 * c1,
                                      H.tout(S["ft.Tt"], N * c1 * c1, c1), s)
        a1, Tt, a1t = self._ft_views()
        H.hfta_fused_linear_fwd(self.B * N, self.L, c1, c1, self.dt, a1, Tt, None, 0, 0, 0, a1t, s)

    def _ft_bwd(self, s, fused):
        """d.c1a holds d(x'); leaves d(a1) (ungated) in d.c1a: the transform's dgrad + STNkd's input
        gradient; adds the regularizer to loss[b]."""
        S, N, R, c1 = self.S, self.N, self.R, self.c1
        a1, Tt, _ = self._ft_views()
        H.hfta_fused_linear_bwd(self.B * N, self.L, c1, c1, self.dt, H.tin(S["d.c1a"], self.L * c1, c1), a1, Tt,
                                H.tout(S["d.a1p"], self.L * c1, c1), H.ptr(S["ft.dTt"]), c1 * c1, c1, None, 0, 0,
                                self.ws.ptr, self.ws.nbytes, s)
        H.hfta_feature_transform_reg(self.B, N, c1, H.ptr(S["fstn.f3"]), N * c1 * c1, H.ptr(S["ft.dTt"]), N * c1 * c1,
                                     self.ft_weight, H.ptr(S["d.ff3"]), N * c1 * c1, H.ptr(self.loss),
                                     H.ptr(self.mean_loss), self.ws.ptr, self.ws.nbytes, s)
        self._stn_head_bwd(s, "fstn")
        if fused:
            self._block_bwd("fstn", A_RELU, s, dx_act=A_RELU)
            self._lbn_bwd("fstn", 2, S["d.c2a"], _in(S["fstn.a1"]), self.c1, S["d.a1q"], A_RELU, s)
            self._lbn_bwd("fstn", 1, S["d.a1q"], _in(S["feat.a1"]), self.c1, S["d.c1a"], A_NONE, s)
        else:
            self._block_bwd("fstn", A_RELU, s)
            self._bn_bwd(S["d.c2a"], S["fstn.y2"], "fstn.bn2", A_RELU, S["d.c2b"], s)
            self._lin_bwd(S["d.c2b"], _in(S["fstn.a1"]), R, "fstn.c2", S["d.a1q"], s)
            self._bn_bwd(S["d.a1q"], S["fstn.y1"], "fstn.bn1", A_RELU, S["d.c1b"], s)
            self._lin_bwd(S["d.c1b"], _in(S["feat.a1"]), R, "fstn.c1", S["d.c1a"], s)
        H.hfta_add(self.B, R, c1, self.dt, _in(S["d.c1a"]), _in(S["d.a1p"]), _out(S["d.c1a"]), s)

    def _stn_feat_fwd(self, x, s):
        S, R = self.S, self.R
        xin = H.tin(self.x_dt, 0, 3)
        # STN3d
        self._lin_fwd(xin, R, "stn.c1", S["stn.y1"], s)
        self._bn_fwd(S["stn.y1"], "stn.bn1", A_RELU, S["stn.a1"], s)
        self._lin_fwd(_in(S["stn.a1"]), R, "stn.c2", S["stn.y2"], s)
        self._bn_fwd(S["stn.y2"], "stn.bn2", A_RELU, S["stn.a2"], s)
        self._block_fwd("stn", A_RELU, s)
        self._lin_fwd(_in(S["stn.g"]), self.N, "stn.fc1", S["stn.f1"], s)
        self._bn_fwd(S["stn.f1"], "stn.bn4", A_RELU, S["stn.h4"], s)
        self._lin_fwd(_in(S["stn.h4"]), self.N, "stn.fc2", S["stn.f2"], s)
        self._bn_fwd(S["stn.f2"], "stn.bn5", A_RELU, S["stn.h5"], s)
        self._lin_fwd(_in(S["stn.h5"]), self.N, "stn.fc3", S["stn.f3"], s)
        # PointNetfeat: x' = x T, T = f3 + I
        H.hfta_transform_points_fwd(self.B, self.N, self.L, self.dt, H.tin(x, 0, 3), _in(S["stn.f3"]), 1,
                                    _out(S["feat.xt"]), s)
        self._lin_fwd(_in(S["feat.xt"]), R, "feat.c1", S["feat.y1"], s)
        self._bn_fwd(S["feat.y1"], "feat.bn1", A_RELU, S["feat.a1"], s)
        if self.ft:
            self._lin_fwd(_in(S["feat.a1"]), R, "fstn.c1", S["fstn.y1"], s)
            self._bn_fwd(S["fstn.y1"], "fstn.bn1", A_RELU, S["fstn.a1"], s)
            self._lin_fwd(_in(S["fstn.a1"]), R, "fstn.c2", S["fstn.y2"], s)
            self._bn_fwd(S["fstn.y2"], "fstn.bn2", A_RELU, S["fstn.a2"], s)
            self._block_fwd("fstn", A_RELU, s)
            self._stn_head_fwd(s, "fstn")
            self._ft_apply(s)
        self._lin_fwd(_in(S[self.pf_key]), R, "feat.c2", S["feat.y2"], s)
        self._bn_fwd(S["feat.y2"], "feat.bn2", A_RELU, S["feat.a2"], s)
        self._block_fwd("feat", A_NONE, s)

    def _stn_feat_bwd(self, x, s):
        S, R, N = self.S, self.R, self.N
        # feat
        self._block_bwd("feat", A_NONE, s)
        self._bn_bwd(S["d.c2a"], S["feat.y2"], "feat.bn2", A_RELU, S["d.c2b"], s)
        self._lin_bwd(S["d.c2b"], _in(S[self.pf_key]), R, "feat.c2", S["d.c1a"], s)
        if self.task == "seg":      # the point feature also feeds the seg head
            H.hfta_add(self.B, R, self.c1, self.dt, _in(S["d.c1a"]), _in(S["d.pf"]), _out(S["d.c1a"]), s)
        if self.ft:
            self._ft_bwd(s, fused=False)
        self._bn_bwd(S["d.c1a"], S["feat.y1"], "feat.bn1", A_RELU, S["d.c1b"], s)
        self._lin_bwd(S["d.c1b"], _in(S["feat.xt"]), R, "feat.c1", S["d.xt"], s)
        H.hfta_transform_points_bwd(self.B, N, self.L, self.dt, H.tin(x, 0, 3), _in(S["d.xt"]), _out(S["d.f3"]), s)
        # STN
        self._lin_bwd(S["d.f3"], _in(S["stn.h5"]), N, "stn.fc3", S["d.sf2a"], s)
        self._bn_bwd(S["d.sf2a"], S["stn.f2"], "stn.bn5", A_RELU, S["d.sf2b"], s)
        self._lin_bwd(S["d.sf2b"], _in(S["stn.h4"]), N, "stn.fc2", S["d.sf1a"], s)
        self._bn_bwd(S["d.sf1a"], S["stn.f1"], "stn.bn4", A_RELU, S["d.sf1b"], s)
        self._lin_bwd(S["d.sf1b"], _in(S["stn.g"]), N, "stn.fc1", S["d.g"], s)
        self._block_bwd("stn", A_RELU, s)
        self._bn_bwd(S["d.c2a"], S["stn.y2"], "stn.bn2", A_RELU, S["d.c2b"], s)
        self._lin_bwd(S["d.c2b"], _in(S["stn.a1"]), R, "stn.c2", S["d.c1a"], s)
        self._bn_bwd(S["d.c1a"], S["stn.y1"], "stn.bn1", A_RELU, S["d.c1b"], s)
        self._lin_bwd(S["d.c1b"], H.tin(self.x_dt, 0, 3), R, "stn.c1", None, s)

    def _cls_head(self, s):
        S, N = self.S, self.N
        self._lin_fwd(_in(S["feat.g"]), N, "head.fc1", S["head.y1"], s)
        self._bn_fwd(S["head.y1"], "head.bn1", A_RELU, S["head.h1"], s)
        self._lin_fwd(_in(S["head.h1"]), N, "head.fc2", S["head.y2"], s)
        # the Philox step comes from the device step counter (+1: it is advanced by the
        # optimizer at the end of the step), so a captured CUDA graph replays correctly
        H.hfta_dropout_fwd(self.B, N, self.f2, H.HFTA_F32, _in(S["head.y2"]), _out(S["head.d2"]), self.dropout_seed,
                           1, H.ptr(self.hv.step), 0, self.p_drop, self.model_offset, H.ptr(self.model_ids), s)
        self._bn_fwd(S["head.d2"], "head.bn2", A_RELU, S["head.h2"], s)
        self._lin_fwd(_in(S["head.h2"]), N, "head.fc3", S["head.logits"], s)
        H.hfta_loss_nll(self.B, N, self.k, H.HFTA_F32, _in(S["head.logits"]), H.ptr(self.labels), 0, H.ptr(self.loss),
                        H.ptr(self.mean_loss), _out(S["d.logits"]), self.ws.ptr, self.ws.nbytes, s)
        self._lin_bwd(S["d.logits"], _in(S["head.h2"]), N, "head.fc3", S["d.f2a"], s)
        self._bn_bwd(S["d.f2a"], S["head.d2"], "head.bn2", A_RELU, S["d.f2b"], s)
        H.hfta_dropout_bwd(self.B, N, self.f2, H.HFTA_F32, _in(S["d.f2b"]), _out(S["d.f2a"]), self.dropout_seed,
                           1, H.ptr(self.hv.step), 0, self.p_drop, self.model_offset, H.ptr(self.model_ids), s)
        self._lin_bwd(S["d.f2a"], _in(S["head.h1"]), N, "head.fc2", S["d.f1a"], s)
        self._bn_bwd(S["d.f1a"], S["head.y1"], "head.bn1", A_RELU, S["d.f1b"], s)
        self._lin_bwd(S["d.f1b"], _in(S["feat.g"]), N, "head.fc1", S["d.g"], s)

    def _seg_head(self, s):
        """PointNetDenseCls head.  Its first layer acts on concat(g repeated over
        the L points, pointfeat) (1088 wide); it is computed with the exact
        split-weight rewrite y1[n*L+l] = (g[n] Wg^T + b) + pf[n*L+l] Wp^T, the
        per-sample part entering the point GEMM as a row-grouped bias table
        (DESIGN.md), so the [R][1088] concat is never materialised."""
        S, N, R, L, B = self.S, self.N, self.R, self.L, self.B
        c1, c3, h1 = self.c1, self.c3, self.h1w
        ar, P = self.arena, self.arena.P
        wld = c3 + c1
        H.hfta_fused_linear_fwd(B, N, h1, c3, H.HFTA_F32, _in(S["feat.g"]), ar.w_in("head.c1.W", H.HFTA_F32, 0, wld),
                                ar.fptr("p", "head.c1.b"), P, 0, 0, _out(S["seg.u"]), s)
        if self._colstat is not None:
            # bf16: each head GEMM's epilogue writes the BN statistics of the y it stores
            # (hfta_fused_linear_fwd_stats), so BN skips its statistics pass over y
            cs = H.ptr(self._colstat)
            H.hfta_fused_linear_fwd_stats(B, R, h1, c1, _in(S[self.pf_key]), ar.w_in("head.c1.W", self.dt, c3, wld),
                                          H.ptr(S["seg.u"]), N * h1, h1, L, _out(S["seg.y1"]), cs, s)
            self._bn_fwd_colstat(S["seg.y1"], "head.bn1", A_RELU, S["seg.h1"], cs, s)
            for src, name, y, bn, h in (("seg.h1", "head.c2", "seg.y2", "head.bn2", "seg.h2"),
                                        ("seg.h2", "head.c3", "seg.y3", "head.bn3", "seg.h3")):
                Nn, K = ar.shape[name + ".W"]
                e0 = self._pbegin(name + ":fwd", s)
                H.hfta_fused_linear_fwd_stats(B, R, Nn, K, _in(S[src]), ar.w_in(name + ".W", self.dt),
                                              ar.fptr("p", name + ".b"), P, 0, 0, _out(S[y]), cs, s)
                self._pend(e0)
                self._bn_fwd_colstat(S[y], bn, A_RELU, S[h], cs, s)
        else:
            H.hfta_fused_linear_fwd(B, R, h1, c1, self.dt, _in(S[self.pf_key]),
                                    ar.w_in("head.c1.W", self.dt, c3, wld), H.ptr(S["seg.u"]), N * h1, h1, L,
                                    _out(S["seg.y1"]), s)
            self._bn_fwd(S["seg.y1"], "head.bn1", A_RELU, S["seg.h1"], s)
            self._lin_fwd(_in(S["seg.h1"]), R, "head.c2", S["seg.y2"], s)
            self._bn_fwd(S["seg.y2"], "head.bn2", A_RELU, S["seg.h2"], s)
            self._lin_fwd(_in(S["seg.h2"]), R, "head.c3", S["seg.y3"], s)
            self._bn_fwd(S["seg.y3"], "head.bn3", A_RELU, S["seg.h3"], s)
        lg, dl = S["seg.logits"], S["d.logits"]
        kp = lg.shape[2]
        H.hfta_fused_linear_fwd(B, R, self.k, self.h3w, self.dt, _in(S["seg.h3"]), ar.w_in("head.c4.W", self.dt),
                                ar.fptr("p", "head.c4.b"), P, 0, 0, H.tout(lg, R * kp, kp), s)
        H.hfta_loss_nll(B, R, self.k, self.dt, H.tin(lg, R * kp, kp), H.ptr(self.labels), 0, H.ptr(self.loss),
                        H.ptr(self.mean_loss), H.tout(dl, R * kp, kp), self.ws.ptr, self.ws.nbytes, s)
        # backward
        self._lin_bwd(dl, _in(S["seg.h3"]), R, "head.c4", S["d.s3a"], s)
        self._bn_bwd(S["d.s3a"], S["seg.y3"], "head.bn3", A_RELU, S["d.s3b"], s)
        self._lin_bwd(S["d.s3b"], _in(S["seg.h2"]), R, "head.c3", S["d.s2a"], s)
        self._bn_bwd(S["d.s2a"], S["seg.y2"], "head.bn2", A_RELU, S["d.s2b"], s)
        self._lin_bwd(S["d.s2b"], _in(S["seg.h1"]), R, "head.c2", S["d.s1a"], s)
        self._bn_bwd(S["d.s1a"], S["seg.y1"], "head.bn1", A_RELU, S["d.s1b"], s)
        dy1 = S["d.s1b"]
        # point part: dWp = dy1^T pf, d pf = dy1 Wp (bias grad identically 0: BN follows)
        H.hfta_fused_linear_bwd(B, R, h1, c1, self.dt, _in(dy1), _in(S[self.pf_key]),
                                ar.w_in("head.c1.W", self.dt, c3, wld), _out(S["d.pf"]),
                                ar.fptr("g", "head.c1.W", c3), P, wld, None, P, 0, self.ws.ptr, self.ws.nbytes, s)
        # per-sample part: S[n] = sum_l dy1[n*L+l]; dWg = S^T g; dg = S Wg
        H.hfta_colsum(B, R, h1, L, self.dt, _in(dy1), H.ptr(S["seg.S"]), N * h1, 0, self.ws.ptr, self.ws.nbytes, s)
        H.hfta_fused_linear_bwd(B, N, h1, c3, H.HFTA_F32, _in(S["seg.S"]), _in(S["feat.g"]),
                                ar.w_in("head.c1.W", H.HFTA_F32, 0, wld), _out(S["d.g"]),
                                ar.fptr("g", "head.c1.W", 0), P, wld, None, P, 0, self.ws.ptr, self.ws.nbytes, s)

    def set_batch(self, x, labels):
        """x: device fp32 [N*L, 3] (shared by all models); labels int32."""
        self.x = x
        self.labels.copy_(labels.reshape(-1).to(torch.int32))

    def forward_backward(self, stream=None):
        """Forward + backward; gradients land in arena.g (before the step)."""
        s = H.stream_ptr(stream)
        x = self.x
        if self.dt == H.HFTA_F32:
            self.x_dt = x
        else:
            H.hfta_cast_f32_bf16(self.R * 3, H.ptr(x), H.ptr(self.x_dt), s)
        fwd, bwd = ((self._stn_feat_fwd_fused, self._stn_feat_bwd_fused) if self.fuse_bn
                    else (self._stn_feat_fwd, self._stn_feat_bwd))
        fwd(x, s)
        if self.task == "cls":
            self._cls_head(s)
        else:
            self._seg_head(s)
        bwd(x, s)

    def step(self, x=None, labels=None, stream=None):
        """One fused training step for all B models; returns the loss vector [B]."""
        if x is not None:
            self.set_batch(x, labels)
        self.t += 1
        s = H.stream_ptr(stream)
        self.forward_backward(stream)
        self.adam(s)
        return self.loss
