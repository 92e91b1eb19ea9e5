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
import numpy as np
import torch

from . import hfta as H
from .fused import ParamArena, HyperVectors, Workspace, fused_adam

A_RELU, A_NONE = H.ACT_RELU, H.ACT_NONE

# Layers whose output feeds a training-mode BatchNorm directly: the gradient
# of their bias is identically zero (BN's input gradient sums to zero over the
# rows: sum_r dx_r = gamma*invstd*(sum dz - dbeta - dgamma*sum(xhat)/R) = 0
# since sum(xhat) = 0), so the fused step writes exact zeros instead of
# reducing a rounding-noise column sum.
BN_FOLLOWED = {"stn.c1", "stn.c2", "stn.c3", "stn.fc1", "stn.fc2", "feat.c1", "feat.c2", "feat.c3",
               "head.fc1", "head.c1", "head.c2", "head.c3"}


class _Acts:
    def __init__(self, B, dtype, device):
        self.B, self.dtype, self.device = B, dtype, device

    def __call__(self, rows, cols, dtype=None):
        return torch.empty(self.B, rows, cols, dtype=dtype or self.dtype, device=self.device)


def _in(t):
    """hfta_in over a model-major [B][rows][cols] tensor."""
    return H.tin(t, t.shape[1] * t.shape[2], t.shape[2])


def _out(t):
    return H.tout(t, t.shape[1] * t.shape[2], t.shape[2])


class FusedPointNet:
    """B fused PointNet models (task 'cls' or 'seg')."""

    def __init__(self, B, param_specs, params, hp, task="cls", dtype="f32", N=32, L=2500, k=40,
                 p_drop=0.3, dropout_seed=42, device="cuda"):
        assert task in ("cls", "seg")
        self.B, self.task, self.N, self.L, self.k = B, task, N, L, k
        self.R = N * L
        self.dt = H.HFTA_F32 if dtype == "f32" else H.HFTA_BF16
        self.tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        self.p_drop, self.dropout_seed = p_drop, dropout_seed
        self.device = torch.device(device)
        self.arena = ParamArena(param_specs, B, self.device, bf16_shadow=(dtype != "f32"))
        self.arena.load(params)
        self.hv = HyperVectors(hp, self.device)
        self.t = 0
        sh = self.arena.shape
        self.c1, self.c2, self.c3 = sh["stn.c1.W"][0], sh["stn.c2.W"][0], sh["stn.c3.W"][0]
        self.f1, self.f2 = sh["stn.fc1.W"][0], sh["stn.fc2.W"][0]
        # BN running statistics and saved batch statistics, [B][C] fp32
        self.bn_names = [n[:-2] for n, _ in param_specs if n.endswith(".g")]
        self.running = {n: (torch.zeros(B, sh[n + ".g"][0], device=self.device),
                            torch.ones(B, sh[n + ".g"][0], device=self.device)) for n in self.bn_names}
        self.saved = {n: (torch.empty(B, sh[n + ".g"][0], device=self.device),
                          torch.empty(B, sh[n + ".g"][0], device=self.device)) for n in self.bn_names}
        self._alloc()

    # ------------------------------------------------------------ buffers --
    def _alloc(self):
        B, N, R = self.B, self.N, self.R
        c1, c2, c3, f1, f2 = self.c1, self.c2, self.c3, self.f1, self.f2
        a = _Acts(B, self.tdt, self.device)          # per-point tensors: dt
        f = _Acts(B, torch.float32, self.device)     # per-sample tensors: fp32 in both modes
        self.x_dt = torch.empty(R, 3, dtype=self.tdt, device=self.device)
        S = {}
        for p in ("stn", "feat"):
            S[p + ".y1"], S[p + ".a1"] = a(R, c1), a(R, c1)
            S[p + ".y2"], S[p + ".a2"] = a(R, c2), a(R, c2)
            S[p + ".y3"] = a(R, c3)
            S[p + ".g"] = f(N, c3)
            S[p + ".amax"] = torch.empty(B, N, c3, dtype=torch.int32, device=self.device)
        S["stn.f1"], S["stn.h4"] = f(N, f1), f(N, f1)
        S["stn.f2"], S["stn.h5"] = f(N, f2), f(N, f2)
        S["stn.f3"] = f(N, 9)
        S["feat.xt"] = a(R, 3)
        if self.task == "cls":
            S["head.y1"], S["head.h1"] = f(N, f1), f(N, f1)
            S["head.y2"], S["head.d2"], S["head.h2"] = f(N, f2), f(N, f2), f(N, f2)
            S["head.logits"] = f(N, self.k)
            S["d.logits"] = f(N, self.k)
            S["d.f2a"], S["d.f2b"] = f(N, f2), f(N, f2)
            S["d.f1a"], S["d.f1b"] = f(N, f1), f(N, f1)
        S["d.big"] = a(R, c3)
        S["d.c2a"], S["d.c2b"] = a(R, c2), a(R, c2)
        S["d.c1a"], S["d.c1b"] = a(R, c1), a(R, c1)
        S["d.g"] = f(N, c3)
        S["d.xt"] = a(R, 3)
        S["d.f3"] = f(N, 9)
        S["d.sf1a"], S["d.sf1b"] = f(N, f1), f(N, f1)
        S["d.sf2a"], S["d.sf2b"] = f(N, f2), f(N, f2)
        self.S = S
        self.loss = torch.zeros(B, device=self.device)
        self.mean_loss = torch.zeros(1, device=self.device)
        self.labels = torch.zeros(N if self.task == "cls" else R, dtype=torch.int32, device=self.device)
        ws = Workspace(self.device)
        for (M, Nn, K) in [(R, c1, 3), (R, c2, c1), (R, c3, c2), (N, f1, c3), (N, f2, f1), (N, 9, f2),
                           (N, self.k, f2)]:
            for dt in (self.dt, H.HFTA_F32):
                ws.reserve(H.hfta_fused_linear_bwd_workspace(B, M, Nn, K, dt))
        for (Rr, Cc) in [(R, c1), (R, c2), (R, c3), (N, f1), (N, f2)]:
            ws.reserve(H.hfta_fused_bn_workspace(B, Rr, Cc))
        ws.reserve(H.hfta_bn_max_bwd_workspace(B, N, c3))
        ws.reserve(H.hfta_loss_workspace(B, N if self.task == "cls" else R))
        ws.alloc()
        self.ws = ws

    # ------------------------------------------------------------- probe --
    # CUDA events around one named contraction inside the timed region (the
    # bench's roofline figure).  name = "<layer>:fwd" or "<layer>:bwd".
    _probe = None

    def probe_arm(self, name):
        self._probe = name
        self._probe_ev = []

    def _pbegin(self, tag, s):
        if self._probe != tag:
            return None
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        return e0

    def _pend(self, e0):
        if e0 is None:
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(torch.cuda.current_stream())
        self._probe_ev.append((e0, e1))

    def probe_collect(self):
        ms = [a.elapsed_time(b) for a, b in getattr(self, "_probe_ev", [])]
        self._probe = None
        return ms

    def probe_roofline(self, name, ms, peaks, path="simt"):
        """Algorithmic work of one launch of the probed contraction / its time."""
        layer, kind = name.split(":")
        Nn, K = self.arena.shape[layer + ".W"]
        M = self.R if (".c" in layer) else self.N
        s = 2 if self.dt == H.HFTA_BF16 and M == self.R else 4
        mult = 1 if kind == "fwd" else 2            # bwd = dgrad + wgrad
        flops = mult * 2.0 * self.B * M * Nn * K
        if kind == "fwd":
            nbytes = self.B * (M * K + Nn * K + M * Nn) * s
        else:   # dgrad reads dY, W, writes dX; wgrad reads dY, X, writes dW fp32
            nbytes = self.B * ((M * Nn + Nn * K + M * K) * s + (M * Nn + M * K) * s + Nn * K * 4)
        t = float(np.mean(ms)) / 1e3 if ms else float("nan")
        if path == "simt":   # FFMA-bound SIMT kernel: 148 SM x 128 FMA/clk x 2 flop x max clock
            peak = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12
            ach = flops / t / 1e12
            return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": None, "kernel": name, "launches_timed": len(ms), "ms_per_launch": t * 1e3,
                    "algorithmic": {"flops": flops, "bytes": nbytes},
                    "peak_source": "FFMA: 148 SM x 128 lanes x 2 flop x %.0f MHz" % peaks["sm_max_mhz"]}
        ridge = peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
        if flops / nbytes >= ridge:
            peak = peaks["bf16_tflops"] if self.dt == H.HFTA_BF16 else peaks["bf16_tflops"] / 4.0
            ach = flops / t / 1e12
            return {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": None, "kernel": name, "launches_timed": len(ms), "ms_per_launch": t * 1e3,
                    "algorithmic": {"flops": flops, "bytes": nbytes}, "peak_source": peaks["source"]}
        ach = nbytes / t / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": None, "kernel": name, "launches_timed": len(ms),
                "ms_per_launch": t * 1e3, "algorithmic": {"flops": flops, "bytes": nbytes},
                "peak_source": peaks["source"]}

    # ----------------------------------------------------------- wrappers --
    def _dt(self, t):
        return H.HFTA_F32 if t.dtype == torch.float32 else H.HFTA_BF16

    def _lin_fwd(self, X, M, name, Y, s):
        Nn, K = self.arena.shape[name + ".W"]
        dt = self._dt(Y)
        e0 = self._pbegin(name + ":fwd", s)
        H.hfta_fused_linear_fwd(self.B, M, Nn, K, dt, X, self.arena.w_in(name + ".W", dt),
                                self.arena.fptr("p", name + ".b"), self.arena.P, 0, 0, _out(Y), s)
        self._pend(e0)

    def _lin_bwd(self, dY, X, M, name, dX, s, accumulate=0):
        Nn, K = self.arena.shape[name + ".W"]
        dt = self._dt(dY)
        e0 = self._pbegin(name + ":bwd", s)
        H.hfta_fused_linear_bwd(self.B, M, Nn, K, dt, _in(dY), X, self.arena.w_in(name + ".W", dt),
                                _out(dX) if dX is not None else H.tout(None, 0, 1),
                                self.arena.fptr("g", name + ".W"), self.arena.P,
                                None if name in BN_FOLLOWED else self.arena.fptr("g", name + ".b"), self.arena.P,
                                accumulate, self.ws.ptr, self.ws.nbytes, s)
        self._pend(e0)

    def _bn_fwd(self, X, name, act, Y, s):
        R, C = X.shape[1], X.shape[2]
        rm, rv = self.running[name]
        sm, si = self.saved[name]
        H.hfta_fused_bn_fwd(self.B, R, C, self._dt(X), _in(X), self.arena.fptr("p", name + ".g"),
                            self.arena.fptr("p", name + ".beta"), self.arena.P, H.ptr(rm), H.ptr(rv), 0.1, 1e-5,
                            act, 0.0, _out(Y) if Y is not None else H.tout(None, 0, 1), H.ptr(sm), H.ptr(si),
                            self.ws.ptr, self.ws.nbytes, s)

    def _bn_bwd(self, dY, X, name, act, dX, s):
        R, C = X.shape[1], X.shape[2]
        sm, si = self.saved[name]
        H.hfta_fused_bn_bwd(self.B, R, C, self._dt(X), _in(dY), _in(X), self.arena.fptr("p", name + ".g"),
                            self.arena.fptr("p", name + ".beta"), self.arena.P, H.ptr(sm), H.ptr(si), act, 0.0,
                            _out(dX), self.arena.fptr("g", name + ".g"), self.arena.fptr("g", name + ".beta"), 0,
                            self.ws.ptr, self.ws.nbytes, s)

    def _bn_max_fwd(self, X, name, act, G, amax, s):
        sm, si = self.saved[name]
        H.hfta_bn_max_fwd(self.B, self.N, self.L, X.shape[2], self.dt, _in(X), self.arena.fptr("p", name + ".g"),
                          self.arena.fptr("p", name + ".beta"), self.arena.P, H.ptr(sm), H.ptr(si), act, 0.0,
                          _out(G), H.ptr(amax), s)

    def _bn_max_bwd(self, dG, X, amax, name, act, dX, s):
        sm, si = self.saved[name]
        H.hfta_bn_max_bwd(self.B, self.N, self.L, X.shape[2], self.dt, _in(dG), _in(X), H.ptr(amax),
                          self.arena.fptr("p", name + ".g"), self.arena.fptr("p", name + ".beta"), self.arena.P,
                          H.ptr(sm), H.ptr(si), act, 0.0, _out(dX), self.arena.fptr("g", name + ".g"),
                          self.arena.fptr("g", name + ".beta"), self.ws.ptr, self.ws.nbytes, s)

    # -------------------------------------------------------------- step --
    def _stn_feat_fwd(self, x, s):
        S, R = self.S, self.R
        xin = H.tin(self.x_dt, 0, 3)
        # STN3d
        self._lin_fwd(xin, R, "stn.c1", S["stn.y1"], s)
        self._bn_fwd(S["stn.y1"], "stn.bn1", A_RELU, S["stn.a1"], s)
        self._lin_fwd(_in(S["stn.a1"]), R, "stn.c2", S["stn.y2"], s)
        self._bn_fwd(S["stn.y2"], "stn.bn2", A_RELU, S["stn.a2"], s)
        self._lin_fwd(_in(S["stn.a2"]), R, "stn.c3", S["stn.y3"], s)
        self._bn_fwd(S["stn.y3"], "stn.bn3", A_RELU, None, s)
        self._bn_max_fwd(S["stn.y3"], "stn.bn3", A_RELU, S["stn.g"], S["stn.amax"], s)
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
        self._lin_fwd(_in(S["feat.a1"]), R, "feat.c2", S["feat.y2"], s)
        self._bn_fwd(S["feat.y2"], "feat.bn2", A_RELU, S["feat.a2"], s)
        self._lin_fwd(_in(S["feat.a2"]), R, "feat.c3", S["feat.y3"], s)
        self._bn_fwd(S["feat.y3"], "feat.bn3", A_NONE, None, s)
        self._bn_max_fwd(S["feat.y3"], "feat.bn3", A_NONE, S["feat.g"], S["feat.amax"], s)

    def _stn_feat_bwd(self, x, s):
        S, R, N = self.S, self.R, self.N
        # feat
        self._bn_max_bwd(S["d.g"], S["feat.y3"], S["feat.amax"], "feat.bn3", A_NONE, S["d.big"], s)
        self._lin_bwd(S["d.big"], _in(S["feat.a2"]), R, "feat.c3", S["d.c2a"], s)
        self._bn_bwd(S["d.c2a"], S["feat.y2"], "feat.bn2", A_RELU, S["d.c2b"], s)
        self._lin_bwd(S["d.c2b"], _in(S["feat.a1"]), R, "feat.c2", S["d.c1a"], s)
        self._bn_bwd(S["d.c1a"], S["feat.y1"], "feat.bn1", A_RELU, S["d.c1b"], s)
        self._lin_bwd(S["d.c1b"], _in(S["feat.xt"]), R, "feat.c1", S["d.xt"], s)
        H.hfta_transform_points_bwd(self.B, N, self.L, self.dt, H.tin(x, 0, 3), _in(S["d.xt"]), _out(S["d.f3"]), s)
        # STN
        self._lin_bwd(S["d.f3"], _in(S["stn.h5"]), N, "stn.fc3", S["d.sf2a"], s)
        self._bn_bwd(S["d.sf2a"], S["stn.f2"], "stn.bn5", A_RELU, S["d.sf2b"], s)
        self._lin_bwd(S["d.sf2b"], _in(S["stn.h4"]), N, "stn.fc2", S["d.sf1a"], s)
        self._bn_bwd(S["d.sf1a"], S["stn.f1"], "stn.bn4", A_RELU, S["d.sf1b"], s)
        self._lin_bwd(S["d.sf1b"], _in(S["stn.g"]), N, "stn.fc1", S["d.g"], s)
        self._bn_max_bwd(S["d.g"], S["stn.y3"], S["stn.amax"], "stn.bn3", A_RELU, S["d.big"], s)
        self._lin_bwd(S["d.big"], _in(S["stn.a2"]), R, "stn.c3", S["d.c2a"], s)
        self._bn_bwd(S["d.c2a"], S["stn.y2"], "stn.bn2", A_RELU, S["d.c2b"], s)
        self._lin_bwd(S["d.c2b"], _in(S["stn.a1"]), R, "stn.c2", S["d.c1a"], s)
        self._bn_bwd(S["d.c1a"], S["stn.y1"], "stn.bn1", A_RELU, S["d.c1b"], s)
        self._lin_bwd(S["d.c1b"], H.tin(self.x_dt, 0, 3), R, "stn.c1", None, s)

    def _cls_head(self, s):
        S, N = self.S, self.N
        self._lin_fwd(_in(S["feat.g"]), N, "head.fc1", S["head.y1"], s)
        self._bn_fwd(S["head.y1"], "head.bn1", A_RELU, S["head.h1"], s)
        self._lin_fwd(_in(S["head.h1"]), N, "head.fc2", S["head.y2"], s)
        H.hfta_dropout_fwd(self.B, N, self.f2, H.HFTA_F32, _in(S["head.y2"]), _out(S["head.d2"]), self.dropout_seed,
                           self.t, 0, self.p_drop, s)
        self._bn_fwd(S["head.d2"], "head.bn2", A_RELU, S["head.h2"], s)
        self._lin_fwd(_in(S["head.h2"]), N, "head.fc3", S["head.logits"], s)
        H.hfta_loss_nll(self.B, N, self.k, H.HFTA_F32, _in(S["head.logits"]), H.ptr(self.labels), 0, H.ptr(self.loss),
                        H.ptr(self.mean_loss), _out(S["d.logits"]), self.ws.ptr, self.ws.nbytes, s)
        self._lin_bwd(S["d.logits"], _in(S["head.h2"]), N, "head.fc3", S["d.f2a"], s)
        self._bn_bwd(S["d.f2a"], S["head.d2"], "head.bn2", A_RELU, S["d.f2b"], s)
        H.hfta_dropout_bwd(self.B, N, self.f2, H.HFTA_F32, _in(S["d.f2b"]), _out(S["d.f2a"]), self.dropout_seed,
                           self.t, 0, self.p_drop, s)
        self._lin_bwd(S["d.f2a"], _in(S["head.h1"]), N, "head.fc2", S["d.f1a"], s)
        self._bn_bwd(S["d.f1a"], S["head.y1"], "head.bn1", A_RELU, S["d.f1b"], s)
        self._lin_bwd(S["d.f1b"], _in(S["feat.g"]), N, "head.fc1", S["d.g"], s)

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
        self._stn_feat_fwd(x, s)
        if self.task == "cls":
            self._cls_head(s)
        else:
            raise NotImplementedError("seg head")
        self._stn_feat_bwd(x, s)

    def step(self, x=None, labels=None, stream=None):
        """One fused training step for all B models; returns the loss vector [B]."""
        if x is not None:
            self.set_batch(x, labels)
        self.t += 1
        s = H.stream_ptr(stream)
        self.forward_backward(stream)
        H.hfta_step_increment(H.ptr(self.hv.step), s)
        fused_adam(self.arena, self.hv, s)
        return self.loss

    # ------------------------------------------------------------ unfuse --
    def params(self, b):
        return {n: self.arena.host_tensor("p", n)[b] for n, _ in self.arena.specs}

    def grads(self, b):
        return {n: self.arena.host_tensor("g", n)[b] for n, _ in self.arena.specs}
