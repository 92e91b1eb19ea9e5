"""Base of the fused-array step drivers: the parameter arena, hyper-vectors,
BN statistics and thin wrappers that marshal one fused layer into one C-ABI
call (`hfta.py`).  Every arithmetic step runs in libhfta's kernels; this
module only computes offsets, strides and shapes.
"""
import numpy as np
import torch

from . import hfta as H
from .fused import ParamArena, HyperVectors, Workspace, fused_adam

A_RELU, A_NONE, A_LEAKY = H.ACT_RELU, H.ACT_NONE, H.ACT_LEAKY_RELU


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



class FusedNet:
    """B fused models of one architecture (see subclasses)."""

    #: layers whose output feeds a training-mode BN (bias gradient identically 0)
    bn_followed = frozenset()

    def _base_init(self, B, param_specs, params, hp, dtype, device):
        self.B = B
        self.dt = H.HFTA_F32 if dtype == "f32" else H.HFTA_BF16
        self.tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        self.device = torch.device(device)
        self.arena = ParamArena(param_specs, B, self.device, bf16_shadow=(dtype != "f32"))
        self.arena.load(params)
        self.hv = HyperVectors(hp, self.device)
        self.t = 0
        sh = self.arena.shape
        self.bn_names = [n[:-2] for n, _ in param_specs if n.endswith(".g")]
        self.running = {n: (torch.zeros(B, sh[n + ".g"][0], dtype=torch.float32, device=self.device),
                            torch.ones(B, sh[n + ".g"][0], dtype=torch.float32, device=self.device)) for n in self.bn_names}
        self.saved = {n: (torch.empty(B, sh[n + ".g"][0], dtype=torch.float32, device=self.device),
                          torch.empty(B, sh[n + ".g"][0], dtype=torch.float32, device=self.device)) for n in self.bn_names}
        self.act_alpha = 0.0

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
        if path == "tf32x3":  # fp32 on the tensor cores: 3 tf32 MMAs per product, tf32 dense = 1/2 of bf16
            peak = peaks["bf16_tflops_sustained"] / 6.0
            ach = flops / t / 1e12
            ridge = peak * 1e12 / (peaks["hbm_gbs"] * 1e9)
            if flops / nbytes < ridge:
                ach_b = nbytes / t / 1e9
                return {"bound": "hbm", "achieved": ach_b, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": ach_b / peaks["hbm_gbs"], "traffic": None, "kernel": name + " (3xTF32)",
                        "launches_timed": len(ms), "ms_per_launch": t * 1e3,
                        "algorithmic": {"flops": flops, "bytes": nbytes}, "peak_source": peaks["source"]}
            return {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": None, "kernel": name + " (3xTF32)", "launches_timed": len(ms), "ms_per_launch": t * 1e3,
                    "algorithmic": {"flops": flops, "bytes": nbytes},
                    "peak_source": "sustained bf16 / 6 (tf32 = 1/2 bf16 rate, 3 MMAs per product); " + peaks["source"]}
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

    def _mixed(self, Y, M, Nn, K, X=None):
        """bf16-AMP contraction of an fp32-activation layer (reading R16b): in
        bf16 mode the per-sample FC layers keep fp32 activations but run
        their GEMMs on the tensor cores with bf16 operands (HFTA_BF16_F32)."""
        if self.dt != H.HFTA_BF16 or Y.dtype != torch.float32 or Nn < 16 or K < 16 or K % 8 or Nn % 8:
            return False
        return X is None or (X.bstride == M * K and X.ld == K)

    def _bf(self, key, rows, cols):
        """Persistent bf16 scratch (graph-capture safe: allocated on first use)."""
        if not hasattr(self, "_bf_bufs"):
            self._bf_bufs = {}
        t = self._bf_bufs.get(key)
        if t is None or t.shape[1] != rows or t.shape[2] != cols:
            t = torch.empty(self.B, rows, cols, dtype=torch.bfloat16, device=self.device)
            self._bf_bufs[key] = t
        return t

    def _lin_fwd(self, X, M, name, Y, s):
        Nn, K = self.arena.shape[name + ".W"]
        dt = self._dt(Y)
        e0 = self._pbegin(name + ":fwd", s)
        if self._mixed(Y, M, Nn, K, X):
            xb = self._bf(name + ".x", M, K)          # kept for the backward's wgrad
            H.hfta_cast_f32_bf16(self.B * M * K, X.ptr, H.ptr(xb), s)
            H.hfta_fused_linear_fwd(self.B, M, Nn, K, H.HFTA_BF16_F32, _in(xb), self.arena.w_in(name + ".W", H.HFTA_BF16),
                                    self.arena.fptr("p", name + ".b"), self.arena.P, 0, 0, _out(Y), s)
        else:
            H.hfta_fused_linear_fwd(self.B, M, Nn, K, dt, X, self.arena.w_in(name + ".W", dt),
                                    self.arena.fptr("p", name + ".b"), self.arena.P, 0, 0, _out(Y), s)
        self._pend(e0)

    def _lin_bwd(self, dY, X, M, name, dX, s, accumulate=0):
        Nn, K = self.arena.shape[name + ".W"]
        dt = self._dt(dY)
        e0 = self._pbegin(name + ":bwd", s)
        xb = getattr(self, "_bf_bufs", {}).get(name + ".x")
        if xb is not None and self._mixed(dY, M, Nn, K) and (dX is None or dX.dtype == torch.float32):
            dyb = self._bf("dy.%d.%d" % (M, Nn), M, Nn)
            H.hfta_cast_f32_bf16(self.B * M * Nn, H.ptr(dY), H.ptr(dyb), s)
            dt, dY_in, X = H.HFTA_BF16_F32, _in(dyb), _in(xb)
            w = self.arena.w_in(name + ".W", H.HFTA_BF16)
        else:
            dY_in, w = _in(dY), self.arena.w_in(name + ".W", dt)
        H.hfta_fused_linear_bwd(self.B, M, Nn, K, dt, dY_in, X, w,
                                _out(dX) if dX is not None else H.tout(None, 0, 1),
                                self.arena.fptr("g", name + ".W"), self.arena.P, K,
                                None if name in self.bn_followed else self.arena.fptr("g", name + ".b"), self.arena.P,
                                accumulate, self.ws.ptr, self.ws.nbytes, s)
        self._pend(e0)

    def _bn_fwd(self, X, name, act, Y, s):
        R, C = X.shape[1], X.shape[2]
        rm, rv = self.running[name]
        sm, si = self.saved[name]
        H.hfta_fused_bn_fwd(self.B, R, C, self._dt(X), _in(X), self.arena.fptr("p", name + ".g"),
                            self.arena.fptr("p", name + ".beta"), self.arena.P, H.ptr(rm), H.ptr(rv), 0.1, 1e-5,
                            act, self.act_alpha, _out(Y) if Y is not None else H.tout(None, 0, 1), H.ptr(sm), H.ptr(si),
                            self.ws.ptr, self.ws.nbytes, s)

    def _bn_fwd_colstat(self, X, name, act, Y, colstat, s):
        """BN forward whose statistics come from the producing GEMM's epilogue."""
        R, C = X.shape[1], X.shape[2]
        rm, rv = self.running[name]
        sm, si = self.saved[name]
        H.hfta_fused_bn_fwd_colstat(self.B, R, C, self._dt(X), _in(X), self.arena.fptr("p", name + ".g"),
                                    self.arena.fptr("p", name + ".beta"), self.arena.P, H.ptr(rm), H.ptr(rv), 0.1,
                                    1e-5, act, self.act_alpha, _out(Y), H.ptr(sm), H.ptr(si), colstat, s)

    def _bn_bwd(self, dY, X, name, act, dX, s):
        R, C = X.shape[1], X.shape[2]
        sm, si = self.saved[name]
        H.hfta_fused_bn_bwd(self.B, R, C, self._dt(X), _in(dY), _in(X), self.arena.fptr("p", name + ".g"),
                            self.arena.fptr("p", name + ".beta"), self.arena.P, H.ptr(sm), H.ptr(si), act, self.act_alpha,
                            _out(dX), self.arena.fptr("g", name + ".g"), self.arena.fptr("g", name + ".beta"), 0,
                            self.ws.ptr, self.ws.nbytes, s)

    def _bn_max_fwd(self, X, name, act, G, amax, s):
        sm, si = self.saved[name]
        H.hfta_bn_max_fwd(self.B, self.N, self.L, X.shape[2], self.dt, _in(X), self.arena.fptr("p", name + ".g"),
                          self.arena.fptr("p", name + ".beta"), self.arena.P, H.ptr(sm), H.ptr(si), act, self.act_alpha,
                          _out(G), H.ptr(amax), s)

    def _bn_max_bwd(self, dG, X, amax, name, act, dX, s):
        sm, si = self.saved[name]
        H.hfta_bn_max_bwd(self.B, self.N, self.L, X.shape[2], self.dt, _in(dG), _in(X), H.ptr(amax),
                          self.arena.fptr("p", name + ".g"), self.arena.fptr("p", name + ".beta"), self.arena.P,
                          H.ptr(sm), H.ptr(si), act, self.act_alpha, _out(dX), self.arena.fptr("g", name + ".g"),
                          self.arena.fptr("g", name + ".beta"), self.ws.ptr, self.ws.nbytes, s)

    def adam(self, s):
        H.hfta_step_increment(H.ptr(self.hv.step), s)
        fused_adam(self.arena, self.hv, s)

    # ------------------------------------------------------------ unfuse --
    def params(self, b):
        return {n: self.arena.host_tensor("p", n)[b] for n, _ in self.arena.specs}

    def grads(self, b):
        return {n: self.arena.host_tensor("g", n)[b] for n, _ in self.arena.specs}
