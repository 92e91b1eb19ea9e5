"""Fused DCGAN training iteration (BJ configs[3]; the DCGAN the paper
benchmarks, model of the cited PyTorch example, reading R1).

B generator/discriminator pairs with per-model hyper-parameters train as one
job: every (de)convolution, BatchNorm2d, activation and loss is one C-ABI call
for all B models.  The iteration follows the cited example (reading R4):
D(real) backward, D(fake.detach) backward accumulating into D's gradients,
Adam(D), D'(fake) backward into G (D's parameter gradients not needed),
Adam(G).  Layouts are NHWC per model; conv weights live in the arena permuted
to [Co][kh][kw][Ci] (Conv2d) / [kh][kw][Co][Ci] (ConvT2d); the generator input
channel count is padded 100 -> 104 and the image channels 3 -> 8 (16-B bf16
rows for TMA and 128-bit gathers); pad values and their weights are zero,
their gradients are exactly zero, so they stay zero.
"""
import numpy as np
import torch

from . import hfta as H
from .fused import ParamArena, HyperVectors, Workspace, fused_adam

NZ, NZP = 100, 104        # generator input channels, padded to 16-B bf16 rows
NC, NCP = 3, 8            # image channels (G output / D input), padded to 16-B bf16 rows
G_LAYERS = [(1, 0), (2, 1), (2, 1), (2, 1), (2, 1)]      # (stride, pad) of t1..t5 (ConvT, k=4)
D_LAYERS = [(2, 1), (2, 1), (2, 1), (2, 1), (1, 0)]      # c1..c5 (Conv, k=4)


def _pad(a, axis, n):
    if a.shape[axis] == n:
        return a
    w = [(0, 0)] * a.ndim
    w[axis] = (0, n - a.shape[axis])
    return np.pad(a, w)


def _to_gpu(name, a):
    """PyTorch layout -> arena layout."""
    if name.startswith("t") and name.endswith(".W"):     # ConvT [Ci][Co][kh][kw] -> [kh][kw][Co][Ci]
        g = np.transpose(a, (2, 3, 1, 0))
        if a.shape[0] == NZ:
            g = _pad(g, 3, NZP)
        if a.shape[1] == NC:
            g = _pad(g, 2, NCP)
        return g
    if name.startswith("c") and name.endswith(".W"):     # Conv [Co][Ci][kh][kw] -> [Co][kh][kw][Ci]
        g = np.transpose(a, (0, 2, 3, 1))
        if a.shape[1] == NC:
            g = _pad(g, 3, NCP)
        return g
    return a


def _to_torch(name, g):
    if name.startswith("t") and name.endswith(".W"):
        if g.shape[3] == NZP:
            g = g[..., :NZ]
        if name == "t5.W":
            g = g[:, :, :NC, :]
        return np.transpose(g, (3, 2, 0, 1))
    if name.startswith("c") and name.endswith(".W"):
        if name == "c1.W":
            g = g[..., :NC]
        return np.transpose(g, (0, 3, 1, 2))
    return g


class _Half:
    """One network (G or D) of the fused array: arena, BN buffers."""

    def __init__(self, B, specs, params, dtype, device):
        self.torch_specs = specs
        gspecs = [(n, _to_gpu(n, np.zeros(s)).shape) for n, s in specs]
        self.arena = ParamArena(gspecs, B, device, bf16_shadow=(dtype == "bf16"))
        self.arena.load([{n: _to_gpu(n, P[n]) for n, _ in specs} for P in params])
        sh = self.arena.shape
        self.bn = [n[:-2] for n, _ in specs if n.endswith(".g")]
        z = lambda c: torch.zeros(B, c, dtype=torch.float32, device=device)
        self.running = {n: (z(sh[n + ".g"][0]), torch.ones(B, sh[n + ".g"][0], dtype=torch.float32, device=device))
                        for n in self.bn}
        self.saved = {n: (z(sh[n + ".g"][0]), z(sh[n + ".g"][0])) for n in self.bn}

    def params(self, b):
        return {n: _to_torch(n, self.arena.host_tensor("p", n)[b]) for n, _ in self.torch_specs}

    def grads(self, b):
        return {n: _to_torch(n, self.arena.host_tensor("g", n)[b]) for n, _ in self.torch_specs}


class FusedDCGAN:
    def __init__(self, B, g_specs, d_specs, G_params, D_params, hp, N=128, dtype="bf16", device="cuda"):
        self.B, self.N = B, N
        self.dt = H.HFTA_F32 if dtype == "f32" else H.HFTA_BF16
        self.tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        self.device = torch.device(device)
        self.G = _Half(B, g_specs, G_params, dtype, self.device)
        self.D = _Half(B, d_specs, D_params, dtype, self.device)
        self.hvG = HyperVectors(hp, self.device)
        self.hvD = HyperVectors(hp, self.device)
        self.t = 0
        self._plan()

    # ------------------------------------------------------------ plan --
    def _desc(self, H_, C_in, C_out, stride, pad, transposed):
        d = H.hfta_conv_desc()
        d.N, d.H, d.W, d.C_in, d.C_out, d.kh, d.kw = self.N, H_, H_, C_in, C_out, 4, 4
        d.stride, d.pad, d.transposed = stride, pad, int(transposed)
        return d

    def _plan(self):
        B, N, dev = self.B, self.N, self.device
        a = lambda *shape: torch.empty((B,) + shape, dtype=self.tdt, device=dev)
        # generator: 1 -> 4 -> 8 -> 16 -> 32 -> 64, channels 104(100) -> 512 -> 256 -> 128 -> 64 -> 3
        gch = [NZP, 512, 256, 128, 64, NCP]
        gsz = [1, 4, 8, 16, 32, 64]
        self.gdesc = [self._desc(gsz[i], gch[i], gch[i + 1], *G_LAYERS[i], True) for i in range(5)]
        self.gch, self.gsz = gch, gsz
        self.z = a(N, NZP)
        self.gy = [a(N, gsz[i + 1], gsz[i + 1], gch[i + 1]) for i in range(5)]     # pre-BN / pre-tanh
        self.gh = [a(N, gsz[i + 1], gsz[i + 1], gch[i + 1]) for i in range(4)]     # post BN+ReLU
        self.fake = a(N, 64, 64, NCP)
        self.dgy = [a(N, gsz[i + 1], gsz[i + 1], gch[i + 1]) for i in range(5)]
        self.dgh = [a(N, gsz[i + 1], gsz[i + 1], gch[i + 1]) for i in range(4)]
        # discriminator: 64 -> 32 -> 16 -> 8 -> 4 -> 1, channels 3 -> 64 -> 128 -> 256 -> 512 -> 1
        dch = [NCP, 64, 128, 256, 512, 1]
        dsz = [64, 32, 16, 8, 4, 1]
        self.ddesc = [self._desc(dsz[i], dch[i], dch[i + 1], *D_LAYERS[i], False) for i in range(5)]
        self.dch, self.dsz = dch, dsz
        self.real = torch.zeros(N, 64, 64, NCP, dtype=self.tdt, device=dev)
        self.dy = [a(N, dsz[i + 1], dsz[i + 1], dch[i + 1]) for i in range(5)]     # pre-activation
        self.dh = [a(N, dsz[i + 1], dsz[i + 1], dch[i + 1]) for i in range(4)]     # post activation
        self.ddy = [a(N, dsz[i + 1], dsz[i + 1], dch[i + 1]) for i in range(5)]
        self.ddh = [a(N, dsz[i + 1], dsz[i + 1], dch[i + 1]) for i in range(4)]
        self.dimg = a(N, 64, 64, NCP)
        f32 = lambda *shape: torch.zeros(shape, dtype=torch.float32, device=dev)
        self.errD_real, self.errD_fake, self.errG = f32(B), f32(B), f32(B)
        self.mean = f32(1)
        ws = Workspace(dev)
        for d in self.gdesc + self.ddesc:
            ws.reserve(H.hfta_fused_conv_workspace(B, d, self.dt))
        for i in range(4):
            ws.reserve(H.hfta_fused_bn_workspace(B, N * gsz[i + 1] ** 2, gch[i + 1]))
            ws.reserve(H.hfta_fused_bn_workspace(B, N * dsz[i + 1] ** 2, dch[i + 1]))
        ws.reserve(H.hfta_loss_workspace(B, N))
        ws.alloc()
        self.ws = ws
        # bf16: D's BN statistics come from the conv epilogues (HFTA_COLSTAT=0 disables)
        import os
        self.colstat = (torch.empty(max([H.hfta_linear_colstat_size(B, N * dsz[i + 1] ** 2, dch[i + 1])
                                         for i in (1, 2, 3)] +
                                        [H.hfta_linear_colstat_size(B, N * gsz[i + 1] ** 2, gch[i + 1])
                                         for i in range(4)]) // 4, dtype=torch.float32, device=dev)
                        if self.dt == H.HFTA_BF16 and os.environ.get("HFTA_COLSTAT", "1") != "0" else None)

    # -------------------------------------------------------- wrappers --
    @staticmethod
    def _in(t):
        return H.tin(t, t[0].numel(), t.shape[-1])

    @staticmethod
    def _out(t):
        return H.tout(t, t[0].numel(), t.shape[-1])

    def _win(self, half, name):
        """Weight operand: Conv2d [Co][kh*kw*Ci] (ld kh*kw*Ci), ConvT2d [kh*kw*Co][Ci] (ld Ci)."""
        ar = half.arena
        src = ar.p if self.dt == H.HFTA_F32 else ar.shadow
        shp = ar.shape[name]
        ld = shp[-1] if name.startswith("t") else int(np.prod(shp[1:]))
        return H.tin(src, ar.P, ld, ar.off[name])

    # CUDA events around one named (de)convolution forward (bench roofline probe):
    # name = "D.c3:fwd" etc.
    _probe = None

    def probe_arm(self, name):
        self._probe, self._probe_ev = name, []

    def probe_collect(self):
        ms = [a.elapsed_time(b) for a, b in getattr(self, "_probe_ev", [])]
        self._probe = None
        return ms

    def probe_roofline(self, name, ms, peaks, path="tc"):
        """Implicit-GEMM (de)convolution: algorithmic flops 2 B M N K of the
        layer (M output pixels, K = 16 C_in); tensor-bound (AI 338-819 for the
        inner layers) against the sustained bf16 peak."""
        layer = name.split(":")[0]
        net, lname = layer.split(".")
        i = int(lname[1:]) - 1
        d = (self.ddesc if net == "D" else self.gdesc)[i]
        if d.transposed:
            Ho = (d.H - 1) * d.stride - 2 * d.pad + d.kh
            flops = 2.0 * self.B * d.N * d.H * d.W * d.C_in * d.C_out * d.kh * d.kw
        else:
            Ho = (d.H + 2 * d.pad - d.kh) // d.stride + 1
            flops = 2.0 * self.B * d.N * Ho * Ho * d.C_out * d.C_in * d.kh * d.kw
        nbytes = self.B * 2 * (d.N * d.H * d.W * d.C_in + d.N * Ho * Ho * d.C_out + d.C_in * d.C_out * d.kh * d.kw)
        t = float(np.mean(ms)) / 1e3 if ms else float("nan")
        ach = flops / t / 1e12
        pk = peaks["bf16_tflops_sustained"] / (1.0 if self.dt == H.HFTA_BF16 else 6.0)
        kind = "implicit-GEMM tcgen05 conv" if self.dt == H.HFTA_BF16 else "patch matrix + 3xTF32 GEMM"
        return {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "traffic": None,
                "kernel": name + " (%s, one call)" % kind, "launches_timed": len(ms),
                "ms_per_launch": t * 1e3, "algorithmic": {"flops": flops, "bytes": nbytes},
                "peak_source": peaks["source"]}

    def _conv_fwd(self, half, name, desc, X, Y, s, act=H.ACT_NONE, alpha=0.0):
        tag = ("G." if half is self.G else "D.") + name.split(".")[0] + ":fwd"
        e0 = None
        if self._probe == tag:
            import torch
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
        H.hfta_fused_conv_fwd(self.B, desc, self.dt, X, self._win(half, name), self._out(Y), act, alpha,
                              self.ws.ptr, self.ws.nbytes, s)
        if e0 is not None:
            import torch
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(torch.cuda.current_stream())
            self._probe_ev.append((e0, e1))

    def _conv_bwd(self, half, name, desc, dY, X, dX, s, wgrad=True, accumulate=0, gate=None):
        """gate: (act, alpha, tensor) -- dX *= act'(tensor), the backward of the
        activation that consumed X (fused into the dgrad epilogue)."""
        ar = half.arena
        act, alpha, g = gate if gate is not None else (H.ACT_NONE, 0.0, None)
        H.hfta_fused_conv_bwd_gated(self.B, desc, self.dt, self._in(dY), X, self._win(half, name),
                                    self._out(dX) if dX is not None else H.hfta_out(None, 0, 1),
                                    ar.fptr("g", name) if wgrad else None, ar.P, accumulate, act, alpha,
                                    self._in(g) if g is not None else H.hfta_in(None, 0, 1), self.ws.ptr,
                                    self.ws.nbytes, s)

    def _bn_fwd(self, half, name, X, act, alpha, Y, s):
        R, C = X[0].numel() // X.shape[-1], X.shape[-1]
        rm, rv = half.running[name]
        sm, si = half.saved[name]
        ar = half.arena
        H.hfta_fused_bn_fwd(self.B, R, C, self.dt, self._in(X), ar.fptr("p", name + ".g"), ar.fptr("p", name + ".beta"),
                            ar.P, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, act, alpha, self._out(Y), H.ptr(sm), H.ptr(si),
                            self.ws.ptr, self.ws.nbytes, s)

    def _bn_bwd(self, half, name, dY, X, act, alpha, dX, s, wgrad=True, accumulate=0):
        R, C = X[0].numel() // X.shape[-1], X.shape[-1]
        sm, si = half.saved[name]
        ar = half.arena
        H.hfta_fused_bn_bwd(self.B, R, C, self.dt, self._in(dY), self._in(X), ar.fptr("p", name + ".g"),
                            ar.fptr("p", name + ".beta"), ar.P, H.ptr(sm), H.ptr(si), act, alpha, self._out(dX),
                            ar.fptr("g", name + ".g") if wgrad else None,
                            ar.fptr("g", name + ".beta") if wgrad else None, accumulate, self.ws.ptr,
                            self.ws.nbytes, s)

    def _act(self, act, alpha, X, Y, s):
        rows = X[0].numel() // X.shape[-1]
        H.hfta_act_fwd(self.B, rows, X.shape[-1], self.dt, act, alpha, self._in(X), self._out(Y), s)

    def _act_bwd(self, act, alpha, XY, dY, dX, s):
        rows = XY[0].numel() // XY.shape[-1]
        H.hfta_act_bwd(self.B, rows, XY.shape[-1], self.dt, act, alpha, self._in(XY), self._in(dY), self._out(dX), s)

    # ---------------------------------------------------------- passes --
    def _bn_fwd_colstat(self, half, name, X, act, alpha, Y, s):
        R, C = X[0].numel() // X.shape[-1], X.shape[-1]
        rm, rv = half.running[name]
        sm, si = half.saved[name]
        ar = half.arena
        H.hfta_fused_bn_fwd_colstat(self.B, R, C, self.dt, self._in(X), ar.fptr("p", name + ".g"),
                                    ar.fptr("p", name + ".beta"), ar.P, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, act, alpha,
                                    self._out(Y), H.ptr(sm), H.ptr(si), H.ptr(self.colstat), s)

    def _D_forward(self, img_in, s):
        D = self.D
        # c1 has no BN: LeakyReLU(0.2) applied in the convolution's epilogue (dh[0] = act(y))
        self._conv_fwd(D, "c1.W", self.ddesc[0], img_in, self.dh[0], s, H.ACT_LEAKY_RELU, 0.2)
        for i in (1, 2, 3):
            name = "c%d.W" % (i + 1)
            if self.colstat is not None:    # BN statistics from the implicit-GEMM conv's epilogue
                tag = "D." + name.split(".")[0] + ":fwd"
                e0 = None
                if self._probe == tag:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e0.record(torch.cuda.current_stream())
                H.hfta_fused_conv_fwd_stats(self.B, self.ddesc[i], self.dt, self._in(self.dh[i - 1]),
                                            self._win(D, name), self._out(self.dy[i]), H.ptr(self.colstat),
                                            self.ws.ptr, self.ws.nbytes, s)
                if e0 is not None:
                    e1 = torch.cuda.Event(enable_timing=True)
                    e1.record(torch.cuda.current_stream())
                    self._probe_ev.append((e0, e1))
                self._bn_fwd_colstat(D, "bn%d" % (i + 1), self.dy[i], H.ACT_LEAKY_RELU, 0.2, self.dh[i], s)
            else:
                self._conv_fwd(D, name, self.ddesc[i], self._in(self.dh[i - 1]), self.dy[i], s)
                self._bn_fwd(D, "bn%d" % (i + 1), self.dy[i], H.ACT_LEAKY_RELU, 0.2, self.dh[i], s)
        self._conv_fwd(D, "c5.W", self.ddesc[4], self._in(self.dh[3]), self.dy[4], s)

    def _D_backward(self, dlogit, img_in, s, wgrad, accumulate, need_dimg):
        """dlogit: [B][N][1][1][1] gradient of the D output logits."""
        D = self.D
        self._conv_bwd(D, "c5.W", self.ddesc[4], dlogit, self._in(self.dh[3]), self.ddh[3], s, wgrad, accumulate)
        for i in (3, 2, 1):
            self._bn_bwd(D, "bn%d" % (i + 1), self.ddh[i], self.dy[i], H.ACT_LEAKY_RELU, 0.2, self.ddy[i], s, wgrad,
                         accumulate)
            if i > 1:
                self._conv_bwd(D, "c%d.W" % (i + 1), self.ddesc[i], self.ddy[i], self._in(self.dh[i - 1]),
                               self.ddh[i - 1], s, wgrad, accumulate)
            else:       # c2's dgrad through c1's LeakyReLU (gate: act(y) > 0 <=> y > 0), one epilogue
                self._conv_bwd(D, "c2.W", self.ddesc[1], self.ddy[1], self._in(self.dh[0]), self.ddy[0], s, wgrad,
                               accumulate, gate=(H.ACT_LEAKY_RELU, 0.2, self.dh[0]))
        self._conv_bwd(D, "c1.W", self.ddesc[0], self.ddy[0], img_in, self.dimg if need_dimg else None, s, wgrad,
                       accumulate)

    def _G_forward(self, s):
        G = self.G
        x = H.tin(self.z, self.N * NZP, NZP)
        for i in range(4):
            if self.colstat is not None:    # BN statistics from the sub-pixel epilogue (t1: one pass over y)
                H.hfta_fused_conv_fwd_stats(self.B, self.gdesc[i], self.dt, x, self._win(G, "t%d.W" % (i + 1)),
                                            self._out(self.gy[i]), H.ptr(self.colstat), self.ws.ptr, self.ws.nbytes,
                                            s)
                self._bn_fwd_colstat(G, "bn%d" % (i + 1), self.gy[i], H.ACT_RELU, 0.0, self.gh[i], s)
            else:
                self._conv_fwd(G, "t%d.W" % (i + 1), self.gdesc[i], x, self.gy[i], s)
                self._bn_fwd(G, "bn%d" % (i + 1), self.gy[i], H.ACT_RELU, 0.0, self.gh[i], s)
            x = self._in(self.gh[i])
        # t5 has no BN: Tanh in the convolution's epilogue (fake = tanh(y))
        self._conv_fwd(G, "t5.W", self.gdesc[4], x, self.fake, s, H.ACT_TANH, 0.0)

    def _G_backward(self, dfake, s):
        G = self.G
        self._act_bwd(H.ACT_TANH, 0.0, self.fake, dfake, self.dgy[4], s)
        for i in range(4, -1, -1):
            X = self._in(self.gh[i - 1]) if i > 0 else H.tin(self.z, self.N * NZP, NZP)
            self._conv_bwd(G, "t%d.W" % (i + 1), self.gdesc[i], self.dgy[i], X, self.dgh[i - 1] if i > 0 else None, s)
            if i > 0:
                self._bn_bwd(G, "bn%d" % i, self.dgh[i - 1], self.gy[i - 1], H.ACT_RELU, 0.0, self.dgy[i - 1], s)

    def _bce(self, target, out_loss, s):
        z = self.dy[4]
        H.hfta_loss_bce_logits(self.B, self.N, self.dt, H.tin(z, self.N, 1), target, H.ptr(out_loss), H.ptr(self.mean),
                               H.tout(self.ddy[4], self.N, 1), self.ws.ptr, self.ws.nbytes, s)

    def set_inputs(self, real_nhwc, z_bn):
        """real: device fp32 [N,64,64,3] (shared); z: device fp32 [B,N,100] (per model)."""
        self.real[..., :NC].copy_(real_nhwc.to(self.tdt))
        self.z.zero_()
        self.z[:, :, :NZ].copy_(z_bn.to(self.tdt))

    def step(self, stream=None):
        """One DCGAN iteration for all B models; returns (errD_real, errD_fake, errG) [B] each."""
        s = H.stream_ptr(stream)
        self.t += 1
        real = H.tin(self.real, 0, NCP)                   # shared by all models
        # (1) D on real, label 1
        self._D_forward(real, s)
        self._bce(1.0, self.errD_real, s)
        self._D_backward(self.ddy[4], real, s, wgrad=True, accumulate=0, need_dimg=False)
        # (2) D on G(z).detach(), label 0, gradients accumulate
        self._G_forward(s)
        fake = self._in(self.fake)
        self._D_forward(fake, s)
        self._bce(0.0, self.errD_fake, s)
        self._D_backward(self.ddy[4], fake, s, wgrad=True, accumulate=1, need_dimg=False)
        # (3) Adam on D
        H.hfta_step_increment(H.ptr(self.hvD.step), s)
        fused_adam(self.D.arena, self.hvD, s)
        # (4) updated D on G(z), label 1, backward into G only
        self._D_forward(fake, s)
        self._bce(1.0, self.errG, s)
        self._D_backward(self.ddy[4], fake, s, wgrad=False, accumulate=0, need_dimg=True)
        self._G_backward(self.dimg, s)
        # (5) Adam on G
        H.hfta_step_increment(H.ptr(self.hvG.step), s)
        fused_adam(self.G.arena, self.hvG, s)
        return self.errD_real, self.errD_fake, self.errG
