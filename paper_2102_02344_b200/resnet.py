"""Fused ResNet-18 training step (the second model family, SURVEY NEXT-4;
the paper's secondary CV benchmark; model: reading R33).

B ResNet-18s with per-model Adadelta hyper-parameters train as one
job: every Conv2d, BatchNorm2d, ReLU, residual add, MaxPool2d,
AdaptiveAvgPool2d, Linear and the cross-entropy loss is one C-ABI call for
all B models (App. B fusion rows P:L1262-1290).  Layouts as in dcgan.py:
NHWC per model, conv weights in the arena as [Co][kh][kw][Ci], the image
channels padded 3 -> 8 (16-B bf16 rows; the pad weights are zero and get
exactly zero gradients).  The CIFAR batch is shared by all models
(bstride 0); labels int32 shared.

Block schedule (BasicBlock, torchvision): y1 = conv3x3_s(h); a1 =
ReLU(BN1(y1)) [one BN call with the ReLU in its apply]; y2 = conv3x3(a1);
z2 = BN2(y2); shortcut = h or BN_d(conv1x1_s(h)); u = z2 + shortcut;
h' = ReLU(u).  Backward: du = ReLU'(u) dh'; BN2/conv2/BN1(+ReLU')/conv1
into dh_main; the shortcut's gradient (du, or through BN_d/conv_d) is added.
"""
import numpy as np
import torch

from . import hfta as H
from .fused import ParamArena, Workspace

NC, NCP = 3, 8            # image channels, padded to 16-B bf16 rows
STAGES = (64, 128, 256, 512)


def block_plan(widths=STAGES):
    """(name, C_in, C_out, stride, has_downsample) of the 8 BasicBlocks."""
    out, cin = [], widths[0]
    for s, w in enumerate(widths):
        for b in range(2):
            stride = 2 if (s > 0 and b == 0) else 1
            out.append(("l%d.%d" % (s + 1, b), cin, w, stride, stride != 1 or cin != w))
            cin = w
    return out


def _to_gpu(name, a):
    if name.endswith(".W") and a.ndim == 4:            # Conv [Co][Ci][kh][kw] -> [Co][kh][kw][Ci]
        g = np.transpose(a, (0, 2, 3, 1))
        if a.shape[1] == NC:
            g = np.pad(g, [(0, 0), (0, 0), (0, 0), (0, NCP - NC)])
        return g
    return a


def _to_torch(name, g):
    if name.endswith(".W") and g.ndim == 4:
        if name == "conv1.W":
            g = g[..., :NC]
        return np.transpose(g, (0, 3, 1, 2))
    return g


class AdadeltaVectors:
    """Per-model Adadelta hyper-parameters on device (lr, rho, eps, wd)."""

    def __init__(self, hp, device):
        self.t = {k: torch.tensor(np.asarray(hp[k], dtype=np.float32), device=device)
                  for k in ("lr", "rho", "eps", "wd")}

    def set(self, name, values):
        self.t[name].copy_(torch.tensor(np.asarray(values, dtype=np.float32)))


class FusedResNet18:
    def __init__(self, B, specs, params, hp, N=128, HW=32, k=10, widths=STAGES, dtype="bf16", device="cuda"):
        self.B, self.N, self.HW, self.k, self.widths = B, N, HW, k, tuple(widths)
        self.dt = H.HFTA_F32 if dtype == "f32" else H.HFTA_BF16
        self.tdt = torch.float32 if dtype == "f32" else torch.bfloat16
        self.device = torch.device(device)
        self.torch_specs = [(n, s) for n, s, *_ in specs]
        gspecs = [(n, _to_gpu(n, np.zeros(s)).shape) for n, s in self.torch_specs]
        self.arena = ParamArena(gspecs, B, self.device, bf16_shadow=(dtype == "bf16"))
        self.arena.load([{n: _to_gpu(n, P[n]) for n, _ in self.torch_specs} for P in params])
        self.hv = AdadeltaVectors(hp, self.device)
        sh = self.arena.shape
        self.bn = [n[:-2] for n, _ in self.torch_specs if n.endswith(".g")]
        z = lambda c: torch.zeros(B, c, dtype=torch.float32, device=self.device)
        self.running = {n: (z(sh[n + ".g"][0]), torch.ones(B, sh[n + ".g"][0], dtype=torch.float32,
                                                           device=self.device)) for n in self.bn}
        self.saved = {n: (z(sh[n + ".g"][0]), z(sh[n + ".g"][0])) for n in self.bn}
        self.t = 0
        self._plan()

    # ------------------------------------------------------------ plan --
    def _desc(self, Hs, cin, cout, k, stride, pad):
        d = H.hfta_conv_desc()
        d.N, d.H, d.W, d.C_in, d.C_out, d.kh, d.kw = self.N, Hs, Hs, cin, cout, k, k
        d.stride, d.pad, d.transposed = stride, pad, 0
        return d

    def _plan(self):
        B, N, dev, w0 = self.B, self.N, self.device, self.widths[0]
        a = lambda *shape: torch.empty((B,) + shape, dtype=self.tdt, device=dev)
        ws = Workspace(dev)
        self.img = torch.zeros(N, self.HW, self.HW, NCP, dtype=self.tdt, device=dev)
        self.labels = torch.zeros(N, dtype=torch.int32, device=dev)
        s1 = (self.HW + 2 * 3 - 7) // 2 + 1                  # stem conv output size
        s2 = (s1 + 2 * 1 - 3) // 2 + 1                       # after the max pool
        self.stem = dict(desc=self._desc(self.HW, NCP, w0, 7, 2, 3), hw=s1, pool_hw=s2,
                         y=a(N, s1, s1, w0), a=a(N, s1, s1, w0), dy=a(N, s1, s1, w0), da=a(N, s1, s1, w0),
                         am=torch.empty((B, N, s2, s2, w0), dtype=torch.uint8, device=dev))
        self.h0, self.dh0 = a(N, s2, s2, w0), a(N, s2, s2, w0)
        ws.reserve(H.hfta_fused_conv_workspace(B, self.stem["desc"], self.dt))
        ws.reserve(H.hfta_fused_bn_workspace(B, N * s1 * s1, w0))
        self.blocks = []
        hw = s2
        for name, cin, cout, stride, down in block_plan(self.widths):
            ho = (hw + 2 - 3) // stride + 1
            blk = dict(name=name, cin=cin, cout=cout, stride=stride, down=down, hin=hw, hout=ho,
                       d1=self._desc(hw, cin, cout, 3, stride, 1), d2=self._desc(ho, cout, cout, 3, 1, 1),
                       y1=a(N, ho, ho, cout), a1=a(N, ho, ho, cout), y2=a(N, ho, ho, cout), z2=a(N, ho, ho, cout),
                       u=a(N, ho, ho, cout), h=a(N, ho, ho, cout),
                       du=a(N, ho, ho, cout), dy2=a(N, ho, ho, cout), da1=a(N, ho, ho, cout),
                       dy1=a(N, ho, ho, cout), dh=a(N, hw, hw, cin))
            ws.reserve(H.hfta_fused_conv_workspace(B, blk["d1"], self.dt))
            ws.reserve(H.hfta_fused_conv_workspace(B, blk["d2"], self.dt))
            ws.reserve(H.hfta_fused_bn_workspace(B, N * ho * ho, cout))
            if down:
                blk.update(dd=self._desc(hw, cin, cout, 1, stride, 0), yd=a(N, ho, ho, cout), zd=a(N, ho, ho, cout),
                           dyd=a(N, ho, ho, cout), dhs=a(N, hw, hw, cin))
                ws.reserve(H.hfta_fused_conv_workspace(B, blk["dd"], self.dt))
            self.blocks.append(blk)
            hw = ho
        self.last_hw = hw
        C = self.widths[-1]
        self.feat, self.dfeat = a(N, C), a(N, C)
        self.logits, self.dlogits = a(N, self.k), a(N, self.k)
        f32 = lambda *shape: torch.zeros(shape, dtype=torch.float32, device=dev)
        self.loss, self.mean_loss = f32(B), f32(1)
        ws.reserve(H.hfta_loss_workspace(B, N))
        ws.reserve(H.hfta_fused_linear_bwd_workspace(B, N, self.k, C, self.dt))
        ws.alloc()
        self.ws = ws
        # bf16: every BN's statistics come from its conv's epilogue (HFTA_COLSTAT=0 disables)
        import os
        sizes = [H.hfta_linear_colstat_size(B, N * s1 * s1, w0)] + \
                [H.hfta_linear_colstat_size(B, N * blk["hout"] ** 2, blk["cout"]) for blk in self.blocks]
        self.colstat = (torch.empty(max(sizes) // 4, dtype=torch.float32, device=dev)
                        if self.dt == H.HFTA_BF16 and os.environ.get("HFTA_COLSTAT", "1") != "0" else None)

    # -------------------------------------------------------- wrappers --
    @staticmethod
    def _in(t):
        return H.tin(t, t[0].numel(), t.shape[-1])

    @staticmethod
    def _out(t):
        return H.tout(t, t[0].numel(), t.shape[-1])

    def _rows(self, t):
        return t[0].numel() // t.shape[-1]

    def _win(self, name):
        ar = self.arena
        src = ar.p if self.dt == H.HFTA_F32 else ar.shadow
        return H.tin(src, ar.P, int(np.prod(ar.shape[name][1:])), ar.off[name])

    # ---- bench roofline probe: CUDA events around one named conv forward ----
    _probe = None

    def probe_arm(self, name):
        self._probe, self._probe_ev = name, []

    def probe_collect(self):
        ms = [a.elapsed_time(b) for a, b in getattr(self, "_probe_ev", [])]
        self._probe = None
        return ms

    def _conv_desc(self, layer):
        if layer == "conv1":
            return self.stem["desc"]
        blk = next(b for b in self.blocks if layer.startswith(b["name"] + "."))
        return blk[{"conv1": "d1", "conv2": "d2", "down": "dd"}[layer.split(".")[-1]]]

    @staticmethod
    def _conv_flops(d, real_cin=None):
        Ho = (d.H + 2 * d.pad - d.kh) // d.stride + 1
        Wo = (d.W + 2 * d.pad - d.kw) // d.stride + 1
        return 2.0 * Ho * Wo * d.C_out * (real_cin or d.C_in) * d.kh * d.kw      # per image

    def flops_per_sample(self):
        """Algorithmic flops of one training step per image (the method's work:
        forward; backward = dgrad + wgrad of every contraction, no stem dgrad;
        the stem counts its 3 real input channels)."""
        stem = self._conv_flops(self.stem["desc"], NC)
        fwd = stem + 2.0 * self.widths[-1] * self.k
        for blk in self.blocks:
            fwd += self._conv_flops(blk["d1"]) + self._conv_flops(blk["d2"])
            if blk["down"]:
                fwd += self._conv_flops(blk["dd"])
        return 3.0 * fwd - stem

    def probe_roofline(self, name, ms, peaks, path="tc"):
        """One conv forward of the ResNet family: patch matrix (im2col) + the
        tcgen05 GEMM; algorithmic flops 2 B N Ho Wo Co Ci k^2."""
        d = self._conv_desc(name.split(":")[0])
        flops = self.B * self.N * self._conv_flops(d)
        t = float(np.mean(ms)) / 1e3 if ms else float("nan")
        ach = flops / t / 1e12
        pk = peaks["bf16_tflops_sustained"] / (1.0 if self.dt == H.HFTA_BF16 else 6.0)
        return {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk, "traffic": None,
                "kernel": name + " (im2col + tcgen05 GEMM, one call)", "launches_timed": len(ms),
                "ms_per_launch": t * 1e3, "algorithmic": {"flops": flops}, "peak_source": peaks["source"]}

    def _conv_fwd(self, name, desc, X, Y, s):
        e0 = None
        if self._probe == name[:-2] + ":fwd":
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
        H.hfta_fused_conv_fwd(self.B, desc, self.dt, X, self._win(name), self._out(Y), H.ACT_NONE, 0.0,
                              self.ws.ptr, self.ws.nbytes, s)
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(torch.cuda.current_stream())
            self._probe_ev.append((e0, e1))

    def _conv_bwd(self, name, desc, dY, X, dX, s):
        H.hfta_fused_conv_bwd(self.B, desc, self.dt, self._in(dY), X, self._win(name),
                              self._out(dX) if dX is not None else H.hfta_out(None, 0, 1),
                              self.arena.fptr("g", name), self.arena.P, 0, self.ws.ptr, self.ws.nbytes, s)

    def _conv_bn_fwd(self, cname, desc, X, y, bname, act, out, s):
        """conv -> BN (-> act): with the bf16 path the BN statistics come from the
        conv's epilogue (hfta_fused_conv_fwd_stats -> hfta_fused_bn_fwd_colstat)."""
        if self.colstat is None:
            self._conv_fwd(cname, desc, X, y, s)
            self._bn_fwd(bname, y, act, out, s)
            return
        e0 = None
        if self._probe == cname[:-2] + ":fwd":
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
        H.hfta_fused_conv_fwd_stats(self.B, desc, self.dt, X, self._win(cname), self._out(y), H.ptr(self.colstat),
                                    self.ws.ptr, self.ws.nbytes, s)
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(torch.cuda.current_stream())
            self._probe_ev.append((e0, e1))
        rm, rv = self.running[bname]
        sm, si = self.saved[bname]
        ar = self.arena
        H.hfta_fused_bn_fwd_colstat(self.B, self._rows(y), y.shape[-1], self.dt, self._in(y), ar.fptr("p", bname + ".g"),
                                    ar.fptr("p", bname + ".beta"), ar.P, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, act, 0.0,
                                    self._out(out), H.ptr(sm), H.ptr(si), H.ptr(self.colstat), s)

    def _bn_fwd(self, name, X, act, Y, s):
        rm, rv = self.running[name]
        sm, si = self.saved[name]
        ar = self.arena
        H.hfta_fused_bn_fwd(self.B, self._rows(X), X.shape[-1], self.dt, self._in(X), ar.fptr("p", name + ".g"),
                            ar.fptr("p", name + ".beta"), ar.P, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, act, 0.0,
                            self._out(Y), H.ptr(sm), H.ptr(si), self.ws.ptr, self.ws.nbytes, s)

    def _bn_bwd(self, name, dY, X, act, dX, s):
        sm, si = self.saved[name]
        ar = self.arena
        H.hfta_fused_bn_bwd(self.B, self._rows(X), X.shape[-1], self.dt, self._in(dY), self._in(X),
                            ar.fptr("p", name + ".g"), ar.fptr("p", name + ".beta"), ar.P, H.ptr(sm), H.ptr(si),
                            act, 0.0, self._out(dX), ar.fptr("g", name + ".g"), ar.fptr("g", name + ".beta"), 0,
                            self.ws.ptr, self.ws.nbytes, s)

    def _add(self, X1, X2, Y, s):
        H.hfta_add(self.B, self._rows(Y), Y.shape[-1], self.dt, X1, X2, self._out(Y), s)

    # ---------------------------------------------------------- passes --
    def forward(self, s):
        st = self.stem
        w0 = self.widths[0]
        img = H.tin(self.img, 0, NCP)                       # shared by all models
        self._conv_bn_fwd("conv1.W", st["desc"], img, st["y"], "bn1", H.ACT_RELU, st["a"], s)
        H.hfta_maxpool2d_fwd(self.B, self.N, st["hw"], st["hw"], w0, 3, 2, 1, self.dt, self._in(st["a"]),
                             self._out(self.h0), H.ptr(st["am"]), st["am"][0].numel(), s)
        h = self.h0
        for blk in self.blocks:
            n = blk["name"]
            self._conv_bn_fwd(n + ".conv1.W", blk["d1"], self._in(h), blk["y1"], n + ".bn1", H.ACT_RELU, blk["a1"], s)
            self._conv_bn_fwd(n + ".conv2.W", blk["d2"], self._in(blk["a1"]), blk["y2"], n + ".bn2", H.ACT_NONE,
                              blk["z2"], s)
            if blk["down"]:
                self._conv_bn_fwd(n + ".down.W", blk["dd"], self._in(h), blk["yd"], n + ".dbn", H.ACT_NONE,
                                  blk["zd"], s)
                sc = blk["zd"]
            else:
                sc = h
            self._add(self._in(blk["z2"]), self._in(sc), blk["u"], s)
            H.hfta_act_fwd(self.B, self._rows(blk["u"]), blk["cout"], self.dt, H.ACT_RELU, 0.0, self._in(blk["u"]),
                           self._out(blk["h"]), s)
            h = blk["h"]
        C = self.widths[-1]
        H.hfta_avgpool2d_fwd(self.B, self.N, self.last_hw * self.last_hw, C, self.dt, self._in(h),
                             self._out(self.feat), s)
        ar = self.arena
        H.hfta_fused_linear_fwd(self.B, self.N, self.k, C, self.dt, self._in(self.feat), ar.w_in("fc.W", self.dt),
                                ar.fptr("p", "fc.b"), ar.P, 0, 0, self._out(self.logits), s)

    def backward(self, s):
        ar, C = self.arena, self.widths[-1]
        H.hfta_fused_linear_bwd(self.B, self.N, self.k, C, self.dt, self._in(self.dlogits), self._in(self.feat),
                                ar.w_in("fc.W", self.dt), self._out(self.dfeat), ar.fptr("g", "fc.W"), ar.P, C,
                                ar.fptr("g", "fc.b"), ar.P, 0, self.ws.ptr, self.ws.nbytes, s)
        last = self.blocks[-1]
        dh = last["dy2"]          # scratch for d(block output): the avg-pool backward
        H.hfta_avgpool2d_bwd(self.B, self.N, self.last_hw * self.last_hw, C, self.dt, self._in(self.dfeat),
                             self._out(dh), s)
        for i in range(len(self.blocks) - 1, -1, -1):
            blk = self.blocks[i]
            n = blk["name"]
            hin = self.blocks[i - 1]["h"] if i > 0 else self.h0
            H.hfta_act_bwd(self.B, self._rows(blk["u"]), blk["cout"], self.dt, H.ACT_RELU, 0.0, self._in(blk["u"]),
                           self._in(dh), self._out(blk["du"]), s)
            self._bn_bwd(n + ".bn2", blk["du"], blk["y2"], H.ACT_NONE, blk["dy2"], s)
            self._conv_bwd(n + ".conv2.W", blk["d2"], blk["dy2"], self._in(blk["a1"]), blk["da1"], s)
            self._bn_bwd(n + ".bn1", blk["da1"], blk["y1"], H.ACT_RELU, blk["dy1"], s)
            self._conv_bwd(n + ".conv1.W", blk["d1"], blk["dy1"], self._in(hin), blk["dh"], s)
            if blk["down"]:
                self._bn_bwd(n + ".dbn", blk["du"], blk["yd"], H.ACT_NONE, blk["dyd"], s)
                self._conv_bwd(n + ".down.W", blk["dd"], blk["dyd"], self._in(hin), blk["dhs"], s)
                self._add(self._in(blk["dh"]), self._in(blk["dhs"]), blk["dh"], s)
            else:
                self._add(self._in(blk["dh"]), self._in(blk["du"]), blk["dh"], s)
            dh = blk["dh"]
        st = self.stem
        w0 = self.widths[0]
        H.hfta_maxpool2d_bwd(self.B, self.N, st["hw"], st["hw"], w0, 3, 2, 1, self.dt, self._in(dh), H.ptr(st["am"]),
                             st["am"][0].numel(), self._out(st["da"]), s)
        self._bn_bwd("bn1", st["da"], st["y"], H.ACT_RELU, st["dy"], s)
        self._conv_bwd("conv1.W", st["desc"], st["dy"], H.tin(self.img, 0, NCP), None, s)

    def adadelta(self, s):
        ar, hv = self.arena, self.hv.t
        H.hfta_fused_adadelta(self.B, ar.P, H.ptr(ar.p), H.ptr(ar.g), H.ptr(ar.m), H.ptr(ar.v), ar.P,
                              H.ptr(hv["lr"]), H.ptr(hv["rho"]), H.ptr(hv["eps"]), H.ptr(hv["wd"]),
                              H.ptr(ar.shadow) if ar.shadow is not None else None, ar.P, s)

    def set_inputs(self, images_nhwc, labels):
        """images: device fp32 [N, HW, HW, 3] (shared); labels: device int [N]."""
        self.img[..., :NC].copy_(images_nhwc.to(self.tdt))
        self.labels.copy_(labels.to(torch.int32))

    def step(self, stream=None):
        """One fused training step of all B models; returns loss [B] (device)."""
        s = H.stream_ptr(stream)
        self.t += 1
        self.forward(s)
        H.hfta_loss_nll(self.B, self.N, self.k, self.dt, self._in(self.logits), H.ptr(self.labels), 0,
                        H.ptr(self.loss), H.ptr(self.mean_loss), self._out(self.dlogits), self.ws.ptr,
                        self.ws.nbytes, s)
        self.backward(s)
        self.adadelta(s)
        return self.loss

    # ---------------------------------------------------------- unfuse --
    def params(self, b):
        return {n: _to_torch(n, self.arena.host_tensor("p", n)[b]) for n, _ in self.torch_specs}

    def grads(self, b):
        return {n: _to_torch(n, self.arena.host_tensor("g", n)[b]) for n, _ in self.torch_specs}

    def running_stats(self, b):
        return {n: (rm[b].double().cpu().numpy(), rv[b].double().cpu().numpy()) for n, (rm, rv) in
                self.running.items()}
