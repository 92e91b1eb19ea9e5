"""Host-side plumbing of a fused model array: the per-model parameter arena,
the fused-Adam state, hyper-parameter vectors and a shared workspace.

The arena is the build's form of the paper's fused parameters ("weights
(filters) and biases [concatenated] along the dimension of the output
channel"): model-major [B][P] fp32 with every tensor of model b at
arena[b, off:off+numel] in PyTorch layout, so one fused-Adam launch updates
all models.  PyTorch only allocates memory here.
"""
import numpy as np
import torch

from . import hfta as H

ALIGN = 32  # elements: 128 B for fp32, 64 B for bf16 -- keeps TMA/vector alignment


def _al(n):
    return (n + ALIGN - 1) // ALIGN * ALIGN


class ParamArena:
    """Flat [B][P] fp32 parameters + grads + Adam m, v (+ bf16 shadow)."""

    def __init__(self, specs, B, device, bf16_shadow=False):
        self.B = B
        self.specs = [(n, tuple(s)) for n, s in specs]
        self.off = {}
        o = 0
        for n, s in self.specs:
            self.off[n] = o
            o += _al(int(np.prod(s)))
        self.P = o
        self.shape = dict(self.specs)
        z = lambda: torch.zeros(B, self.P, dtype=torch.float32, device=device)
        self.p, self.g, self.m, self.v = z(), z(), z(), z()
        self.shadow = torch.zeros(B, self.P, dtype=torch.bfloat16, device=device) if bf16_shadow else None

    def load(self, params_per_model):
        host = torch.zeros(self.B, self.P, dtype=torch.float32)
        for b, P in enumerate(params_per_model):
            for n, s in self.specs:
                a = np.asarray(P[n], dtype=np.float32).reshape(-1)
                host[b, self.off[n]:self.off[n] + a.size] = torch.from_numpy(a)
        self.p.copy_(host)
        self.sync_shadow()

    def sync_shadow(self, stream=None):
        if self.shadow is not None:
            H.hfta_cast_f32_bf16(self.B * self.P, H.ptr(self.p), H.ptr(self.shadow), H.stream_ptr(stream))

    def numel(self, n):
        return int(np.prod(self.shape[n]))

    def host_tensor(self, which, n):
        """Per-model values of tensor n as numpy [B, *shape] (for tests / unfuse)."""
        src = dict(p=self.p, g=self.g, m=self.m, v=self.v)[which]
        k = self.numel(n)
        return src[:, self.off[n]:self.off[n] + k].detach().cpu().numpy().astype(np.float64).reshape(
            (self.B,) + self.shape[n])

    # ---- ABI views (element offsets into the arena; bstride = P) ----
    def w_in(self, n, dt, col_off=0, ld=None):
        """Weight operand of dtype dt: fp32 master or the bf16 shadow."""
        src = self.p if dt == H.HFTA_F32 else self.shadow
        ld = self.shape[n][-1] if ld is None else ld
        return H.tin(src, self.P, ld, self.off[n] + col_off)

    def fptr(self, which, n, col_off=0):
        src = dict(p=self.p, g=self.g, m=self.m, v=self.v)[which]
        return src.data_ptr() + 4 * (self.off[n] + col_off)


class HyperVectors:
    """Per-model hyper-parameter vectors on device (HyperVector)."""

    def __init__(self, hp, device):
        self.t = {k: torch.tensor(np.asarray(hp[k], dtype=np.float32), device=device)
                  for k in ("lr", "beta1", "beta2", "eps", "wd")}
        self.step = torch.zeros(1, dtype=torch.int64, device=device)

    def set(self, name, values):
        self.t[name].copy_(torch.tensor(np.asarray(values, dtype=np.float32)))


def fused_adam(arena, hv, stream):
    H.hfta_fused_adam(arena.B, arena.P, H.ptr(arena.p), H.ptr(arena.g), H.ptr(arena.m), H.ptr(arena.v),
                      arena.P, H.ptr(hv.t["lr"]), H.ptr(hv.t["beta1"]), H.ptr(hv.t["beta2"]),
                      H.ptr(hv.t["eps"]), H.ptr(hv.t["wd"]), H.ptr(hv.step),
                      H.ptr(arena.shadow) if arena.shadow is not None else None, arena.P, stream)


class Workspace:
    """One scratch buffer shared by all calls of a step (they are stream-ordered)."""

    def __init__(self, device):
        self.device = device
        self.need = 0
        self.buf = None

    def reserve(self, nbytes):
        self.need = max(self.need, int(nbytes))

    def alloc(self):
        self.buf = torch.empty(max(self.need, 256), dtype=torch.uint8, device=self.device)

    @property
    def ptr(self):
        return self.buf.data_ptr()

    @property
    def nbytes(self):
        return self.buf.numel()
