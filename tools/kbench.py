"""Per-kernel microbenchmark at the PointNet-cls B=64 bf16 shapes (through the
C ABI), CUDA-event timed after warm-up; prints achieved GB/s vs the measured
HBM peak.  Usage: python tools/kbench.py [B]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H  # noqa: E402

H.hfta_init(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
R, N, L = 80000, 32, 2500
dev = "cuda"
s = torch.cuda.current_stream().cuda_stream
try:
    PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except Exception:
    PEAK = 6450.0
bf = torch.bfloat16
ws = torch.empty(2 << 30, dtype=torch.uint8, device=dev)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rep(name, ms, nbytes):
    gbs = nbytes / ms / 1e6
    print("%-34s %8.3f ms  %7.0f GB/s  %5.1f%% of %.0f" % (name, ms, gbs, 100 * gbs / PEAK, PEAK), flush=True)


def T(*shape, dtype=bf):
    return torch.randn(*shape, device=dev).to(dtype)


def tin(x):
    return H.tin(x, x[0].numel(), x.shape[-1])


def tout(x):
    return H.tout(x, x[0].numel(), x.shape[-1])


g = torch.rand(B, 1024, device=dev) + 0.5
be = torch.rand(B, 1024, device=dev) - 0.5
sm, si = torch.empty(B, 1024, device=dev), torch.empty(B, 1024, device=dev)
for C in (64, 128, 1024):
    X, Y, D = T(B, R, C), T(B, R, C), T(B, R, C)
    el = B * R * C * 2
    rep("bn_fwd stats+apply C=%d" % C, t(lambda: H.hfta_fused_bn_fwd(
        B, R, C, 1, tin(X), H.ptr(g), H.ptr(be), 1024, None, None, 0.1, 1e-5, 1, 0.0, tout(Y), H.ptr(sm), H.ptr(si),
        H.ptr(ws), ws.numel(), s)), 3 * el)
    rep("bn_bwd reduce+apply C=%d" % C, t(lambda: H.hfta_fused_bn_bwd(
        B, R, C, 1, tin(D), tin(X), H.ptr(g), H.ptr(be), 1024, H.ptr(sm), H.ptr(si), 1, 0.0, tout(Y), H.ptr(g), H.ptr(be),
        0, H.ptr(ws), ws.numel(), s)), 5 * el)
    del X, Y, D
X = T(B, R, 1024)
G = torch.empty(B, N, 1024, device=dev)
am = torch.empty(B, N, 1024, dtype=torch.int32, device=dev)
rep("bn_max_fwd C=1024", t(lambda: H.hfta_bn_max_fwd(B, N, L, 1024, 1, tin(X), H.ptr(g), H.ptr(be), 1024, H.ptr(sm),
                                                    H.ptr(si), 1, 0.0, tout(G), H.ptr(am), s)), B * R * 1024 * 2)
H.hfta_bn_max_fwd(B, N, L, 1024, 1, tin(X), H.ptr(g), H.ptr(be), 1024, H.ptr(sm), H.ptr(si), 1, 0.0, tout(G), H.ptr(am), s)
dX = T(B, R, 1024)
rep("bn_max_bwd C=1024", t(lambda: H.hfta_bn_max_bwd(B, N, L, 1024, 1, tin(G), tin(X), H.ptr(am), H.ptr(g), H.ptr(be),
                                                    1024, H.ptr(sm), H.ptr(si), 1, 0.0, tout(dX), H.ptr(g), H.ptr(be),
                                                    H.ptr(ws), ws.numel(), s)), 2 * B * R * 1024 * 2)
del dX
for (K, Nn) in ((128, 1024), (64, 128)):
    A = T(B, R, K)
    Wt = T(B, Nn, K)
    Y = T(B, R, Nn)
    bias = torch.zeros(B, Nn, device=dev)
    rep("linear fwd %dx%d" % (K, Nn), t(lambda: H.hfta_fused_linear_fwd(B, R, Nn, K, 1, tin(A), tin(Wt), H.ptr(bias), Nn,
                                                                        0, 0, tout(Y), s)), B * R * (K + Nn) * 2)
    dW = torch.empty(B, Nn, K, device=dev)
    dA = T(B, R, K)
    rep("linear bwd (dgrad+wgrad) %dx%d" % (K, Nn), t(lambda: H.hfta_fused_linear_bwd(
        B, R, Nn, K, 1, tin(Y), tin(A), tin(Wt), tout(dA), H.ptr(dW), Nn * K, K, None, 0, 0, H.ptr(ws), ws.numel(), s)),
        B * R * (2 * Nn + 2 * K) * 2)
    del A, Y, dA
x = torch.randn(R, 3, device=dev).to(bf)
W1 = T(B, 64, 3)
b1 = torch.zeros(B, 64, device=dev)
Y1 = T(B, R, 64)
rep("skinny fwd 3->64", t(lambda: H.hfta_fused_linear_fwd(B, R, 64, 3, 1, H.tin(x, 0, 3), tin(W1), H.ptr(b1), 64, 0, 0,
                                                          tout(Y1), s)), B * R * 64 * 2)
dW1 = torch.empty(B, 64, 3, device=dev)
dx = T(B, R, 3)
rep("skinny bwd 3->64 (dgrad+wgrad)", t(lambda: H.hfta_fused_linear_bwd(
    B, R, 64, 3, 1, tin(Y1), H.tin(x, 0, 3), tin(W1), tout(dx), H.ptr(dW1), 192, 3, None, 0, 0, H.ptr(ws), ws.numel(),
    s)), B * R * (2 * 64 + 3) * 2)
