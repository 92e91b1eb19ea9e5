"""Microbenchmark of the fused Linear->BN->max block (K10) at the bench shape
(B models x N=32 clouds x L=2500 points, K=128 -> C=1024, bf16), CUDA-event
timed after warm-up; prints ms and TFLOP/s per pass.  Usage:
  python tools/kbench_lbm.py [B] [reps]      (reps=1: one launch each, for ncu)"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H  # noqa: E402

H.hfta_init(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
N, L, C, K = 32, 2500, 1024, 128
R = N * L
dev = "cuda"
s = torch.cuda.current_stream().cuda_stream
X = torch.relu(torch.randn(B, R, K, device=dev)).to(torch.bfloat16)
W = (torch.randn(B, C, K, device=dev) / K ** 0.5).to(torch.bfloat16)
bias = torch.zeros(B, C, device=dev)
g = torch.rand(B, C, device=dev) + 0.5
be = torch.rand(B, C, device=dev) - 0.5
rm, rv = torch.zeros(B, C, device=dev), torch.ones(B, C, device=dev)
G, ext = torch.empty(B, N, C, device=dev), torch.empty(B, N, C, device=dev)
am = torch.empty(B, N, C, dtype=torch.int32, device=dev)
sm, si = torch.empty(B, C, device=dev), torch.empty(B, C, device=dev)
ws = torch.empty(H.hfta_fused_linear_bn_max_workspace(B, N, L, C, K), dtype=torch.uint8, device=dev)
dG = torch.randn(B, N, C, device=dev)
dX = torch.empty(B, R, K, dtype=torch.bfloat16, device=dev)
gram, xsum = torch.empty(B, K, K, device=dev), torch.empty(B, K, device=dev)
dW = torch.empty(B, C, K, device=dev)
dg, db, dbias = torch.empty(B, C, device=dev), torch.empty(B, C, device=dev), torch.empty(B, C, device=dev)


def fwd():
    H.hfta_fused_linear_bn_max_fwd(B, N, L, C, K, 1, H.tin(X, R * K, K), H.tin(W, C * K, K), H.ptr(bias), C, H.ptr(g),
                                   H.ptr(be), C, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, 1, 0.0, H.tout(G, N * C, C),
                                   H.ptr(am), H.tout(ext, N * C, C), H.ptr(sm), H.ptr(si), H.ptr(gram), H.ptr(xsum), H.ptr(ws),
                                   ws.numel(), s)


def bwd():
    H.hfta_fused_linear_bn_max_bwd(B, N, L, C, K, 1, H.tin(dG, N * C, C), H.tin(X, R * K, K), H.tin(W, C * K, K),
                                   H.ptr(am), H.tin(ext, N * C, C), H.ptr(bias), C, H.ptr(g), H.ptr(be), C, H.ptr(sm),
                                   H.ptr(si), H.ptr(gram), H.ptr(xsum), 1, 0.0, H.tout(dX, R * K, K), 1, 0.0, H.ptr(dW), C * K, K, H.ptr(dbias), C,
                                   H.ptr(dg), H.ptr(db), 0, H.ptr(ws), ws.numel(), s)


def t(fn):
    fn()
    torch.cuda.synchronize()
    if reps <= 1:
        return float("nan")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


fl = 2.0 * B * R * C * K
tf = t(fwd)
tb = t(bwd)
print("lbm fwd  %.3f ms  %.0f TFLOP/s (1x contraction)" % (tf, fl / tf / 1e9))
print("lbm bwd  %.3f ms  %.0f TFLOP/s (2x contraction; 4x incl. recompute: %.0f)" % (tb, 2 * fl / tb / 1e9,
                                                                                   4 * fl / tb / 1e9))
