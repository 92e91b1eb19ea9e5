"""Microbenchmark of the Gram-form Linear->BN->ReLU layer (K11) at the
PointNet c2 shape (B models x R = 80 000 points, K = 64 -> N = 128, bf16),
CUDA-event timed.  Usage: python tools/kbench_bnl.py [B] [reps] [K] [N]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H  # noqa: E402

H.hfta_init(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
K = int(sys.argv[3]) if len(sys.argv) > 3 else 64
N = int(sys.argv[4]) if len(sys.argv) > 4 else 128
R = 32 * 2500
dev = "cuda"
s = torch.cuda.current_stream().cuda_stream
X = torch.relu(torch.randn(B, R, K, device=dev)).to(torch.bfloat16)
W = (torch.randn(B, N, K, device=dev) / K ** 0.5).to(torch.bfloat16)
bias = torch.zeros(B, N, device=dev)
g = torch.rand(B, N, device=dev) + 0.5
be = torch.rand(B, N, device=dev) - 0.5
rm, rv = torch.zeros(B, N, device=dev), torch.ones(B, N, device=dev)
A = torch.empty(B, R, N, dtype=torch.bfloat16, device=dev)
sm, si = torch.empty(B, N, device=dev), torch.empty(B, N, device=dev)
G, sv = torch.empty(B, K, K, device=dev), torch.empty(B, K, device=dev)
ws = torch.empty(H.hfta_fused_linear_bn_workspace(B, R, N, K), dtype=torch.uint8, device=dev)
dZ = torch.randn(B, R, N, device=dev).to(torch.bfloat16)
dX = torch.empty(B, R, K, dtype=torch.bfloat16, device=dev)
dW = torch.empty(B, N, K, device=dev)
dg, db, dbias = torch.empty(B, N, device=dev), torch.empty(B, N, device=dev), torch.empty(B, N, device=dev)


def fwd():
    H.hfta_fused_linear_bn_fwd(B, R, N, K, 1, H.tin(X, R * K, K), H.tin(W, N * K, K), H.ptr(bias), N, H.ptr(g),
                               H.ptr(be), N, H.ptr(rm), H.ptr(rv), 0.1, 1e-5, 1, 0.0, H.tout(A, R * N, N), H.ptr(sm),
                               H.ptr(si), H.ptr(G), H.ptr(sv), H.ptr(ws), ws.numel(), s)


def bwd():
    H.hfta_fused_linear_bn_bwd(B, R, N, K, 1, H.tin(dZ, R * N, N), H.tin(X, R * K, K), H.tin(W, N * K, K), H.ptr(bias),
                               N, H.ptr(g), N, H.ptr(sm), H.ptr(si), H.ptr(G), H.ptr(sv), H.tout(dX, R * K, K), 1, 0.0,
                               H.ptr(dW), N * K, K, H.ptr(dbias), N, H.ptr(dg), H.ptr(db), 0, H.ptr(ws), ws.numel(), s)


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


tf, tb = t(fwd), t(bwd)
gb = B * R * 2 / 1e9
print("bnl fwd %.3f ms (X %.2f GB + A %.2f GB)" % (tf, gb * K, gb * N))
print("bnl bwd %.3f ms (dZ %.2f GB, X %.2f GB, dX %.2f GB)" % (tb, gb * N, gb * K, gb * K))
