"""Quick numeric check of the fp32 (3xTF32) contraction in all operand
majornesses: linear fwd (K/K), dgrad (K/MN), wgrad (MN/MN) vs float64 numpy."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H

H.hfta_init(0)
rng = np.random.default_rng(0)
s = torch.cuda.current_stream().cuda_stream
for (B, M, N, K) in [(1, 256, 64, 64), (1, 256, 128, 64), (2, 1000, 64, 128), (1, 300, 128, 256), (2, 777, 96, 40)]:
    X = rng.standard_normal((B, M, K)).astype(np.float32)
    W = rng.standard_normal((B, N, K)).astype(np.float32)
    dY = rng.standard_normal((B, M, N)).astype(np.float32)
    Xd, Wd, dYd = (torch.tensor(a, device="cuda") for a in (X, W, dY))
    Y = torch.zeros(B, M, N, device="cuda")
    dX = torch.zeros(B, M, K, device="cuda")
    dW = torch.zeros(B, N, K, device="cuda")
    ws = torch.empty(H.hfta_fused_linear_bwd_workspace(B, M, N, K, 0) + 256, dtype=torch.uint8, device="cuda")
    H.hfta_fused_linear_fwd(B, M, N, K, 0, H.tin(Xd, M * K, K), H.tin(Wd, N * K, K), None, 0, 0, 0,
                            H.tout(Y, M * N, N), s)
    H.hfta_fused_linear_bwd(B, M, N, K, 0, H.tin(dYd, M * N, N), H.tin(Xd, M * K, K), H.tin(Wd, N * K, K),
                            H.tout(dX, M * K, K), H.ptr(dW), N * K, K, None, 0, 0, H.ptr(ws), ws.numel(), s)
    torch.cuda.synchronize()
    X64, W64, dY64 = X.astype(np.float64), W.astype(np.float64), dY.astype(np.float64)
    ry = X64 @ W64.transpose(0, 2, 1)
    rdx = dY64 @ W64
    rdw = dY64.transpose(0, 2, 1) @ X64
    e = lambda a, r: float(np.linalg.norm(a.cpu().numpy() - r) / np.linalg.norm(r))
    print("B%d M%d N%d K%d  Y %.2e  dX %.2e  dW %.2e  |dX| %.3g" % (B, M, N, K, e(Y, ry), e(dX, rdx), e(dW, rdw),
                                                                    float(dX.abs().max())), flush=True)
