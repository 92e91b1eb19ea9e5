"""Quick tcgen05 GEMM check through the C ABI (bf16) against numpy fp64."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H
H.hfta_init(0)
R = np.random.default_rng(0)
s = torch.cuda.current_stream().cuda_stream


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


for (B, M, N, K) in [(1, 128, 128, 64), (2, 300, 128, 64), (3, 1000, 1024, 128), (2, 777, 64, 128),
                     (2, 1000, 256, 512), (2, 1000, 40, 256), (3, 2000, 128, 1024)]:
    X = torch.tensor(R.standard_normal((B, M, K)), dtype=torch.bfloat16, device="cuda")
    W = torch.tensor(R.standard_normal((B, N, K)) / np.sqrt(K), dtype=torch.bfloat16, device="cuda")
    bias = torch.tensor(R.standard_normal((B, N)), dtype=torch.float32, device="cuda")
    dY = torch.tensor(R.standard_normal((B, M, N)), dtype=torch.bfloat16, device="cuda")
    Y = torch.empty(B, M, N, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(B, M, K, dtype=torch.bfloat16, device="cuda")
    dW = torch.empty(B, N, K, dtype=torch.float32, device="cuda")
    ws = torch.empty(max(H.hfta_fused_linear_bwd_workspace(B, M, N, K, 1), 1), dtype=torch.uint8, device="cuda")
    H.hfta_fused_linear_fwd(B, M, N, K, 1, H.tin(X, M * K, K), H.tin(W, N * K, K), H.ptr(bias), N, 0, 0,
                            H.tout(Y, M * N, N), s)
    H.hfta_fused_linear_bwd(B, M, N, K, 1, H.tin(dY, M * N, N), H.tin(X, M * K, K), H.tin(W, N * K, K),
                            H.tout(dX, M * K, K), H.ptr(dW), N * K, K, None, 0, 0, H.ptr(ws), ws.numel(), s)
    torch.cuda.synchronize()
    x, w, dy = (t.double().cpu().numpy() for t in (X, W, dY))
    e = [rel(Y[b].double().cpu().numpy(), x[b] @ w[b].T + bias[b].double().cpu().numpy()) for b in range(B)]
    ed = [rel(dX[b].double().cpu().numpy(), dy[b] @ w[b]) for b in range(B)]
    ew = [rel(dW[b].double().cpu().numpy(), dy[b].T @ x[b]) for b in range(B)]
    print("B=%d M=%d N=%d K=%d  fwd %.1e  dgrad %.1e  wgrad %.1e" % (B, M, N, K, max(e), max(ed), max(ew)), flush=True)
