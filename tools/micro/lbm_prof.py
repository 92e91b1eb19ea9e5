"""Per-role wait-cycle attribution of k_lbm_fwd (developer build with
HFTA_NVCC_EXTRA=-DHFTA_LBM_PROF).  Usage: python tools/micro/lbm_prof.py [B]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H  # noqa: E402

H.hfta_init(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
N, L, C, K = 32, 2500, 1024, 128
R = N * L
X = torch.relu(torch.randn(B, R, K, device="cuda")).to(torch.bfloat16)
W = (torch.randn(B, C, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
g = torch.rand(B, C, device="cuda") + 0.5
be = torch.zeros(B, C, device="cuda")
G = torch.empty(B, N, C, device="cuda"); ext = torch.empty(B, N, C, device="cuda")
am = torch.empty(B, N, C, dtype=torch.int32, device="cuda")
sm, si = torch.empty(B, C, device="cuda"), torch.empty(B, C, device="cuda")
ws = torch.empty(H.hfta_fused_linear_bn_max_workspace(B, N, L, C, K), dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
gram, xsum = torch.empty(B, K, K, device="cuda"), torch.empty(B, K, device="cuda")
for _ in range(3):
    H.hfta_fused_linear_bn_max_fwd(B, N, L, C, K, 1, H.tin(X, R * K, K), H.tin(W, C * K, K), None, 0, H.ptr(g),
                                   H.ptr(be), C, None, None, 0.1, 1e-5, 1, 0.0, H.tout(G, N * C, C), H.ptr(am),
                                   H.tout(ext, N * C, C), H.ptr(sm), H.ptr(si), H.ptr(gram), H.ptr(xsum), H.ptr(ws),
                                   ws.numel(), s)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (512 * 8))()
H._lib.hfta_lbm_prof_dump(buf, 512)
a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 8).astype(np.float64)
a = a[a[:, 7] > 0]
units = B * N / (a.shape[0] / 4)
nch = units * ((L + 127) // 128)
print("CTAs %d, ~%.0f chunks per CTA" % (a.shape[0], nch))
names = ["prod empty wait", "-", "mma tempty wait", "mma full wait", "epi tfull wait", "epi hold", "-", "total"]
lead = a[a[:, 2] + a[:, 3] > 0]
for i, nm in enumerate(names):
    if nm == "-":
        continue
    src = lead if i in (2, 3) else a
    print("%-16s mean %10.0f cyc  per chunk %7.1f" % (nm, src[:, i].mean(), src[:, i].mean() / nch))
