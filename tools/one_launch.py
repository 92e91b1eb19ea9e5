"""One launch of a hot kernel at the bench shape, for `ncu --set full -c 1`.
Usage: python tools/one_launch.py c3fwd [B]   (PointNet c3: 128->1024 over
R = 32*2500 points per model, bf16, as in the bench's feat.c3:fwd probe)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H  # noqa: E402

H.hfta_init(0)
which = sys.argv[1] if len(sys.argv) > 1 else "c3fwd"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
R = 32 * 2500
s = torch.cuda.current_stream().cuda_stream
bf = torch.bfloat16
if which == "c3fwd":
    K, N = 128, 1024
    A = torch.randn(B, R, K, device="cuda").to(bf)
    W = torch.randn(B, N, K, device="cuda").to(bf)
    Y = torch.empty(B, R, N, device="cuda", dtype=bf)
    H.hfta_fused_linear_fwd(B, R, N, K, 1, H.tin(A, R * K, K), H.tin(W, N * K, K), None, 0, 0, 0,
                            H.tout(Y, R * N, N), s)
torch.cuda.synchronize()
print("ok", which, B)
