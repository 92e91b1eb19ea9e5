import sys, torch
sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H
H.hfta_init(0)
B, R = 64, 80000
s = torch.cuda.current_stream().cuda_stream
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for (K, N) in [(64, 128), (128, 128), (128, 64), (64, 64)]:
    X = torch.randn(B, R, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(B, N, K, device="cuda").to(torch.bfloat16)
    Y = torch.empty(B, R, N, device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(B, N, device="cuda")
    ms = t(lambda: H.hfta_fused_linear_fwd(B, R, N, K, 1, H.tin(X, R*K, K), H.tin(W, N*K, K), H.ptr(bias), N, 0, 0, H.tout(Y, R*N, N), s))
    gb = B * R * (K + N) * 2 / 1e9
    print("plain fwd K=%d N=%d: %.3f ms  %.0f GB/s" % (K, N, ms, gb / ms * 1e3))
    del X, W, Y
