"""PointNet-seg head forward GEMM microbenchmark through the C ABI (bf16):
the point part of head c1 (K = 64 -> N = 512 over R = 80 000 rows per model,
row-grouped bias table: one bias row per cloud of L = 2500 points) and c2
(512 -> 256), each with and without the epilogue BN statistics; CUDA-event
timed, HBM GB/s from the bytes each call must move.
Usage: python tools/kbench_head.py [B]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2102_02344_b200.hfta as H  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    H.hfta_init(0)
    R, L, dev, bf = 80000, 2500, "cuda", torch.bfloat16
    s = torch.cuda.current_stream().cuda_stream
    g = torch.Generator(device=dev).manual_seed(0)

    def t(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out = {}
    for name, K, N, table in (("c1_point", 64, 512, True), ("c2", 512, 256, False), ("c3", 256, 128, False)):
        X = torch.randn(B, R, K, device=dev, generator=g).to(bf)
        W = (torch.randn(B, N, K, device=dev, generator=g) / K ** 0.5).to(bf)
        Y = torch.empty(B, R, N, device=dev, dtype=bf)
        if table:
            bias = torch.randn(B, R // L, N, device=dev, generator=g)
            bargs = (H.ptr(bias), (R // L) * N, N, L)
        else:
            bias = torch.randn(B, N, device=dev, generator=g)
            bargs = (H.ptr(bias), N, 0, 0)
        cs = torch.empty(H.hfta_linear_colstat_size(B, R, N) // 4, device=dev)
        xi, wi, yo = H.tin(X, R * K, K), H.tin(W, N * K, K), H.tout(Y, R * N, N)
        plain = t(lambda: H.hfta_fused_linear_fwd(B, R, N, K, H.HFTA_BF16, xi, wi, *bargs, yo, s))
        stats = t(lambda: H.hfta_fused_linear_fwd_stats(B, R, N, K, xi, wi, *bargs, yo, H.ptr(cs), s))
        byt = B * R * (K + N) * 2
        out[name] = {"ms_plain": round(plain, 4), "ms_stats": round(stats, 4),
                     "gbs_plain": round(byt / plain / 1e6, 1),
                     "gbs_stats": round((byt + cs.numel() * 4) / stats / 1e6, 1)}
        del X, W, Y, cs
    print(json.dumps({"B": B, "R": R, **out}))


if __name__ == "__main__":
    main()
