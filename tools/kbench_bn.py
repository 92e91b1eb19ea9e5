"""BatchNorm kernel microbenchmark at the PointNet-seg head shapes (bf16,
B models x R = 80 000 rows, C in {512, 256, 128}) through the C ABI,
CUDA-event timed.  The knobs HFTA_BN_RUN / _S1 / _S2 / _BWD_BPS / _BPS are read
once per process, so `--sweep` re-runs this script per configuration.
Usage: python tools/kbench_bn.py [B] | python tools/kbench_bn.py --sweep [B]"""
import json
import os
import subprocess
import sys

CONFIGS = [
    {},
    {"HFTA_BN_S1": "8"},
    {"HFTA_BN_S2": "4"},
    {"HFTA_BN_RUN": "32"},
    {"HFTA_BN_RUN": "512"},
    {"HFTA_BN_RUN": "0"},
    {"HFTA_BN_BWD_BPS": "8"},
    {"HFTA_BN_BPS": "8"},
    {"HFTA_BN_BPS": "16"},
]


def run_one(B):
    import torch
    sys.path.insert(0, ".")
    import paper_2102_02344_b200.hfta as H
    H.hfta_init(0)
    R, dev, bf = 80000, "cuda", torch.bfloat16
    s = torch.cuda.current_stream().cuda_stream
    ws = torch.empty(1 << 30, dtype=torch.uint8, device=dev)

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

    g = torch.rand(B, 512, device=dev) + 0.5
    be = torch.rand(B, 512, device=dev) - 0.5
    sm, si = torch.empty(B, 512, device=dev), torch.empty(B, 512, device=dev)
    out = {}
    for C in (512, 256, 128):
        X, Y, D = [torch.randn(B, R, C, device=dev).to(bf) for _ in range(3)]
        tin = lambda x: H.tin(x, x[0].numel(), C)  # noqa: E731
        tout = lambda x: H.tout(x, x[0].numel(), C)  # noqa: E731
        el = B * R * C * 2
        st = t(lambda: H.hfta_fused_bn_fwd(B, R, C, 1, tin(X), H.ptr(g), H.ptr(be), 512, None, None, 0.1, 1e-5, 1, 0.0,
                                           H.tout(None, 0, C), H.ptr(sm), H.ptr(si), H.ptr(ws), ws.numel(), s))
        fw = t(lambda: H.hfta_fused_bn_fwd(B, R, C, 1, tin(X), H.ptr(g), H.ptr(be), 512, None, None, 0.1, 1e-5, 1, 0.0,
                                           tout(Y), H.ptr(sm), H.ptr(si), H.ptr(ws), ws.numel(), s))
        bw = t(lambda: H.hfta_fused_bn_bwd(B, R, C, 1, tin(D), tin(X), H.ptr(g), H.ptr(be), 512, H.ptr(sm), H.ptr(si),
                                           1, 0.0, tout(Y), H.ptr(g), H.ptr(be), 0, H.ptr(ws), ws.numel(), s))
        out[C] = {"stats_gbs": el / st / 1e6, "apply_gbs": 2 * el / max(fw - st, 1e-6) / 1e6,
                  "fwd_gbs": 3 * el / fw / 1e6, "bwd_gbs": 5 * el / bw / 1e6, "fwd_ms": fw, "bwd_ms": bw}
        del X, Y, D
    tot = sum(v["fwd_ms"] + v["bwd_ms"] for v in out.values())
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("HFTA_BN")}, "total_ms": tot,
                      "per_C": {c: {k: round(x, 3) for k, x in v.items()} for c, v in out.items()}}),
          flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--sweep":
        B = sys.argv[2] if len(sys.argv) > 2 else "64"
        for cfg in CONFIGS:
            env = {k: v for k, v in os.environ.items() if not k.startswith("HFTA_BN")}
            env.update(cfg)
            subprocess.run([sys.executable, __file__, B], env=env, timeout=300)
    else:
        run_one(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
