"""B sweep of the fused training step until HBM is full (BJ metric "vs B
(peak)"; the paper's curves run until the GPU is out of memory),
3 repeats per point with mean / min / max, peak
torch.cuda.max_memory_allocated per B.

  python tools/sweep.py --workload pointnet_cls --dtype bf16 [--steps 10] [--Bs 1,2,4,...]

Prints one JSON line per B and a final summary line {"peak": ...}; each point
replays a captured CUDA graph of the whole step (inputs resident), timed with
CUDA events on the compute stream.
"""
import argparse
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

DEFAULT_BS = [1, 2, 4, 8, 16, 32, 64, 96, 128, 192, 256, 384, 512, 768, 1024, 1536, 2048]


def point(args, B, device):
    import torch
    a = argparse.Namespace(**vars(args))
    a.B = B
    a.fast_init = B > 64          # identical initial parameters beyond 64 models (init cost only)
    torch.cuda.reset_peak_memory_stats(device)
    wl = bench.build_net(a, 0, 1, device)
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        wl.step()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    vals = []
    for _ in range(args.repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        vals.append(B * wl.samples * args.steps / (e0.elapsed_time(e1) / 1e3))
    mem = torch.cuda.max_memory_allocated(device)
    samples = wl.samples
    del g, wl
    gc.collect()
    torch.cuda.empty_cache()
    return dict(B=B, value=sum(vals) / len(vals), min=min(vals), max=max(vals), repeats=len(vals),
                ms_per_step=B * samples * 1e3 / (sum(vals) / len(vals)),
                peak_mem_gb=mem / 1e9)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="pointnet_cls", choices=["pointnet_cls", "pointnet_seg", "dcgan", "resnet18"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--Bs", default=",".join(map(str, DEFAULT_BS)))
    ap.add_argument("--N", type=int, default=32)
    ap.add_argument("--L", type=int, default=2500)
    ap.add_argument("--k", type=int, default=40)
    ap.add_argument("--k-seg", type=int, default=50)
    ap.add_argument("--N-dcgan", type=int, default=128)
    ap.add_argument("--N-resnet", type=int, default=128)
    ap.add_argument("--max-seconds", type=float, default=900.0)
    args = ap.parse_args()
    import torch
    import paper_2102_02344_b200.hfta as H
    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    H.hfta_init(0)
    t0 = time.time()
    rows = []
    oom_at = None
    for B in [int(b) for b in args.Bs.split(",")]:
        if time.time() - t0 > args.max_seconds:
            break
        try:
            r = point(args, B, device)
        except torch.cuda.OutOfMemoryError:
            oom_at = B
            gc.collect()
            torch.cuda.empty_cache()
            break
        except RuntimeError as e:          # allocator failures inside libhfta workspaces
            if "out of memory" in str(e).lower() or "CUDA" in str(e):
                oom_at = B
                gc.collect()
                torch.cuda.empty_cache()
                break
            raise
        r.update(workload=args.workload, dtype=args.dtype)
        rows.append(r)
        print(json.dumps(r), flush=True)
    best = max(rows, key=lambda r: r["value"]) if rows else None
    print(json.dumps({"summary": True, "workload": args.workload, "dtype": args.dtype, "peak": best,
                      "B1": rows[0] if rows else None, "first_oom_B": oom_at,
                      "B_max_fitted": rows[-1]["B"] if rows else None}), flush=True)


if __name__ == "__main__":
    main()
