#!/usr/bin/env python
"""Benchmark of the HFTA fused training step on B200 (BJ metric: fused
models x samples / sec per B200).

Workload (BJ configs[1]): PointNet-cls, ModelNet40-shaped synthetic point
clouds (batch N=32, L=2500 points, k=40 classes), B fused models with
per-model hyper-parameters, bf16-AMP (per-point tensors bf16, per-sample
tensors/statistics/optimizer fp32), one step = forward + backward + fused
Adam over all B models.  Default B = the peak of the measured B sweep
(tools/sweep.py, profiles/sweep_r02_*.jsonl): 256 models per GPU for cls.  `value` = B * N * steps / time (device-timed, inputs
resident in HBM), summed over ranks (weak scaling: B models per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--B 256] [--dtype bf16|f32]
  python bench.py --impl reference ...   (the CPU oracle, bounded sample)
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused models x samples/sec per B200 (HFTA fused training step)"
UNIT = "model-samples/s"


def peaks():
    p = dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, sm_max_mhz=1965.0,
             source="fallback (B200_PROFILING.md)")
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: float(m[k]) for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained", "sm_max_mhz") if k in m})
        p["source"] = "measured (MEASURED_PEAKS.json)"
    except Exception:
        pass
    return p


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region (the
    recipe's clocks line) through NVML every 20 ms in a background thread;
    nvidia-smi as the fallback sampler."""
    BITS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device):
        self.device, self.rows, self.stop_ev = device, [], threading.Event()
        self.max_mhz = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def loop():
                while not self.stop_ev.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((float(sm), int(rs)))
                    except Exception:
                        pass
                    self.stop_ev.wait(0.02)
            self.th = threading.Thread(target=loop, daemon=True)
            self.th.start()
        except Exception:
            self.th = None

    def stop(self):
        if self.th is None:
            return None
        self.stop_ev.set()
        self.th.join(timeout=2)
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for _, m in self.rows for k, bit in self.BITS.items() if m & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "sampler": "nvml 20 ms"}


# ------------------------------------------------------------------ oracle --

def cpu_oracle_sample(n_samples=8, L=2500, k=40, steps=1):
    """The oracle as it stands (one model trained alone, NumPy fp64) on a
    bounded sample of the workload: n_samples point clouds of cfg2."""
    import synth
    from oracle import models as OM
    P = synth.init_params("pointnet_cls", 1000, k)
    x, y = synth.points_cls(0, N=n_samples, L=L, k=k)
    hp = synth.hparams_pointnet(7, 1)
    t0 = time.perf_counter()
    for t in range(1, steps + 1):
        OM.train_step("pointnet_cls", P, {}, {}, (x, y), t, OM.hp_of(hp, 0))
    dt = time.perf_counter() - t0
    return n_samples * steps / dt, dt


def run_reference(args, rank):
    if rank != 0:
        return
    n = args.ref_samples
    for _ in range(args.warmup):
        cpu_oracle_sample(n, args.L, args.k)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_oracle_sample(n, args.L, args.k)
    dt = time.perf_counter() - t0
    v = n * args.steps / dt
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "pointnet_cls cfg2 (BJ configs[1]) sample: 1 model x %d samples x %d points, "
                                   "k=%d, fp64 NumPy oracle (one model trained alone)" % (n, args.L, args.k)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "1 model x %d samples of cfg2 per step" % n},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------- step roofline --

def step_roofline(workload, dtype, value, pk, args):
    """Whole-step fraction of roofline: the method's algorithmic
    flops per model-sample (cls 4.1908, seg 15.0962 GFLOP,
    DCGAN 2.2746 GFLOP) at the sustained bf16 peak give the compute ceiling;
    the HBM ceiling of the deepest fusion schedule (S3, App. B5: 17.4 MB per
    model-sample for PointNet bf16) is the bytes floor.  frac = achieved /
    min(ceilings): the step's time vs the larger of its two lower bounds."""
    gf = {"pointnet_cls": 4.1908, "pointnet_seg": 15.0962, "dcgan": 2.2746,
          "resnet18": getattr(args, "resnet_gflop", None)}[workload]
    if workload == "pointnet_cls" and (args.N, args.L) != (32, 2500):
        return None
    peak_tf = pk["bf16_tflops_sustained"] if dtype == "bf16" else pk["bf16_tflops_sustained"] / 6.0
    comp = peak_tf * 1e12 / (gf * 1e9)
    hbm_mb = {"pointnet_cls": 17.4}.get(workload)
    hbm = pk["hbm_gbs"] * 1e9 / (hbm_mb * 1e6 * (1 if dtype == "bf16" else 2)) if hbm_mb else None
    ceiling = min(c for c in (comp, hbm) if c)
    return {"gflop_per_model_sample": gf, "compute_ceiling": comp, "hbm_ceiling_S3": hbm,
            "achieved_tflops": value * gf * 1e9 / 1e12, "frac": value / ceiling, "unit": UNIT,
            "peak": "sustained bf16 %.1f TF/s%s" % (pk["bf16_tflops_sustained"],
                                                   "" if dtype == "bf16" else " / 6 (fp32 = 3 tf32 MMAs at 1/2 rate)"),
            "note": "algorithmic flops of the method (fusion does no extra work, P:L729)"}


# -------------------------------------------------------------------- ours --

def build_net(args, rank, world, device):
    """Workload adapter: .net, .step() (inputs resident), .e2e_step() (pinned host
    inputs copied in, per-model losses read back), .loss (device [B]), h2d/d2h bytes."""
    import torch
    import synth
    from paper_2102_02344_b200 import shard
    B = args.B
    base, _ = shard.model_range(rank, world, B * world)   # weak scaling: B models per GPU

    class W:
        pass
    w = W()
    if args.workload in ("pointnet_cls", "pointnet_seg"):
        from paper_2102_02344_b200.pointnet import FusedPointNet
        task = args.workload.split("_")[1]
        k = args.k if task == "cls" else args.k_seg
        arch = "pointnet_" + task
        specs = [(n, s) for n, s, _ in synth.param_specs(arch, k)]
        if args.fast_init:   # identical initial parameters, different hyper-parameters
            P0 = synth.init_params(arch, 1000, k)
            Ps = [P0] * B
        else:
            Ps = [synth.init_params(arch, 1000 + base + b, k) for b in range(B)]
        hp = shard.slice_hparams(synth.hparams_pointnet(7, B * world), base, base + B)
        net = FusedPointNet(B, specs, Ps, hp, task=task, dtype=args.dtype, N=args.N, L=args.L, k=k, device=device,
                            model_offset=base)
        x, y = (synth.points_cls if task == "cls" else synth.points_seg)(0, N=args.N, L=args.L, k=k)
        net.set_batch(torch.tensor(x.reshape(-1, 3), dtype=torch.float32, device=device),
                      torch.tensor(y, dtype=torch.int32, device=device))
        xh = torch.from_numpy(x.reshape(-1, 3).astype(np.float32)).pin_memory()
        yh = torch.from_numpy(y.astype(np.int32).reshape(-1)).pin_memory()
        lh = torch.empty(B, dtype=torch.float32).pin_memory()
        xd, yd = torch.empty_like(xh, device=device), torch.empty_like(yh, device=device)

        def e2e_step():
            xd.copy_(xh, non_blocking=True)
            yd.copy_(yh, non_blocking=True)
            lh.copy_(net.step(xd, yd), non_blocking=True)
        w.net, w.step, w.e2e_step, w.loss = net, net.step, e2e_step, lambda: net.loss
        w.samples = args.N
        w.h2d, w.d2h = xh.numel() * 4 + yh.numel() * 4, B * 4
        w.x_host, w.y_host = x, y
        w.desc = "%s (BJ configs[%d]), N=%d clouds x %d points, k=%d" % (arch, 1 if task == "cls" else 2, args.N,
                                                                       args.L, k)
    elif args.workload == "resnet18":
        from paper_2102_02344_b200.resnet import FusedResNet18
        Nr = args.N_resnet
        specs = synth.param_specs("resnet18")
        if args.fast_init:
            Ps = [synth.init_params("resnet18", 1000)] * B
        else:
            Ps = [synth.init_params("resnet18", 1000 + base + b) for b in range(B)]
        hp = shard.slice_hparams(synth.hparams_resnet(3, B * world), base, base + B)
        net = FusedResNet18(B, specs, Ps, hp, N=Nr, dtype=args.dtype, device=device)
        x, y = synth.cifar(0, N=Nr)
        xh = torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 3, 1))).pin_memory()
        yh = torch.from_numpy(y.astype(np.int32)).pin_memory()
        xd, yd = torch.empty_like(xh, device=device), torch.empty_like(yh, device=device)
        xd.copy_(xh)
        yd.copy_(yh)
        net.set_inputs(xd, yd)
        lh = torch.empty(B, dtype=torch.float32).pin_memory()

        def e2e_step():
            xd.copy_(xh, non_blocking=True)
            yd.copy_(yh, non_blocking=True)
            net.set_inputs(xd, yd)
            lh.copy_(net.step(), non_blocking=True)
        w.net, w.step, w.e2e_step, w.loss = net, net.step, e2e_step, lambda: net.loss
        w.samples = Nr
        w.h2d, w.d2h = xh.numel() * 4 + yh.numel() * 4, B * 4
        args.resnet_gflop = net.flops_per_sample() / 1e9
        w.desc = "resnet18 (NEXT-4; torchvision BasicBlock, 10 classes), N=%d CIFAR-shaped 32x32 images, Adadelta" % Nr
    else:
        from paper_2102_02344_b200.dcgan import FusedDCGAN
        Nd = args.N_dcgan
        gs = [(n, s) for n, s, _ in synth.param_specs("dcgan_g")]
        ds = [(n, s) for n, s, _ in synth.param_specs("dcgan_d")]
        if args.fast_init:   # identical initial parameters, different hyper-parameters
            PG = [synth.init_params("dcgan_g", 1000)] * B
            PD = [synth.init_params("dcgan_d", 2000)] * B
        else:
            PG = [synth.init_params("dcgan_g", 1000 + base + b) for b in range(B)]
            PD = [synth.init_params("dcgan_d", 2000 + base + b) for b in range(B)]
        hp = shard.slice_hparams(synth.hparams_dcgan(3, B * world), base, base + B)
        net = FusedDCGAN(B, gs, ds, PG, PD, hp, N=Nd, dtype=args.dtype, device=device)
        real = synth.images(0, N=Nd).transpose(0, 2, 3, 1).astype(np.float32)
        z = np.stack([synth.noise(0, base + b, 1, N=Nd) for b in range(B)]).astype(np.float32)
        rh, zh = torch.from_numpy(np.ascontiguousarray(real)).pin_memory(), torch.from_numpy(z).pin_memory()
        rd, zd = torch.empty_like(rh, device=device), torch.empty_like(zh, device=device)
        rd.copy_(rh)
        zd.copy_(zh)
        net.set_inputs(rd, zd)
        lh = torch.empty(3, B, dtype=torch.float32).pin_memory()

        def e2e_step():
            rd.copy_(rh, non_blocking=True)
            zd.copy_(zh, non_blocking=True)
            net.set_inputs(rd, zd)
            e = net.step()
            for i in range(3):
                lh[i].copy_(e[i], non_blocking=True)
        w.net, w.step, w.e2e_step, w.loss = net, net.step, e2e_step, lambda: net.errG
        w.samples = Nd
        w.h2d, w.d2h = rh.numel() * 4 + zh.numel() * 4, 3 * B * 4
        w.desc = "dcgan 64x64 G+D (BJ configs[3]), N=%d images, per-model noise" % Nd
    return w


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2102_02344_b200.hfta as H
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    H.hfta_init(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    wl = build_net(args, rank, world, device)
    net = wl.net
    stream = torch.cuda.current_stream()
    B, N = args.B, wl.samples
    from paper_2102_02344_b200 import shard

    gatherer = shard.LossGather(B * world, world, device) if world > 1 else None

    def gather_losses():
        if gatherer is not None:
            gatherer.launch(wl.loss())      # C1: per-model losses only, on a side stream after an event

    # ---- device-timed region (inputs resident in HBM) ----
    for _ in range(args.warmup):
        wl.step()
        gather_losses()
    torch.cuda.synchronize()
    # The whole training step (all B models: forward, backward, optimizer) is
    # captured once as a CUDA graph and replayed (--no-graph: eager launches).
    graph = None
    l0 = H.hfta_launch_count()
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            wl.step()
        torch.cuda.synchronize()
        launches_per_step = H.hfta_launch_count() - l0
        graph.replay()                     # (warm replay; the captured step is a real step)
        torch.cuda.synchronize()

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            wl.step()
        gather_losses()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local_rank)
    clocks.start()
    l0 = H.hfta_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        run_step()
    if gatherer is not None:
        gatherer.wait()                 # the last step's gather belongs to the timed work
    e1.record(stream)
    torch.cuda.synchronize()
    launches = (launches_per_step * args.steps) if graph is not None else H.hfta_launch_count() - l0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = B * N * args.steps * world / (ms_max / 1e3)
    mem_peak = torch.cuda.max_memory_allocated(device)

    # ---- roofline probe: CUDA events around the probed kernel in eager steps ----
    probe_name = args.probe or {"pointnet_cls": "feat.c3:fwd", "pointnet_seg": "head.c2:fwd",
                                "dcgan": "D.c3:fwd", "resnet18": "l1.1.conv1:fwd"}[args.workload]
    probe_ms = []
    if probe_name:
        net.probe_arm(probe_name)
        for _ in range(3):
            wl.step()
        torch.cuda.synchronize()
        probe_ms = net.probe_collect()
        if args.workload == "dcgan":      # D runs 3 times per iteration: one launch per pass
            probe_ms = probe_ms[:3 * 3]

    # ---- end to end through the public API: pinned host inputs in, losses out ----
    graph_e2e = None
    if not args.no_graph:
        graph_e2e = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_e2e):
            wl.e2e_step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        if graph_e2e is not None:
            graph_e2e.replay()
        else:
            wl.e2e_step()
        gather_losses()
        stream.synchronize()            # the host reads the step's per-model losses
    f1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([f0.elapsed_time(f1)], device=device, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = B * N * args.steps * world / (float(te.item()) / 1e3)

    if rank == 0:
        pk = peaks()
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if args.dtype == "bf16" else "f32",
                "data": "synthetic (seeded inputs, random-init models of the named architecture)",
                "config": {"workload": wl.desc, "B_per_gpu": B, "batch": N, "precision": args.dtype,
                           "l2": "working set >> L2 (activations ~%.0f GB/step)" % (mem_peak / 1e9),
                           "parallelism": "model-array sharding, %d x %d models" % (world, B)},
                "gpu_launches": int(launches),
                "cuda_graph": graph is not None,
                "peak_mem_gb": mem_peak / 1e9,
                "clocks": clk,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(wl.h2d),
                        "d2h_bytes_per_step": int(wl.d2h)}}
        path = "tc" if args.dtype == "bf16" else "tf32x3"
        roof = net.probe_roofline(probe_name, probe_ms, pk, path=path) if probe_name else None
        line["step_roofline"] = step_roofline(args.workload, args.dtype, value, pk, args)
        try:   # DRAM traffic of the probed kernel from the committed ncu --set full capture
            key = probe_name + (":lbm" if getattr(net, "fuse_lbm", False) and ".c3:" in probe_name else "")
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic_r02.json")))[key]
            if path == "tc":
                roof["traffic"] = tr["dram_bytes_per_model"] * B
                roof["traffic_source"] = tr["source"]
        except Exception:
            pass
        line["roofline"] = roof
        if world == 1 and not args.no_serial and args.workload == "pointnet_cls":
            import serial_baselines as SB
            xd = torch.tensor(wl.x_host, dtype=torch.float32, device=device)
            yd = torch.tensor(wl.y_host, dtype=torch.int64, device=device)
            v_pt = SB.serial_pytorch(xd, yd, n_models=4, steps=3, warmup=2, dtype=args.dtype, device=device)
            import copy
            a1 = copy.copy(args)
            a1.B = 1
            w1 = build_net(a1, 0, 1, device)
            v_b1 = SB.serial_libhfta_b1(w1.net, steps=3, warmup=2)
            del w1
            line["serial"] = {"pytorch_eager_per_model_loop": v_pt, "libhfta_B1_loop": v_b1, "unit": UNIT,
                              "speedup_vs_pytorch_serial": value / v_pt, "speedup_vs_libhfta_B1": value / v_b1,
                              "note": "same-precision (%s) serial loops on this GPU, 4 / 1 models timed" % args.dtype}
        if world == 1 and not args.no_cpu_baseline and args.workload == "pointnet_cls":
            v, dt = cpu_oracle_sample(args.ref_samples, args.L, args.k)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                                    "sample": "1 model x %d samples of cfg2, one fp64 step (%.1f s)" %
                                              (args.ref_samples, dt)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--B", type=int, default=None,
                    help="models per GPU (default: the peak of the B sweep, profiles/sweep_r02_*.jsonl)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--N", type=int, default=32)
    ap.add_argument("--L", type=int, default=2500)
    ap.add_argument("--k", type=int, default=40)
    ap.add_argument("--k-seg", type=int, default=50)
    ap.add_argument("--N-dcgan", type=int, default=128)
    ap.add_argument("--N-resnet", type=int, default=128, help="ResNet-18 batch (P:L937: 128)")
    ap.add_argument("--probe", default=None, help="layer:fwd|bwd timed for the roofline (default: the workload's "
                    "dominant contraction)")
    ap.add_argument("--ref-samples", type=int, default=8)
    ap.add_argument("--fast-init", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-serial", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of the captured step graph")
    ap.add_argument("--workload", default="pointnet_cls", choices=["pointnet_cls", "pointnet_seg", "dcgan", "resnet18"])
    args = ap.parse_args()
    if args.B is None:      # peak of the measured B sweep (throughput flat within 1% beyond it)
        # (final sweeps profiles/sweep_r02c_*.jsonl: seg flat 58-59k from B = 32 to 192,
        # DCGAN 213k from 128, ResNet-18 705k at 512)
        args.B = {("pointnet_cls", "bf16"): 256, ("pointnet_seg", "bf16"): 96, ("dcgan", "bf16"): 128,
                  ("pointnet_cls", "f32"): 64, ("pointnet_seg", "f32"): 64, ("dcgan", "f32"): 64,
                  ("resnet18", "bf16"): 512, ("resnet18", "f32"): 128}[(args.workload, args.dtype)]
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
