"""Launch-list roofline of a step: for every launch k of an ncu --csv launch
list collected with
  gpu__time_duration.sum, sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,
  dram__bytes_read.sum, dram__bytes_write.sum
(tools/final_job.sh), the least time the launch could take on this GPU is
  t_k = max(TC_k * dur_k,  bytes_k / BW)
-- the tensor-pipe work it executed at 100% pipe activity, or its DRAM
traffic at the measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs) -- and
the step's roofline fraction is sum_k t_k / sum_k dur_k.  Executed work, not
algorithmic (the Gram-form rewrites execute fewer flops than the method,
im2col-free convs no extra bytes); cold-cache, serialised launches with
clock-control none, so this is a property of the kernels, not of the graph
replay bench.py times.
usage: python tools/steproof.py launches.csv [launches.csv ...]"""
import collections
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "KB": 1e3, "MB": 1e6, "GB": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "B": 1, "%": 1.0}
TC = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
BW = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: j for j, h in enumerate(hdr)}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        lid = int(r[ix["ID"]])
        per[lid][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * UNITS.get(
            r[ix["Metric Unit"]], 1.0)
        names[lid] = r[ix["Kernel Name"]].replace("(anonymous namespace)::", "").split("(")[0][:80]
    return per, names


def main():
    for path in sys.argv[1:]:
        per, names = load(path)
        T = Tt = Tm = Tmin = 0.0
        bound = collections.defaultdict(float)
        worst = collections.defaultdict(lambda: [0.0, 0.0])
        for lid, m in per.items():
            dur = m.get("gpu__time_duration.sum", 0.0)
            tt = m.get(TC, 0.0) / 100.0 * dur
            tm = (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / BW
            t = max(tt, tm)
            T += dur; Tt += tt; Tm += tm; Tmin += t
            bound["tensor" if tt >= tm else "hbm"] += dur
            w = worst[names[lid]]
            w[0] += dur; w[1] += dur - t
        print(json.dumps({"launch_list": os.path.basename(path), "launches": len(per), "step_ms": round(T * 1e3, 3),
                          "min_ms": round(Tmin * 1e3, 3), "roofline_frac": round(Tmin / T, 4) if T else None,
                          "tensor_bound_share": round(bound["tensor"] / T, 4) if T else None,
                          "hbm_gbs": BW / 1e9}))
        print("   %8s %8s  kernel (largest gaps to their own bound)" % ("ms", "gap ms"))
        for k, (d, g) in sorted(worst.items(), key=lambda kv: -kv[1][1])[:6]:
            print("   %8.2f %8.2f  %s" % (d * 1e3, g * 1e3, k))


if __name__ == "__main__":
    main()
