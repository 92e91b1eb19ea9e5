"""Time-weighted tensor-pipe utilisation of a step (the analogue of DCGM
tensor_active) from an ncu --csv launch list collected with
  --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
usage: python tools/tcutil.py launches.csv [skip_launches]
Prints per-kernel time / TC-active % and the step's time-weighted TC %."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: j for j, h in enumerate(hdr)}
per = collections.defaultdict(dict)
names = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    lid = int(r[ix["ID"]])
    v = float(r[ix["Metric Value"]].replace(",", ""))
    m = r[ix["Metric Name"]]
    u = r[ix["Metric Unit"]]
    if m == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    per[lid][m] = v
    n = r[ix["Kernel Name"]]
    names[lid] = n.replace("(anonymous namespace)::", "").split("(")[0] + (
        "<" + n.split("<", 1)[1].split(">(")[0] + ">" if "<" in n else "")
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
T = W = 0.0
for lid in sorted(per)[skip:]:
    t = per[lid].get("gpu__time_duration.sum", 0.0)
    u = per[lid].get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    a = agg[names[lid]]
    a[0] += t
    a[1] += t * u
    a[2] += 1
    T += t
    W += t * u
print("%8s %8s %6s %5s  %s" % ("us", "share", "TC%", "n", "kernel"))
for k, (t, w, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
    print("%8.1f %7.2f%% %6.1f %5d  %s" % (t, 100 * t / T, w / t if t else 0, n, k[:100]))
print(json.dumps({"step_time_us": T, "tc_util_time_weighted_pct": W / T if T else 0.0, "launches": sum(a[2] for a in agg.values())}))
