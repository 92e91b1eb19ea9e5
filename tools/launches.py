"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
idx = {h: j for j, h in enumerate(hdr)}
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[start + 1:]:
    if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[idx["Kernel Name"]]
    name = name.replace("(anonymous namespace)::", "").split("(")[0] + ("<" + name.split("<", 1)[1].split(">(")[0] + ">" if "<" in name else "")
    v = float(r[idx["Metric Value"]].replace(",", ""))
    u = r[idx["Metric Unit"]]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}.get(u, 1.0)
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print("%-8s %12s %5s  %s" % ("share", "total_us", "n", "kernel"))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%6.2f%% %12.1f %5d  %s" % (100 * t / tot, t, n, k[:110]))
print("total_us %.1f over %d launches" % (tot, sum(n for n, _ in agg.values())))
