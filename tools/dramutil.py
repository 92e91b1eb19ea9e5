"""Per-kernel DRAM bandwidth from an ncu --csv launch list collected with
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum (the
profile job's metric set).  usage: python tools/dramutil.py launches.csv [top]"""
import collections
import csv
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "KB": 1e3, "MB": 1e6, "GB": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "B": 1}
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: j for j, h in enumerate(hdr)}
per = collections.defaultdict(dict)
names = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    lid = int(r[ix["ID"]])
    v = float(r[ix["Metric Value"]].replace(",", "")) * UNITS.get(r[ix["Metric Unit"]], 1.0)
    per[lid][r[ix["Metric Name"]]] = v
    n = r[ix["Kernel Name"]].replace("(anonymous namespace)::", "")
    names[lid] = n.split("(")[0][:90]
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
T = 0.0
for lid, m in per.items():
    a = agg[names[lid]]
    t = m.get("gpu__time_duration.sum", 0.0)
    a[0] += t
    a[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a[2] += 1
    T += t
print("%9s %7s %9s %8s %4s  kernel" % ("ms", "share", "GB", "GB/s", "n"))
for k, (t, b, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%9.2f %6.2f%% %9.2f %8.0f %4d  %s" % (t * 1e3, 100 * t / T, b / 1e9, b / t / 1e9 if t else 0, n, k))
print("total %.2f ms" % (T * 1e3))
