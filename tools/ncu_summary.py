"""One-line-per-kernel summary of ncu --set full captures (profiles/ncu_r02/*.ncu-rep)."""
import csv
import glob
import io
import subprocess
import sys

W = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size"]
for f in sorted(glob.glob(sys.argv[1] + "/*.ncu-rep")):
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")].split("(")[0].replace("unnamed>::", "")
    print("%s: %s" % (f.split("/")[-1], name))
    print("   " + "  ".join("%s=%s%s" % (w.split(".")[0].replace("__", ".") if "pct" not in w else w.split("__")[1].split(".")[0] + "%",
                                        v[h.index(w)], u[h.index(w)] if "pct" not in w else "") for w in W if w in h))
