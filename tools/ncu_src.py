"""Per-SASS-line warp-stall samples of one kernel in an ncu report (needs
--import-source / source page).  Prints the top lines and the lines around
mbarrier waits (SYNCS) with their samples.  Usage: python tools/ncu_src.py rep kernel-regex [N] [skip]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0      # which matching launch (0 = first)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
seen = {}
for r in rows[2:]:
    seen.setdefault(r[0], r)
data = list(seen.values())
si = hdr.index("Warp Stall Sampling (All Samples)")
ex = hdr.index("Instructions Executed")
tot = sum(int(r[si]) for r in data if r[si].isdigit())
print("total samples", tot)
for i, r in sorted(enumerate(data), key=lambda t: -int(t[1][si]) if t[1][si].isdigit() else 0)[:top]:
    print("%5d %6s %5.1f%% %9s  %s" % (i, r[si], 100 * int(r[si]) / tot, r[ex], r[1][:100]))
