"""Summarise one kernel of an ncu report: headline metrics + top stall reasons + busiest units.
Usage: python tools/ncu_sum.py report.ncu-rep [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ki = h.index("Kernel Name")
for row in rows[2:]:
    if sub not in row[ki]:
        continue
    d = {}
    for i, k in enumerate(h):
        try:
            d[k] = float(row[i].replace(",", ""))
        except ValueError:
            pass
    print("kernel:", row[ki][:100])
    for k in ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "lts__t_bytes.sum", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread"]:
        if k in d:
            print("  %-75s %g" % (k, d[k]))
    st = sorted(((v, k) for k, v in d.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")),
                reverse=True)[:8]
    print("  top stall samples:")
    for v, k in st:
        print("    %-70s %g" % (k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v))
    top = sorted(((v, k) for k, v in d.items() if k.endswith(".avg.pct_of_peak_sustained_elapsed") and v > 30),
                 reverse=True)[:10]
    print("  busiest units (% of peak, elapsed):")
    for v, k in top:
        print("    %-70s %.1f" % (k, v))
