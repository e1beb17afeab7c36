"""Key metrics + top stall reasons of every kernel in an ncu report (dev tool)."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
for row in r[2:]:
    print(row[hdr.index("ID")], row[hdr.index("Kernel Name")][:60])
    for w in WANT:
        if w in hdr:
            print("   ", w, row[hdr.index(w)], r[1][hdr.index(w)])
    vals = []
    for i, k in enumerate(hdr):
        if "average_warps_issue_stalled" in k and "per_issue_active" in k:
            try:
                vals.append((float(row[i].replace(",", "")), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("    stalls", [(k, round(v, 2)) for v, k in sorted(vals, reverse=True)[:7]])
