#!/usr/bin/env python
"""Summarise ncu reports for profiles/: key metrics per kernel as JSON.

usage: python tools/ncu_summary.py OUT.json REPORT.ncu-rep [REPORT2 ...]
       python tools/ncu_summary.py --launches OUT.json LAUNCHES.csv
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1.0, "ms": 1e-3,
        "us": 1e-6, "ns": 1e-9, "s": 1.0}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    d[k] = float(v) * UNIT.get(units[i], 1.0)
                except ValueError:
                    d[k] = v
        stalls = {h.split("stalled_")[1]: float(vals[i] or 0) for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        d["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        res.append(d)
    return res


def main():
    if sys.argv[1] == "--launches":
        out, path = sys.argv[2], sys.argv[3]
        agg = {}
        with open(path) as f:
            lines = [l for l in f if l.startswith('"')]
        for r in csv.DictReader(io.StringIO("".join(lines))):
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0][:120]
            ns = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1e-9) * 1e9
            a = agg.setdefault(name, {"launches": 0, "total_ns": 0.0})
            a["launches"] += 1
            a["total_ns"] += ns
        tot = sum(a["total_ns"] for a in agg.values())
        for a in agg.values():
            a["share"] = a["total_ns"] / tot if tot else 0.0
        json.dump({"source": path, "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["total_ns"]))},
                  open(out, "w"), indent=1)
        return
    out = sys.argv[1]
    kernels = {}
    for rep in sys.argv[2:]:
        per = {}
        for d in raw(rep):
            short = d["kernel"].split("(")[0].split("::")[-1].split("<")[0]
            rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
            d["dram_bytes_per_launch"] = (rd or 0) + (wr or 0)
            d["report"] = rep
            per.setdefault(short, []).append(d)
        for short, ds in per.items():
            if len(ds) == 1:
                kernels[short] = ds[0]
                continue
            # several launches of one kernel in one report (e.g. the level
            # launches of one set-major evaluation): metrics of the longest
            # launch, times and DRAM bytes summed over the captured launches
            big = dict(max(ds, key=lambda d: d.get("gpu__time_duration.sum", 0)))
            big["launches_summed"] = len(ds)
            big["time_sum_s"] = sum(d.get("gpu__time_duration.sum", 0) for d in ds)
            big["dram_bytes_per_launch"] = sum(d["dram_bytes_per_launch"] for d in ds)
            big["dram_bytes_note"] = "summed over the captured launches (one evaluation)"
            kernels[short] = big
    json.dump({"kernels": kernels}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
