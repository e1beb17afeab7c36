#!/usr/bin/env python
"""Copy one tools/round_measure.sh session (gpurun_out/r/) into profiles/.

usage: python tools/update_profiles.py [ROUND_TAG]   (default r01)
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = os.path.join(ROOT, "gpurun_out", "r")
P = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "": 1}


def last_json(path):
    lines = [l for l in open(path) if l.startswith("{")]
    return lines[-1] if lines else None


def summary(rep):
    out = os.path.join("/tmp", os.path.basename(rep) + ".json")
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), out, rep],
                   check=True)
    (k, v), = json.load(open(out))["kernels"].items()
    v["report"] = os.path.basename(v["report"])
    return v


def launch_eval(path):
    """Per-launch time/DRAM of the first complete evaluation in an ncu launch list."""
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    ids = {}
    for r in rows:
        d = ids.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"].split("(")[0].split("::")[-1]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1)
    keys = sorted(ids)
    start = [k for k in keys if "tensorgen" in ids[k]["kernel"]][0]
    end = [k for k in keys if "energy" in ids[k]["kernel"] and k > start][0]
    ev = [ids[k] for k in keys if start <= k <= end]
    agg = {}
    for v in ev:
        a = agg.setdefault(v["kernel"], {"launches": 0, "time_s": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["time_s"] += v["gpu__time_duration.sum"]
        a["dram_bytes"] += v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
    return agg, [{"kernel": v["kernel"], "time_us": v["gpu__time_duration.sum"] * 1e6,
                  "dram_MB": (v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / 1e6}
                 for v in ev]


def main():
    for src, dst in [("bench_config1", "config1"), ("bench_default", "config2"), ("bench_reference", "reference_config2"),
                     ("bench_config3", "config3"), ("bench_config3d", "config3d"),
                     ("bench_config4", "config4"), ("bench_config4_k3", "config4_k3")]:
        line = last_json(os.path.join(R, src + ".json"))
        if line:
            open(os.path.join(P, f"bench_{TAG}_{dst}.json"), "w").write(line)
    with open(os.path.join(P, f"config5_sweep_{TAG}.jsonl"), "w") as f:
        f.writelines(l for l in open(os.path.join(R, "config5_sweep.json")) if l.startswith("{"))
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), "--launches",
                    os.path.join(P, f"launches_{TAG}_config2.json"),
                    os.path.join(R, "launches_config2.csv")], check=True)
    agg, launches = launch_eval(os.path.join(R, "launches_config4.csv"))
    json.dump({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                         "dram__bytes_write.sum (serialised), one config-4 evaluation",
               "kernels": agg, "launches": launches},
              open(os.path.join(P, f"launches_{TAG}_config4.json"), "w"), indent=1)
    sm = summary(os.path.join(R, "prof_setmajor.ncu-rep"))
    smem = summary(os.path.join(R, "prof_smem.ncu-rep"))
    c5 = summary(os.path.join(R, "prof_stream_c5.ncu-rep"))
    s4 = agg.get("stream_kernel", {"launches": 0, "time_s": 0.0, "dram_bytes": 0.0})
    for src, dst in [("bench_config3d_noxt", "config3d_noxt"), ("bench_config4_noxt", "config4_noxt"),
                     ("bench_config3d_nowsum", "config3d_nowsum"), ("bench_config4_nowsum", "config4_nowsum")]:
        line = last_json(os.path.join(R, src + ".json")) if os.path.exists(os.path.join(R, src + ".json")) else None
        if line:
            open(os.path.join(P, f"bench_{TAG}_{dst}.json"), "w").write(line)
    f7 = os.path.join(R, "prof_fused_c3d.ncu-rep")
    y4 = agg.get("xt_kernel")
    x4 = agg.get("expand_kernel")
    out = {"note": "dram_bytes_per_launch: DRAM bytes (read+write) of the kernel for one "
                   "evaluation of the workload; for multi-launch executors (set-major levels, "
                   "streaming levels) summed over the launches of one evaluation",
           "kernels": {
               "sm_level_kernel_c64@config2": dict(sm, workload="config2: 150 edges x 1024 angle "
                                                              "sets, complex64 rows, one evaluation "
                                                              "= 15 level launches"),
               "xt_kernel@config4": dict(summary(os.path.join(R, "prof_xt_c4.ncu-rep")),
                                         workload="config4 edge #1058: the chain [1,22,21]->26, "
                                                  "[2,16,26]->25, three traces ->22 as one launch"),
               "smem_net_kernel@config2-16sets": dict(smem, workload="config2, 16 angle sets "
                                                                     "(warp-resident executor)"),
               "stream_kernel@config5": dict(c5, workload="config5 w=30 m=16, one launch"),
               "stream_kernel@config4": {"kernel": "stream_kernel",
                                         "workload": "config4 edge #1058, one contraction: its "
                                                     "stream_kernel level launches",
                                         "launches_summed": s4["launches"],
                                         "time_sum_s": s4["time_s"],
                                         "dram_bytes_per_launch": s4["dram_bytes"],
                                         "source": f"launches_{TAG}_config4.json"}}}
    out["kernels"]["hbm_executor@config4"] = {
        "kernel": "hbm_executor", "workload": "config4 edge #1058, one contraction: every "
                                              "launch of the evaluation",
        "launches_summed": sum(v["launches"] for v in agg.values()),
        "time_sum_s": sum(v["time_s"] for v in agg.values()),
        "dram_bytes_per_launch": sum(v["dram_bytes"] for v in agg.values()),
        "by_kernel": agg, "source": f"launches_{TAG}_config4.json"}
    c3d = os.path.join(R, "launches_config3d.csv")
    if os.path.exists(c3d):
        agg3, launches3 = launch_eval(c3d)
        json.dump({"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                             "dram__bytes_write.sum (serialised), one config-3-default evaluation",
                   "kernels": agg3, "launches": launches3},
                  open(os.path.join(P, f"launches_{TAG}_config3d.json"), "w"), indent=1)
        out["kernels"]["hbm_executor@config3-default"] = {
            "kernel": "hbm_executor", "workload": "config3 default, 366 edges, one evaluation",
            "launches_summed": sum(v["launches"] for v in agg3.values()),
            "time_sum_s": sum(v["time_s"] for v in agg3.values()),
            "dram_bytes_per_launch": sum(v["dram_bytes"] for v in agg3.values()),
            "by_kernel": agg3, "source": f"launches_{TAG}_config3d.json"}
    w4 = os.path.join(R, "prof_wsum_c4.ncu-rep")
    if os.path.exists(w4):
        out["kernels"]["wsum_kernel@config4"] = dict(summary(w4), workload="config4 edge #1058: the tail chain (rank-22 "
                                                     "intermediate, 22 buckets down to the scalar) as one weighted sum")
    if os.path.exists(f7):
        out["kernels"]["fused_kernel@config3-default"] = dict(summary(f7), workload="config3 default: one fused_kernel launch")
    if y4:
        out["kernels"]["xt_kernel@config4-all"] = {
            "kernel": "xt_kernel", "workload": "config4 edge #1058, one contraction: its xt_kernel launches",
            "launches_summed": y4["launches"], "time_sum_s": y4["time_s"],
            "dram_bytes_per_launch": y4["dram_bytes"], "source": f"launches_{TAG}_config4.json"}
    if x4:
        out["kernels"]["expand_kernel@config4-all"] = {
            "kernel": "expand_kernel", "workload": "config4 edge #1058, one contraction: its "
                                                   "expand_kernel launches",
            "launches_summed": x4["launches"], "time_sum_s": x4["time_s"],
            "dram_bytes_per_launch": x4["dram_bytes"], "source": f"launches_{TAG}_config4.json"}
    json.dump(out, open(os.path.join(P, f"ncu_full_{TAG}.json"), "w"), indent=1)
    for name in sorted(os.listdir(P)):
        if name.startswith("bench_"):
            d = json.loads(open(os.path.join(P, name)).read())
            print(name, round(d["value"], 1), (d.get("e2e") or {}).get("value"),
                  (d.get("roofline") or {}).get("frac"), (d.get("clocks") or {}).get("sm_mhz"))


if __name__ == "__main__":
    main()
