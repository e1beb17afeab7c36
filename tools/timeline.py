#!/usr/bin/env python
"""Kernel timeline of one evaluation (CUPTI via torch.profiler): every
kernel launch with its start/duration, also inside the captured graph.

usage: python tools/timeline.py WORKLOAD [--sets A] [--slices k] [--out FILE.json]

Prints per kernel name: launches, summed duration, and the evaluation's
wall span; writes the raw event list (name, ts_us, dur_us, stream) to --out.
"""
import argparse
import re
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("--sets", type=int, default=0)
    ap.add_argument("--slices", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_2106_15740_b200 as Q

    wl = bench.WORKLOADS[a.workload]
    args = bench.parse_args(["--workload", a.workload, "--slices", str(a.slices)])
    graph, jobs, _ = bench.plan_jobs(wl, args, wl["dtype"], 1, 0)
    plan = Q.EnergyPlan(graph, wl["p"], wl["mode"], dtype=wl["dtype"], jobs=jobs)
    A = a.sets or wl["sets"]
    ang = torch.from_numpy(bench.angle_sets(wl["p"], A)).cuda()
    st = torch.cuda.current_stream()
    for _ in range(5):
        plan.execute_only(ang, st)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            plan.execute_only(ang, st)
            torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        m = re.search(r"(\w+_kernel\w*)", e.name)
        ev.append({"name": m.group(1) if m else e.name[:40],
                   "ts": e.time_range.start, "dur": e.time_range.end - e.time_range.start})
    ev.sort(key=lambda x: x["ts"])
    # split into evaluations at gaps > 50 us
    runs, cur = [], []
    for x in ev:
        if cur and x["ts"] - max(c["ts"] + c["dur"] for c in cur[-8:]) > 50:
            runs.append(cur)
            cur = []
        cur.append(x)
    if cur:
        runs.append(cur)
    last = runs[-1]
    t0 = last[0]["ts"]
    span = max(x["ts"] + x["dur"] for x in last) - t0
    tot = {}
    for x in last:
        d = tot.setdefault(x["name"], [0, 0.0])
        d[0] += 1
        d[1] += x["dur"]
    print(f"{a.workload}: {len(last)} kernels, span {span:.1f} us, summed {sum(d[1] for d in tot.values()):.1f} us")
    for k, (n, d) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:28s} {n:5d} launches {d:9.1f} us")
    if a.out:
        with open(a.out, "w") as f:
            json.dump([{"name": x["name"], "ts_us": x["ts"] - t0, "dur_us": x["dur"]} for x in last], f)


if __name__ == "__main__":
    main()
