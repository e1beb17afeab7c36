import csv, io, json
for f in ["gpurun_out/b_c4.json", "gpurun_out/b_c3d.json"]:
    try:
        d = json.load(open(f))
        print(f, round(d["value"], 1), round(d["ms_per_step"], 3), d["config"]["energy_set0"])
    except Exception as e:
        print(f, "ERR", e)
for l in open("gpurun_out/c5_sweep.json"):
    try:
        d = json.loads(l); print("c5", d["w"], d["m"], round(d["gbs"]), round(d["frac"], 3))
    except Exception:
        pass
lines = [l for l in open("gpurun_out/launches_c4b.csv") if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
by = {}
for r in rows:
    by.setdefault(r["ID"], {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
tot = 0
for i, (k, v) in enumerate(sorted(by.items(), key=lambda kv: int(kv[0]))):
    t = v["gpu__time_duration.sum"][0] * (1e-3 if v["gpu__time_duration.sum"][1] == "ns" else 1)
    tot += t
    if t > 30:
        print(i, round(t, 1), "us", v["dram__bytes_read.sum"][0] / 1e6, v["dram__bytes_write.sum"][0] / 1e6)
print("total us", tot)
