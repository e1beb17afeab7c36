"""Print one evaluation (tensorgen/gate rows .. energy kernel) of an ncu launch list CSV."""
import csv
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "": 1}
path = sys.argv[1]
min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
ids = {}
for r in rows:
    d = ids.setdefault(int(r["ID"]), {"k": r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1)
ks = sorted(ids)
st = [k for k in ks if "tensorgen" in ids[k]["k"] or "gate_rows" in ids[k]["k"]][0]
en = ([k for k in ks if "energy" in ids[k]["k"] and k > st] or [ks[-1]])[0]
tot = {}
for k in ks:
    if k < st or k > en:
        continue
    v = ids[k]
    t = v["gpu__time_duration.sum"]
    dr = v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
    a = tot.setdefault(v["k"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += t
    a[2] += dr
    if t * 1e6 >= min_us:
        print(f"{k:4d} {v['k']:24s} {t*1e6:8.1f} us {dr/1e6:9.1f} MB {dr/t/1e9 if t else 0:7.0f} GB/s")
for k, (n, t, dr) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:24s} launches {n:3d}  {t*1e6:8.1f} us  {dr/1e6:9.1f} MB")
print("total us", sum(v[1] for v in tot.values()) * 1e6)
