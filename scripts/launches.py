"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
idx = {h: k for k, h in enumerate(hdr)}
agg = defaultdict(lambda: [0.0, 0.0])
names = {}
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    key = int(r[idx["ID"]])
    names[key] = r[idx["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "")[:60]
    val = float(r[idx["Metric Value"]].replace(",", ""))
    met = r[idx["Metric Name"]]
    if met == "gpu__time_duration.sum":
        agg[key][0] = val / 1e3
    elif met.startswith("dram__bytes"):
        agg[key][1] += val / 1e6
for k in sorted(agg):
    t, b = agg[k]
    print(f"{k:3d} {names[k]:60s} {t:9.1f} us {b:9.1f} MB {b / t * 1e3 if t else 0:7.0f} GB/s")
if len(sys.argv) > 2 and sys.argv[2] == "--by-name":
    tot = defaultdict(lambda: [0, 0.0])
    for k in agg:
        tot[names[k]][0] += 1
        tot[names[k]][1] += agg[k][0]
    print("---- by kernel name ----")
    for n, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{n:60s} {c:6d} launches {t / 1e3:9.2f} ms  {t / c:8.1f} us avg")
