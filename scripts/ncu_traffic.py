"""Per-launch DRAM traffic of a kernel from an ncu --set full report.
usage: python scripts/ncu_traffic.py REPORT.ncu-rep NNZ OUT.json
Writes {kernel, launches, dram_bytes_per_launch, duration_us_per_launch, nnz}."""
import csv
import io
import json
import subprocess
import sys

rep, nnz, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
metrics = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
units = rows[1]
data = rows[2:]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
per = []
for r in data:
    rd = float(r[col["dram__bytes_read.sum"]].replace(",", "")) * scale[units[col["dram__bytes_read.sum"]]]
    wr = float(r[col["dram__bytes_write.sum"]].replace(",", "")) * scale[units[col["dram__bytes_write.sum"]]]
    du = float(r[col["gpu__time_duration.sum"]].replace(",", "")) * scale[units[col["gpu__time_duration.sum"]]]
    per.append((r[col["Kernel Name"]], rd, wr, du))
k = len(per)
res = {"kernel": per[0][0].split("(")[0] if per else None, "launches": k, "nnz": nnz,
       "dram_bytes_per_launch": sum(p[1] + p[2] for p in per) / k,
       "dram_read_bytes_per_launch": sum(p[1] for p in per) / k,
       "dram_write_bytes_per_launch": sum(p[2] for p in per) / k,
       "duration_us_per_launch_ncu": sum(p[3] for p in per) / k,
       "per_launch": [{"read": p[1], "write": p[2], "us": p[3]} for p in per],
       "source": rep}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k_: v for k_, v in res.items() if k_ != "per_launch"}))
