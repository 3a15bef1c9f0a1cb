"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum csv).
    python tools/launch_table.py gpurun_out/l_dc2.csv [steps]"""
import csv, io, re, sys
from collections import defaultdict
path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
txt = open(path).read()
txt = txt[txt.index('"ID"'):]
tot, cnt = defaultdict(float), defaultdict(int)
for row in csv.DictReader(io.StringIO(txt)):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    m = re.search(r"(\w+_kernel)", row["Kernel Name"])
    k = m.group(1) if m else row["Kernel Name"][:40]
    v = float(row["Metric Value"].replace(",", ""))
    unit = row.get("Metric Unit", "ns")
    v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    tot[k] += v
    cnt[k] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:32s} {cnt[k]:5d} {v:10.1f} us  {v / steps:9.1f} us/step  {100 * v / s:5.1f}%")
print(f"{'total':32s} {sum(cnt.values()):5d} {s:10.1f} us  {s / steps:9.1f} us/step")
