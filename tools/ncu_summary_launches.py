"""Sum an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import csv
import sys
from collections import defaultdict

tot = defaultdict(float)
cnt = defaultdict(int)
with open(sys.argv[1]) as f:
    rows = [l for l in f if l.startswith('"')]
for r in csv.DictReader(rows):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.2f} ms over {sum(cnt.values())} launches")
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{tot[k]:10.3f} ms {100 * tot[k] / T:5.1f}%  {cnt[k]:5d}  {k}")
