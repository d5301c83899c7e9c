"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total time per
kernel name, count, share. Usage: ncu_sum.py launches.csv [skip_first_n]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = defaultdict(lambda: [0, 0.0])
for r in rows[skip:]:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0][:90]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v = v / 1000.0 if unit == "ns" else (v if unit == "us" else v * 1000.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:10.1f} us {100 * t / tot:5.1f}% n={n:5d} avg={t / n:8.2f}  {k}")
