"""Summarise an ncu --metrics gpu__time_duration.sum CSV over ALL launches:
per-kernel count, total and average time, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hdr_i]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if not r[vi]:
        continue
    s = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:64]
    agg[s][0] += 1
    agg[s][1] += float(r[vi].replace(",", ""))
tot = sum(v for _, v in agg.values())
print(f"{'kernel':64s} {'n':>6s} {'sum_ms':>9s} {'avg_us':>8s} {'share':>6s}")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{k:64s} {c:6d} {v / 1e6:9.2f} {v / c / 1e3:8.2f} {100 * v / tot:5.1f}%")
print(f"total {sum(c for c, _ in agg.values())} launches, {tot / 1e6:.1f} ms (ncu: serialized, cold L2)")
