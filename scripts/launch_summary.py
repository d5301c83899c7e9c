"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel share of
one decode step (the launches between the last two `advance` kernels)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hdr_i]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ks = [(r[ki], float(r[vi])) for r in rows[hdr_i + 1:] if r[vi]]
idx = [i for i, (k, _) in enumerate(ks) if "advance" in k]
step = ks[idx[-2] + 1: idx[-1] + 1]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in step:
    s = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:64]
    agg[s][0] += 1
    agg[s][1] += v
tot = sum(v for _, v in step)
print(f"{'kernel':64s} {'n':>4s} {'sum_us':>9s} {'avg_us':>8s} {'share':>6s}")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:64s} {c:4d} {v / 1e3:9.1f} {v / c / 1e3:8.2f} {100 * v / tot:5.1f}%")
print(f"one decode step: {len(step)} launches, {tot / 1e3:.1f} us (ncu: serialized, cold L2)")
