"""Key counters of one kernel from an `ncu --set full` report, in the
`metric value unit` text format committed under profiles/ (bench.py reads the
dram__bytes lines as roofline.traffic). Usage: ncu_summary.py rep.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__shared_mem_per_block_static"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, d = rows[0], rows[1], rows[2]
col = {k: i for i, k in enumerate(h)}
if len(sys.argv) > 2:
    print("#", sys.argv[2])
print(f"{'Kernel Name':70s} {d[col['Kernel Name']][:150]}")
for k in KEYS:
    if k in col:
        print(f"{k:70s} {d[col[k]]} {units[col[k]]}")
stalls = []
for k, i in col.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            stalls.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[i])))
        except ValueError:
            pass
tot = sum(v for _, v in stalls) or 1.0
print("top stall reasons (share of warp samples):",
      [(k, round(v / tot, 3)) for k, v in sorted(stalls, key=lambda x: -x[1])[:8]])
