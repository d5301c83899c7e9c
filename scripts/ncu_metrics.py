"""Key metrics of an `ncu --page raw --csv` export (one kernel): time, DRAM
bytes, tensor-pipe / issue / warps-active utilisation, registers, smem, and
the top warp-stall reasons. Usage: ncu_metrics.py raw.csv [label]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
label = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tc.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x"]
print(f"== {label}")
for k in KEYS:
    for i, h in enumerate(hdr):
        if h == k or (k.endswith("*") and h.startswith(k[:-1])):
            print(f"  {h:72s} {vals[i][:110]} {units[i]}")
tc = [(h, vals[i]) for i, h in enumerate(hdr) if "pipe_tc" in h or "tcgen05" in h or "utcmma" in h.lower()]
for h, v in tc[:12]:
    print(f"  {h:72s} {v}")
st = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
        try:
            st.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in st) or 1.0
print("  top stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:6]))
