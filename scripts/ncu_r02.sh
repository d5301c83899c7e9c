#!/bin/bash
# Round-2 ncu captures (one GPU, one kernel each), summarised into
# gpurun_out/ncu_r02.txt with scripts/ncu_metrics.py; reports are deleted
# after export to keep gpurun_out under the 64 MiB merge cap.
mkdir -p gpurun_out
out=gpurun_out/ncu_r02.txt; : > $out
cap() {  # tag, kernel regex, skip, command...
  tag=$1; rx=$2; skip=$3; shift 3
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 \
      -o gpurun_out/$tag "$@" > gpurun_out/$tag.log 2>&1
  ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.csv 2>/dev/null
  python scripts/ncu_metrics.py gpurun_out/$tag.csv "$tag" >> $out
  python - "$tag" >> $out <<'PY'
import csv, sys
tag = sys.argv[1]
try:
    rows = list(csv.reader(open(f"gpurun_out/{tag}.csv")))
    h, v = rows[0], rows[2]
    for k in ("lts__t_bytes.sum", "lts__t_sectors_srcunit_tex.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
        if k in h: print(f"  {k:72s} {v[h.index(k)]}")
except Exception as ex:
    print("  (no report)", ex)
PY
  rm -f gpurun_out/$tag.ncu-rep gpurun_out/$tag.csv
}
cap w4_gemv_gate_up gemv_w4_kernel 12 python scripts/gemv_micro.py 2 gate_up
cap gemm_f16_t1024 gemm_tc_kernel 2 python scripts/gemm_tc_probe.py 0 28672 4096 1024 1
cap gemm_f16_t4096 gemm_tc_kernel 2 python scripts/gemm_tc_probe.py 0 28672 4096 4096 1
cap gemm_w4_t1024 gemm_tc_kernel 2 python scripts/gemm_tc_probe.py 2 28672 4096 1024 1
cap attn_prefill_tc05_1900 attn_prefill_tc05 8 python scripts/decode_once.py --mode 0 --prompt 1900 --new 2
