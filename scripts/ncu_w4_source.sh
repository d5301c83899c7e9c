#!/bin/bash
# W4 gate_up decode GEMV: one ncu --set full capture with source import;
# exports the per-SASS-line source page (stall samples) and raw metrics to
# CSV, then drops the report (gpurun_out merge cap).
mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemv_w4_kernel -s 12 -c 1 \
    -o gpurun_out/w4src python scripts/gemv_micro.py 2 gate_up > gpurun_out/w4src.log 2>&1
ncu -i gpurun_out/w4src.ncu-rep --page source --csv --print-source sass > gpurun_out/w4src_sass.csv 2>/dev/null
ncu -i gpurun_out/w4src.ncu-rep --page raw --csv > gpurun_out/w4src_raw.csv 2>/dev/null
ncu -i gpurun_out/w4src.ncu-rep --page details --csv > gpurun_out/w4src_details.csv 2>/dev/null
rm -f gpurun_out/w4src.ncu-rep
ls -la gpurun_out/w4src*
