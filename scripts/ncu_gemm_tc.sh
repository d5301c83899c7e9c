#!/bin/bash
# ncu --set full captures of the tcgen05 GEMM at 8B shapes (prefill T=128 and
# T=1024, continuous-batching T=64) for FP16 / INT8 / W4: one capture per
# case, metric summary into gpurun_out/gemm_tc_ncu.txt.
mkdir -p gpurun_out
out=gpurun_out/gemm_tc_ncu.txt; : > $out
for fmt in 0 1 2; do
  for case in "28672 4096 128" "28672 4096 1024" "4096 14336 64"; do
    set -- $case
    tag=gemm_tc_f${fmt}_n$1_k$2_t$3
    python scripts/gemm_tc_probe.py $fmt $1 $2 $3 5 >> $out 2>&1
    ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 2 -c 1 \
        -o gpurun_out/$tag python scripts/gemm_tc_probe.py $fmt $1 $2 $3 1 > /dev/null 2>&1
    ncu -i gpurun_out/$tag.ncu-rep --page raw --csv > gpurun_out/$tag.csv 2>/dev/null
    python scripts/ncu_metrics.py gpurun_out/$tag.csv "$tag" >> $out
    rm -f gpurun_out/$tag.ncu-rep gpurun_out/$tag.csv  # keep gpurun_out small (64 MiB merge cap)
  done
done
