ncu --set full --import-source on --clock-control none -k regex:gemv_tf_kernel -s 12 -c 1 -o gpurun_out/w4_gu_l2 python scripts/gemv_micro.py 2 gate_up --l2 > gpurun_out/ncu_l2.log 2>&1
ncu -i gpurun_out/w4_gu_l2.ncu-rep --page raw --csv > gpurun_out/w4_gu_l2_raw.csv
ncu -i gpurun_out/w4_gu_l2.ncu-rep --page source --csv > gpurun_out/w4_gu_l2_src.csv 2>/dev/null
ls -la gpurun_out
