ncu --set full --import-source on --clock-control none -k regex:gemv_w4 -s 3 -c 1 -o gpurun_out/w4_gu python scripts/gemv_micro.py 2 gate_up > gpurun_out/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w4.csv python scripts/decode_once.py --mode 2 --new 4 > gpurun_out/ncu2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_int8.csv python scripts/decode_once.py --mode 1 --new 4 > gpurun_out/ncu3.log 2>&1
timeout 300 python scripts/gemv_micro.py 2,1,0 > gpurun_out/gemv_micro_all.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 900 python bench.py --workload configs > gpurun_out/bench_configs.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
