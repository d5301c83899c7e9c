mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout -s KILL 300 python scripts/gemv_micro.py 2,1,0 > gpurun_out/gemv_micro_all.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w4.csv python scripts/decode_once.py --mode 2 --new 4 > gpurun_out/ncu2.log 2>&1
