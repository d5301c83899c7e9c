mkdir -p gpurun_out
timeout -s KILL 300 python scripts/cb_once.py --n 64 --prompt 1024 --new 6 > gpurun_out/cb_once.txt 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cb.csv python scripts/cb_once.py --n 64 --prompt 1024 --new 6 > gpurun_out/ncu_cb.log 2>&1
