timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout -s KILL 900 python bench.py --workload configs > gpurun_out/bench_configs.log 2>&1
timeout -s KILL 1200 python bench.py --workload profile --profile-out gpurun_out/b200_profile.json > gpurun_out/bench_profile.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w4.csv python scripts/decode_once.py --mode 2 --new 4 > gpurun_out/ncu2.log 2>&1
timeout -s KILL 300 python scripts/attn_timeline.py 2 200 > gpurun_out/attn_tl.txt 2>&1
