timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout -s KILL 900 python bench.py --workload configs > gpurun_out/bench_configs.log 2>&1
timeout -s KILL 900 python bench.py --workload mix --mix-per-class 2 > gpurun_out/bench_mix.log 2>&1
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout -s KILL 1200 python bench.py --workload profile --profile-out gpurun_out/b200_profile.json > gpurun_out/bench_profile.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w4.csv python scripts/decode_once.py --mode 2 --new 4 > gpurun_out/ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 40 -c 1 -o gpurun_out/attn_dec2 python scripts/decode_once.py --mode 2 --new 4 --graphs 0 > gpurun_out/ncu3.log 2>&1
