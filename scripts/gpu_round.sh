timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout -s KILL 900 python bench.py --workload mix --mix-per-class 4 --decisions-out gpurun_out/mix_decisions.csv > gpurun_out/bench_mix.log 2>&1
