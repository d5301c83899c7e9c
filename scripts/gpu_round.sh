timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout -s KILL 1200 python bench.py --workload profile --profile-out gpurun_out/b200_profile.json > gpurun_out/bench_profile.log 2>&1
