mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py tests/test_executor_gpu.py tests/test_dispatch_gpu.py -m gpu -x -q > gpurun_out/pytest_cb.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_cb.log
timeout -s KILL 1200 python bench.py --workload configs > gpurun_out/bench_configs3.log 2>&1
timeout -s KILL 1200 python bench.py --workload configs --no-cpu-baseline > gpurun_out/bench_configs4.log 2>&1
