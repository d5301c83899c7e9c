nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "EXIT $?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --workload configs > gpurun_out/bench_configs.log 2>&1; echo "EXIT $?" >> gpurun_out/bench_configs.log
