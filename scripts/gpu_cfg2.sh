mkdir -p gpurun_out
timeout -s KILL 1200 python bench.py --workload configs --no-cpu-baseline > gpurun_out/bench_configs_nocpu.log 2>&1
timeout -s KILL 1200 python bench.py --workload configs > gpurun_out/bench_configs2.log 2>&1
