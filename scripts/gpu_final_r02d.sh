mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
timeout -s KILL 900 python bench.py --workload mix --mix-per-class 4 --decisions-out gpurun_out/mix_decisions.csv > gpurun_out/bench_mix.log 2>&1
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.log 2>&1
