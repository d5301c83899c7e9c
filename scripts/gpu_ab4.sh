mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_gpu.log
bash scripts/ab_decode.sh 2 3 main prev > gpurun_out/ab_w4.txt 2>&1
bash scripts/ab_decode.sh 1 1 main prev > gpurun_out/ab_i8.txt 2>&1
bash scripts/ab_decode.sh 0 1 main prev > gpurun_out/ab_f16.txt 2>&1
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
