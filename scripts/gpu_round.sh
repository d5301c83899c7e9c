for t in 6 5; do timeout -s KILL 300 python scripts/repro_gemv_t6.py 4096 200 $t > gpurun_out/repro_$t.txt 2>&1; done
timeout -s KILL 300 python scripts/repro_gemv_t6.py 256 300 6 >> gpurun_out/repro_6.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "EXIT $?" >> gpurun_out/smoke.log
