mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py tests/test_attention_gpu.py -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_k.log
bash scripts/ab_cb.sh 3 main prev > gpurun_out/ab_cb.txt 2>&1
