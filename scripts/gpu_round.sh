timeout -s KILL 600 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
for m in 2 1 0; do timeout -s KILL 200 python scripts/decode_once.py --mode $m --new 129 --reps 2 > gpurun_out/dec_m$m.txt 2>&1; done
for m in 2 1 0; do MSW_NO_L2_PREFETCH=1 timeout -s KILL 200 python scripts/decode_once.py --mode $m --new 129 --reps 2 > gpurun_out/dec_m${m}_nopf.txt 2>&1; done
