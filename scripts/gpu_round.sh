MSW_MK=1 timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout 300 python scripts/mk_timeline.py 2 > gpurun_out/mk_timeline_m2.txt 2>&1
for m in 2 1 0; do MSW_MK=1 timeout 300 python scripts/decode_once.py --mode $m --new 129 --reps 2 > gpurun_out/mk_decode_m$m.txt 2>&1; done
