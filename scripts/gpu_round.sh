timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
for m in 2 1 0; do timeout -s KILL 200 python scripts/decode_once.py --mode $m --new 129 --reps 2 > gpurun_out/dec_m$m.txt 2>&1; done
MSW_ATTN_MERGE_O=1 timeout -s KILL 200 python scripts/decode_once.py --mode 2 --new 129 --reps 2 > gpurun_out/dec_m2_mo.txt 2>&1
timeout -s KILL 300 python scripts/gemv_micro.py 2 > gpurun_out/gemv_micro_w4.txt 2>&1
