timeout -s KILL 60 python scripts/decode_once.py --mode 0 --target tiny --prompt 20 --new 5 --graphs 0 > gpurun_out/t1.log 2>&1; echo "EXIT $?" >> gpurun_out/t1.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
for m in 2 1 0; do timeout -s KILL 200 python scripts/decode_once.py --mode $m --new 129 --reps 2 > gpurun_out/dec_m$m.txt 2>&1; done
MSW_NO_ATTN_TAIL=1 timeout -s KILL 200 python scripts/decode_once.py --mode 2 --new 129 --reps 2 > gpurun_out/dec_m2_notail.txt 2>&1
