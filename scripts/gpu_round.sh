timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
for m in 2 1 0; do timeout -s KILL 200 python scripts/decode_once.py --mode $m --new 129 --reps 2 > gpurun_out/dec_m$m.txt 2>&1; done
timeout -s KILL 200 python scripts/decode_once.py --mode 2 --prompt 900 --new 129 --reps 1 > gpurun_out/dec_m2_long.txt 2>&1
timeout -s KILL 300 python scripts/attn_timeline.py 2 200 > gpurun_out/attn_tl.txt 2>&1
