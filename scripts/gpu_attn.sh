mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_attention_gpu.py tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q > gpurun_out/pytest_attn.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_attn.log
timeout -s KILL 300 python scripts/attn_timeline.py 2 129 > gpurun_out/attn_tl129.txt 2>&1
timeout -s KILL 300 python scripts/attn_timeline.py 2 200 > gpurun_out/attn_tl.txt 2>&1
timeout -s KILL 300 python scripts/decode_once.py --mode 2 --new 129 --reps 2 > gpurun_out/dec_w4.txt 2>&1
timeout -s KILL 300 python scripts/decode_once.py --mode 0 --new 129 --reps 2 > gpurun_out/dec_f16.txt 2>&1
timeout -s KILL 300 python scripts/decode_once.py --mode 1 --new 129 --reps 2 > gpurun_out/dec_i8.txt 2>&1
