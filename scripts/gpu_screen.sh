# AWQ4 and KV-compression screening modes on the closing build: 8B batch-1
# decode per-token ms (decode_once), KV compression vs FP16 at 8K context.
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/decode_once.py --mode 3 --new 129 --reps 3 > gpurun_out/dec_awq.txt 2>&1
timeout -s KILL 600 python scripts/decode_once.py --mode 9 --prompt 8192 --new 65 --reps 2 > gpurun_out/dec_kv8.txt 2>&1
timeout -s KILL 600 python scripts/decode_once.py --mode 0 --prompt 8192 --new 65 --reps 2 > gpurun_out/dec_f16_8k.txt 2>&1
timeout -s KILL 600 python scripts/decode_once.py --mode 2 --prompt 8192 --new 65 --reps 2 > gpurun_out/dec_w4_8k.txt 2>&1
