mkdir -p gpurun_out
MSW_ENGINE_SO=libmsw_engine_probe.so timeout -s KILL 300 python scripts/attn_timeline.py 2 129 > gpurun_out/attn_probe.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_attention_gpu.py -m gpu -x -q > gpurun_out/pytest_attn.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_attn.log
for v in main w8 main w8; do
  if [ $v = main ]; then so=libmsw_engine.so; else so=libmsw_engine_$v.so; fi
  echo "== $v" >> gpurun_out/ab.txt
  MSW_ENGINE_SO=$so timeout -s KILL 300 python scripts/decode_once.py --mode 2 --new 129 --reps 2 >> gpurun_out/ab.txt 2>&1
done
