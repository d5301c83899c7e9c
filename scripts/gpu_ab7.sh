mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_attention_gpu.py tests/test_engine_gpu.py tests/test_engine_8b_gpu.py -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; echo "EXIT $?" >> gpurun_out/pytest_k.log
bash scripts/ab_cb.sh 2 main prev > gpurun_out/ab_cb.txt 2>&1
for r in 1 2; do for v in main prev; do
  if [ $v = main ]; then so=libmsw_engine.so; else so=libmsw_engine_$v.so; fi
  echo "== $v $(MSW_ENGINE_SO=$so timeout -s KILL 600 python scripts/decode_once.py --mode 2 --prompt 8192 --new 65 --reps 2 2>&1 | tail -1)" >> gpurun_out/ab_8k.txt
done; done
