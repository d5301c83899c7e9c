# A/B of the next-linear L2 prefetch (MSW_L2NEXT_KB) on 8B batch-1 decode, per mode
out=gpurun_out/l2next_ab.txt
: > $out
for mode in 2 1 0; do
for kb in 0 32 64 128 256 0 64; do
  r=$(MSW_ENGINE_SO=libmsw_engine_trace.so MSW_L2NEXT_KB=$kb timeout 300 python scripts/decode_once.py --mode $mode --new 129 --reps 3 2>&1 | tail -1)
  echo "mode=$mode kb=$kb $r" >> $out
done; done
