# In-graph attribution of the batch-1 decode step: per-token time with
# kernel classes dropped from the captured step (MSW_SKIP, diagnostics only).
mode=${1:-2}
out=gpurun_out/step_attrib_m${mode}.txt
: > $out
for sk in "" attn argmax head "qkv" "o,oonly" gu down "qkv,o,oonly,gu,down" "qkv,o,oonly,gu,down,attn,head,argmax"; do
  r=$(MSW_ENGINE_SO=libmsw_engine_trace.so MSW_SKIP="$sk" timeout 300 python scripts/decode_once.py --mode $mode --new 129 --reps 2 2>&1 | tail -1)
  echo "skip=[$sk] $r" >> $out
done
