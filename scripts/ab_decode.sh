# A/B of engine library variants on 8B batch-1 decode (prompt 128 -> 129 new):
# per-token ms of repeated requests, variants interleaved.
# usage: bash scripts/ab_decode.sh <mode> <rounds> <variant> ...  ("main" = lib/libmsw_engine.so)
mode=$1; rounds=$2; shift 2
for r in $(seq $rounds); do
  for v in "$@"; do
    if [ "$v" = main ]; then so=libmsw_engine.so; else so=libmsw_engine_$v.so; fi
    echo "== $v $(MSW_ENGINE_SO=$so timeout -s KILL 300 python scripts/decode_once.py --mode $mode --new 129 --reps 4 2>&1 | awk '/per_token_ms/{print $(NF-4)}' | tail -3 | tr '\n' ' ')"
  done
done
