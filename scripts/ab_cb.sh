# A/B of engine library variants on one 8B INT8 + continuous-batching cohort
# (64 requests, prompt 1024 -> 64 new): mean request ms and prefill ms.
# usage: bash scripts/ab_cb.sh <rounds> <variant> ...  ("main" = lib/libmsw_engine.so)
rounds=$1; shift
for r in $(seq $rounds); do
  for v in "$@"; do
    if [ "$v" = main ]; then so=libmsw_engine.so; else so=libmsw_engine_$v.so; fi
    echo "== $v $(MSW_ENGINE_SO=$so timeout -s KILL 300 python scripts/cb_once.py --n 64 --prompt 1024 --new 64 2>&1 | tail -1)"
  done
done
