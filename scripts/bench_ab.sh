# A/B of engine library variants on the default decode bench (no CPU leg):
# bash scripts/bench_ab.sh <variant> ...  ("main" = lib/libmsw_engine.so)
for v in "$@"; do
  if [ "$v" = main ]; then so=libmsw_engine.so; else so=libmsw_engine_$v.so; fi
  echo "== $v"
  MSW_ENGINE_SO=$so bash "$(dirname "$0")/bench_quick.sh"
done
