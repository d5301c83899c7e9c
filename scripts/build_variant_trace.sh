#!/bin/bash
# Trace-build variant of build_variant.sh: links against build/engine_trace objects (-DMSW_TRACE).
# build/engine with ONE source file replaced by <file.cu> (compiled with the
# product flags). Select it at run time with MSW_ENGINE_SO=libmsw_engine_<name>.so.
# EXTRA="-DMSW_TRACE" adds flags (e.g. the timeline probes).
# usage: scripts/build_variant.sh <name> <variant.cu> <replaced basename, e.g. gemv.cu>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; src=$2; repl=$3
E=$ROOT/paper_2605_23057_b200/csrc/engine
mkdir -p $ROOT/build/variant
o=$ROOT/build/variant/$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr $EXTRA -I $ROOT/include -I $E -c $src -o $o
objs=$(ls $ROOT/build/engine_trace/*.o | grep -v "/$repl.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o $ROOT/paper_2605_23057_b200/lib/libmsw_engine_$name.so $objs $o -lpthread -ldl -lrt
echo built lib/libmsw_engine_$name.so
