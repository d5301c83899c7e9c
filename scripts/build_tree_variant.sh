#!/bin/bash
# A/B helper: build lib/libmsw_engine_<name>.so from a whole source tree
# (e.g. `git archive <rev> paper_2605_23057_b200/csrc include | tar -x -C <dir>`),
# product flags. usage: scripts/build_tree_variant.sh <name> <tree dir>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; tree=$2
E=$tree/paper_2605_23057_b200/csrc/engine
mkdir -p $ROOT/build/variant_$name
objs=""
for s in $E/*.cu; do
  o=$ROOT/build/variant_$name/$(basename $s).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I $tree/include -I $E -c $s -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o $ROOT/paper_2605_23057_b200/lib/libmsw_engine_$name.so $objs -lpthread -ldl -lrt
echo built lib/libmsw_engine_$name.so
