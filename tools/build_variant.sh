#!/bin/bash
# Build a tuning variant of libls_eval.so into ab/libls_eval_<name>.so:
#   tools/build_variant.sh g12f2r48 "-DLS_GATE_WARPS=12 -DLS_FP_WARPS=2 -DLS_RING_KB=48"
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2509_00217_b200/csrc
OUT=/tmp/variant_$NAME; mkdir -p $OUT $ROOT/ab
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v $DEFS"
rm -f $OUT/*.o
pids=()
for f in ls_tables ls_memo ls_evaluate ls_select ls_search ls_policy ls_capi; do
  nvcc $FLAGS -c -o $OUT/$f.o $SRC/$f.cu 2> $OUT/$f.ptxas &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "$NAME: compile failed (see $OUT/*.ptxas)" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/ab/libls_eval_$NAME.so $OUT/*.o -lcudart
grep -A2 "eval_ws_kernelILb1ELb0ELb1ELb1ELi4E" $OUT/ls_evaluate.ptxas | grep -E "registers|spill" | sed "s/^/$NAME: /"
