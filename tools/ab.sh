#!/bin/bash
# A/B timing of two builds of libls_eval.so on the same box:
#   tools/ab.sh ab/libls_eval_base.so paper_2509_00217_b200/libls_eval.so [prof_eval args...]
A=$1; B=$2; shift 2
for r in 1 2; do
  for L in "$A" "$B"; do
    echo "== $L"
    LS_EVAL_LIB=$(realpath "$L") python tools/prof_eval.py "$@" 2>&1 | grep evaluate | tail -n 3
  done
done
