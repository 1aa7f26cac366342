#!/bin/bash
# Experiment builds: bench-path-only libraries with different batching / occupancy macros.
# usage: scripts/build_variants.sh "tag:-DFLAGS ..." ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  tag="${spec%%:*}"; flags="${spec#*:}"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -DAB_BENCH_ONLY -diag-suppress 177,550 $flags \
    -o paper_2306_15685_b200/libarcboost_b200_$tag.so paper_2306_15685_b200/csrc/arcboost_b200.cu &
done
wait
