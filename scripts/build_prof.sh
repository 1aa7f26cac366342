#!/bin/bash
# Phase-profiling variant of the library (clock64 per phase, printed per ab_decode).
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -DAB_PROFILE -diag-suppress 177,550 \
  -o paper_2306_15685_b200/libarcboost_b200_prof.so paper_2306_15685_b200/csrc/arcboost_b200.cu
