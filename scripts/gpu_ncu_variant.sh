#!/bin/bash
# one full ncu capture of the decode kernel for a variant library: $1 = tag
mkdir -p gpurun_out
ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_$1.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/prof_$1 python bench.py --frames 20 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_$1.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_$1.log
