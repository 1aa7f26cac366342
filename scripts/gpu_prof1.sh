#!/bin/bash
mkdir -p gpurun_out
ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_prof.so timeout 300 python bench.py --frames 100 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof1.log 2>&1
ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_prof.so AB_GRID=148 timeout 300 python bench.py --frames 100 --segments 1 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof1_g148.log 2>&1
