#!/bin/bash
mkdir -p gpurun_out
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))"; }
: > gpurun_out/blocks.log
echo "== B512 m2 : $(AB_BLOCK=512 ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_B512.so run)" >> gpurun_out/blocks.log
echo "== B512 m3 : $(AB_BLOCK=512 ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_B512m3.so run)" >> gpurun_out/blocks.log
echo "== B128 m8 : $(AB_BLOCK=128 ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_B128.so run)" >> gpurun_out/blocks.log
echo "== B256 m5 : $(ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_A5.so run)" >> gpurun_out/blocks.log
echo "== B256 m4 default : $(run)" >> gpurun_out/blocks.log
