#!/bin/bash
mkdir -p gpurun_out
run() { timeout 300 python bench.py --frames 100 --segments 1 --steps 2 --warmup 1 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))"; }
: > gpurun_out/sweep15.log
echo "== default : $(run)" >> gpurun_out/sweep15.log
for v in U2m4 U2m3 Q4 PQ4 m5; do
  echo "== $v : $(ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_$v.so run)" >> gpurun_out/sweep15.log
done
echo "== default again : $(run)" >> gpurun_out/sweep15.log
