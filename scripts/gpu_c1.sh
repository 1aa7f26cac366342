#!/bin/bash
mkdir -p gpurun_out
run() { timeout 300 python bench.py --workload $1 --steps 3 --warmup 2 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))"; }
: > gpurun_out/c1.log
for B in 256 512 1024; do
  echo "== c1 B$B : $(AB_BLOCK=$B ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_B1k.so run c1)" >> gpurun_out/c1.log
  echo "== c2 B$B : $(AB_BLOCK=$B ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_B1k.so run c2)" >> gpurun_out/c1.log
done
