#!/bin/bash
# C4 5% words / arcs with 2-bit vs 8-bit per-state slack (experiment libraries hq2 / hq8).
mkdir -p gpurun_out
: > gpurun_out/hq_ab.log
for rep in 1 2; do
for t in hq2 hq8; do
  for k in words arcs; do
    ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_$t.so timeout 600 python bench.py --workload c4 --density 0.05 --c4-kind $k --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); b=d['biasing_overhead']
print('$t $k', round(d['value']), 'overhead', round(b['discount_overhead_pct'],2), 'zero', round(b['zero_discount_overhead_pct'],2))" >> gpurun_out/hq_ab.log 2>&1
  done
done
done
