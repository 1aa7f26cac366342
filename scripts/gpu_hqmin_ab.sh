#!/bin/bash
# C4 0.1% / 1% contexts: per-state slack for every negative context (hm0) vs only above 24k flagged states (hm24).
mkdir -p gpurun_out
: > gpurun_out/hqmin_ab.log
for t in hm24 hm0; do
  for d in 0.001 0.01; do
    for k in words arcs; do
      ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_$t.so timeout 600 python bench.py --workload c4 --density $d --c4-kind $k --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); b=d['biasing_overhead']
print('$t $d $k', round(d['value']), 'overhead', round(b['discount_overhead_pct'],2), 'zero', round(b['zero_discount_overhead_pct'],2))" >> gpurun_out/hqmin_ab.log 2>&1
    done
  done
done
ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_hm0.so timeout 900 python bench.py --ctx-kind entities --steps 2 --warmup 2 --no-e2e --no-cpu 2>/dev/null | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); b=d['biasing_overhead']
print('hm0 entities', round(d['value']), 'overhead', round(b['discount_overhead_pct'],2), 'zero', round(b['zero_discount_overhead_pct'],2))" >> gpurun_out/hqmin_ab.log 2>&1
