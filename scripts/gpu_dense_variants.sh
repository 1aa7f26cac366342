#!/bin/bash
# C4 5% (words, arcs) with experiment libraries: biased / unbiased / zero legs
mkdir -p gpurun_out
: > gpurun_out/dense_variants.log
for t in "$@"; do
  if [ "$t" = main ]; then lib=paper_2306_15685_b200/libarcboost_b200.so; else lib=paper_2306_15685_b200/libarcboost_b200_$t.so; fi
  for k in words arcs; do
    ARCBOOST_B200_LIB=$lib timeout 600 python bench.py --workload c4 --density 0.05 --c4-kind $k --steps 2 --warmup 2 --no-e2e --no-cpu 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); b=d['biasing_overhead']
print('$t $k', round(d['value']), 'unbiased_ms', round(b['unbiased_ms_per_step'],1), 'biased_ms', round(b['biased_ms_per_step'],1), 'zero_ms', round(b['zero_discount_ms_per_step'],1), 'ovh %.1f%%' % b['discount_overhead_pct'])" >> gpurun_out/dense_variants.log 2>&1
  done
done
