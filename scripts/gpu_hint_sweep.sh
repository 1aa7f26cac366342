#!/bin/bash
# Cutoff hint margin sweep (C3, kernel-only legs): AB_CUT_HINT_EXTRA values
mkdir -p gpurun_out
: > gpurun_out/hint_sweep.log
for x in "$@"; do
  AB_CUT_HINT_EXTRA=$x timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); b=d['biasing_overhead']
print('extra $x', round(d['value']), 'unbiased_ms', round(b['unbiased_ms_per_step'],1), 'biased_ms', round(b['biased_ms_per_step'],1), 'zero_ms', round(b['zero_discount_ms_per_step'],1), 'redos', d['cutoff']['frames_redone_per_step'])" >> gpurun_out/hint_sweep.log 2>&1
done
