#!/bin/bash
# Full C3 bench (kernel-only legs: biased, unbiased, zero-discount) of experiment libraries.
# usage: scripts/gpu_variants_full.sh TAG...   (main = the in-tree library)
mkdir -p gpurun_out
: > gpurun_out/variants_full.log
for t in "$@"; do
  if [ "$t" = main ]; then lib=paper_2306_15685_b200/libarcboost_b200.so; else lib=paper_2306_15685_b200/libarcboost_b200_$t.so; fi
  ARCBOOST_B200_LIB=$lib timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); b=d['biasing_overhead']
print('$t', round(d['value']), 'unbiased_ms', round(b['unbiased_ms_per_step'],1), 'biased_ms', round(b['biased_ms_per_step'],1), 'zero_ms', round(b['zero_discount_ms_per_step'],1), 'redos', d['cutoff']['frames_redone_per_step'])" >> gpurun_out/variants_full.log 2>&1
done
