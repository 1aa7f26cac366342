#!/bin/bash
# C3 launch-shape / shared-memory sweep (kernel-only legs)
mkdir -p gpurun_out
: > gpurun_out/shape_sweep.log
run() { tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); b=d['biasing_overhead']
print('$tag', round(d['value']), 'unbiased_ms', round(b['unbiased_ms_per_step'],1), 'biased_ms', round(b['biased_ms_per_step'],1), 'zero_ms', round(b['zero_discount_ms_per_step'],1), 'redos', d['cutoff']['frames_redone_per_step'])" >> gpurun_out/shape_sweep.log 2>&1
}
run main A=1
run rowglobal AB_ROW_GLOBAL=1
run n2k ARCBOOST_B200_LIB=paper_2306_15685_b200/libarcboost_b200_n2k.so
run b512 AB_BLOCK=512
run b1024 AB_BLOCK=1024
run grid444 AB_GRID=444
