#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/warm_sweep.log
run() { tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-overhead 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('$tag', round(d['value']), 'redos', d['cutoff']['frames_redone_per_step'])" >> gpurun_out/warm_sweep.log 2>&1
}
run base A=1
run w1x4 AB_CUT_HINT_WARM=1.0 AB_CUT_HINT_WARM_FRAMES=4
run w2x6 AB_CUT_HINT_WARM=2.0 AB_CUT_HINT_WARM_FRAMES=6
run w1x10 AB_CUT_HINT_WARM=1.0 AB_CUT_HINT_WARM_FRAMES=10
run w05x6_e015 AB_CUT_HINT_WARM=0.5 AB_CUT_HINT_WARM_FRAMES=6 AB_CUT_HINT_EXTRA=0.15
run w1x6_e01 AB_CUT_HINT_WARM=1.0 AB_CUT_HINT_WARM_FRAMES=6 AB_CUT_HINT_EXTRA=0.1
